// Reference-produced option documents and solve results for the reference's
// own chain fixtures (proj/tests/fixtures/*_chain.json).  Built against the
// reference ALONE (tests/dropin/Makefile; nlohmann json from the image's
// cudnn_frontend third-party tree stands in for the absent vendor/), run here
// on the CPU:
//   remat::load_chain                     ingest.hpp:495-503
//   remat::build_menus (ILP options)      pipeline.hpp:144-185
//   the `--save-options` document         tools/remat.cpp:72-89 (framing) +
//                                         ingest.hpp:409-436 (encode_options)
//   schedule_with_menu + flatten_schedule pipeline.hpp:194-247 (cmd_solve,
//                                         tools/remat.cpp:158-188) per budget
// Output: <out>/ref_chain_<name>.json (the chain as the reference encodes
// it), <out>/ref_options_<name>.json (the options document, byte for byte
// what `remat solve --save-options` writes) and <out>/ref_solve_<name>.json
// (per budget: opt_time, makespan, peak, overhead, block-level ops, or the
// min-feasible budget).  tests/test_options_io.py reads the documents with
// options_io and solves them on the GPU against these results.
#include <cstdio>
#include <string>
#include <vector>

#include "remat/ingest.hpp"
#include "remat/pipeline.hpp"

using namespace remat;

namespace {

void write_options_doc(const Chain& chain, const MenuSet& menus, const std::string& path) {
    Json j;  // tools/remat.cpp:72-89
    j["format_version"] = kFormatVersion;
    j["kind"] = "options";
    Json classes = Json::array();
    for (const ClassMenu& c : menus.classes) {
        Json jc;
        jc["class_id"] = c.class_id;
        jc["representative"] = c.representative;
        jc["members"] = c.members;
        jc["options"] = encode_options(chain.blocks[c.representative], c.options);
        classes.push_back(jc);
    }
    j["classes"] = classes;
    detail::write_document(j, path);
}

const char* kind_name(ScheduleOp::Kind k) {
    switch (k) {
        case ScheduleOp::Compute: return "compute";
        case ScheduleOp::Forget: return "forget";
        case ScheduleOp::BlockFwd: return "block_fwd";
        default: return "block_bwd";
    }
}

}  // namespace

int main(int argc, char** argv) {
    if (argc < 4) {
        std::fprintf(stderr, "usage: options_ref <out-dir> <name> <chain.json> [n_peak n_save]\n");
        return 2;
    }
    const std::string out = argv[1], name = argv[2], chain_path = argv[3];
    SolveSettings st;  // the CLI defaults (pipeline.hpp:21-29) unless overridden
    if (argc >= 6) {
        st.n_peak = std::stoi(argv[4]);
        st.n_save = std::stoi(argv[5]);
    }
    Chain chain = load_chain(chain_path);
    save_chain(chain, out + "/ref_chain_" + name + ".json");  // re-encoded by ingest.hpp:505-507
    MenuSet menus = build_menus(chain, st);
    write_options_doc(chain, menus, out + "/ref_options_" + name + ".json");

    const Bytes ceiling = chain_max_peak(chain, menus.menu);
    Json res;
    res["chain"] = name;
    res["n_peak"] = st.n_peak;
    res["n_save"] = st.n_save;
    res["units"] = st.units;
    res["chain_max_peak"] = ceiling;
    res["timeout_pairs"] = menus.timeout_pairs;
    Json rows = Json::array();
    std::vector<Bytes> budgets;
    for (int q = 0; q <= 24; ++q) budgets.push_back(ceiling * q / 20);
    budgets.push_back(300);  // SURVEY.md 6.2's tiny_chain figure
    for (Bytes b : budgets) {
        Json r;
        r["budget"] = b;
        try {
            ScheduledRun run = schedule_with_menu(chain, menus.menu, b, st.units);
            Schedule flat = flatten_schedule(run.schedule, chain, menus.menu);
            r["opt_time"] = run.opt_time;
            r["makespan"] = run.report.makespan;
            r["peak"] = run.report.peak_mem;
            r["overhead"] = run.report.overhead;
            Json ops = Json::array();
            for (const ScheduleOp& op : run.schedule.ops)
                ops.push_back(Json::array({kind_name(op.kind), op.block, op.option, op.target}));
            r["ops"] = ops;
            r["flat_ops"] = static_cast<int>(flat.ops.size());
        } catch (const InfeasibleBudget& e) {
            r["infeasible"] = true;
            r["min_feasible"] = e.min_feasible_budget;
        }
        rows.push_back(r);
    }
    res["rows"] = rows;
    detail::write_document(res, out + "/ref_solve_" + name + ".json");
    std::printf("%s: %zu classes, ceiling %lld\n", name.c_str(), menus.classes.size(),
                static_cast<long long>(ceiling));
    return 0;
}
