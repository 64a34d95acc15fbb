// The reference pipeline's schedule gate around the DP, run on fixtures from
// the reference's own test helpers: build_menus (rk-Checkmate ILP option
// generation, pipeline.hpp:144-185) -> schedule_with_menu (solve_chain +
// simulate, :194-205) over a budget ladder incl. infeasible budgets ->
// flatten_schedule (:224-247) replayed without menus -> chain_max_peak
// (:251-274).  Compiled three times by tests/dropin/Makefile: against the
// reference alone (CPU; its output is tests/golden/dropin_pipeline.txt),
// against this repo's drop-in (include/ first: the DP and the simulator of
// this repo, the fill and walk on the GPU), and with -DRKR_B200_GATE, where
// build_menus / schedule_with_menu / flatten_schedule / chain_max_peak are
// this repo's own (include/remat_b200/menus.hpp, gate.hpp).  All outputs must
// be equal, line for line.
#include <cstdio>
#include <random>
#include <string>
#include <vector>

#include "remat/pipeline.hpp"
#include "test_helpers.hpp"
#ifdef RKR_B200_GATE  // this repo's own gate and menu builder (include/remat_b200/)
#include "remat_b200/gate.hpp"
#include "remat_b200/menus.hpp"
namespace gate = remat::b200;
#else  // pipeline.hpp's
namespace gate = remat;
#endif

using namespace remat;

namespace {

unsigned long long fnv(const Schedule& s) {
    unsigned long long h = 1469598103934665603ull;
    auto mix = [&](long long v) {
        h ^= (unsigned long long)v;
        h *= 1099511628211ull;
    };
    for (const ScheduleOp& op : s.ops) {
        mix(op.kind);
        mix(op.block);
        mix(op.option);
        for (char c : op.target) mix(c);
    }
    return h;
}

void run_chain(const char* name, const Chain& chain, int units) {
    SolveSettings st;
    st.n_peak = 3;
    st.n_save = 3;
    st.units = units;
    st.time_limit_seconds = 60.0;
    MenuSet ms = gate::build_menus(chain, st);
    const OptionMenu& menu = ms.menu;
    int nopt = 0;
    for (const auto& b : menu.options) nopt += (int)b.size();
    Bytes ceiling = -1;
    try {
        ceiling = gate::chain_max_peak(chain, menu);
    } catch (const ValidationError& e) {
        std::printf("%s blocks=%d options=%d timeouts=%d chain_max_peak: %s\n", name, chain.length(),
                    nopt, ms.timeout_pairs, e.what());
        return;
    }
    std::printf("%s blocks=%d options=%d timeouts=%d ceiling=%lld\n", name, chain.length(), nopt,
                ms.timeout_pairs, (long long)ceiling);
    // budgets from well below the input up to the no-recompute ceiling
    for (int q = 0; q <= 28; ++q) {
        const Bytes budget = ceiling * q / 24;
        try {
            auto run = gate::schedule_with_menu(chain, menu, budget, units);
            Schedule flat = gate::flatten_schedule(run.schedule, chain, menu);
            SimulateOptions plain;  // the flat schedule stands alone
            SimReport again = simulate(flat, chain, budget, plain);
            std::printf("  budget=%lld opt=%lld makespan=%lld peak=%lld at_loss=%lld overhead=%lld "
                        "ops=%zu flat=%zu hash=%016llx flat_makespan=%lld flat_peak=%lld\n",
                        (long long)budget, (long long)run.opt_time, (long long)run.report.makespan,
                        (long long)run.report.peak_mem, (long long)run.report.mem_at_loss,
                        (long long)run.report.overhead, run.schedule.ops.size(), flat.ops.size(),
                        fnv(run.schedule), (long long)again.makespan, (long long)again.peak_mem);
        } catch (const InfeasibleBudget& e) {
            std::printf("  budget=%lld infeasible min_feasible=%lld\n", (long long)budget,
                        (long long)e.min_feasible_budget);
        } catch (const BudgetExceeded& e) {
            std::printf("  budget=%lld budget_exceeded excess=%lld\n", (long long)budget,
                        (long long)e.excess);
        }
    }
}

}  // namespace

int main() {
    {  // the toy block twice, seams matched (test_chain_dp.cpp:203-210)
        Chain chain;
        chain.blocks = {testing::toy_block(4), testing::toy_block(4)};
        chain.equiv_class = {0, 0};
        run_chain("toy2", chain, 500);
    }
    std::mt19937 rng(2024);
    for (int i = 0; i < 10; ++i) {  // random seam-compatible chains
        Chain chain = testing::random_chain(rng, 5, i < 5 ? 2 : 3);
        run_chain(("random" + std::to_string(i)).c_str(), chain, 64);
    }
    return 0;
}
