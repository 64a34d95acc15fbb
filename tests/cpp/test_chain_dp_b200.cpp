// C++ drop-in check: the known-answer cases of the reference's
// proj/tests/test_chain_dp.cpp (:9-107, :203-221), written against
// include/remat_b200/chain_dp.hpp (namespace remat, same names) and run on
// the GPU through librkr.  Exit status 0 iff every check passes.
//
// Catch2 is not in the image, so this file carries a 10-line harness.
#include <cstdio>
#include <string>
#include <vector>

#include "remat_b200/chain_dp.hpp"

using namespace remat;

static int g_checks = 0, g_fail = 0;
#define CHECK(cond)                                                          \
    do {                                                                     \
        ++g_checks;                                                          \
        if (!(cond)) {                                                       \
            ++g_fail;                                                        \
            std::fprintf(stderr, "FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond); \
        }                                                                    \
    } while (0)

// Two forwards, a loss and two backwards; ids as in the reference's toy block.
static CDGraph toy_block(Bytes sz) {
    CDGraph g;
    const char* dn[] = {"d0", "d1", "d2", "g2", "g1", "g0"};
    for (int i = 0; i < 6; ++i) {
        DNode d;
        d.id = dn[i];
        d.size = sz;
        d.kind = i < 3 ? DNodeKind::Data : DNodeKind::Grad;
        g.dnodes.push_back(d);
    }
    const char* cn[] = {"f1", "f2", "loss", "b2", "b1"};
    CNodeKind kinds[] = {CNodeKind::Forward, CNodeKind::Forward, CNodeKind::Loss,
                         CNodeKind::Backward, CNodeKind::Backward};
    for (int i = 0; i < 5; ++i) {
        CNode c;
        c.id = cn[i];
        c.kind = kinds[i];
        g.cnodes.push_back(c);
    }
    g.input_data = 0;
    g.output_data = 2;
    g.loss_index = 2;
    return g;
}

static BlockOption mk(int id, Micros ef, Micros eb, Bytes save, Bytes pf, Bytes pre, Bytes pb) {
    BlockOption o;
    o.option_id = id;
    o.time_fwd = ef;
    if (id != 0) o.time_bwd = eb;
    o.save_mem = save;
    o.peak_fwd = pf;
    o.peak_fwd_pre = pre;
    o.peak_bwd = pb;
    return o;
}

// a = (4, 4, 2); block 0 saves 10, block 1 saves 8 (reference test_helpers.hpp:64-82)
static OptionMenu tiny_menu() {
    OptionMenu menu;
    menu.act_sizes = {4, 4, 2};
    menu.options = {{mk(0, 10, 0, 4, 8, 8, 0), mk(1, 10, 12, 10, 10, 10, 14)},
                    {mk(0, 8, 0, 4, 6, 6, 0), mk(1, 8, 9, 8, 8, 8, 10)}};
    return menu;
}

static Chain tiny_chain() {
    Chain chain;
    chain.blocks = {toy_block(4), toy_block(4)};
    chain.blocks[1].dnodes[chain.blocks[1].dnode_index("d2")].size = 2;
    chain.blocks[1].dnodes[chain.blocks[1].dnode_index("g2")].size = 2;
    chain.equiv_class = {0, 1};
    return chain;
}

static void quantization() {
    Quantization q = quantize(1000, 10);
    CHECK(q.unit == 100);
    CHECK(q.budget_units == 10);
    CHECK(to_units(100, q.unit) == 1);
    CHECK(to_units(250, q.unit) == 3);
    CHECK(to_units(300, q.unit) == 3);
    Quantization one = quantize(7, 1);
    CHECK(one.unit == 7 && one.budget_units == 1);
    bool threw = false;
    try {
        quantize(10, 0);
    } catch (const ValidationError&) {
        threw = true;
    }
    CHECK(threw);
}

static void single_block() {
    OptionMenu menu;
    menu.act_sizes = {4, 4};
    menu.options = {{mk(0, 10, 0, 4, 8, 8, 0), mk(1, 10, 12, 10, 10, 10, 14)}};
    DpTable table(menu, 1, 100);
    CHECK(table.opt(0, 0, 100) == 22);
}

static void tiny_optima(bool force64) {
    ExecConfig cfg;
    cfg.force_int64 = force64;
    OptionMenu menu = tiny_menu();
    DpTable table(menu, 1, 64, cfg);
    CHECK(table.opt(0, 1, 64) == 39);
    CHECK(table.opt(0, 1, 12) == 39);
    CHECK(table.opt(0, 1, 11) == 49);
    CHECK(table.opt(0, 1, 10) == 49);
    CHECK(table.opt(0, 1, 9) >= kInfTime);
    DpArg a = table.arg(0, 1, 10);
    CHECK(a.kind == DpArg::Cut);
    CHECK(a.value == 1);
    CHECK(table.opt(0, 0, 5) >= kInfTime);
    CHECK(table.opt(0, 1, -1) >= kInfTime);
    CHECK(table.opt(0, 1, 1000) == 39);  // clamps to m_max
    CHECK(table.worst_cell_allowance <= 0);
}

static void tiny_schedules() {
    OptionMenu menu = tiny_menu();
    Chain chain = tiny_chain();
    DpTable ample(menu, 1, 12);
    std::vector<ScheduleOp> ops;
    build_schedule_rec(ample, menu, chain, 0, 1, 12, ops);
    std::vector<ScheduleOp> expect = {
        ScheduleOp::block_fwd(0, 1), ScheduleOp::block_fwd(1, 1), ScheduleOp::compute(1, "loss"),
        ScheduleOp::block_bwd(1, 1), ScheduleOp::block_bwd(0, 1)};
    CHECK(ops == expect);

    DpTable tight(menu, 1, 10);
    ops.clear();
    build_schedule_rec(tight, menu, chain, 0, 1, 10, ops);
    int fwd0 = 0, fwd0_opt0 = 0;
    for (const ScheduleOp& op : ops)
        if (op.kind == ScheduleOp::BlockFwd && op.block == 0) {
            ++fwd0;
            if (op.option == 0) ++fwd0_opt0;
        }
    CHECK(fwd0 == 2);
    CHECK(fwd0_opt0 == 1);

    DpTable none(menu, 1, 9);
    ops.clear();
    bool threw = false;
    try {
        build_schedule_rec(none, menu, chain, 0, 1, 9, ops);
    } catch (const InfeasibleBudget&) {
        threw = true;
    }
    CHECK(threw);
}

static void solve_and_min_feasible() {
    OptionMenu menu = tiny_menu();
    Chain chain = tiny_chain();
    ChainSolution sol = solve_chain(chain, menu, 16, 16);
    CHECK(sol.opt_time == 39);
    CHECK(sol.m_top == 12);
    CHECK(sol.schedule.ops.size() == 5);
    ChainSolution tight = solve_chain(chain, menu, 14, 14);
    CHECK(tight.opt_time == 49);
    bool threw = false;
    try {
        solve_chain(chain, menu, 12, 12);
    } catch (const InfeasibleBudget& e) {
        threw = true;
        CHECK(e.min_feasible_budget == 14);
    }
    CHECK(threw);
    threw = false;
    try {
        solve_chain(chain, menu, 3, 3);  // cannot even hold a_0
    } catch (const InfeasibleBudget& e) {
        threw = true;
        CHECK(e.min_feasible_budget == -1);
    }
    CHECK(threw);
}

static void validation() {
    OptionMenu menu = tiny_menu();
    menu.options[1].erase(menu.options[1].begin());  // block 1 loses option 0
    bool threw = false;
    try {
        DpTable t(menu, 1, 8);
    } catch (const ValidationError&) {
        threw = true;
    }
    CHECK(threw);
    OptionMenu nob = tiny_menu();
    nob.options[0][1].time_bwd.reset();
    threw = false;
    try {
        DpTable t(nob, 1, 8);
    } catch (const ValidationError&) {
        threw = true;
    }
    CHECK(threw);
}

static void b200_extensions() {
    OptionMenu menu = tiny_menu();
    Chain chain = tiny_chain();
    // batched tables agree with single tables
    b200::Batch batch({menu, menu}, {1, 1}, {64, 10});
    CHECK(batch.size() == 2);
    CHECK(batch.table(0).opt(0, 1, 64) == 39);
    CHECK(batch.table(1).opt(0, 1, 10) == 49);
    // the sweep: per-budget solve_chain results, sorted, monotone
    auto rows = b200::sweep(chain, menu, {16, 14, 12, 16, 40}, 16);
    CHECK(rows.size() == 4);
    CHECK(rows[0].budget == 12 && !rows[0].feasible && rows[0].min_feasible > 0);
    CHECK(rows[1].budget == 14 && rows[1].feasible);
    CHECK(rows[3].feasible && rows[3].opt_time == 39);
    ChainSolution one = solve_chain(chain, menu, 16, 16);
    CHECK(rows[2].schedule.ops == one.schedule.ops);
    // a 2-shard table equals the unsharded one
    b200::ShardedTable sh(menu, 1, 64, 2);
    DpTable whole(menu, 1, 64);
    bool same = true;
    for (int m = 0; m <= 64; ++m) same = same && sh.opt(0, 1, m) == whole.opt(0, 1, m);
    CHECK(same);
    std::vector<ScheduleOp> a, b;
    sh.build_schedule(chain, 0, 1, 10, a);
    build_schedule_rec(whole, menu, chain, 0, 1, 10, b);
    CHECK(a == b);
}

int main() {
    quantization();
    single_block();
    tiny_optima(false);
    tiny_optima(true);
    tiny_schedules();
    solve_and_min_feasible();
    validation();
    b200_extensions();
    std::printf("%d checks, %d failed\n", g_checks, g_fail);
    return g_fail == 0 ? 0 : 1;
}
