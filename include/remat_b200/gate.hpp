// remat_b200/gate.hpp -- the schedule validation gate around the device DP
// (SURVEY.md 8(f) rank 2), for callers that do not build the reference's
// pipeline.hpp (which drags in the ILP option generator):
//   schedule_with_menu  pipeline.hpp:187-205  solve_chain + simulate, meta filled
//   flatten_schedule    pipeline.hpp:222-247  block ops -> compute / forget ops
//   chain_max_peak      pipeline.hpp:249-274  the no-recompute budget ceiling
// Same semantics and messages as the reference, in namespace remat::b200 so
// that a caller may include both this and the reference's pipeline.hpp.  With
// the reference tree on the include path the reference's functions run the
// same code path anyway (this repo's remat/chain_dp.hpp + remat/simulate.hpp);
// tests/dropin/pipeline_check.cpp checks the two line for line.
#pragma once

#include <utility>
#include <vector>

#include "remat/chain_dp.hpp"
#include "remat/simulate.hpp"

namespace remat {
namespace b200 {

struct ScheduledRun {
    Schedule schedule;
    SimReport report;
    Micros opt_time = 0;
};

// DP (on the device) + reconstruction + the exact replay for one budget.
inline ScheduledRun schedule_with_menu(const Chain& chain, const OptionMenu& menu, Bytes memory,
                                       int units, const ExecConfig& cfg = {}) {
    ChainSolution sol = solve_chain(chain, menu, memory, units, cfg);
    ScheduledRun run;
    run.opt_time = sol.opt_time;
    run.schedule = std::move(sol.schedule);
    SimulateOptions sim;
    sim.menus = &menu.options;
    run.report = simulate(run.schedule, chain, memory, sim);  // throws BudgetExceeded / ValidationError
    run.schedule.meta = ScheduleMeta{memory, run.report.makespan, run.report.peak_mem};
    return run;
}

// Every BlockFwd / BlockBwd replaced by its option's local ops, so the
// schedule replays without a menu.  The option is the LAST one of the block
// with the op's id (the reference's lookup loop has no break, :231-233).
inline Schedule flatten_schedule(const Schedule& s, const Chain& chain, const OptionMenu& menu) {
    Schedule flat;
    flat.meta = s.meta;
    flat.ops.reserve(s.ops.size() * 4);
    for (const ScheduleOp& op : s.ops) {
        if (op.kind != ScheduleOp::BlockFwd && op.kind != ScheduleOp::BlockBwd) {
            flat.ops.push_back(op);
            continue;
        }
        const BlockOption* pick = nullptr;
        for (const BlockOption& o : menu.options[op.block])
            if (o.option_id == op.option) pick = &o;
        if (!pick) throw ValidationError("schedule references a missing option");
        const CDGraph& g = chain.blocks[op.block];
        for (const BlockLocalOp& lo : op.kind == ScheduleOp::BlockFwd ? pick->fwd_ops : pick->bwd_ops)
            flat.ops.push_back(lo.kind == BlockLocalOp::Compute
                                   ? ScheduleOp::compute(op.block, g.cnodes[lo.node].id)
                                   : ScheduleOp::forget(op.block, g.dnodes[lo.node].id));
    }
    return flat;
}

// Peak of the one-pass schedule that saves every block with its fastest
// saved option (first of equal totals): forwards 0..L-1, the loss of the last
// block, backwards L-1..0.  The budget above which recomputation never pays.
inline Bytes chain_max_peak(const Chain& chain, const OptionMenu& menu,
                            std::vector<int>* chosen = nullptr) {
    const int L = chain.length();
    std::vector<int> pick(L, -1);
    Schedule s;
    s.ops.reserve(2 * static_cast<size_t>(L) + 1);
    for (int i = 0; i < L; ++i) {
        Micros best = kInfTime;
        for (const BlockOption& o : menu.options[i])
            if (o.has_bwd() && o.total_time() < best) {
                best = o.total_time();
                pick[i] = o.option_id;
            }
        if (pick[i] < 0) throw ValidationError("block without a saved option");
        s.ops.push_back(ScheduleOp::block_fwd(i, pick[i]));
    }
    const CDGraph& last = chain.blocks[L - 1];
    s.ops.push_back(ScheduleOp::compute(L - 1, last.cnodes[last.loss_index].id));
    for (int i = L - 1; i >= 0; --i) s.ops.push_back(ScheduleOp::block_bwd(i, pick[i]));
    SimulateOptions sim;
    sim.menus = &menu.options;
    const Bytes peak = simulate(s, chain, -1, sim).peak_mem;
    if (chosen) *chosen = std::move(pick);
    return peak;
}

}  // namespace b200
}  // namespace remat
