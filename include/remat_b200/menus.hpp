// remat_b200/menus.hpp -- option generation (rk-Checkmate's ILP per block
// class) on a host thread pool: SURVEY.md 8(f) rank 4.
//
// The reference's build_menus (pipeline.hpp:144-185) solves its block classes
// one after another, and each class's budget-pair lattice one pair after
// another (solve_block_class, :57-134); it ignores SolveSettings::threads
// (`int /*threads*/`, :58).  Here every (class, budget pair) solve is a task on
// one pool of `threads` workers (0 = the hardware concurrency), with the
// lattice's own dependencies and nothing more:
//   * pair i reads, in the reference's order, the records of the pairs solved
//     before it that are TIGHTER (both budgets <=: the warm start and upper
//     bound, :86-92) or LOOSER (lower bound / known infeasible).  In the
//     sorted order with the loosest pair rotated to the front (:61-71) the
//     only looser one is pair 0, so pair i waits for pair 0 and its tighter
//     predecessors -- an anti-diagonal wavefront over the grid;
//   * the upper bound is chosen by scanning those records in the reference's
//     order (first minimum), so every solve gets the same warm start as in the
//     sequential run, and the branch-and-bound is deterministic
//     (ilp_solver.hpp:31): the menus come out identical, member for member
//     (tests/dropin/menus_check.cpp), as long as no solve hits its time limit.
//
// Needs the reference's ILP layer on the include path (remat/pipeline.hpp:
// ilp_model.hpp, ilp_solver.hpp, options.hpp); tests/dropin builds it against
// a scratch copy.
#pragma once

#include <algorithm>
#include <condition_variable>
#include <deque>
#include <exception>
#include <mutex>
#include <thread>
#include <utility>
#include <vector>

#include "remat/pipeline.hpp"

namespace remat {
namespace b200 {

namespace menus_detail {

struct PairRec {
    BudgetPair pair;
    bool feasible = false, timed_out = false, done = false;
    Micros objective = 0;
    std::vector<signed char> assignment;
};

struct ClassWork {
    const CDGraph* g = nullptr;
    std::vector<PairRec> rec;                // the reference's solve order
    std::vector<std::vector<int>> waiters;   // pair -> pairs waiting on it
    std::vector<int> pending;                // unfinished dependencies per pair
    std::vector<BlockOption> options;        // extracted answers, in order (after all pairs)
};

// pipeline.hpp:60-71: the grid in the reference's solve order
inline std::vector<BudgetPair> solve_order(const CDGraph& g, int n_peak, int n_save) {
    BudgetGrid grid = budget_grid(g, n_peak, n_save);
    auto& p = grid.pairs;
    std::sort(p.begin(), p.end(), [](const BudgetPair& a, const BudgetPair& b) {
        return a.m_peak != b.m_peak ? a.m_peak < b.m_peak : a.m_save < b.m_save;
    });
    p.erase(std::unique(p.begin(), p.end(),
                        [](const BudgetPair& a, const BudgetPair& b) {
                            return a.m_peak == b.m_peak && a.m_save == b.m_save;
                        }),
            p.end());
    std::rotate(p.begin(), p.end() - 1, p.end());
    return p;
}

inline bool tighter(const BudgetPair& a, const BudgetPair& b) {  // a <= b in both
    return a.m_peak <= b.m_peak && a.m_save <= b.m_save;
}

// pipeline.hpp:73-119 for pair i of one class, its predecessors done.
inline void solve_pair(ClassWork& w, int i, double time_limit) {
    PairRec& r = w.rec[i];
    const PairRec* upper = nullptr;
    Micros lower = -1;
    bool known_infeasible = false;
    for (int j = 0; j < i; ++j) {
        const PairRec& s = w.rec[j];
        const bool t = tighter(s.pair, r.pair), l = tighter(r.pair, s.pair);
        if (!t && !l) continue;  // incomparable: not read (and maybe not solved yet)
        if (t && s.feasible && (!upper || s.objective < upper->objective)) upper = &s;
        if (l && s.feasible) lower = std::max(lower, s.objective);
        if (l && !s.feasible) known_infeasible = true;
    }
    if (known_infeasible) return;
    if (upper && lower >= 0 && upper->objective == lower) {
        r.feasible = true;
        r.objective = upper->objective;
        r.assignment = upper->assignment;
        return;
    }
    IlpModel model = build_model(*w.g, r.pair);
    SolveResult res = upper ? solve(model, time_limit, &upper->assignment, upper->objective)
                            : solve(model, time_limit);
    if (res.status == SolveStatus::TimedOut) {
        r.timed_out = true;
        return;
    }
    if (res.status == SolveStatus::Optimal) {
        r.feasible = true;
        r.objective = res.objective;
        r.assignment = std::move(res.assignment);
    }
}

}  // namespace menus_detail

// pipeline.hpp:144-185 with the (class, pair) solves on a thread pool.
inline MenuSet build_menus(const Chain& chain, const SolveSettings& settings) {
    using namespace menus_detail;
    MenuSet out;
    std::vector<int> cls = settings.use_classes ? chain.equiv_class : std::vector<int>{};
    if (cls.empty()) {
        cls.resize(chain.length());
        for (int i = 0; i < chain.length(); ++i) cls[i] = i;
    }
    verify_equiv_classes(chain);
    std::vector<int> reps, class_of_block(chain.length(), -1);  // :153-164
    for (int i = 0; i < chain.length(); ++i) {
        int found = -1;
        for (size_t r = 0; r < reps.size(); ++r)
            if (cls[reps[r]] == cls[i]) found = static_cast<int>(r);
        if (found < 0) {
            found = static_cast<int>(reps.size());
            reps.push_back(i);
        }
        class_of_block[i] = found;
    }
    const int nc = static_cast<int>(reps.size());
    std::vector<ClassWork> work(nc);
    std::deque<std::pair<int, int>> ready;  // (class, pair)
    size_t total = 0;
    for (int c = 0; c < nc; ++c) {
        ClassWork& w = work[c];
        w.g = &chain.blocks[reps[c]];
        const std::vector<BudgetPair> order = solve_order(*w.g, settings.n_peak, settings.n_save);
        const int P = static_cast<int>(order.size());
        w.rec.resize(P);
        w.waiters.assign(P, {});
        w.pending.assign(P, 0);
        for (int i = 0; i < P; ++i) {
            w.rec[i].pair = order[i];
            for (int j = 0; j < i; ++j)
                if (j == 0 || tighter(order[j], order[i]) || tighter(order[i], order[j])) {
                    w.waiters[j].push_back(i);
                    ++w.pending[i];
                }
        }
        for (int i = 0; i < P; ++i)
            if (w.pending[i] == 0) ready.emplace_back(c, i);
        total += P;
    }
    std::mutex mu;
    std::condition_variable cv;
    size_t finished = 0;
    std::exception_ptr err;
    auto worker = [&] {
        std::unique_lock<std::mutex> lk(mu);
        for (;;) {
            cv.wait(lk, [&] { return !ready.empty() || finished == total || err; });
            if (finished == total || err) return;
            auto [c, i] = ready.front();
            ready.pop_front();
            lk.unlock();
            try {
                solve_pair(work[c], i, settings.time_limit_seconds);
            } catch (...) {
                lk.lock();
                if (!err) err = std::current_exception();
                cv.notify_all();
                return;
            }
            lk.lock();
            work[c].rec[i].done = true;
            ++finished;
            for (int k : work[c].waiters[i])
                if (--work[c].pending[k] == 0) ready.emplace_back(c, k);
            cv.notify_all();
        }
    };
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    const int nt = std::max(1, std::min<int>(static_cast<int>(total),
                                             settings.threads > 0 ? settings.threads : static_cast<int>(hw)));
    if (total > 0) {
        std::vector<std::thread> pool;
        for (int t = 1; t < nt; ++t) pool.emplace_back(worker);
        worker();
        for (auto& t : pool) t.join();
    }
    if (err) std::rethrow_exception(err);
    for (int c = 0; c < nc; ++c) {  // :121-133 and :166-175, in class order
        ClassWork& w = work[c];
        ClassMenu menu;
        std::vector<BlockOption> opts;
        opts.push_back(option_zero(*w.g));
        for (const PairRec& r : w.rec) {
            if (r.timed_out) ++menu.timed_out_pairs;
            if (!r.feasible) continue;
            IlpModel model = build_model(*w.g, r.pair);
            opts.push_back(extract_option(*w.g, model, r.assignment, 1));
        }
        menu.options = dedup_options(std::move(opts));
        menu.solved_pairs = static_cast<int>(w.rec.size());
        menu.class_id = c;
        menu.representative = reps[c];
        for (int i = 0; i < chain.length(); ++i)
            if (class_of_block[i] == c) menu.members.push_back(i);
        out.timeout_pairs += menu.timed_out_pairs;
        out.classes.push_back(std::move(menu));
    }
    out.class_solves = nc;
    out.menu.options.resize(chain.length());
    for (int i = 0; i < chain.length(); ++i) out.menu.options[i] = out.classes[class_of_block[i]].options;
    out.menu.act_sizes.resize(chain.length() + 1);
    for (int i = 0; i <= chain.length(); ++i) out.menu.act_sizes[i] = chain.act_size(i);
    return out;
}

}  // namespace b200
}  // namespace remat
