// ref_driver.cpp -- C-ABI shim around the UNMODIFIED reference solver.
//
// TEST INFRASTRUCTURE ONLY.  Compiled by oracle/Makefile against the
// reference headers where they lie (/root/reference/proj/include and
// /root/reference/proj/tests); the output goes to oracle/_ref/ (git-ignored).
// No reference source is copied into this repository.  Used by tests/ to pin
// oracle/rotor_oracle.c, by tests/golden/gen_golden.py to produce fixtures,
// and by bench.py's CPU legs ("kind": "reference").
//
// Reference entry points wrapped: remat::DpTable (chain_dp.hpp:54-196),
// remat::build_schedule_rec (:211-246), remat::solve_chain (:255-296),
// remat::quantize (:32-39), testing::random_menu (test_helpers.hpp:197-232),
// testing::tiny_chain_menu (:64-82), testing::chain_oracle (:370-383),
// testing::chain_oracle_dijkstra (:385-550), testing::atomic_replay (:249-322).
#include <chrono>
#include <cstdint>
#include <cstring>
#include <random>
#include <string>
#include <thread>
#include <vector>

#include "remat/chain_dp.hpp"
#include "test_helpers.hpp"

using namespace remat;

namespace {

thread_local std::string g_err;

struct FlatMenu {
    int32_t n_blocks;
    const int32_t* option_offsets;
    const int32_t* option_id;
    const int64_t* time_fwd;
    const int64_t* time_bwd;
    const uint8_t* has_bwd;
    const int64_t* save_mem;
    const int64_t* peak_fwd;
    const int64_t* peak_fwd_pre;
    const int64_t* peak_bwd;
    const int64_t* act_sizes;
};

OptionMenu to_menu(const FlatMenu* f) {
    OptionMenu menu;
    menu.options.resize(f->n_blocks);
    menu.act_sizes.assign(f->act_sizes, f->act_sizes + f->n_blocks + 1);
    for (int i = 0; i < f->n_blocks; ++i)
        for (int o = f->option_offsets[i]; o < f->option_offsets[i + 1]; ++o) {
            BlockOption b;
            b.option_id = f->option_id[o];
            b.time_fwd = f->time_fwd[o];
            if (f->has_bwd[o]) b.time_bwd = f->time_bwd[o];
            b.save_mem = f->save_mem[o];
            b.peak_fwd = f->peak_fwd[o];
            b.peak_fwd_pre = f->peak_fwd_pre[o];
            b.peak_bwd = f->peak_bwd[o];
            menu.options[i].push_back(b);
        }
    return menu;
}

// Skeleton chain: block i has input dnode "b<i>_in" and loss cnode "b<i>_loss".
Chain skeleton_chain(int L) {
    Chain chain;
    for (int i = 0; i < L; ++i) {
        CDGraph g;
        DNode d;
        d.id = "b" + std::to_string(i) + "_in";
        g.dnodes.push_back(d);
        CNode c;
        c.id = "b" + std::to_string(i) + "_loss";
        c.kind = CNodeKind::Loss;
        g.cnodes.push_back(c);
        g.input_data = 0;
        g.output_data = 0;
        g.loss_index = 0;
        chain.blocks.push_back(g);
        chain.equiv_class.push_back(i);
    }
    return chain;
}

int64_t ops_to_triples(const std::vector<ScheduleOp>& ops, int32_t* out, int64_t cap) {
    int64_t n = 0;
    for (const ScheduleOp& op : ops) {
        if (n >= cap) return -1;
        int32_t k = op.kind == ScheduleOp::Compute ? 0
                    : op.kind == ScheduleOp::Forget ? 1
                    : op.kind == ScheduleOp::BlockFwd ? 2 : 3;
        out[3 * n] = k;
        out[3 * n + 1] = op.block;
        out[3 * n + 2] = (k >= 2) ? op.option : -1;
        ++n;
    }
    return n;
}

size_t tri_row(int L, int s, int t) { return (size_t)s * L - (size_t)s * (s - 1) / 2 + (t - s); }

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_quantize(int64_t budget, int32_t units, int64_t* unit, int64_t* budget_units) {
    try {
        Quantization q = quantize(budget, units);
        *unit = q.unit;
        *budget_units = q.budget_units;
        return 0;
    } catch (const ValidationError& e) {
        g_err = e.what();
        return 1;
    }
}

// Full table in the s-major triangular layout (row tri_row(s,t), column m).
int ref_table_fill(const FlatMenu* f, int64_t unit, int32_t m_max, int64_t* opt, int8_t* kind,
                   int32_t* value, int64_t* max_cands, int64_t* worst_allow) {
    try {
        OptionMenu menu = to_menu(f);
        DpTable table(menu, unit, m_max);
        const int L = table.length();
        for (int s = 0; s < L; ++s)
            for (int t = s; t < L; ++t) {
                size_t r = tri_row(L, s, t) * (size_t)(m_max + 1);
                for (int m = 0; m <= m_max; ++m) {
                    opt[r + m] = table.opt(s, t, m);
                    DpArg a = table.arg(s, t, m);
                    kind[r + m] = (int8_t)a.kind;
                    value[r + m] = a.value;
                }
            }
        if (max_cands) *max_cands = table.max_candidates_per_cell;
        if (worst_allow) *worst_allow = table.worst_cell_allowance;
        return 0;
    } catch (const ValidationError& e) {
        g_err = e.what();
        return 1;
    }
}

// DpTable construction time only (the reference hot path), n_threads
// independent concurrent fills of the same menu.  Returns the wall seconds
// of the slowest thread; *top receives opt(0, L-1, m_max).
double ref_table_bench(const FlatMenu* f, int64_t unit, int32_t m_max, int32_t n_threads,
                       int64_t* top) {
    OptionMenu menu = to_menu(f);
    if (n_threads < 1) n_threads = 1;
    std::vector<double> secs(n_threads, 0.0);
    std::vector<int64_t> tops(n_threads, 0);
    auto work = [&](int i) {
        auto t0 = std::chrono::steady_clock::now();
        DpTable table(menu, unit, m_max);
        auto t1 = std::chrono::steady_clock::now();
        secs[i] = std::chrono::duration<double>(t1 - t0).count();
        tops[i] = table.opt(0, table.length() - 1, m_max);
    };
    if (n_threads == 1) {
        work(0);
    } else {
        std::vector<std::thread> th;
        for (int i = 0; i < n_threads; ++i) th.emplace_back(work, i);
        for (auto& x : th) x.join();
    }
    double worst = 0;
    for (double s : secs) worst = s > worst ? s : worst;
    if (top) *top = tops[0];
    return worst;
}

// remat::solve_chain (DpTable + top cell + build_schedule_rec, chain_dp.hpp:
// 255-296) -- the same work as the device solve -- run n_threads times
// concurrently (one independent solve per host thread; the reference itself
// is single-threaded).  Returns the wall seconds of the slowest thread;
// *opt_time / *n_ops / *m_top describe thread 0's solution (status in *status).
double ref_solve_bench(const FlatMenu* f, int64_t budget, int32_t units, int32_t n_threads,
                       int64_t* opt_time, int64_t* n_ops, int32_t* m_top, int32_t* status) {
    OptionMenu menu = to_menu(f);
    Chain chain = skeleton_chain(menu.length());
    if (n_threads < 1) n_threads = 1;
    std::vector<double> secs(n_threads, 0.0);
    std::vector<int64_t> ot(n_threads, -1), no(n_threads, 0);
    std::vector<int32_t> mt(n_threads, -1), st(n_threads, 0);
    auto work = [&](int i) {
        auto t0 = std::chrono::steady_clock::now();
        try {
            ChainSolution sol = solve_chain(chain, menu, budget, units);
            ot[i] = sol.opt_time;
            no[i] = (int64_t)sol.schedule.ops.size();
            mt[i] = sol.m_top;
        } catch (const InfeasibleBudget&) {
            st[i] = 2;
        } catch (const ValidationError&) {
            st[i] = 1;
        }
        auto t1 = std::chrono::steady_clock::now();
        secs[i] = std::chrono::duration<double>(t1 - t0).count();
    };
    if (n_threads == 1) {
        work(0);
    } else {
        std::vector<std::thread> th;
        for (int i = 0; i < n_threads; ++i) th.emplace_back(work, i);
        for (auto& x : th) x.join();
    }
    double worst = 0;
    for (double s : secs) worst = s > worst ? s : worst;
    if (opt_time) *opt_time = ot[0];
    if (n_ops) *n_ops = no[0];
    if (m_top) *m_top = mt[0];
    if (status) *status = st[0];
    return worst;
}

// One DpTable, then build_schedule_rec from n cells (stm = {s, t, m} triples):
// the whole table (as ref_table_fill) and every walk's ops, concatenated in
// ops (ops_off[i] .. ops_off[i+1]); status[i] = 0 / 2 (InfeasibleBudget).
// Returns 0, 1 (ValidationError) or 5 (ops_cap too small).
int ref_fill_and_walk(const FlatMenu* f, int64_t unit, int32_t m_max, int64_t* opt, int8_t* kind,
                      int32_t* value, int64_t* max_cands, int32_t n, const int32_t* stm,
                      int32_t* status, int32_t* ops, int64_t ops_cap, int64_t* ops_off) {
    try {
        OptionMenu menu = to_menu(f);
        DpTable table(menu, unit, m_max);
        const int L = table.length();
        if (opt)
            for (int s = 0; s < L; ++s)
                for (int t = s; t < L; ++t) {
                    size_t r = tri_row(L, s, t) * (size_t)(m_max + 1);
                    for (int m = 0; m <= m_max; ++m) {
                        opt[r + m] = table.opt(s, t, m);
                        DpArg a = table.arg(s, t, m);
                        kind[r + m] = (int8_t)a.kind;
                        value[r + m] = a.value;
                    }
                }
        if (max_cands) *max_cands = table.max_candidates_per_cell;
        Chain chain = skeleton_chain(L);
        int64_t pos = 0;
        ops_off[0] = 0;
        for (int i = 0; i < n; ++i) {
            std::vector<ScheduleOp> out;
            status[i] = 0;
            try {
                build_schedule_rec(table, menu, chain, stm[3 * i], stm[3 * i + 1], stm[3 * i + 2], out);
            } catch (const InfeasibleBudget&) {
                status[i] = 2;
                out.clear();
            }
            int64_t k = ops_to_triples(out, ops + 3 * pos, ops_cap - pos);
            if (k < 0) return 5;
            pos += k;
            ops_off[i + 1] = pos;
        }
        return 0;
    } catch (const ValidationError& e) {
        g_err = e.what();
        return 1;
    }
}

int ref_build_schedule(const FlatMenu* f, int64_t unit, int32_t m_max, int32_t s, int32_t t,
                       int32_t m, int32_t* ops, int64_t cap, int64_t* n_ops) {
    try {
        OptionMenu menu = to_menu(f);
        DpTable table(menu, unit, m_max);
        Chain chain = skeleton_chain(menu.length());
        std::vector<ScheduleOp> out;
        build_schedule_rec(table, menu, chain, s, t, m, out);
        *n_ops = ops_to_triples(out, ops, cap);
        return *n_ops < 0 ? 5 : 0;
    } catch (const InfeasibleBudget& e) {
        g_err = e.what();
        return 2;
    } catch (const ValidationError& e) {
        g_err = e.what();
        return 1;
    }
}

int ref_solve_chain(const FlatMenu* f, int64_t budget, int32_t units, int32_t* ops, int64_t cap,
                    int64_t* n_ops, int64_t* opt_time, int64_t* unit, int32_t* m_top,
                    int64_t* min_feasible) {
    *n_ops = 0;
    *min_feasible = -1;
    try {
        OptionMenu menu = to_menu(f);
        Chain chain = skeleton_chain(menu.length());
        ChainSolution sol = solve_chain(chain, menu, budget, units);
        *opt_time = sol.opt_time;
        *unit = sol.unit;
        *m_top = sol.m_top;
        *n_ops = ops_to_triples(sol.schedule.ops, ops, cap);
        return *n_ops < 0 ? 5 : 0;
    } catch (const InfeasibleBudget& e) {
        g_err = e.what();
        *min_feasible = e.min_feasible_budget;
        return 2;
    } catch (const ValidationError& e) {
        g_err = e.what();
        return 1;
    }
}

// --- generators and oracles from the reference test helpers ---------------

void* ref_rng_new(uint32_t seed) { return new std::mt19937(seed); }
void ref_rng_free(void* rng) { delete static_cast<std::mt19937*>(rng); }

// Draws one testing::random_menu(rng, max_blocks, max_options) and writes it
// in flat form.  Capacity: blocks <= cap_blocks, options <= cap_options.
// Returns the number of blocks or -1 on overflow.
int32_t ref_random_menu(void* rng, int32_t max_blocks, int32_t max_options, int32_t cap_blocks,
                        int32_t cap_options, int32_t* option_offsets, int32_t* option_id,
                        int64_t* time_fwd, int64_t* time_bwd, uint8_t* has_bwd, int64_t* save_mem,
                        int64_t* peak_fwd, int64_t* peak_fwd_pre, int64_t* peak_bwd,
                        int64_t* act_sizes) {
    OptionMenu menu = testing::random_menu(*static_cast<std::mt19937*>(rng), max_blocks, max_options);
    const int L = menu.length();
    if (L > cap_blocks) return -1;
    int k = 0;
    for (int i = 0; i < L; ++i) {
        option_offsets[i] = k;
        for (const BlockOption& o : menu.options[i]) {
            if (k >= cap_options) return -1;
            option_id[k] = o.option_id;
            time_fwd[k] = o.time_fwd;
            time_bwd[k] = o.time_bwd.value_or(0);
            has_bwd[k] = o.has_bwd() ? 1 : 0;
            save_mem[k] = o.save_mem;
            peak_fwd[k] = o.peak_fwd;
            peak_fwd_pre[k] = o.peak_fwd_pre;
            peak_bwd[k] = o.peak_bwd;
            ++k;
        }
    }
    option_offsets[L] = k;
    for (int i = 0; i <= L; ++i) act_sizes[i] = menu.act_sizes[i];
    return L;
}

int64_t ref_chain_oracle(const FlatMenu* f, int64_t budget_units) {
    return testing::chain_oracle(to_menu(f), budget_units);
}

int64_t ref_chain_oracle_dijkstra(const FlatMenu* f, int64_t budget_units, int32_t fwd_cap) {
    return testing::chain_oracle_dijkstra(to_menu(f), budget_units, fwd_cap);
}

// testing::atomic_replay on schedule-op triples (BlockFwd->Fwd, Compute->Loss,
// BlockBwd->Bwd, Forget->ForgetAct).
int64_t ref_atomic_replay(const FlatMenu* f, const int32_t* ops, int64_t n, int64_t* time_out) {
    std::vector<testing::AtomicOp> seq;
    for (int64_t i = 0; i < n; ++i) {
        testing::AtomicOp a{};
        switch (ops[3 * i]) {
            case 0: a.kind = testing::AtomicOp::Loss; break;
            case 1: a.kind = testing::AtomicOp::ForgetAct; break;
            case 2: a.kind = testing::AtomicOp::Fwd; break;
            default: a.kind = testing::AtomicOp::Bwd; break;
        }
        a.block = ops[3 * i + 1];
        a.option = ops[3 * i + 2];
        seq.push_back(a);
    }
    return testing::atomic_replay(to_menu(f), seq, time_out);
}

}  // extern "C"
