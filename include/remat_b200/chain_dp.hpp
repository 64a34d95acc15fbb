// remat_b200/chain_dp.hpp -- the reference's rk-Rotor C++ API
// (include/remat/chain_dp.hpp, the drop-in) plus the B200 extensions that
// have no reference counterpart: batched fills, the device budget sweep
// (cmd_sweep, tools/remat.cpp:217-263) and budget-axis sharding.
// Link with -lrkr (paper_2307_01236_b200/librkr.so).
#pragma once

#include <algorithm>
#include <memory>
#include <stdexcept>
#include <vector>

#include "remat/chain_dp.hpp"

namespace remat {

// ---------------------------------------------------------------------------
// B200 extensions (no reference counterpart): batched fills, the device
// budget sweep (cmd_sweep, tools/remat.cpp:217-263), budget-axis sharding.
// ---------------------------------------------------------------------------
namespace b200 {

// Many independent tables filled by ONE persistent launch.
class Batch {
public:
    Batch(const std::vector<OptionMenu>& menus, const std::vector<Bytes>& units,
          const std::vector<int>& m_max, const ExecConfig& cfg = {}) {
        std::vector<detail::FlatMenu> flats;
        flats.reserve(menus.size());
        for (const OptionMenu& m : menus) flats.emplace_back(m);
        std::vector<const rkr_menu*> views;
        for (const auto& f : flats) views.push_back(&f.view);
        std::vector<int64_t> u(units.begin(), units.end());
        std::vector<int32_t> mm(m_max.begin(), m_max.end());
        rkr_exec ex = cfg.to_exec();
        rkr_batch* b = nullptr;
        detail::check(rkr_batch_create(views.data(), u.data(), mm.data(),
                                       static_cast<int32_t>(views.size()), &ex, &b));
        b_.reset(b);
    }
    int size() const { return rkr_batch_size(b_.get()); }
    DpTable table(int i) const { return DpTable::borrow(rkr_batch_table(b_.get(), i)); }
    void refill() { detail::check(rkr_batch_refill(b_.get())); }

private:
    struct Del {
        void operator()(rkr_batch* b) const { rkr_batch_destroy(b); }
    };
    std::unique_ptr<rkr_batch, Del> b_;
};

struct SweepRow {
    Bytes budget = 0;
    bool feasible = false;
    Micros opt_time = 0;
    Bytes unit = 1;
    int m_top = 0;
    Bytes min_feasible = -1;
    Schedule schedule;
};

// cmd_sweep's loop: budgets sorted and de-duplicated, every solve_chain on
// the device in batched calls, then the monotonicity check.
inline std::vector<SweepRow> sweep(const Chain& chain, const OptionMenu& menu,
                                   std::vector<Bytes> budgets, int units,
                                   const ExecConfig& cfg = {}) {
    std::sort(budgets.begin(), budgets.end());
    budgets.erase(std::unique(budgets.begin(), budgets.end()), budgets.end());
    const int32_t n = static_cast<int32_t>(budgets.size());
    if (n == 0) return {};
    detail::FlatMenu flat(menu);
    const rkr_exec ex = cfg.to_exec();
    std::vector<int32_t> status(n), mtop(n);
    std::vector<int64_t> opt(n), unit(n), minf(n), offs(n + 1);
    std::vector<rkr_op> ops(4096);
    rkr_status st;
    for (;;) {
        st = rkr_sweep(&flat.view, budgets.data(), n, units, &ex, status.data(), opt.data(),
                       unit.data(), mtop.data(), minf.data(), ops.data(),
                       static_cast<int64_t>(ops.size()), offs.data());
        if (st == RKR_ERR_CAPACITY && offs[n] > static_cast<int64_t>(ops.size())) {
            ops.resize(static_cast<size_t>(offs[n]));
            continue;
        }
        break;
    }
    detail::check(st);
    std::vector<SweepRow> rows(n);
    Micros prev = kInfTime;
    for (int32_t i = 0; i < n; ++i) {
        SweepRow& r = rows[i];
        r.budget = budgets[i];
        r.feasible = status[i] == RKR_OK;
        r.unit = unit[i];
        r.min_feasible = minf[i];
        if (!r.feasible) continue;
        r.opt_time = opt[i];
        r.m_top = mtop[i];
        std::vector<rkr_op> mine(ops.begin() + offs[i], ops.begin() + offs[i + 1]);
        detail::append_ops(mine, static_cast<int64_t>(mine.size()), chain, r.schedule.ops);
        // optimality implies the makespan curve never rises with budget (remat.cpp:256-263)
        if (r.opt_time > prev) throw std::logic_error("sweep makespan increased with budget");
        prev = r.opt_time;
    }
    return rows;
}

// One table split along the budget axis across devices (config 5).
class ShardedTable {
public:
    ShardedTable(const OptionMenu& menu, Bytes unit, int m_max, int n_shards,
                 const std::vector<int>& devices = {}, const ExecConfig& cfg = {}) {
        detail::FlatMenu flat(menu);
        rkr_exec ex = cfg.to_exec();
        ex.stream = nullptr;  // per-device library streams
        std::vector<int32_t> dv(devices.begin(), devices.end());
        rkr_sharded* h = nullptr;
        detail::check(rkr_sharded_create(&flat.view, unit, m_max, n_shards,
                                         dv.empty() ? nullptr : dv.data(), &ex, &h));
        h_.reset(h);
        L_ = menu.length();
        m_max_ = m_max;
    }
    Micros opt(int s, int t, int m) const {
        int64_t v = 0;
        detail::check(rkr_sharded_opt(h_.get(), s, t, m, &v));
        return v;
    }
    void build_schedule(const Chain& chain, int s, int t, int m, std::vector<ScheduleOp>& out) {
        std::vector<rkr_op> raw(4096);
        int64_t n = 0;
        rkr_status st;
        for (;;) {
            st = rkr_sharded_backtrack(h_.get(), s, t, m, raw.data(),
                                       static_cast<int64_t>(raw.size()), &n);
            if (st != RKR_ERR_CAPACITY) break;
            raw.resize(static_cast<size_t>(n));
        }
        if (st == RKR_OK || st == RKR_ERR_INFEASIBLE)
            detail::append_ops(raw, std::min<int64_t>(n, static_cast<int64_t>(raw.size())), chain, out);
        detail::check(st);
    }
    int shards() const { return rkr_sharded_count(h_.get()); }

private:
    struct Del {
        void operator()(rkr_sharded* h) const { rkr_sharded_destroy(h); }
    };
    std::unique_ptr<rkr_sharded, Del> h_;
    int L_ = 0, m_max_ = 0;
};

}  // namespace b200

}  // namespace remat
