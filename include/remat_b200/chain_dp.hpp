// chain_dp.hpp -- the reference's rk-Rotor C++ API, backed by librkr (sm_100a).
//
// Drop-in for /root/reference/proj/include/remat/chain_dp.hpp: same
// namespace, names and signatures.  Differences a
// caller can observe are limited to:
//   * the table lives in device memory; opt()/arg() are served from a host
//     mirror that is downloaded once, on first access;
//   * build_schedule_rec walks the table on the device (the table's own copy
//     of the menu is used; pass the menu the table was built from, as the
//     reference requires implicitly);
//   * menus whose shifts would make the reference read outside its vectors
//     (save_mem < input size, negative activation sizes) are rejected with
//     ValidationError instead of being undefined behaviour;
//   * device failures raise remat::DeviceError.  There is no CPU fallback.
// Link with -lrkr (paper_2307_01236_b200/librkr.so).
#pragma once

#include <algorithm>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "rkr.h"
#include "remat_b200/errors.hpp"
#include "remat_b200/types.hpp"

namespace remat {

// chain_dp.hpp:16-21
struct OptionMenu {
    std::vector<std::vector<BlockOption>> options;  // per block
    std::vector<Bytes> act_sizes;                   // a_0..a_L, bytes

    int length() const { return static_cast<int>(options.size()); }
};

inline constexpr Micros kInfTime = RKR_INF_TIME;  // chain_dp.hpp:23

struct Quantization {  // chain_dp.hpp:25-28
    Bytes unit = 1;
    Bytes budget_units = 0;
};

namespace detail {

[[noreturn]] inline void raise(rkr_status st, Bytes min_feasible = -1) {
    std::string msg = rkr_last_error();
    switch (st) {
        case RKR_ERR_INVALID: throw ValidationError(msg);
        case RKR_ERR_INFEASIBLE: throw InfeasibleBudget(msg, min_feasible);
        case RKR_ERR_ARGUMENT: throw std::out_of_range(msg);
        default: throw DeviceError(msg);
    }
}

inline void check(rkr_status st) {
    if (st != RKR_OK) raise(st);
}

// OptionMenu -> rkr_menu (CSR); owns the flat arrays.
struct FlatMenu {
    std::vector<int32_t> offsets, ids;
    std::vector<int64_t> tf, tb, save, pf, pre, pb, act;
    std::vector<uint8_t> hb;
    rkr_menu view{};

    explicit FlatMenu(const OptionMenu& m) {
        offsets.push_back(0);
        for (const auto& blk : m.options) {
            for (const BlockOption& o : blk) {
                ids.push_back(o.option_id);
                tf.push_back(o.time_fwd);
                tb.push_back(o.time_bwd.value_or(0));
                hb.push_back(o.has_bwd() ? 1 : 0);
                save.push_back(o.save_mem);
                pf.push_back(o.peak_fwd);
                pre.push_back(o.peak_fwd_pre);
                pb.push_back(o.peak_bwd);
            }
            offsets.push_back(static_cast<int32_t>(ids.size()));
        }
        act = m.act_sizes;
        // act_sizes must cover a_0..a_L; the reference indexes it unchecked
        if (act.size() < m.options.size() + 1) act.resize(m.options.size() + 1, 0);
        view.n_blocks = m.length();
        view.option_offsets = offsets.data();
        view.option_id = ids.data();
        view.time_fwd = tf.data();
        view.time_bwd = tb.data();
        view.has_bwd = hb.data();
        view.save_mem = save.data();
        view.peak_fwd = pf.data();
        view.peak_fwd_pre = pre.data();
        view.peak_bwd = pb.data();
        view.act_sizes = act.data();
    }
};

}  // namespace detail

// chain_dp.hpp:32-39
inline Quantization quantize(Bytes budget_bytes, int units) {
    Quantization q;
    detail::check(rkr_quantize(budget_bytes, units, &q.unit, &q.budget_units));
    return q;
}

// chain_dp.hpp:41
inline Bytes to_units(Bytes bytes, Bytes unit) { return rkr_to_units(bytes, unit); }

// chain_dp.hpp:44-47
struct DpArg {
    enum Kind : std::uint8_t { None, Option, Cut } kind = None;
    int value = -1;
};

// Device execution knobs (no reference equivalent; defaults = device 0, auto width).
struct ExecConfig {
    int device = 0;
    void* stream = nullptr;
    bool force_int64 = false;
    int kernel = RKR_KERNEL_PERSISTENT;  // or _TILES, _QUEUE, _DIAGONAL (include/rkr.h)
};

// chain_dp.hpp:54-196.  Construction fills every cell on the GPU.
class DpTable {
    struct Del {
        bool owns;
        Del() noexcept : owns(true) {}
        explicit Del(bool o) noexcept : owns(o) {}
        void operator()(rkr_table* t) const {
            if (owns) rkr_table_destroy(t);
        }
    };

public:
    DpTable(const OptionMenu& menu, Bytes unit, int m_max, const ExecConfig& cfg = {}) {
        detail::FlatMenu flat(menu);
        rkr_exec ex{};
        ex.device = cfg.device;
        ex.stream = cfg.stream;
        ex.width = cfg.force_int64 ? RKR_WIDTH_64 : RKR_WIDTH_AUTO;
        ex.kernel = cfg.kernel;
        rkr_table* h = nullptr;
        detail::check(rkr_table_create(&flat.view, unit, m_max, &ex, &h));
        h_.reset(h);
        L_ = rkr_table_length(h);
        m_max_ = m_max;
        unit_ = unit;
        detail::check(rkr_table_work_bound(h, &max_candidates_per_cell, &worst_cell_allowance));
    }

    Micros opt(int s, int t, int m) const {
        if (m < 0) return kInfTime;
        if (m > m_max_) m = m_max_;
        mirror();
        return opt_[cell(s, t) * (m_max_ + 1) + m];
    }
    DpArg arg(int s, int t, int m) const {
        if (m < 0) return {};
        if (m > m_max_) m = m_max_;
        mirror();
        const size_t i = cell(s, t) * (m_max_ + 1) + m;
        return {static_cast<DpArg::Kind>(kind_[i]), value_[i]};
    }
    int length() const { return L_; }
    Bytes unit() const { return unit_; }
    int m_max() const { return m_max_; }
    Bytes act_units(int i) const { return rkr_table_act_units(h_.get(), i); }

    // instrumentation for the per-cell work bound (t-s) + B + 1 (chain_dp.hpp:118-120)
    long max_candidates_per_cell = 0;
    long worst_cell_allowance = 0;

    // the device table, for callers that want the C ABI directly
    rkr_table* device_handle() const { return h_.get(); }

    // A non-owning view of a table that lives in a batch (b200::Batch).
    static DpTable borrow(rkr_table* h) {
        DpTable t;
        t.h_ = std::unique_ptr<rkr_table, Del>(h, Del{false});
        t.L_ = rkr_table_length(h);
        t.m_max_ = rkr_table_m_max(h);
        t.unit_ = rkr_table_unit(h);
        detail::check(rkr_table_work_bound(h, &t.max_candidates_per_cell, &t.worst_cell_allowance));
        return t;
    }

private:
    DpTable() = default;
    size_t cell(int s, int t) const {
        if (s < 0 || t < s || t >= L_) throw std::out_of_range("DpTable cell outside s <= t < L");
        return static_cast<size_t>(s) * L_ - static_cast<size_t>(s) * (s - 1) / 2 + (t - s);
    }
    void mirror() const {
        if (!opt_.empty()) return;
        const size_t n = static_cast<size_t>(L_) * (L_ + 1) / 2 * (m_max_ + 1);
        opt_.resize(n);
        kind_.resize(n);
        value_.resize(n);
        detail::check(rkr_table_download(h_.get(), opt_.data(), kind_.data(), value_.data()));
    }

    std::unique_ptr<rkr_table, Del> h_;
    int L_ = 0;
    int m_max_ = 0;
    Bytes unit_ = 1;
    mutable std::vector<int64_t> opt_;
    mutable std::vector<int8_t> kind_;
    mutable std::vector<int32_t> value_;
};

namespace detail {

inline void append_ops(const std::vector<rkr_op>& raw, int64_t n, const Chain& chain,
                       std::vector<ScheduleOp>& out) {
    for (int64_t i = 0; i < n; ++i) {
        const rkr_op& o = raw[i];
        switch (o.kind) {
            case RKR_OP_COMPUTE: {
                const CDGraph& g = chain.blocks[o.block];
                out.push_back(ScheduleOp::compute(o.block, g.cnodes[g.loss_index].id));
                break;
            }
            case RKR_OP_FORGET: {
                const CDGraph& g = chain.blocks[o.block];
                out.push_back(ScheduleOp::forget(o.block, g.dnodes[g.input_data].id));
                break;
            }
            case RKR_OP_BLOCK_FWD: out.push_back(ScheduleOp::block_fwd(o.block, o.option)); break;
            default: out.push_back(ScheduleOp::block_bwd(o.block, o.option)); break;
        }
    }
}

}  // namespace detail

// chain_dp.hpp:211-246, walked on the device; only the ops come back.
inline void build_schedule_rec(const DpTable& table, const OptionMenu& /*menu*/, const Chain& chain,
                               int s, int t, int m, std::vector<ScheduleOp>& out) {
    std::vector<rkr_op> raw(1024);
    int64_t n = 0;
    rkr_status st;
    for (;;) {
        st = rkr_backtrack(table.device_handle(), s, t, m, raw.data(),
                           static_cast<int64_t>(raw.size()), &n);
        if (st != RKR_ERR_CAPACITY) break;
        raw.resize(static_cast<size_t>(n));
    }
    if (st == RKR_OK || st == RKR_ERR_INFEASIBLE)
        detail::append_ops(raw, std::min<int64_t>(n, static_cast<int64_t>(raw.size())), chain, out);
    detail::check(st);
}

// chain_dp.hpp:248-253
struct ChainSolution {
    Schedule schedule;
    Micros opt_time = 0;
    Bytes unit = 1;
    int m_top = 0;
};

// chain_dp.hpp:255-296 in one device-side call.
inline ChainSolution solve_chain(const Chain& chain, const OptionMenu& menu, Bytes budget_bytes,
                                 int units, const ExecConfig& cfg = {}) {
    detail::FlatMenu flat(menu);
    rkr_exec ex{};
    ex.device = cfg.device;
    ex.stream = cfg.stream;
    ex.width = cfg.force_int64 ? RKR_WIDTH_64 : RKR_WIDTH_AUTO;
    ex.kernel = cfg.kernel;
    std::vector<rkr_op> raw(4096);
    int64_t n = 0, opt_time = 0, unit = 1, min_feasible = -1;
    int32_t m_top = 0;
    rkr_status st;
    for (;;) {
        st = rkr_solve_chain(&flat.view, budget_bytes, units, &ex, raw.data(),
                             static_cast<int64_t>(raw.size()), &n, &opt_time, &unit, &m_top,
                             &min_feasible);
        if (st != RKR_ERR_CAPACITY) break;
        raw.resize(static_cast<size_t>(n));
    }
    if (st != RKR_OK) detail::raise(st, min_feasible);
    ChainSolution sol;
    sol.opt_time = opt_time;
    sol.unit = unit;
    sol.m_top = m_top;
    detail::append_ops(raw, n, chain, sol.schedule.ops);
    return sol;
}


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
        rkr_exec ex{};
        ex.device = cfg.device;
        ex.stream = cfg.stream;
        ex.width = cfg.force_int64 ? RKR_WIDTH_64 : RKR_WIDTH_AUTO;
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
    rkr_exec ex{};
    ex.device = cfg.device;
    ex.stream = cfg.stream;
    ex.width = cfg.force_int64 ? RKR_WIDTH_64 : RKR_WIDTH_AUTO;
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
        rkr_exec ex{};
        ex.device = cfg.device;
        ex.width = cfg.force_int64 ? RKR_WIDTH_64 : RKR_WIDTH_AUTO;
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
