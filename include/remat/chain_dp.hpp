// remat/chain_dp.hpp -- drop-in replacement for the reference's header of the
// same path (/root/reference/proj/include/remat/chain_dp.hpp), backed by
// librkr (sm_100a).  Same namespace, names, signatures and exceptions
// (SURVEY.md section 8(b)); the DP fill and the schedule walk run on the GPU.
//
// Switching: put this repo's include/ directory BEFORE the reference's on the
// include path and link -lrkr.  Every `#include "remat/chain_dp.hpp"` -- the
// caller's, pipeline.hpp's (:10), the reference tests' -- then resolves here,
// while remat/types.hpp and remat/errors.hpp still resolve to the
// reference's own (this directory does not shadow them), so Chain,
// BlockOption, ScheduleOp, ValidationError, InfeasibleBudget ... are the
// caller's types, not copies.  Without the reference tree on the path the
// standalone vocabulary in remat_b200/ is used instead (same members).
//
// Differences a caller can observe:
//   * opt()/arg() read the device table one row at a time (each row is
//     copied on its first access and cached);
//   * menus whose shifts would make the reference read outside its vectors
//     (save_mem < input size, negative activation sizes) are rejected with
//     ValidationError instead of being undefined behaviour;
//   * device failures raise remat::DeviceError.  There is no CPU fallback.
#pragma once

#include <algorithm>
#include <cstdint>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <utility>
#include <vector>

#if __has_include("remat/types.hpp")
#include "remat/errors.hpp"
#include "remat/types.hpp"
#else
#include "remat_b200/errors.hpp"
#include "remat_b200/types.hpp"
#endif
#include "remat_b200/device_error.hpp"
#include "rkr.h"

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

// Device execution knobs (no reference equivalent; defaults = device 0, auto
// width, the library's measured kernel choices).
struct ExecConfig {
    int device = 0;
    void* stream = nullptr;
    bool force_int64 = false;
    int kernel = RKR_KERNEL_PERSISTENT;  // or _TILES, _QUEUE, _DIAGONAL (include/rkr.h)
    int tune = 0;                        // rkr_tune bits (A/B only)
    int tile_rows = 0;

    rkr_exec to_exec() const {
        rkr_exec ex{};
        ex.device = device;
        ex.stream = stream;
        ex.width = force_int64 ? RKR_WIDTH_64 : RKR_WIDTH_AUTO;
        ex.kernel = kernel;
        ex.tune = tune;
        ex.tile_rows = tile_rows;
        return ex;
    }
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
    struct Row {
        std::vector<int64_t> opt;
        std::vector<int8_t> kind;
        std::vector<int32_t> value;
    };

public:
    DpTable(const OptionMenu& menu, Bytes unit, int m_max, const ExecConfig& cfg = {}) {
        detail::FlatMenu flat(menu);
        const rkr_exec ex = cfg.to_exec();
        rkr_table* h = nullptr;
        detail::check(rkr_table_create(&flat.view, unit, m_max, &ex, &h));
        h_.reset(h);
        L_ = rkr_table_length(h);
        m_max_ = m_max;
        unit_ = unit;
        detail::check(rkr_table_work_bound(h, &max_candidates_per_cell, &worst_cell_allowance));
    }
    DpTable(DpTable&& o) noexcept
        : max_candidates_per_cell(o.max_candidates_per_cell),
          worst_cell_allowance(o.worst_cell_allowance),
          h_(std::move(o.h_)),
          L_(o.L_),
          m_max_(o.m_max_),
          unit_(o.unit_),
          rows_(std::move(o.rows_)) {}

    // chain_dp.hpp:103-112: m < 0 -> kInfTime / {None, -1}; m > m_max clamps.
    Micros opt(int s, int t, int m) const {
        if (m < 0) return kInfTime;
        if (m > m_max_) m = m_max_;
        return row(s, t).opt[m];
    }
    DpArg arg(int s, int t, int m) const {
        if (m < 0) return {};
        if (m > m_max_) m = m_max_;
        const Row& r = row(s, t);
        return {static_cast<DpArg::Kind>(r.kind[m]), r.value[m]};
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
    // One row (s, t), m = 0..m_max, copied from the device on first access.
    // Guarded: const reads of one table from several threads stay safe, as
    // the reference's immutable DpTable is.
    const Row& row(int s, int t) const {
        if (s < 0 || t < s || t >= L_) throw std::out_of_range("DpTable cell outside s <= t < L");
        const int64_t key = static_cast<int64_t>(s) * L_ + t;
        std::lock_guard<std::mutex> g(*mu_);
        auto it = rows_.find(key);
        if (it != rows_.end()) return it->second;
        Row r;
        r.opt.resize(static_cast<size_t>(m_max_) + 1);
        r.kind.resize(r.opt.size());
        r.value.resize(r.opt.size());
        detail::check(rkr_table_row(h_.get(), s, t, r.opt.data(), r.kind.data(), r.value.data()));
        return rows_.emplace(key, std::move(r)).first->second;
    }

    std::unique_ptr<rkr_table, Del> h_;
    int L_ = 0;
    int m_max_ = 0;
    Bytes unit_ = 1;
    mutable std::unique_ptr<std::mutex> mu_ = std::make_unique<std::mutex>();
    mutable std::unordered_map<int64_t, Row> rows_;
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

// chain_dp.hpp:211-246, walked on the device; only the ops come back.  The
// decisions come from the table, the option lookups and pack shifts from the
// caller's `menu` (detail::menu_option, :200-205, :228), as in the reference;
// on a throw, `out` holds the ops emitted before it.
inline void build_schedule_rec(const DpTable& table, const OptionMenu& menu, const Chain& chain,
                               int s, int t, int m, std::vector<ScheduleOp>& out) {
    detail::FlatMenu flat(menu);
    std::vector<rkr_op> raw(1024);
    int64_t n = 0;
    rkr_status st;
    for (;;) {
        st = rkr_backtrack_menu(table.device_handle(), &flat.view, s, t, m, raw.data(),
                                static_cast<int64_t>(raw.size()), &n);
        if (st != RKR_ERR_CAPACITY) break;
        raw.resize(static_cast<size_t>(n));
    }
    if (st == RKR_OK || st == RKR_ERR_INFEASIBLE || st == RKR_ERR_INVALID)
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
    const rkr_exec ex = cfg.to_exec();
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

}  // namespace remat
