// rkr_internal.h -- device-side table layout shared by the kernels and the
// host half of librkr.so.  Not installed; include/rkr.h is the public ABI.
#pragma once

#include <cstdint>

namespace rkr {

// Cost infinities.  The 64-bit path keeps the reference's sentinel
// (remat::kInfTime, chain_dp.hpp:23).  The 32-bit path stores costs as
// uint32 with INF32 = 2^30; it is only selected when the host proves every
// finite candidate total is < 2^30, so
// sum-of-three-operands never wraps and "total < INF32" <=> all operands finite.
constexpr int64_t kInf64 = INT64_MAX / 4;
constexpr uint32_t kInf32 = 1u << 30;

// Arg codes (uint16, 0 = none).  Saved option oi (menu order) -> oi + 1;
// cut c -> 0x8000 | c.  Numeric order == the reference's candidate order
// (options in menu order, then cuts ascending, chain_dp.hpp:139-174).
constexpr uint16_t kCutBit = 0x8000;

// Per-table menu data in units (the DpTable ctor precompute, chain_dp.hpp:56-95),
// device resident.  Saved options of block s: [blk_off[s], blk_off[s+1]).
struct DevMenu {
    const int32_t* blk_off;      // [L+1]
    const int64_t* fwd_req;      // per saved option
    const int64_t* fwd_req_pre;
    const int64_t* bwd_req;
    const int64_t* pack_chg;     // >= 0 (validated)
    const int64_t* tftb;         // time_fwd + time_bwd
    const int64_t* chg_bt;       // build_schedule_rec's chg (chain_dp.hpp:228)
    const int32_t* ids;          // option ids
    const int64_t* act_u;        // [L+1]
    const int64_t* fwd0_own;     // [L]
    const int64_t* fwd0_full;    // [L]
    const int64_t* tf0;          // [L]
};

// Table geometry.  Rows are stored diagonal-major: row id of (s, t) is
// off(k) + s with k = t - s and off(k) = k*L - k(k-1)/2.  Each opt row holds
// PAD infinity slots and then m = 0..M, padded to a multiple of 32 elements
// (row stride SR).  Arg rows are uint16, stride SA, no pad.
struct Geometry {
    int32_t L;
    int32_t M;
    int32_t pad;       // >= every clamped shift (pack_chg, act_u), <= M + 1
    int64_t sr;        // opt row stride (elements)
    int64_t sa;        // arg row stride (elements)
    int64_t rows;      // L(L+1)/2
};

__host__ __device__ inline int64_t diag_off(int32_t L, int32_t k) {
    return (int64_t)k * L - (int64_t)k * (k - 1) / 2;
}
__host__ __device__ inline int64_t row_id(int32_t L, int32_t s, int32_t t) {
    return diag_off(L, t - s) + s;
}

// Launch entry points (rkr_kernels.cu).
struct LaunchCtx {
    Geometry g;
    DevMenu dm;
    void* opt;          // uint32_t* (width 32) or int64_t* (width 64)
    uint16_t* arg;
    int32_t width;      // 32 or 64
    int32_t max_opts;   // max saved options per block
    void* stream;       // cudaStream_t
    int32_t kernel;     // 0 = persistent dataflow fill (K1p), 1 = one launch per diagonal (K1)
    void* sched;        // K1p scheduler state: counter + per-(diagonal, tile) done flags
    size_t sched_bytes;
};

// K1p (rkr_persist.cu)
size_t persistent_sched_bytes(const Geometry& g);
int launch_fill_persistent(const LaunchCtx& c);
constexpr int64_t kOptSlack = 4096;  // elements past the last row (tile over-reads)

int launch_init_pads(const LaunchCtx& c);
int launch_fill_all(const LaunchCtx& c);
// backtrack: ops as int32 triples; dev_out = {n_ops (int64), status (int64), bad_s, bad_t}
int launch_backtrack(const LaunchCtx& c, int32_t s, int32_t t, int32_t m, int32_t* dev_ops,
                     int64_t cap, int32_t* dev_stack, int64_t* dev_out);
int launch_first_feasible(const LaunchCtx& c, int32_t s, int32_t t, int32_t* dev_m);
// export rows [r0, r1) of the s-major triangular order to reference-layout buffers
int launch_export(const LaunchCtx& c, int64_t r0, int64_t r1, int64_t* opt, int8_t* kind,
                  int32_t* value);

}  // namespace rkr
