// rkr_internal.h -- device-side table layout shared by the kernels and the
// host half of librkr.so.  Not installed; include/rkr.h is the public ABI.
#pragma once

#include <cuda_runtime.h>

#include <climits>
#include <cstdint>
#include <mutex>
#include <unordered_map>
#include <vector>

#include "../../include/rkr.h"

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

// A walk with the CALLER's menu (rkr_backtrack_menu) marks the table's saved
// options that the caller's menu lacks with this pack shift: the reference's
// detail::menu_option throws ValidationError at them (chain_dp.hpp:200-205),
// before it emits anything for the cell.  A table's own shifts are >= 0.
constexpr int32_t kMissingShift = INT32_MIN;

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
    int32_t M;         // last LOCAL budget slot (a shard holds global m_base .. m_base + M)
    int32_t pad;       // >= every clamped shift (pack_chg, act_u), <= global M + 1
    int64_t sr;        // opt row stride (elements)
    int64_t sa;        // arg row stride (elements)
    int64_t rows;      // L(L+1)/2
    int32_t m_base;    // global budget slot of local slot 0 (0 unless budget-sharded)
};

__host__ __device__ inline int64_t diag_off(int32_t L, int32_t k) {
    return (int64_t)k * L - (int64_t)k * (k - 1) / 2;
}
__host__ __device__ inline int64_t row_id(int32_t L, int32_t s, int32_t t) {
    return diag_off(L, t - s) + s;
}
// First cell-program cut entry of diagonal k: sum_{k' < k} (L - k') k'.
// Cell (s, s + k) owns entries [diag_cut_off(L, k) + s * k, + k).
__host__ __device__ inline int64_t diag_cut_off(int64_t L, int64_t k) {
    return L * k * (k - 1) / 2 - (k - 1) * k * (2 * k - 1) / 6;
}

// K1p schedule (rkr_persist.cu).  Work items are (column group g, diagonal k,
// tile j in the group, s).  Groups are GW = 1 tile wide; their diagonal
// sweeps are interleaved with a lag of `lambda` diagonals (item order key
// tau = lambda * g + k), so about L / lambda groups are in flight: enough
// items to fill the GPU, few enough that their rows stay in L2.
struct PersistPlan {
    int32_t R = 1, TM = 256, J = 1, dj = 0, lambda = 1;
    int32_t j_offset = 0;        // global tile index of local tile 0 (sharded tables)
    int64_t total = 0;
    std::vector<int64_t> start;  // first item index of each (g, k) plan entry, in key order
    std::vector<int32_t> g, k;   // the entry's group and diagonal
};
struct PlanDev {
    int32_t R, TM, J, dj, n_plan;
    int64_t total;
    const int64_t* start;
    const int32_t* g;
    const int32_t* k;
    int32_t* done;                   // [L * J] rows completed per (diagonal, tile)
    unsigned long long* counter;     // unused (the launch owns the item counter)
    unsigned long long* trace;       // optional: 6 globaltimer stamps per item (nullptr = off)
};
// Per-table cell programs (K1p), filled by launch_prep_programs.
struct ProgDev {
    void* ptr;        // longlong2 [cut entries]
    void* sweep;      // V [cut entries]
    int32_t* gate;    // [cut entries]
    int32_t* thr;     // [rows * max_opts]
    int32_t* pc;      // [saved options]
    void* otot;       // V [saved options]
    int64_t nq;
    int32_t ocap;     // row stride of thr (the table's max saved options, >= 1; K1t: rounded to 4)
    int32_t tiles;    // 1: ptr holds K1t cut programs, int4 {off_l, off_r, sweep, gate}
};
int64_t program_cut_entries(const Geometry& g);

// One table of a (possibly batched) persistent fill, as the kernel sees it.
struct InstDesc {
    Geometry g;
    DevMenu dm;
    void* opt;
    uint16_t* arg;
    PlanDev plan;
    ProgDev prog;
    void* stack;        // backtrack stack (int4[2L + 16])
    int64_t item_base;  // unused by the kernel (kept for diagnostics)
    // Budget-axis sharding (config 5).  This shard's local slots [M+1-pad, M]
    // are the halo of the next shard (slots [-pad, 0) of its rows): the item
    // that computes them also stores them there (next_opt may be peer memory)
    // and counts them in next_halo[k].  halo_need > 0: items whose reads
    // reach below local slot 0 also wait for halo[k-1] >= (L-k+1) * halo_need.
    void* next_opt;
    int64_t next_sr;
    int32_t* next_halo;
    int32_t* halo;
    int32_t halo_need;
    int32_t next_peer;  // 1: next shard lives on another GPU (system-scope fences)
    // Walk mirror (process shards): every tile also stores its arg codes into
    // shard 0's full-width copy (peer memory), so the walk runs on one GPU
    // with local reads instead of one NVLink round trip per hop.
    uint16_t* arg_mirror;
    int64_t mirror_sa;
    int32_t mirror_base;  // global slot of this shard's local slot 0
};
// The launch-wide item order: entry e covers items [start[e], start[e] +
// L_inst - k[e]) = rows s = 0.. of (instance inst[e], diagonal k[e], tile
// j[e]).  Entries are sorted by (lambda_inst * j + k, inst, j), so tables of
// a batch advance their wavefronts together and every item only waits on
// items of smaller index.
struct LaunchPlan {
    const int64_t* start;
    const int32_t* inst;
    const int32_t* k;
    const int32_t* j;
    int32_t n;
    int64_t total;
};
// Host side: merge per-table plans into one launch order.
struct HostLaunchPlan {
    std::vector<int64_t> start;
    std::vector<int32_t> inst, k, j;
    int64_t total = 0;
};
void merge_plans(const std::vector<const PersistPlan*>& plans, const std::vector<int32_t>& L,
                 HostLaunchPlan& out);
int launch_batch_walk(const InstDesc* d, const int32_t* m_at, const uint8_t* active, int n,
                      int width, int32_t* ops, int64_t cap, int64_t* out, void* stream);
// A budget shard as the cross-shard walk reads it.
struct ShardView {
    const void* opt;
    const uint16_t* arg;
    int64_t sr, sa;
    int32_t pad, lo;   // local slot 0 = global slot lo
};
int launch_walk_sharded(const ShardView* sv, int n, const DevMenu& dm, int L, int M, int width,
                        int s, int t, int m, int32_t* ops, int64_t cap, int32_t* stack,
                        int64_t* out, void* stream);
int launch_batch_tops(const InstDesc* d, const int32_t* m_at, int n, int width, int64_t* out,
                      void* stream);
int launch_batch_first_feasible(const InstDesc* d, int n, int width, int32_t* out, void* stream);
// min-feasible thresholds thr(0, L-1) of the tables d[which[i]] (rkr_kernels.cu);
// scratch + scr_off[i]: L(L+1)/2 int64 per instance
int launch_batch_thresholds(const InstDesc* d, const int32_t* which, int n, int64_t* scratch,
                            const int64_t* scr_off, int64_t* out, void* stream);
// Fill n tables with ONE persistent launch.  All tables share the cost
// width and the plan's R.  The counter and every table's done flags must be
// zeroed on `stream` before the call (they are, by the callers in rkr_table.cu / rkr_batch.cu).
// single != nullptr: a one-table launch whose descriptor is passed by value.
int launch_fill_batch(const InstDesc* dev_desc, const InstDesc* single, const LaunchPlan& lp,
                      int width, int R, int kcap, int ocap, unsigned long long* counter,
                      void* stream);
void persistent_plan(const Geometry& g, int width, int R, PersistPlan& p);
int persistent_choose_r(int32_t M);
size_t persistent_state_bytes(const Geometry& g, const PersistPlan& p);  // counter + flags

// K1t schedule (rkr_tiles.cu): CTA j owns budget slots [jW, (j+1)W) of every
// row; done[k * T + j] != 0 once diagonal k of tile j is stored.
// K1t reads option thresholds and (shift, pass time) pairs in whole batches
// of kTileOptBatch: thr rows and option slots are padded to a multiple.
constexpr int kTileOptBatch = 8;  // the smallest K1t option batch (tile_plan pads to its kernel's batch)
struct TileSmem {  // shared-memory carve-up of K1t (byte offsets)
    uint32_t best, code, blk, split, thx, opd, pru, prog, thr, xch, bar, total;
    uint32_t prog_bytes, thr_bytes;  // one buffer of each (two of each are kept)
};
struct TilePlan {
    int32_t rpw = 0, W = 0, T = 0, d = 0;  // rows per warp; W = 32 / rpw; d = lower tiles read (ceil(pad / W))
    int32_t cap = 0;                      // bulk partials (values + codes) in shared memory
    int32_t L = 0, nq = 0, ocap = 0;      // blocks, saved options, thr row stride
    TileSmem sm{};
    int32_t comm = 0;                     // 1: a dedicated communication warp (latency-bound tables)
    int32_t jobs = 0;                     // 1: more tiles than SMs: run as tile jobs (one-table batch)
    int32_t split = 0;                    // 1 (with comm): late diagonals split each tail over 2 warps
    int32_t stream = 0;                   // 1: programs / thresholds / options read from global (long chains)
    int32_t halo = 0;                     // 1: a budget shard (halo wait / push compiled in; comm, no split)
    int32_t prune = 0;                    // 1: open rows scan each block's undominated options only
    // mixed tile widths (single tables as tile jobs): tiles j >= j1 are
    // 16-slot (two rows per warp) tiles after j1 32-slot ones, so the last
    // wave of jobs is made of half jobs
    int32_t j1 = INT32_MAX;
    // fused K2 (per launch): the last CTA walks from (ws, wt, wm) into wops /
    // wout = {n_ops, status, bad_s, bad_t, top} (rkr_walk.cuh)
    int32_t walk = 0, ws = 0, wt = 0, wm = 0;
    int32_t* wops = nullptr;
    int64_t wcap = 0;
    int64_t* wout = nullptr;
    int4* wstack = nullptr;
    int* fin = nullptr;                   // CTAs finished (zeroed with the flags)
    int32_t* done = nullptr;              // [L * T]
    unsigned long long* trace = nullptr;  // optional: 6 stamps per (k, j)
};
// The rkr_exec tuning fields a plan honours (include/rkr.h; 0 = defaults).
struct TileKnobs {
    int32_t tune = 0;  // rkr_tune bits
    int32_t rows = 0;  // K1t rows per warp: 0 auto, 1 or 2
    bool mixed = false;  // a plain single table: may end its tile jobs with half tiles
};
// 1 = eligible.  Long chains, whose per-step programs do not fit shared
// memory, get the streamed-program variant (tp.stream = 1) by default.
int tile_plan(const Geometry& g, int width, int sms, int64_t nq, int ocap, const TileKnobs& kn,
              TilePlan& tp);
// K1t rows per warp for a table (or shard) of `slots` budget slots.
int tile_rows_for(int64_t slots, int sms, const TileKnobs& kn);
int launch_fill_tiles(const InstDesc& d, const TilePlan& tp, int width, void* stream);
// One table as tile jobs (tp.jobs), descriptor and plan as kernel parameters.
int launch_fill_tiles_jobs1(const InstDesc& d, const TilePlan& tp, unsigned int* counter, void* stream);
// Batches: jobs (table, tile) in queue order; tps[i].sm is the batch-wide
// layout (tile_batch_smem of a plan with every table's maxima).
TileSmem tile_batch_smem(const TilePlan& proto);
int launch_fill_tiles_batch(const InstDesc* descs, const TilePlan* tps, const int2* jobs,
                            int njobs, unsigned int* counter, const TilePlan& proto, void* stream,
                            const TilePlan* walk = nullptr);

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
    int32_t nq;         // saved options in the menu (walk staging)
    PlanDev plan;       // K1p schedule + state (device pointers)
    ProgDev prog;       // K1p cell programs
    size_t state_bytes; // bytes of counter + flags to zero before each fill
    int32_t prep_zero = 0;  // 1: the program launch also zeroes that state
};

int launch_prep_programs(const LaunchCtx& c);
// cell programs (and pads) of n tables whose descriptors are in d (device)
int launch_prep_programs_batch(const InstDesc* d, int n, int64_t max_rows, int width, void* stream);
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

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize, smem) for a launch of
// `smem` bytes.  The attribute only ever GROWS (per kernel and device): a
// launch with a smaller size runs under a larger limit, so a thread that
// checked the limit for its launch can never have it lowered underneath it by
// another thread's table (the check-then-launch race of a set-to-exact-size
// scheme).  The call is skipped when the limit already covers the request
// (it costs host time on every launch otherwise).
inline cudaError_t set_dyn_smem(const void* kern, size_t smem) {
    // (no "<= 48 KB needs nothing" shortcut: the default limit covers
    // dynamic + static shared memory, so 48 KB of dynamic alone can exceed it)
    int dev = 0;
    cudaGetDevice(&dev);
    static std::mutex mu;
    static std::unordered_map<const void*, int> limit[64];
    std::lock_guard<std::mutex> g(mu);  // held across the set: the map and the attribute agree
    auto& m = limit[dev & 63];
    auto it = m.find(kern);
    if (it != m.end() && it->second >= (int)smem) return cudaSuccess;
    const cudaError_t e =
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e == cudaSuccess) m[kern] = (int)smem;
    return e;
}

}  // namespace rkr
