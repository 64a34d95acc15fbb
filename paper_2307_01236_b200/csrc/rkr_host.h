// rkr_host.h -- host-side internals of librkr.so shared by its C-ABI
// translation units: rkr_table.cu (tables, walks, solve_chain),
// rkr_batch.cu (batches, sweeps), rkr_shard.cu (budget-axis shards) and
// rkr_replay.cu (the chain-level replay).  Not installed; include/rkr.h is
// the public ABI.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/rkr.h"
#include "rkr_internal.h"

namespace rkr {
namespace host {

extern thread_local std::string g_err;  // rkr_last_error()

// fn(i) for i in [0, n) on up to 16 host threads (batched table setup: the
// per-table host precompute of the DpTable constructor is independent).
template <typename F>
void parallel_for(int n, F fn) {
    int nt = (int)std::min<unsigned>(16u, std::max(1u, std::thread::hardware_concurrency()));
    nt = std::min(nt, std::max(1, n / 8));
    if (nt <= 1) {
        for (int i = 0; i < n; ++i) fn(i);
        return;
    }
    std::vector<std::thread> pool;
    for (int w = 0; w < nt; ++w)
        pool.emplace_back([&, w] {
            for (int i = w; i < n; i += nt) fn(i);
        });
    for (auto& th : pool) th.join();
}

// rkr_exec.tune & RKR_TUNE_PROFILE: host phase timings of the batched entry
// points on stderr (each mark synchronises the stream first, so only for
// diagnostics).
struct PhaseTimer {
    bool on = false;
    explicit PhaseTimer(const rkr_exec* ex) : on(ex && (ex->tune & RKR_TUNE_PROFILE)) {}
    cudaStream_t st = nullptr;
    std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
    void mark(const char* what) {
        if (!on) return;
        if (st) cudaStreamSynchronize(st);
        const auto t1 = std::chrono::steady_clock::now();
        fprintf(stderr, "[rkr] %-28s %9.3f ms\n", what,
                std::chrono::duration<double, std::milli>(t1 - t0).count());
        t0 = t1;
    }
};

rkr_status fail(rkr_status st, const char* fmt, ...);
rkr_status cuda_fail(cudaError_t e, const char* where);

#define CK(call)                                          \
    do {                                                  \
        cudaError_t e_ = (call);                          \
        if (e_ != cudaSuccess) return cuda_fail(e_, #call); \
    } while (0)

inline int64_t to_units(int64_t b, int64_t unit) {  // chain_dp.hpp:41 (unit 1: no division)
    return unit == 1 ? b : (b + unit - 1) / unit;
}

// to_units by one fixed unit, for the host precompute's hot loop: a
// double-precision quotient corrected to the exact floor for numerators in
// [0, 2^52) (one multiply instead of a 64-bit division), the plain
// truncating division otherwise.
struct UnitDiv {
    int64_t u;
    double inv;
    explicit UnitDiv(int64_t unit) : u(unit), inv(1.0 / (double)unit) {}
    int64_t operator()(int64_t b) const {
        if (u == 1) return b;
        const int64_t n = b + u - 1;
        if (n < 0 || n >= (int64_t(1) << 52)) return n / u;
        int64_t q = (int64_t)((double)n * inv);
        if (q * u > n) --q;
        else if ((q + 1) * u <= n) ++q;
        return q;
    }
};

inline int64_t round_up(int64_t x, int64_t a) { return (x + a - 1) / a * a; }

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        int cur = -1;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

// Host image of the DpTable constructor's precompute (chain_dp.hpp:56-95).
struct HostMenu {
    int32_t L = 0;
    std::vector<int32_t> blk_off;  // saved options per block, CSR
    std::vector<int64_t> fwd_req, fwd_req_pre, bwd_req, pack_chg, tftb, chg_bt;
    std::vector<int32_t> ids;
    std::vector<int64_t> act_u, fwd0_own, fwd0_full, tf0;
    int32_t max_opts = 0;
    bool bounded32 = false;  // the 32-bit overflow proof holds
    bool bounded64 = false;  // ... below kInfTime: feasibility is time-free (min-feasible thresholds)
};

rkr_status build_host_menu(const rkr_menu* m, int64_t unit, HostMenu& h);

// the per-device library stream (and the warm memory pool)
cudaError_t device_ctx(int dev, cudaStream_t* st);

// Thread-local pinned staging for the menu upload and small readbacks; an
// event guards reuse while an earlier async copy may still read it.
struct Staging {
    void* ptr = nullptr;
    size_t cap = 0;
    cudaEvent_t done = nullptr;
    ~Staging() {
        if (done) cudaEventDestroy(done);
        if (ptr) cudaFreeHost(ptr);
    }
    cudaError_t get(size_t n, void** out) {
        cudaError_t e = cudaSuccess;
        if (done) {
            e = cudaEventSynchronize(done);
            if (e != cudaSuccess) return e;
        } else {
            e = cudaEventCreateWithFlags(&done, cudaEventDisableTiming);
            if (e != cudaSuccess) return e;
        }
        if (n > cap) {
            if (ptr) cudaFreeHost(ptr);
            ptr = nullptr;
            size_t c = std::max<size_t>(n, 1 << 16);
            e = cudaMallocHost(&ptr, c);
            if (e != cudaSuccess) {
                cap = 0;
                return e;
            }
            cap = c;
        }
        *out = ptr;
        return cudaSuccess;
    }
};
extern thread_local Staging t_stage;
extern thread_local Staging t_back;   // pinned D2H staging (walk results)
extern thread_local Staging t_sweep;  // pinned D2H staging (a sweep's walks; outlives nested fetches)
extern thread_local Staging t_desc;   // pinned H2D staging of batch descriptors

}  // namespace host
}  // namespace rkr

using namespace rkr;
using namespace rkr::host;

struct rkr_table {
    int device = 0;
    cudaStream_t stream = nullptr;
    int64_t unit = 1;
    int width = 64;
    HostMenu hm;
    Geometry g{};
    DevMenu dm{};
    void* block = nullptr;        // one pooled allocation: menu | scratch | opt | arg
    size_t block_bytes = 0, work_bytes = 0;
    size_t block_cap = 0, mirror_cap = 0;  // process shards: bytes of the cudaMalloc blocks (reused)
    size_t off_tp = 0, off_jobs = 0;  // K1t tile jobs: plan and job list in the menu blob
    TilePlan* dtp = nullptr;
    int2* djobs = nullptr;
    std::vector<size_t> off;      // layout_sizes: menu-blob offsets, then work-area offsets
    bool owns_block = true;       // false: carved out of a batch's blocks
    size_t menu_bytes = 0;        // H2D bytes per create
    void* opt = nullptr;
    uint16_t* arg = nullptr;
    int4* stack = nullptr;
    int64_t* dout = nullptr;      // device scratch: backtrack result / first-feasible
    int64_t hout[8] = {};
    int64_t* wrec = nullptr;      // walk record (8 x int64) | op buffer: one allocation, one D2H
    int32_t* dops = nullptr;      // device op buffer (wrec + 64 B, grows on demand)
    int64_t dops_cap = 0;
    bool bt_pending = false;
    int kernel = 0;               // RKR_KERNEL_PERSISTENT or RKR_KERNEL_DIAGONAL
    bool tiles = false;           // persistent fill by budget tiles (K1t) instead of the queue (K1p)
    TilePlan tplan;
    int32_t flag_cols = 0;        // done-flag columns: max(K1p tiles J, K1t tiles T)
    PersistPlan plan;
    PlanDev pdev{};
    ProgDev prog{};
    size_t state_bytes = 0;
    bool state_clean = false;     // the program launch zeroed the fill state
    bool self_reset = false;      // the last co-resident K1t launch re-zeroed its state
    unsigned long long* trace = nullptr;
    int32_t bt_s = 0, bt_t = 0, bt_m = 0;
    InstDesc hdesc{};             // this table as the persistent kernel sees it
    bool ipc = false;             // block from cudaMalloc (multi-process shard)
    int32_t shard_lo = 0, shard_hi = 0;
    std::vector<void*> ipc_open;  // peer blocks opened with cudaIpcOpenMemHandle
    // process shards: shard 0's walk mirror (owned: cudaMalloc, IPC-exported)
    // and the cross-shard walk's cached views and scratch
    uint16_t* mirror = nullptr;
    int64_t mirror_sa = 0;
    int32_t mirror_M = -1;        // last global budget slot
    std::vector<unsigned char> walk_key;  // the handles the cached views were opened from
    void* walk_scratch = nullptr; // ShardView[n] | out[8] | stack | ops[cap]
    int64_t walk_cap = 0;
    int32_t walk_n = 0;
    InstDesc* ddesc = nullptr;    // device copy (single-table fills)
    LaunchPlan lplan{};           // single-table launch order (device pointers)

    // rkr_backtrack_menu: the caller's menu's pack shifts for the walk
    // (device, nq entries; nullptr = the table's own)
    int64_t* walk_chg = nullptr;
    LaunchCtx ctx() const {
        LaunchCtx c;
        c.g = g;
        c.dm = dm;
        if (walk_chg) c.dm.chg_bt = walk_chg;
        c.opt = opt;
        c.arg = arg;
        c.width = width;
        c.max_opts = hm.max_opts;
        c.nq = (int32_t)hm.ids.size();
        c.stream = stream;
        c.kernel = kernel;
        c.plan = pdev;
        c.prog = prog;
        c.state_bytes = state_bytes;
        return c;
    }
};

namespace rkr {
namespace host {

struct ShardSpec {
    int32_t m_base, pad, j_offset;
    bool ipc = false;
};

// Everything rkr_table_create does except the fill: validation and unit
// precompute, geometry, plan, one pooled allocation + one H2D copy, pads,
// cell programs.  R = 0 lets the plan choose the per-thread slot count.
rkr_status prepare_table(const rkr_menu* menu, int64_t unit, int32_t m_max, const rkr_exec* exec,
                         int R, rkr_table** out, const ShardSpec* spec = nullptr,
                         bool batch_tiles = false, bool defer = false);
void free_table(rkr_table* t);
// reusable cudaMalloc blocks of process shards (IPC-exportable), per device
void* ipc_block_take(int dev, size_t need, size_t* cap);
void ipc_block_give(int dev, void* block, size_t bytes);
// solve_chain's min-feasible search by thresholds (rkr_kernels.cu
// batch_thresholds): thr(0, L-1) of the tables d[which[i]] (device
// descriptors), L[i] blocks each; kInf64 when never feasible.
rkr_status min_feasible_thresholds(const InstDesc* d, const std::vector<int32_t>& which,
                                   const std::vector<int32_t>& L, cudaStream_t st,
                                   std::vector<int64_t>& thr);
// the wide table's budget cap of solve_chain's infeasible branch (:267-278)
int64_t feasibility_cap(const rkr_menu* menu, int64_t unit);
void bind_block(rkr_table* t, unsigned char* mb, unsigned char* wb);
void stage_menu(const rkr_table* t, unsigned char* blob);

}  // namespace host
}  // namespace rkr

// ---------------------------------------------------------------------------
// Batches: many independent tables, one persistent fill (config 4 sweeps).
// ---------------------------------------------------------------------------
struct rkr_batch {
    int device = 0;
    cudaStream_t stream = nullptr;
    int width = 32, R = 1, kcap = 1, ocap = 1;
    int32_t tune = 0;                    // rkr_exec.tune of the creating call
    std::vector<rkr_table*> tables;
    void* block = nullptr;               // desc array | counter | flags of every table
    InstDesc* ddesc = nullptr;
    unsigned long long* counter = nullptr;
    size_t state_bytes = 0;              // counter + flags
    int64_t total = 0;
    LaunchPlan lplan{};                  // merged launch order (device pointers)
    HostLaunchPlan hp;
    std::vector<InstDesc> hd;            // host copies of the descriptors
    size_t desc_bytes = 0, plan_bytes = 0, o_inst = 0, o_k = 0, o_j = 0;
    bool owns_tables = true;
    // budget-tile batches (K1t jobs): per-table plans, the job queue
    bool tiles = false;
    TilePlan proto{};                    // batch-wide WC / comm / shared-memory layout
    std::vector<TilePlan> htp;
    std::vector<int2> hjobs;
    TilePlan* dtps = nullptr;
    int2* djobs = nullptr;
    size_t tps_bytes = 0, jobs_bytes = 0;
    bool ordered = false;                // tile jobs in table order (budget shards)
    void* mblock = nullptr;              // every table's menu blob (one H2D copy)
    void* wblock = nullptr;              // every table's work area
};

namespace rkr {
namespace host {

void free_batch(rkr_batch* b);
rkr_status batch_zero(rkr_batch* b);
rkr_status batch_launch(rkr_batch* b);
rkr_status batch_layout(rkr_batch* b);
rkr_status batch_upload(rkr_batch* b);

}  // namespace host
}  // namespace rkr
