// rkr_capi.cu -- host half of librkr.so: the C ABI of include/rkr.h.
//
// Host work here is exactly the reference's host-side bookkeeping (menu
// validation and the per-block unit precompute of the DpTable constructor,
// chain_dp.hpp:56-95; quantize/to_units :32-41; solve_chain's control flow
// :255-296).  Every table cell is computed on the device (rkr_kernels.cu);
// there is no CPU fallback.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <mutex>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "../../include/rkr.h"
#include "rkr_internal.h"

using namespace rkr;

namespace {

thread_local std::string g_err;

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

rkr_status fail(rkr_status st, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return st;
}

rkr_status cuda_fail(cudaError_t e, const char* where) {
    cudaGetLastError();  // clear sticky-free errors
    return fail(e == cudaErrorMemoryAllocation ? RKR_ERR_OOM : RKR_ERR_CUDA, "%s: %s", where,
                cudaGetErrorString(e));
}

#define CK(call)                                          \
    do {                                                  \
        cudaError_t e_ = (call);                          \
        if (e_ != cudaSuccess) return cuda_fail(e_, #call); \
    } while (0)

int64_t to_units(int64_t b, int64_t unit) {  // chain_dp.hpp:41 (unit 1: no division)
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

int64_t round_up(int64_t x, int64_t a) { return (x + a - 1) / a * a; }

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
};

rkr_status build_host_menu(const rkr_menu* m, int64_t unit, HostMenu& h) {
    if (!m) return fail(RKR_ERR_ARGUMENT, "null menu");
    const int32_t L = m->n_blocks;
    if (L <= 0) return fail(RKR_ERR_INVALID, "empty option menu");      // chain_dp.hpp:58
    if (!m->option_offsets || !m->option_id || !m->time_fwd || !m->time_bwd || !m->has_bwd ||
        !m->save_mem || !m->peak_fwd || !m->peak_fwd_pre || !m->peak_bwd || !m->act_sizes)
        return fail(RKR_ERR_ARGUMENT, "null menu array");
    if (unit < 1) return fail(RKR_ERR_INVALID, "unit must be >= 1");
    if (L > 0x7fff) return fail(RKR_ERR_INVALID, "chains longer than 32767 blocks are not supported");
    for (int32_t i = 0; i < L; ++i)
        if (m->option_offsets[i + 1] < m->option_offsets[i])
            return fail(RKR_ERR_ARGUMENT, "option_offsets not monotone at block %d", i);
    h.L = L;
    const UnitDiv tu(unit);
    const size_t nopt = (size_t)m->option_offsets[L] - (size_t)m->option_offsets[0];
    // sized for every option up front (indexed writes, trimmed at the end)
    for (auto* v : {&h.fwd_req, &h.fwd_req_pre, &h.bwd_req, &h.pack_chg, &h.tftb, &h.chg_bt})
        v->resize(nopt);
    h.ids.resize(nopt);
    int64_t* const fwd_req = h.fwd_req.data();
    int64_t* const fwd_req_pre = h.fwd_req_pre.data();
    int64_t* const bwd_req = h.bwd_req.data();
    int64_t* const pack_chg = h.pack_chg.data();
    int64_t* const tftb = h.tftb.data();
    int64_t* const chg_bt = h.chg_bt.data();
    int32_t* const ids = h.ids.data();
    int32_t nq = 0;  // saved options so far
    h.act_u.resize(L + 1);
    for (int32_t i = 0; i <= L; ++i) h.act_u[i] = tu(m->act_sizes[i]);  // :59-60
    h.blk_off.assign(L + 1, 0);
    h.fwd0_own.assign(L, 0);
    h.fwd0_full.assign(L, 0);
    h.tf0.assign(L, 0);
    bool nonneg = true;
    long double F = 0, Bk = 0;
    std::vector<std::pair<int32_t, int32_t>> first;  // (option id, first position) of a block
    for (int32_t i = 0; i < L; ++i) {                                         // :72-95
        const int64_t a_i = m->act_sizes[i];
        bool saw_zero = false;
        // build_schedule_rec looks an option up by id, first match in menu
        // order (chain_dp.hpp:200-205, :228): first position of every id --
        // a backward scan for blocks of <= 32 options, else sorted
        // (id, position) pairs (a plain sort keeps the first position of an
        // id first, without stable_sort's allocation)
        const int32_t o_lo = m->option_offsets[i], o_hi = m->option_offsets[i + 1];
        const bool small = o_hi - o_lo <= 32;
        auto first_pos = [&](int32_t o) {
            if (small) {
                for (int32_t q = o_lo; q < o; ++q)
                    if (m->option_id[q] == m->option_id[o]) return q;
                return o;
            }
            return std::lower_bound(first.begin(), first.end(),
                                    std::make_pair(m->option_id[o], INT32_MIN))->second;
        };
        if (!small) {
            first.clear();
            for (int32_t o = o_lo; o < o_hi; ++o) first.emplace_back(m->option_id[o], o);
            std::sort(first.begin(), first.end());
        }
        h.blk_off[i] = nq;
        int64_t fmax = 0, bmax = 0;
        for (int32_t o = m->option_offsets[i]; o < m->option_offsets[i + 1]; ++o) {
            if (m->time_fwd[o] < 0) nonneg = false;
            fmax = std::max(fmax, m->time_fwd[o]);
            if (m->option_id[o] == 0) {                                       // :76-81
                h.fwd0_own[i] = tu(m->peak_fwd[o] - a_i);
                h.fwd0_full[i] = tu(m->peak_fwd[o]);
                h.tf0[i] = m->time_fwd[o];
                saw_zero = true;
                continue;
            }
            if (!m->has_bwd[o])                                               // :83-85
                return fail(RKR_ERR_INVALID, "saved option without a backward in block %d", i);
            if (m->time_bwd[o] < 0) nonneg = false;
            bmax = std::max(bmax, m->time_bwd[o]);
            ids[nq] = m->option_id[o];                                        // :86-92
            fwd_req[nq] = tu(m->peak_fwd[o] - a_i);
            fwd_req_pre[nq] = tu(m->peak_fwd_pre[o] - a_i);
            bwd_req[nq] = tu(m->peak_bwd[o] - a_i);
            pack_chg[nq] = tu(m->save_mem[o] - a_i);
            tftb[nq] = m->time_fwd[o] + m->time_bwd[o];
            chg_bt[nq] = tu(m->save_mem[first_pos(o)] - a_i);
            ++nq;
        }
        if (!saw_zero) return fail(RKR_ERR_INVALID, "block %d lacks option 0", i);  // :94
        const int32_t n = nq - h.blk_off[i];
        if (n > 0x7ffe) return fail(RKR_ERR_INVALID, "block %d has more than 32766 options", i);
        h.max_opts = std::max(h.max_opts, n);
        F += (long double)fmax;
        Bk += (long double)bmax;
    }
    h.blk_off[L] = nq;
    for (auto* v : {&h.fwd_req, &h.fwd_req_pre, &h.bwd_req, &h.pack_chg, &h.tftb, &h.chg_bt})
        v->resize(nq);
    h.ids.resize(nq);
    // Shifts index earlier budget columns; a negative one would read past
    // m_max, which is undefined behaviour in the reference (vector overrun).
    for (size_t q = 0; q < h.pack_chg.size(); ++q)
        if (h.pack_chg[q] < 0)
            return fail(RKR_ERR_INVALID,
                        "saved option with save_mem below its input size (negative pack shift)");
    for (int32_t c = 1; c < L; ++c)
        if (h.act_u[c] < 0) return fail(RKR_ERR_INVALID, "negative activation size a_%d", c);
    // Overflow proof for 32-bit costs: every finite candidate total is at most
    // L * sum_j max time_fwd_j + sum_j max time_bwd_j when times are >= 0
    // (induction over span).  Require it below INF32 = 2^30.
    h.bounded32 = nonneg && ((long double)L * F + Bk) < (long double)kInf32;
    return RKR_OK;
}

}  // namespace

namespace {

// Per-device state shared by all tables: a non-blocking stream for handles
// created without one, and the default memory pool kept warm (release
// threshold = max) so per-table cudaMallocAsync is a pool hit after warm-up.
struct DeviceCtx {
    std::once_flag once;
    cudaStream_t stream = nullptr;
    cudaError_t err = cudaSuccess;
};
DeviceCtx g_dev[64];

cudaError_t device_ctx(int dev, cudaStream_t* st) {
    if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
    DeviceCtx& c = g_dev[dev];
    std::call_once(c.once, [&] {
        c.err = cudaStreamCreateWithFlags(&c.stream, cudaStreamNonBlocking);
        if (c.err != cudaSuccess) return;
        cudaMemPool_t pool;
        c.err = cudaDeviceGetDefaultMemPool(&pool, dev);
        if (c.err != cudaSuccess) return;
        uint64_t thr = UINT64_MAX;
        c.err = cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    });
    *st = c.stream;
    return c.err;
}

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
thread_local Staging t_stage;
thread_local Staging t_back;   // pinned D2H staging (walk results)
thread_local Staging t_sweep;  // pinned D2H staging (a sweep's walks; outlives nested fetches)
thread_local Staging t_desc;   // pinned H2D staging of batch descriptors (overlaps the menu upload)

}  // namespace

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

namespace {

void free_table(rkr_table* t) {
    if (!t) return;
    DeviceGuard dg(t->device);
    if (t->trace) cudaFreeAsync(t->trace, t->stream);
    for (void* p : t->ipc_open) {
        cudaStreamSynchronize(t->stream);
        cudaIpcCloseMemHandle(p);
    }
    if (t->block && t->ipc) {
        cudaStreamSynchronize(t->stream);
        cudaFree(t->block);
        t->block = nullptr;
    }
    if (t->block && t->owns_block) cudaFreeAsync(t->block, t->stream);
    if (t->wrec) cudaFreeAsync(t->wrec, t->stream);
    delete t;
}

rkr_status check_cell(const rkr_table* t, int32_t s, int32_t tt) {
    if (!t) return fail(RKR_ERR_ARGUMENT, "null table");
    if (s < 0 || tt < s || tt >= t->g.L)
        return fail(RKR_ERR_ARGUMENT, "cell (%d, %d) outside 0 <= s <= t < %d", s, tt, t->g.L);
    return RKR_OK;
}

// Device layout of one table: a menu blob (uploaded once: the unit
// precompute, the K1p plan, the kernel descriptor) and a work area (scratch,
// opt rows, arg rows, state, cell programs).  A single table keeps both in
// one block; a batch carves every table's menu blob out of one region (one
// H2D copy) and its work area out of another.
void layout_sizes(rkr_table* t) {
    const HostMenu& h = t->hm;
    const size_t nq = std::max<size_t>(h.ids.size(), 1);
    const size_t L = h.L;
    std::vector<size_t>& off = t->off;
    off.clear();
    size_t bytes = 0;
    auto take = [&](size_t n) {
        off.push_back(bytes);
        bytes += round_up((int64_t)n, 256);
    };
    take((L + 1) * 4);                         // 0 blk_off
    for (int i = 0; i < 6; ++i) take(nq * 8);  // 1..6 fwd_req..chg_bt
    take(nq * 4);                              // 7 ids
    take((L + 1) * 8);                         // 8 act_u
    for (int i = 0; i < 3; ++i) take(L * 8);   // 9..11 fwd0_own, fwd0_full, tf0
    const size_t np = t->plan.start.size();
    take(np * 8);                              // 12 plan start
    take(np * 4);                              // 13 plan g
    take(np * 4);                              // 14 plan k
    take(sizeof(InstDesc));                    // 15 kernel descriptor
    take(np * 4);                              // 16 plan instance ids (all 0)
    // K1t as tile jobs (more tiles than SMs): its plan and job list travel
    // with the menu blob
    const bool jobs = t->tiles && t->tplan.jobs;
    t->off_tp = bytes;
    bytes += jobs ? round_up((int64_t)sizeof(TilePlan), 256) : 0;
    t->off_jobs = bytes;
    bytes += jobs ? round_up((int64_t)t->tplan.T * (int64_t)sizeof(int2), 256) : 0;
    t->menu_bytes = bytes;
    bytes = 0;                                 // work area offsets from here
    take(sizeof(int4) * (2 * L + 16));         // 17 backtrack stack
    take(8 * sizeof(int64_t));                 // 18 dout
    const size_t vbytes = t->width == 32 ? 4 : 8;
    take(((size_t)t->g.rows * t->g.sr + kOptSlack) * vbytes);  // 19 opt
    take((size_t)t->g.rows * t->g.sa * 2);       // 20 arg
    // counter | done flags [L x flag_cols] (K1p tiles or K1t tiles) | halo [L]
    // | CTAs finished (K1t fused walk)
    t->flag_cols = std::max<int32_t>(t->plan.J, t->tplan.T);
    t->state_bytes = 8 + ((size_t)t->g.L * t->flag_cols + t->g.L + 1) * sizeof(int);
    take(t->state_bytes);                        // 21 K1p counter + done flags
    const bool progs = t->kernel == RKR_KERNEL_PERSISTENT;
    const size_t nc = progs ? (size_t)program_cut_entries(t->g) : 0;
    // thr row stride; K1t copies thr rows with bulk copies and reads whole option batches
    t->prog.ocap = (int32_t)(t->tiles ? round_up(std::max<int32_t>(h.max_opts, 1), kTileOptBatch)
                                      : std::max<int32_t>(h.max_opts, 1));
    take(nc * 16);                               // 22 program ptr
    take(nc * vbytes);                           // 23 program sweep
    take(nc * 4);                                // 24 program gate
    take(progs ? (size_t)t->g.rows * t->prog.ocap * 4 : 0);  // 25 program thr
    take(progs ? nq * 4 : 0);                    // 26 program pc
    take(progs ? nq * vbytes : 0);               // 27 program otot
    t->work_bytes = bytes;
    t->block_bytes = t->menu_bytes + t->work_bytes;
}

// Device pointers of the table (and its descriptor) inside menu blob `mb`
// and work area `wb`.
void bind_block(rkr_table* t, unsigned char* mb, unsigned char* wb) {
    const HostMenu& h = t->hm;
    const std::vector<size_t>& off = t->off;
    const size_t np = t->plan.start.size();
    auto at = [&](int idx) { return idx <= 16 ? mb + off[idx] : wb + off[idx]; };
    t->dm.blk_off = reinterpret_cast<const int32_t*>(at(0));
    t->dm.fwd_req = reinterpret_cast<const int64_t*>(at(1));
    t->dm.fwd_req_pre = reinterpret_cast<const int64_t*>(at(2));
    t->dm.bwd_req = reinterpret_cast<const int64_t*>(at(3));
    t->dm.pack_chg = reinterpret_cast<const int64_t*>(at(4));
    t->dm.tftb = reinterpret_cast<const int64_t*>(at(5));
    t->dm.chg_bt = reinterpret_cast<const int64_t*>(at(6));
    t->dm.ids = reinterpret_cast<const int32_t*>(at(7));
    t->dm.act_u = reinterpret_cast<const int64_t*>(at(8));
    t->dm.fwd0_own = reinterpret_cast<const int64_t*>(at(9));
    t->dm.fwd0_full = reinterpret_cast<const int64_t*>(at(10));
    t->dm.tf0 = reinterpret_cast<const int64_t*>(at(11));
    t->ddesc = reinterpret_cast<InstDesc*>(at(15));
    t->dtp = reinterpret_cast<TilePlan*>(mb + t->off_tp);
    t->djobs = reinterpret_cast<int2*>(mb + t->off_jobs);
    t->lplan.start = reinterpret_cast<const int64_t*>(at(12));
    t->lplan.j = reinterpret_cast<const int32_t*>(at(13));
    t->lplan.k = reinterpret_cast<const int32_t*>(at(14));
    t->lplan.inst = reinterpret_cast<const int32_t*>(at(16));
    t->lplan.n = (int32_t)np;
    t->lplan.total = t->plan.total;
    t->stack = reinterpret_cast<int4*>(at(17));
    t->dout = reinterpret_cast<int64_t*>(at(18));
    t->opt = at(19);
    t->arg = reinterpret_cast<uint16_t*>(at(20));
    PlanDev& pd = t->pdev;
    pd.R = t->plan.R;
    pd.TM = t->plan.TM;
    pd.J = t->plan.J;
    pd.dj = t->plan.dj;
    pd.n_plan = (int32_t)np;
    pd.total = t->plan.total;
    pd.start = reinterpret_cast<const int64_t*>(at(12));
    pd.g = reinterpret_cast<const int32_t*>(at(13));
    pd.k = reinterpret_cast<const int32_t*>(at(14));
    pd.counter = reinterpret_cast<unsigned long long*>(at(21));
    pd.done = reinterpret_cast<int32_t*>(at(21) + 8);
    pd.trace = nullptr;
    t->hdesc.halo = pd.done + (size_t)t->g.L * t->flag_cols;
    t->tplan.done = pd.done;
    t->tplan.fin = t->hdesc.halo + t->g.L;
    t->prog.ptr = at(22);
    t->prog.sweep = at(23);
    t->prog.gate = reinterpret_cast<int32_t*>(at(24));
    t->prog.thr = reinterpret_cast<int32_t*>(at(25));
    t->prog.pc = reinterpret_cast<int32_t*>(at(26));
    t->prog.otot = at(27);
    t->prog.nq = (int64_t)h.ids.size();
    t->prog.tiles = t->tiles ? 1 : 0;
    t->hdesc.g = t->g;
    t->hdesc.dm = t->dm;
    t->hdesc.opt = t->opt;
    t->hdesc.arg = t->arg;
    t->hdesc.plan = t->pdev;
    t->hdesc.prog = t->prog;
    t->hdesc.stack = t->stack;
    t->hdesc.item_base = 0;
}

// The menu blob's host image (menu_bytes) for the pinned staging buffer.
void stage_menu(const rkr_table* t, unsigned char* blob) {
    const HostMenu& h = t->hm;
    const std::vector<size_t>& off = t->off;
    const size_t L = h.L, np = t->plan.start.size();
    // every region is written below; only the alignment gaps between them
    // are zeroed (the blob is uploaded whole)
    auto put = [&](int idx, const void* src, size_t n) {
        if (n) std::memcpy(blob + off[idx], src, n);
        const size_t end = off[idx] + n, next = idx + 1 < 17 ? off[idx + 1] : t->off_tp;
        if (next > end) std::memset(blob + end, 0, next - end);
    };
    put(0, h.blk_off.data(), (L + 1) * 4);
    put(1, h.fwd_req.data(), h.fwd_req.size() * 8);
    put(2, h.fwd_req_pre.data(), h.fwd_req_pre.size() * 8);
    put(3, h.bwd_req.data(), h.bwd_req.size() * 8);
    put(4, h.pack_chg.data(), h.pack_chg.size() * 8);
    put(5, h.tftb.data(), h.tftb.size() * 8);
    put(6, h.chg_bt.data(), h.chg_bt.size() * 8);
    put(7, h.ids.data(), h.ids.size() * 4);
    put(8, h.act_u.data(), (L + 1) * 8);
    put(9, h.fwd0_own.data(), L * 8);
    put(10, h.fwd0_full.data(), L * 8);
    put(11, h.tf0.data(), L * 8);
    put(12, t->plan.start.data(), np * 8);
    put(13, t->plan.g.data(), np * 4);
    put(14, t->plan.k.data(), np * 4);
    put(15, &t->hdesc, sizeof(InstDesc));
    std::memset(blob + off[16], 0, t->off_tp - off[16]);  // 16: plan instance ids (all 0)
    if (t->tiles && t->tplan.jobs) {
        std::memcpy(blob + t->off_tp, &t->tplan, sizeof(TilePlan));
        int2* jb = reinterpret_cast<int2*>(blob + t->off_jobs);
        for (int32_t j = 0; j < t->tplan.T; ++j) jb[j] = make_int2(0, j);
    }
}

// One pooled allocation (menu blob | work area), pinned staging, one H2D copy.
rkr_status alloc_and_upload(rkr_table* t) {
    layout_sizes(t);
    if (t->ipc) {  // exportable to other processes (cudaIpcGetMemHandle needs cudaMalloc)
        CK(cudaMalloc(&t->block, t->block_bytes));
    } else {
        CK(cudaMallocAsync(&t->block, t->block_bytes, t->stream));
    }
    unsigned char* b = static_cast<unsigned char*>(t->block);
    bind_block(t, b, b + t->menu_bytes);
    void* stage = nullptr;
    CK(t_stage.get(t->menu_bytes, &stage));
    stage_menu(t, static_cast<unsigned char*>(stage));
    CK(cudaMemcpyAsync(t->block, stage, t->menu_bytes, cudaMemcpyHostToDevice, t->stream));
    CK(cudaEventRecord(t_stage.done, t->stream));
    return RKR_OK;
}

rkr_status ensure_ops(rkr_table* t) {
    if (t->dops_cap == 0) {
        const int64_t cap = std::max<int64_t>(4096, 8 * (int64_t)t->g.L + 64);
        CK(cudaMallocAsync(reinterpret_cast<void**>(&t->wrec), 64 + (size_t)cap * 12, t->stream));
        t->dops = reinterpret_cast<int32_t*>(t->wrec + 8);
        t->dops_cap = cap;
    }
    return RKR_OK;
}

// Fill, then (walk) the schedule walk from (s, tt, m): fused into the K1t
// launch (its last CTA walks), or as the K2 launch after the fill.
rkr_status enqueue_fill(rkr_table* t, bool walk = false, int32_t s = 0, int32_t tt = 0,
                        int32_t m = 0) {
    if (walk) {
        rkr_status st = ensure_ops(t);
        if (st) return st;
    }
    if (walk && !t->tiles) {
        rkr_status st = enqueue_fill(t);
        if (st) return st;
        if (launch_backtrack(t->ctx(), s, tt, m, t->dops, t->dops_cap,
                             reinterpret_cast<int32_t*>(t->stack), t->wrec))
            return cuda_fail(cudaGetLastError(), "backtrack launch");
        return RKR_OK;
    }
    if (t->kernel != RKR_KERNEL_PERSISTENT) {
        if (launch_init_pads(t->ctx())) return cuda_fail(cudaGetLastError(), "pad launch");
        if (launch_fill_all(t->ctx())) return cuda_fail(cudaGetLastError(), "fill launch");
        return RKR_OK;
    }
    if (t->state_clean || t->self_reset) {  // zeroed by the program launch (first
        t->state_clean = false;             // fill) or by the previous co-resident
        t->self_reset = false;              // K1t launch's last CTA
    } else {
        CK(cudaMemsetAsync(t->pdev.counter, 0, t->state_bytes, t->stream));
    }
    if (t->tiles) {
        TilePlan tp = t->tplan;
        tp.walk = walk ? 1 : 0;
        tp.ws = s;
        tp.wt = tt;
        tp.wm = m;
        tp.wops = t->dops;
        tp.wcap = t->dops_cap;
        tp.wout = t->wrec;
        tp.wstack = reinterpret_cast<int4*>(t->stack);
        if (tp.jobs) {  // more tiles than SMs: one-table tile jobs
            if (launch_fill_tiles_batch(t->ddesc, t->dtp, t->djobs, tp.T,
                                        reinterpret_cast<unsigned int*>(t->pdev.counter), tp,
                                        t->stream, &tp))  // (a single table: its plan)
                return cuda_fail(cudaGetLastError(), "tile job launch");
            return RKR_OK;
        }
        if (launch_fill_tiles(t->hdesc, tp, t->width, t->stream))
            return cuda_fail(cudaGetLastError(), "tile fill launch");
        // the last CTA re-zeroes the done flags and its counter -- but not a
        // budget shard's halo counters, so shard tables memset before a refill
        t->self_reset = !tp.halo;
        return RKR_OK;
    }
    if (launch_fill_batch(t->ddesc, &t->hdesc, t->lplan, t->width, t->plan.R,
                          std::max(t->g.L - 1, 1), std::max(t->hm.max_opts, 1), t->pdev.counter,
                          t->stream))
        return cuda_fail(cudaGetLastError(), "fill launch");
    return RKR_OK;
}

// Budget-axis shard of a table: local slot 0 is global slot m_base; pad is
// common to all shards; j_offset = global tile index of local tile 0.
struct ShardSpec {
    int32_t m_base, pad, j_offset;
    bool ipc = false;
};

// Everything rkr_table_create does except the fill: validation and unit
// precompute, geometry, plan, one pooled allocation + one H2D copy, pads,
// cell programs.  R = 0 lets the plan choose the per-thread slot count.
rkr_status prepare_table(const rkr_menu* menu, int64_t unit, int32_t m_max, const rkr_exec* exec,
                         int R, rkr_table** out, const ShardSpec* spec = nullptr,
                         bool batch_tiles = false, bool defer = false) {
    if (!out) return fail(RKR_ERR_ARGUMENT, "null output handle");
    *out = nullptr;
    if (m_max < 0) return fail(RKR_ERR_INVALID, "m_max must be >= 0");
    PhaseTimer ppt(exec);
    rkr_table* t = new rkr_table();
    rkr_status st = build_host_menu(menu, unit, t->hm);
    ppt.mark("  prepare: build_host_menu");
    if (st != RKR_OK) {
        delete t;
        return st;
    }
    t->unit = unit;
    t->device = exec ? exec->device : 0;
    const int want = exec ? exec->width : RKR_WIDTH_AUTO;
    const int kreq = exec ? exec->kernel : RKR_KERNEL_PERSISTENT;
    if (kreq < RKR_KERNEL_PERSISTENT || kreq > RKR_KERNEL_TILES) {
        delete t;
        return fail(RKR_ERR_ARGUMENT, "unknown kernel %d", kreq);
    }
    t->kernel = kreq == RKR_KERNEL_DIAGONAL ? RKR_KERNEL_DIAGONAL : RKR_KERNEL_PERSISTENT;
    t->width = (want != RKR_WIDTH_64 && t->hm.bounded32) ? 32 : 64;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev <= t->device || t->device < 0) {
        cudaGetLastError();
        delete t;
        return fail(RKR_ERR_CUDA, "no CUDA device %d visible (librkr has no CPU fallback)",
                    exec ? exec->device : 0);
    }
    DeviceGuard dg(t->device);
    cudaStream_t shared = nullptr;
    cudaError_t e = device_ctx(t->device, &shared);
    if (e != cudaSuccess) {
        delete t;
        return cuda_fail(e, "device context");
    }
    t->stream = (exec && exec->stream) ? static_cast<cudaStream_t>(exec->stream) : shared;
    // geometry
    const HostMenu& h = t->hm;
    int64_t maxshift = 0;
    for (int64_t p : h.pack_chg) maxshift = std::max(maxshift, p);
    for (int32_t c = 1; c < h.L; ++c) maxshift = std::max(maxshift, h.act_u[c]);
    t->g.L = h.L;
    t->g.M = m_max;
    t->g.pad = (int32_t)std::min<int64_t>(maxshift, (int64_t)m_max + 1);
    t->g.pad = (int32_t)round_up(t->g.pad, 8);
    if (spec) {
        t->g.pad = spec->pad;
        t->g.m_base = spec->m_base;
        t->ipc = spec->ipc;
    }
    t->g.sr = round_up((int64_t)t->g.pad + m_max + 1, 32);
    t->g.sa = round_up((int64_t)m_max + 1, 64);
    t->g.rows = (int64_t)h.L * (h.L + 1) / 2;
    ppt.mark("  prepare: device ctx + geometry");
    if (t->kernel == RKR_KERNEL_PERSISTENT) {
        // budget tiles (K1t) for unsharded tables; the queue (K1p) otherwise
        // or on request -- its work-item plan is only built when it runs
        if ((!spec || kreq == RKR_KERNEL_TILES) && kreq != RKR_KERNEL_QUEUE) {
            int sms = 0;
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, t->device);
            // batch tables need no co-residency (their tiles are queued jobs)
            TileKnobs kn;
            kn.tune = exec ? exec->tune : 0;
            // batches run 32-slot tiles unless told otherwise (their jobs
            // already fill the GPU); shards get the rows of their sharding
            kn.rows = exec && exec->tile_rows ? exec->tile_rows : (batch_tiles ? 1 : 0);
            t->tiles = tile_plan(t->g, t->width, batch_tiles ? INT32_MAX : sms, (int64_t)h.ids.size(),
                                 (int)round_up(std::max<int32_t>(h.max_opts, 1), kTileOptBatch), kn,
                                 t->tplan) == 1;
        }
        if (kreq == RKR_KERNEL_TILES && !t->tiles) {
            delete t;
            return fail(RKR_ERR_INVALID, "kernel TILES: the table does not fit the budget-tile "
                        "kernel (64-bit costs, or too many rows for its shared memory)");
        }
        if (t->tiles && spec && !batch_tiles) {  // a process shard: the halo variant
            t->tplan.comm = 1;
            t->tplan.split = 0;
            t->tplan.halo = 1;
            t->tplan.sm = tile_batch_smem(t->tplan);
        }
        if (!t->tiles) {
            t->tplan = TilePlan{};
            persistent_plan(t->g, t->width, R > 0 ? R : persistent_choose_r(m_max), t->plan);
            if (spec) t->plan.j_offset = spec->j_offset;
        }
        ppt.mark("  prepare: plans");
    }
    if (defer) {  // the caller (a batch) allocates, binds, uploads and preps
        layout_sizes(t);
        t->owns_block = false;
        *out = t;
        return RKR_OK;
    }
    ppt.mark("  prepare: host menu + geometry + plans");
    st = alloc_and_upload(t);
    ppt.mark("  prepare: alloc + stage + H2D enqueue");
    // (the persistent kernels' program launch also writes the pads)
    if (st == RKR_OK && t->kernel != RKR_KERNEL_PERSISTENT && launch_init_pads(t->ctx()))
        st = cuda_fail(cudaGetLastError(), "pad launch");
    if (st == RKR_OK && t->kernel == RKR_KERNEL_PERSISTENT) {
        // a plain table (every fill goes through enqueue_fill) has its first
        // fill's state zeroed by this launch
        LaunchCtx c = t->ctx();
        c.prep_zero = spec ? 0 : 1;
        if (launch_prep_programs(c)) st = cuda_fail(cudaGetLastError(), "program launch");
        else t->state_clean = !spec;
    }
    ppt.mark("  prepare: program launch");
    if (st != RKR_OK) {
        free_table(t);
        return st;
    }
    *out = t;
    return RKR_OK;
}

rkr_status create_impl(const rkr_menu* menu, int64_t unit, int32_t m_max, const rkr_exec* exec,
                       rkr_table** out) {
    rkr_status st = prepare_table(menu, unit, m_max, exec, 0, out);
    if (st != RKR_OK) return st;
    DeviceGuard dg((*out)->device);
    st = enqueue_fill(*out);
    if (st != RKR_OK) {
        free_table(*out);
        *out = nullptr;
    }
    return st;
}

template <typename V>
rkr_status read_cell(const rkr_table* t, int32_t s, int32_t tt, int32_t m, int64_t* val,
                     uint16_t* code) {
    const int64_t rid = row_id(t->g.L, s, tt);
    V v{};
    const V* o = static_cast<const V*>(t->opt);
    CK(cudaMemcpyAsync(&v, o + rid * t->g.sr + t->g.pad + m, sizeof(V), cudaMemcpyDeviceToHost,
                       t->stream));
    uint16_t c = 0;
    CK(cudaMemcpyAsync(&c, t->arg + rid * t->g.sa + m, 2, cudaMemcpyDeviceToHost, t->stream));
    CK(cudaStreamSynchronize(t->stream));
    if (t->width == 32)
        *val = (uint64_t)v >= kInf32 ? kInf64 : (int64_t)v;
    else
        *val = (int64_t)v;
    *code = c;
    return RKR_OK;
}

rkr_status cell(const rkr_table* t, int32_t s, int32_t tt, int32_t m, int64_t* val,
                uint16_t* code) {
    return t->width == 32 ? read_cell<uint32_t>(t, s, tt, m, val, code)
                          : read_cell<int64_t>(t, s, tt, m, val, code);
}

void decode(const rkr_table* t, int32_t s, int64_t val, uint16_t code, int32_t* kind,
            int32_t* value) {
    if (val >= kInf64 || code == 0) {  // chain_dp.hpp:177
        *kind = RKR_ARG_NONE;
        *value = -1;
    } else if (code & kCutBit) {
        *kind = RKR_ARG_CUT;
        *value = code & 0x7fff;
    } else {
        *kind = RKR_ARG_OPTION;
        *value = t->hm.ids[t->hm.blk_off[s] + code - 1];
    }
}

}  // namespace

extern "C" {

const char* rkr_last_error(void) { return g_err.c_str(); }
int32_t rkr_abi_version(void) { return RKR_ABI_VERSION; }

int32_t rkr_device_ok(int32_t device) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || device < 0 || device >= n) {
        cudaGetLastError();
        return 0;
    }
    cudaDeviceProp p;
    if (cudaGetDeviceProperties(&p, device) != cudaSuccess) return 0;
    return p.major == 10 ? 1 : 0;
}

rkr_status rkr_quantize(int64_t budget_bytes, int32_t units, int64_t* unit,
                        int64_t* budget_units) {
    if (!unit || !budget_units) return fail(RKR_ERR_ARGUMENT, "null output");
    if (units < 1) return fail(RKR_ERR_INVALID, "quantization needs at least one unit");  // :33
    int64_t u = (budget_bytes + units - 1) / units;                                       // :35
    if (u < 1) u = 1;
    *unit = u;
    *budget_units = budget_bytes / u;
    return RKR_OK;
}

int64_t rkr_to_units(int64_t bytes, int64_t unit) { return to_units(bytes, unit); }

rkr_status rkr_table_create(const rkr_menu* menu, int64_t unit, int32_t m_max,
                            const rkr_exec* exec, rkr_table** out) {
    return create_impl(menu, unit, m_max, exec, out);
}

void rkr_table_destroy(rkr_table* table) { free_table(table); }

int32_t rkr_table_length(const rkr_table* t) { return t ? t->g.L : 0; }
int64_t rkr_table_unit(const rkr_table* t) { return t ? t->unit : 0; }
int32_t rkr_table_m_max(const rkr_table* t) { return t ? t->g.M : -1; }
int32_t rkr_table_width(const rkr_table* t) { return t ? t->width : 0; }
int32_t rkr_table_kernel(const rkr_table* t) {
    if (!t) return -1;
    if (t->kernel == RKR_KERNEL_DIAGONAL) return RKR_KERNEL_DIAGONAL;
    return t->tiles ? RKR_KERNEL_TILES : RKR_KERNEL_QUEUE;
}
int64_t rkr_table_act_units(const rkr_table* t, int32_t i) {
    return (t && i >= 0 && i <= t->g.L) ? t->hm.act_u[i] : 0;
}

rkr_status rkr_table_work_bound(const rkr_table* t, int64_t* max_cands, int64_t* worst_allow) {
    if (!t || !max_cands || !worst_allow) return fail(RKR_ERR_ARGUMENT, "null argument");
    // Candidates per cell are non-decreasing in m (every test is "x <= m"),
    // so the maximum sits at m = m_max (counting as chain_dp.hpp:140,161).
    const HostMenu& h = t->hm;
    const int L = h.L;
    const int64_t M = t->g.M;
    // For a fixed t (fixed seed), the cut loop of cell (s, t) counts
    // min(t, j + 1) - s candidates, j = first block > s whose bare forward
    // does not fit (the `break`, counted before it fires); nxt[] gives j for
    // every s in one backward scan, so the whole bound is O(L^2).
    int64_t best = 0, worst = 0;  // both start at 0 as in chain_dp.hpp:119-120
    std::vector<int> nxt(L + 1);
    for (int tt = 0; tt < L; ++tt) {
        const int64_t seed = tt < L - 1 ? 2 * h.act_u[tt + 1] : 0;
        nxt[L - 1] = L;  // none
        for (int s = L - 2; s >= 0; --s)
            nxt[s] = (h.fwd0_full[s + 1] + seed > M) ? s + 1 : nxt[s + 1];
        for (int s = 0; s <= tt; ++s) {
            const int64_t nopt = h.blk_off[s + 1] - h.blk_off[s];
            int64_t cands = nopt;
            if (h.fwd0_own[s] + seed <= M) cands += std::min<int64_t>(tt, (int64_t)nxt[s] + 1) - s;
            best = std::max(best, cands);
            worst = std::max(worst, cands - ((tt - s) + nopt + 1));
        }
    }
    *max_cands = best;
    *worst_allow = worst;
    return RKR_OK;
}

rkr_status rkr_table_opt(const rkr_table* t, int32_t s, int32_t tt, int32_t m, int64_t* out) {
    rkr_status st = check_cell(t, s, tt);
    if (st) return st;
    if (!out) return fail(RKR_ERR_ARGUMENT, "null output");
    if (m < 0) {  // chain_dp.hpp:104
        *out = RKR_INF_TIME;
        return RKR_OK;
    }
    if (m > t->g.M) m = t->g.M;  // :105
    DeviceGuard dg(t->device);
    uint16_t code;
    return cell(t, s, tt, m, out, &code);
}

rkr_status rkr_table_arg(const rkr_table* t, int32_t s, int32_t tt, int32_t m, int32_t* kind,
                         int32_t* value) {
    rkr_status st = check_cell(t, s, tt);
    if (st) return st;
    if (!kind || !value) return fail(RKR_ERR_ARGUMENT, "null output");
    if (m < 0) {  // chain_dp.hpp:109
        *kind = RKR_ARG_NONE;
        *value = -1;
        return RKR_OK;
    }
    if (m > t->g.M) m = t->g.M;
    DeviceGuard dg(t->device);
    int64_t v;
    uint16_t code;
    st = cell(t, s, tt, m, &v, &code);
    if (st) return st;
    decode(t, s, v, code, kind, value);
    return RKR_OK;
}

static rkr_status export_rows_host(const rkr_table* t, int64_t r0, int64_t r1, int64_t* opt,
                                   int8_t* kind, int32_t* value) {
    // Device-side conversion in chunks of rows, then D2H.
    const int64_t W = t->g.M + 1;
    const int64_t per_row = W * (8 + 1 + 4);
    int64_t chunk = std::max<int64_t>(1, (int64_t)(256ll << 20) / per_row);
    chunk = std::min<int64_t>(chunk, 65535);
    chunk = std::min<int64_t>(chunk, r1 - r0);
    void* buf = nullptr;
    CK(cudaMalloc(&buf, (size_t)(chunk * per_row)));
    int64_t* dopt = static_cast<int64_t*>(buf);
    int32_t* dval = reinterpret_cast<int32_t*>(dopt + chunk * W);
    int8_t* dkind = reinterpret_cast<int8_t*>(dval + chunk * W);
    LaunchCtx c = t->ctx();
    rkr_status st = RKR_OK;
    for (int64_t r = r0; r < r1 && st == RKR_OK; r += chunk) {
        const int64_t n = std::min(chunk, r1 - r);
        if (launch_export(c, r, r + n, opt ? dopt : nullptr, kind ? dkind : nullptr,
                          value ? dval : nullptr)) {
            st = cuda_fail(cudaGetLastError(), "export launch");
            break;
        }
        const int64_t o = (r - r0) * W;
        cudaError_t e = cudaSuccess;
        if (opt && e == cudaSuccess)
            e = cudaMemcpyAsync(opt + o, dopt, n * W * 8, cudaMemcpyDeviceToHost, t->stream);
        if (value && e == cudaSuccess)
            e = cudaMemcpyAsync(value + o, dval, n * W * 4, cudaMemcpyDeviceToHost, t->stream);
        if (kind && e == cudaSuccess)
            e = cudaMemcpyAsync(kind + o, dkind, n * W, cudaMemcpyDeviceToHost, t->stream);
        if (e == cudaSuccess) e = cudaStreamSynchronize(t->stream);
        if (e != cudaSuccess) st = cuda_fail(e, "export copy");
    }
    cudaStreamSynchronize(t->stream);
    cudaFree(buf);
    return st;
}

rkr_status rkr_table_row(const rkr_table* t, int32_t s, int32_t tt, int64_t* opt, int8_t* kind,
                         int32_t* value) {
    rkr_status st = check_cell(t, s, tt);
    if (st) return st;
    DeviceGuard dg(t->device);
    const int64_t r = (int64_t)s * t->g.L - (int64_t)s * (s - 1) / 2 + (tt - s);
    return export_rows_host(t, r, r + 1, opt, kind, value);
}

rkr_status rkr_table_download(const rkr_table* t, int64_t* opt, int8_t* kind, int32_t* value) {
    if (!t) return fail(RKR_ERR_ARGUMENT, "null table");
    DeviceGuard dg(t->device);
    return export_rows_host(t, 0, t->g.rows, opt, kind, value);
}

rkr_status rkr_backtrack_async(rkr_table* t, int32_t s, int32_t tt, int32_t m) {
    rkr_status st = check_cell(t, s, tt);
    if (st) return st;
    DeviceGuard dg(t->device);
    st = ensure_ops(t);
    if (st) return st;
    if (launch_backtrack(t->ctx(), s, tt, m, t->dops, t->dops_cap,
                         reinterpret_cast<int32_t*>(t->stack), t->wrec))
        return cuda_fail(cudaGetLastError(), "backtrack launch");
    t->bt_s = s;
    t->bt_t = tt;
    t->bt_m = m;
    t->bt_pending = true;
    return RKR_OK;
}

rkr_status rkr_backtrack_fetch(rkr_table* t, rkr_op* ops, int64_t cap, int64_t* n_ops) {
    if (!t) return fail(RKR_ERR_ARGUMENT, "null table");
    if (!n_ops || (cap > 0 && !ops)) return fail(RKR_ERR_ARGUMENT, "null output");
    if (!t->bt_pending) return fail(RKR_ERR_ARGUMENT, "no backtrack enqueued on this table");
    DeviceGuard dg(t->device);
    *n_ops = 0;
    // one round trip for the usual case: the walk record and the first `est`
    // ops come back together through pinned memory
    const int64_t est = std::min<int64_t>({cap, t->dops_cap, 16 * (int64_t)t->g.L + 64});
    void* pin = nullptr;
    CK(t_back.get(64 + (size_t)std::max<int64_t>(est, 0) * 12, &pin));
    // (the record and the ops are adjacent: one copy)
    CK(cudaMemcpyAsync(pin, t->wrec, 64 + (size_t)std::max<int64_t>(est, 0) * 12,
                       cudaMemcpyDeviceToHost, t->stream));
    CK(cudaStreamSynchronize(t->stream));
    std::memcpy(t->hout, pin, 5 * sizeof(int64_t));
    int64_t n = t->hout[0];
    const bool have = n <= est;  // ops already on the host
    if (n > t->dops_cap) {  // grow the device op buffer and walk again (rare)
        CK(cudaFreeAsync(t->wrec, t->stream));
        CK(cudaMallocAsync(reinterpret_cast<void**>(&t->wrec), 64 + (size_t)n * 12, t->stream));
        t->dops = reinterpret_cast<int32_t*>(t->wrec + 8);
        t->dops_cap = n;
        if (launch_backtrack(t->ctx(), t->bt_s, t->bt_t, t->bt_m, t->dops, t->dops_cap,
                             reinterpret_cast<int32_t*>(t->stack), t->wrec))
            return cuda_fail(cudaGetLastError(), "backtrack launch");
        CK(cudaMemcpyAsync(t->hout, t->wrec, 4 * sizeof(int64_t), cudaMemcpyDeviceToHost,
                           t->stream));
        CK(cudaStreamSynchronize(t->stream));
        n = t->hout[0];
    }
    t->bt_pending = false;
    const int64_t status = t->hout[1];
    const int64_t ncopy = std::min(n, cap);
    if (ncopy > 0 && have) {
        std::memcpy(ops, static_cast<char*>(pin) + 64, (size_t)ncopy * 12);
    } else if (ncopy > 0) {
        CK(cudaMemcpyAsync(ops, t->dops, (size_t)ncopy * 12, cudaMemcpyDeviceToHost, t->stream));
        CK(cudaStreamSynchronize(t->stream));
    }
    *n_ops = n;
    if (status == 2)
        return fail(RKR_ERR_INFEASIBLE, "no feasible schedule for blocks %lld..%lld",
                    (long long)t->hout[2], (long long)t->hout[3]);
    if (status == 3)  // chain_dp.hpp:203-204, the reference's message
        return fail(RKR_ERR_INVALID, "menu for block %lld lacks option %lld",
                    (long long)t->hout[2], (long long)t->hout[3]);
    if (n > cap) return fail(RKR_ERR_CAPACITY, "schedule needs %lld ops", (long long)n);
    return RKR_OK;
}

rkr_status rkr_backtrack(const rkr_table* tc, int32_t s, int32_t tt, int32_t m, rkr_op* ops,
                         int64_t cap, int64_t* n_ops) {
    rkr_table* t = const_cast<rkr_table*>(tc);  // scratch buffers only
    if (!n_ops || (cap > 0 && !ops)) return fail(RKR_ERR_ARGUMENT, "null output");
    rkr_status st = rkr_backtrack_async(t, s, tt, m);
    if (st) return st;
    return rkr_backtrack_fetch(t, ops, cap, n_ops);
}

rkr_status rkr_backtrack_menu(const rkr_table* tc, const rkr_menu* menu, int32_t s, int32_t tt,
                              int32_t m, rkr_op* ops, int64_t cap, int64_t* n_ops) {
    rkr_table* t = const_cast<rkr_table*>(tc);  // scratch buffers only
    if (!menu) return rkr_backtrack(tc, s, tt, m, ops, cap, n_ops);
    rkr_status st = check_cell(t, s, tt);
    if (st) return st;
    if (!n_ops || (cap > 0 && !ops)) return fail(RKR_ERR_ARGUMENT, "null output");
    const HostMenu& h = t->hm;
    if (menu->n_blocks < h.L || !menu->option_offsets || !menu->option_id || !menu->save_mem ||
        !menu->act_sizes)
        return fail(RKR_ERR_INVALID, "menu has %d blocks, the table %d", menu->n_blocks, h.L);
    // build_schedule_rec's per-option shift from the caller's menu: the first
    // option with the decided id (detail::menu_option, chain_dp.hpp:200-205)
    // and to_units(save_mem - act_sizes[s], table unit) (:228)
    const UnitDiv tu(t->unit);
    std::vector<int64_t> chg(h.ids.size());
    bool same = true;
    for (int32_t b = 0; b < h.L; ++b) {
        const int32_t o_lo = menu->option_offsets[b], o_hi = menu->option_offsets[b + 1];
        for (int32_t q = h.blk_off[b]; q < h.blk_off[b + 1]; ++q) {
            int64_t c = (int64_t)kMissingShift;
            for (int32_t o = o_lo; o < o_hi; ++o)
                if (menu->option_id[o] == h.ids[q]) {
                    c = tu(menu->save_mem[o] - menu->act_sizes[b]);
                    break;
                }
            chg[q] = c;
            same = same && c == h.chg_bt[q];
        }
    }
    if (same) return rkr_backtrack(tc, s, tt, m, ops, cap, n_ops);
    DeviceGuard dg(t->device);
    int64_t* dchg = nullptr;
    CK(cudaMallocAsync(reinterpret_cast<void**>(&dchg), std::max<size_t>(chg.size(), 1) * 8, t->stream));
    CK(cudaMemcpyAsync(dchg, chg.data(), chg.size() * 8, cudaMemcpyHostToDevice, t->stream));
    t->walk_chg = dchg;
    st = rkr_backtrack_async(t, s, tt, m);
    if (st == RKR_OK) st = rkr_backtrack_fetch(t, ops, cap, n_ops);
    t->walk_chg = nullptr;
    cudaFreeAsync(dchg, t->stream);
    cudaStreamSynchronize(t->stream);  // chg lives on the host stack
    return st;
}

rkr_status rkr_table_refill(rkr_table* t) {
    if (!t) return fail(RKR_ERR_ARGUMENT, "null table");
    DeviceGuard dg(t->device);
    return enqueue_fill(t);
}

rkr_status rkr_table_refill_walk(rkr_table* t, int32_t s, int32_t tt, int32_t m) {
    rkr_status st = check_cell(t, s, tt);
    if (st) return st;
    DeviceGuard dg(t->device);
    st = enqueue_fill(t, true, s, tt, m);
    if (st) return st;
    t->bt_s = s;
    t->bt_t = tt;
    t->bt_m = m;
    t->bt_pending = true;
    return RKR_OK;
}

static int64_t rkr_trace_slots(const rkr_table* t) {
    return t->tiles ? (int64_t)t->g.L * t->tplan.T : t->plan.total;
}

rkr_status rkr_debug_trace(rkr_table* t, int32_t enable) {
    if (!t) return fail(RKR_ERR_ARGUMENT, "null table");
    DeviceGuard dg(t->device);
    if (enable && !t->trace && t->kernel == RKR_KERNEL_PERSISTENT) {
        const size_t n = (size_t)rkr_trace_slots(t) * 48;
        CK(cudaMallocAsync(reinterpret_cast<void**>(&t->trace), n, t->stream));
        CK(cudaMemsetAsync(t->trace, 0, n, t->stream));
    } else if (!enable && t->trace) {
        CK(cudaFreeAsync(t->trace, t->stream));
        t->trace = nullptr;
    }
    t->pdev.trace = t->trace;
    t->hdesc.plan.trace = t->trace;
    t->tplan.trace = t->trace;
    if (t->tiles && t->tplan.jobs)
        CK(cudaMemcpyAsync(t->dtp, &t->tplan, sizeof(TilePlan), cudaMemcpyHostToDevice, t->stream));
    CK(cudaMemcpyAsync(t->ddesc, &t->hdesc, sizeof(InstDesc), cudaMemcpyHostToDevice, t->stream));
    CK(cudaStreamSynchronize(t->stream));
    return RKR_OK;
}

int64_t rkr_debug_trace_items(const rkr_table* t) {
    return (t && t->trace) ? rkr_trace_slots(t) : 0;
}

rkr_status rkr_debug_trace_read(const rkr_table* t, uint64_t* out, int32_t* item_k,
                                int32_t* item_j) {
    if (!t || !t->trace) return fail(RKR_ERR_ARGUMENT, "tracing not enabled");
    DeviceGuard dg(t->device);
    CK(cudaStreamSynchronize(t->stream));
    CK(cudaMemcpy(out, t->trace, (size_t)rkr_trace_slots(t) * 48, cudaMemcpyDeviceToHost));
    if (t->tiles) {  // one slot per (diagonal k, tile j), k-major
        for (int64_t q = 0; q < rkr_trace_slots(t); ++q) {
            if (item_k) item_k[q] = (int32_t)(q / t->tplan.T);
            if (item_j) item_j[q] = (int32_t)(q % t->tplan.T);
        }
        return RKR_OK;
    }
    // item -> (k, j) from the host copy of the plan
    const PersistPlan& p = t->plan;
    for (size_t e = 0; e < p.start.size(); ++e) {
        const int64_t n = t->g.L - p.k[e];
        for (int64_t i = 0; i < n; ++i) {
            if (item_k) item_k[p.start[e] + i] = p.k[e];
            if (item_j) item_j[p.start[e] + i] = p.g[e];
        }
    }
    return RKR_OK;
}

void* rkr_table_stream(const rkr_table* t) { return t ? (void*)t->stream : nullptr; }

int64_t rkr_table_h2d_bytes(const rkr_table* t) { return t ? (int64_t)t->menu_bytes : 0; }

int64_t rkr_table_device_bytes(const rkr_table* t) { return t ? (int64_t)t->block_bytes : 0; }

rkr_status rkr_first_feasible(const rkr_table* t, int32_t s, int32_t tt, int32_t* m_out) {
    rkr_status st = check_cell(t, s, tt);
    if (st) return st;
    if (!m_out) return fail(RKR_ERR_ARGUMENT, "null output");
    DeviceGuard dg(t->device);
    int32_t* dm = reinterpret_cast<int32_t*>(t->dout);
    const int32_t big = 0x7fffffff;
    CK(cudaMemcpyAsync(dm, &big, 4, cudaMemcpyHostToDevice, t->stream));
    if (launch_first_feasible(t->ctx(), s, tt, dm))
        return cuda_fail(cudaGetLastError(), "first_feasible launch");
    int32_t hm = big;
    CK(cudaMemcpyAsync(&hm, dm, 4, cudaMemcpyDeviceToHost, t->stream));
    CK(cudaStreamSynchronize(t->stream));
    *m_out = hm == big ? -1 : hm;
    return RKR_OK;
}

rkr_status rkr_table_sync(const rkr_table* t) {
    if (!t) return fail(RKR_ERR_ARGUMENT, "null table");
    DeviceGuard dg(t->device);
    CK(cudaStreamSynchronize(t->stream));
    return RKR_OK;
}

rkr_status rkr_solve_chain(const rkr_menu* menu, int64_t budget_bytes, int32_t units,
                           const rkr_exec* exec, rkr_op* ops, int64_t cap, int64_t* n_ops,
                           int64_t* opt_time, int64_t* unit_out, int32_t* m_top_out,
                           int64_t* min_feasible) {
    if (!menu || !n_ops || !opt_time || !unit_out || !m_top_out || !min_feasible)
        return fail(RKR_ERR_ARGUMENT, "null argument");
    *n_ops = 0;
    *min_feasible = -1;
    int64_t unit, bu;
    rkr_status st = rkr_quantize(budget_bytes, units, &unit, &bu);        // :257
    if (st) return st;
    if (menu->n_blocks <= 0 || !menu->act_sizes)
        return fail(RKR_ERR_INVALID, "empty option menu");
    const int64_t a0_u = to_units(menu->act_sizes[0], unit);              // :258
    const int64_t m_top = bu - a0_u;                                       // :259
    if (m_top < 0) return fail(RKR_ERR_INFEASIBLE, "budget cannot hold the chain input");
    if (m_top > 0x7ffffffe) return fail(RKR_ERR_INVALID, "budget slots exceed int range");
    rkr_table* t = nullptr;
    PhaseTimer pt(exec);  // host-side enqueue costs (no synchronisation)
    st = prepare_table(menu, unit, (int32_t)m_top, exec, 0, &t);          // :262
    pt.mark("solve: prepare_table (+H2D, programs)");
    if (st) return st;
    const int L = t->g.L;
    // fill + one device walk from the top cell (fused into the K1t launch):
    // its first read is opt(0, L-1, m_top) (chain_dp.hpp:264), returned with
    // the ops, so a feasible solve needs a single host synchronisation
    st = rkr_table_refill_walk(t, 0, L - 1, (int32_t)m_top);
    pt.mark("solve: fill + walk enqueued");
    if (st == RKR_OK) st = rkr_backtrack_fetch(t, ops, cap, n_ops);
    pt.mark("solve: fetch (sync + D2H)");
    const int64_t best = t->hout[4];
    if (st != RKR_OK && best < RKR_INF_TIME) {
        rkr_table_destroy(t);
        return st;
    }
    if (best >= RKR_INF_TIME) *n_ops = 0;
    if (best >= RKR_INF_TIME) {                                            // :265-288
        int64_t capu = 0;
        for (int i = 0; i < L; ++i) {
            int64_t worst = 0;
            for (int o = menu->option_offsets[i]; o < menu->option_offsets[i + 1]; ++o)
                worst = std::max({worst, to_units(menu->peak_fwd[o], unit),
                                  to_units(menu->peak_bwd[o], unit),
                                  to_units(menu->save_mem[o], unit)});
            capu += worst;
        }
        for (int i = 0; i <= L; ++i) capu += 2 * to_units(menu->act_sizes[i], unit);
        rkr_table_destroy(t);
        if (capu > 0x7ffffffe) return fail(RKR_ERR_INVALID, "feasibility cap exceeds int range");
        rkr_table* wide = nullptr;
        st = rkr_table_create(menu, unit, (int32_t)capu, exec, &wide);
        if (st) return st;
        int32_t m = -1;
        st = rkr_first_feasible(wide, 0, L - 1, &m);
        rkr_table_destroy(wide);
        if (st) return st;
        if (m >= 0) *min_feasible = (m + a0_u) * unit;
        return fail(RKR_ERR_INFEASIBLE, "budget of %lld bytes is infeasible for this chain",
                    (long long)budget_bytes);
    }
    *opt_time = best;
    *unit_out = unit;
    *m_top_out = (int32_t)m_top;
    rkr_table_destroy(t);
    pt.mark("solve: destroy");
    return st;
}

}  // extern "C"

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

namespace {

void free_batch(rkr_batch* b) {
    if (!b) return;
    DeviceGuard dg(b->device);
    if (b->owns_tables)
        for (rkr_table* t : b->tables) free_table(t);
    if (b->block) cudaFreeAsync(b->block, b->stream);
    if (b->mblock) cudaFreeAsync(b->mblock, b->stream);
    if (b->wblock) cudaFreeAsync(b->wblock, b->stream);
    delete b;
}

rkr_status batch_zero(rkr_batch* b) {
    CK(cudaMemsetAsync(b->counter, 0, b->state_bytes, b->stream));
    return RKR_OK;
}

rkr_status batch_launch(rkr_batch* b) {
    if (b->tiles) {
        if (launch_fill_tiles_batch(b->ddesc, b->dtps, b->djobs, (int)b->hjobs.size(),
                                    reinterpret_cast<unsigned int*>(b->counter), b->proto,
                                    b->stream))
            return cuda_fail(cudaGetLastError(), "tile batch launch");
        return RKR_OK;
    }
    if (launch_fill_batch(b->ddesc, nullptr, b->lplan, b->width, b->R, b->kcap, b->ocap,
                          b->counter, b->stream))
        return cuda_fail(cudaGetLastError(), "batch fill launch");
    return RKR_OK;
}

rkr_status batch_fill(rkr_batch* b) {
    CK(cudaMemsetAsync(b->counter, 0, b->state_bytes, b->stream));
    if (b->tiles) {
        if (launch_fill_tiles_batch(b->ddesc, b->dtps, b->djobs, (int)b->hjobs.size(),
                                    reinterpret_cast<unsigned int*>(b->counter), b->proto,
                                    b->stream))
            return cuda_fail(cudaGetLastError(), "tile batch launch");
        return RKR_OK;
    }
    if (launch_fill_batch(b->ddesc, nullptr, b->lplan, b->width, b->R, b->kcap, b->ocap,
                          b->counter, b->stream))
        return cuda_fail(cudaGetLastError(), "batch fill launch");
    return RKR_OK;
}

// Allocate a batch's descriptor array, merged plan and state (counter, done
// flags and halo counters of every table) and fill the host descriptors
// (b->hd); batch_upload copies them to the device.
rkr_status batch_layout(rkr_batch* b) {
    const int n = (int)b->tables.size();
    b->stream = b->tables[0]->stream;
    b->width = b->tables[0]->width;
    size_t flags = 0, halos = 0;
    for (rkr_table* t : b->tables) {
        b->kcap = std::max(b->kcap, t->g.L - 1);
        b->ocap = std::max(b->ocap, t->hm.max_opts);
        flags += (size_t)t->g.L * t->flag_cols;
        halos += (size_t)t->g.L;
    }
    // merged launch order: tables advance their wavefronts together
    std::vector<const PersistPlan*> plans;
    std::vector<int32_t> Ls;
    for (rkr_table* t : b->tables) {
        plans.push_back(&t->plan);
        Ls.push_back(t->g.L);
    }
    merge_plans(plans, Ls, b->hp);
    const size_t np = b->hp.start.size();
    b->desc_bytes = (size_t)round_up((int64_t)(sizeof(InstDesc) * n), 256);
    b->o_inst = round_up((int64_t)(np * 8), 256);
    b->o_k = b->o_inst + round_up((int64_t)(np * 4), 256);
    b->o_j = b->o_k + round_up((int64_t)(np * 4), 256);
    b->plan_bytes = b->o_j + round_up((int64_t)(np * 4), 256);
    if (b->tiles) {
        // job queue: tables by decreasing work (the long ones start first),
        // each table's tiles ascending (a job only waits on earlier ones)
        std::vector<int> order(n);
        for (int i = 0; i < n; ++i) order[i] = i;
        auto work = [&](int i) {
            const rkr_table* t = b->tables[i];
            return (double)t->g.L * t->g.L * (t->g.M + 1) * (t->g.L + t->hm.max_opts);
        };
        if (!b->ordered)  // (budget shards keep chain order: shard r+1 waits on shard r)
            std::stable_sort(order.begin(), order.end(), [&](int x, int y) { return work(x) > work(y); });
        b->hjobs.clear();
        for (int i : order)
            for (int jt = 0; jt < b->tables[i]->tplan.T; ++jt) b->hjobs.push_back(make_int2(i, jt));
        b->tps_bytes = (size_t)round_up((int64_t)(sizeof(TilePlan) * n), 256);
        b->jobs_bytes = (size_t)round_up((int64_t)(sizeof(int2) * b->hjobs.size()), 256);
    }
    const size_t extra = b->tps_bytes + b->jobs_bytes;
    b->state_bytes = 8 + (flags + halos) * sizeof(int);
    CK(cudaMallocAsync(&b->block, b->desc_bytes + b->plan_bytes + extra + b->state_bytes,
                       b->stream));
    unsigned char* base = static_cast<unsigned char*>(b->block);
    b->ddesc = reinterpret_cast<InstDesc*>(base);
    unsigned char* pb = base + b->desc_bytes;
    b->lplan.start = reinterpret_cast<const int64_t*>(pb);
    b->lplan.inst = reinterpret_cast<const int32_t*>(pb + b->o_inst);
    b->lplan.k = reinterpret_cast<const int32_t*>(pb + b->o_k);
    b->lplan.j = reinterpret_cast<const int32_t*>(pb + b->o_j);
    b->lplan.n = (int32_t)np;
    b->lplan.total = b->hp.total;
    b->dtps = reinterpret_cast<TilePlan*>(base + b->desc_bytes + b->plan_bytes);
    b->djobs = reinterpret_cast<int2*>(base + b->desc_bytes + b->plan_bytes + b->tps_bytes);
    b->counter = reinterpret_cast<unsigned long long*>(base + b->desc_bytes + b->plan_bytes + extra);
    int32_t* flag = reinterpret_cast<int32_t*>(base + b->desc_bytes + b->plan_bytes + extra + 8);
    int32_t* halo = flag + flags;
    b->hd.assign(n, InstDesc{});
    if (b->tiles) {
        // one shared-memory layout for every job: the tables' maxima (create)
        TilePlan& pr = b->proto;
        if (b->tune & RKR_TUNE_COMM_OFF) pr.comm = 0;
        pr.sm = tile_batch_smem(pr);
        b->htp.assign(n, TilePlan{});
    }
    int64_t item = 0;
    for (int32_t i = 0; i < n; ++i) {
        rkr_table* t = b->tables[i];
        b->hd[i] = t->hdesc;
        b->hd[i].plan.done = flag;
        b->hd[i].plan.trace = nullptr;
        b->hd[i].halo = halo;
        b->hd[i].item_base = item;
        if (b->tiles) {
            TilePlan tp = t->tplan;
            tp.done = flag;
            tp.trace = nullptr;
            tp.walk = 0;
            tp.fin = nullptr;
            tp.comm = b->proto.comm;
            tp.split = 0;  // measured slower for batches (throughput-bound)
            tp.stream = 0;
            tp.sm = b->proto.sm;
            b->htp[i] = tp;
        }
        flag += (size_t)t->g.L * t->flag_cols;
        halo += t->g.L;
        item += t->plan.total;
    }
    b->total = item;
    return RKR_OK;
}

// Deferred tables of a batch: one menu region + one work region for all,
// every menu blob staged into one pinned buffer, one H2D copy.
rkr_status batch_tables_upload(rkr_batch* b) {
    b->stream = b->tables[0]->stream;
    std::vector<size_t> mo, wo;
    size_t mt = 0, wt = 0;
    for (rkr_table* t : b->tables) {
        mo.push_back(mt);
        wo.push_back(wt);
        mt += (size_t)round_up((int64_t)t->menu_bytes, 256);
        wt += (size_t)round_up((int64_t)t->work_bytes, 256);
    }
    CK(cudaMallocAsync(&b->mblock, mt, b->stream));
    CK(cudaMallocAsync(&b->wblock, wt, b->stream));
    unsigned char* mb = static_cast<unsigned char*>(b->mblock);
    unsigned char* wb = static_cast<unsigned char*>(b->wblock);
    for (size_t i = 0; i < b->tables.size(); ++i) {
        rkr_table* t = b->tables[i];
        t->block = mb + mo[i];
        bind_block(t, mb + mo[i], wb + wo[i]);
    }
    void* stage = nullptr;
    CK(t_stage.get(mt, &stage));
    unsigned char* sb = static_cast<unsigned char*>(stage);
    // staged and copied in chunks of ~16 MB: the DMA of one chunk overlaps
    // the (16-thread) staging of the next
    const int nt = (int)b->tables.size();
    constexpr size_t kChunk = size_t(16) << 20;
    for (int i0 = 0; i0 < nt;) {
        int i1 = i0 + 1;
        while (i1 < nt && mo[i1] - mo[i0] < kChunk) ++i1;
        parallel_for(i1 - i0, [&](int i) { stage_menu(b->tables[i0 + i], sb + mo[i0 + i]); });
        const size_t end = i1 < nt ? mo[i1] : mt;
        CK(cudaMemcpyAsync(mb + mo[i0], sb + mo[i0], end - mo[i0], cudaMemcpyHostToDevice,
                           b->stream));
        i0 = i1;
    }
    CK(cudaEventRecord(t_stage.done, b->stream));
    return RKR_OK;
}

rkr_status batch_upload(rkr_batch* b) {
    const int n = (int)b->tables.size();
    const size_t np = b->hp.start.size();
    const size_t up = b->desc_bytes + b->plan_bytes + b->tps_bytes + b->jobs_bytes;
    void* stage = nullptr;
    CK(t_desc.get(up, &stage));
    unsigned char* sb = static_cast<unsigned char*>(stage);
    std::memcpy(sb, b->hd.data(), sizeof(InstDesc) * n);
    unsigned char* pb = sb + b->desc_bytes;
    std::memcpy(pb, b->hp.start.data(), np * 8);
    std::memcpy(pb + b->o_inst, b->hp.inst.data(), np * 4);
    std::memcpy(pb + b->o_k, b->hp.k.data(), np * 4);
    std::memcpy(pb + b->o_j, b->hp.j.data(), np * 4);
    if (b->tiles) {
        std::memcpy(pb + b->plan_bytes, b->htp.data(), sizeof(TilePlan) * n);
        std::memcpy(pb + b->plan_bytes + b->tps_bytes, b->hjobs.data(),
                    sizeof(int2) * b->hjobs.size());
    }
    CK(cudaMemcpyAsync(b->block, stage, up, cudaMemcpyHostToDevice, b->stream));
    CK(cudaEventRecord(t_desc.done, b->stream));
    return RKR_OK;
}

rkr_status batch_create_impl(const rkr_menu* const* menus, const int64_t* units,
                             const int32_t* m_max, int32_t n, const rkr_exec* exec,
                             rkr_batch** out) {
    if (!out || !menus || !units || !m_max) return fail(RKR_ERR_ARGUMENT, "null argument");
    *out = nullptr;
    if (n < 1) return fail(RKR_ERR_ARGUMENT, "empty batch");
    int32_t min_m = INT32_MAX;
    for (int32_t i = 0; i < n; ++i) {
        if (m_max[i] < 0) return fail(RKR_ERR_INVALID, "m_max must be >= 0");
        min_m = std::min(min_m, m_max[i]);
    }
    rkr_exec ex{};
    if (exec) ex = *exec;
    const int kreq = exec ? exec->kernel : RKR_KERNEL_PERSISTENT;
    bool want_tiles = kreq != RKR_KERNEL_QUEUE && kreq != RKR_KERNEL_DIAGONAL;
    if (ex.tune & RKR_TUNE_BATCH_QUEUE) want_tiles = false;
    // One pass normally: every table's host side prepared in parallel as
    // budget-tile jobs (K1t).  A common cost width is needed (32 only if every
    // table's overflow proof holds) and the batch-wide shared-memory layout
    // must fit; otherwise a second pass prepares them for the row-segment
    // queue (K1p), in the common width.
    rkr_batch* b = nullptr;
    PhaseTimer pt0(exec);
    for (int attempt = want_tiles ? 0 : 1; attempt < 2; ++attempt) {
        ex.kernel = attempt == 0 ? RKR_KERNEL_TILES : RKR_KERNEL_QUEUE;
        b = new rkr_batch();
        b->device = ex.device;
        b->R = persistent_choose_r(min_m);
        b->tune = ex.tune;
        b->tiles = attempt == 0;
        DeviceGuard dg0(b->device);
        std::vector<rkr_table*> ts(n, nullptr);
        std::vector<rkr_status> sts(n, RKR_OK);
        std::vector<std::string> errs(n);
        parallel_for(n, [&](int i) {
            sts[i] = prepare_table(menus[i], units[i], m_max[i], &ex, b->R, &ts[i], nullptr,
                                   attempt == 0, /*defer=*/true);
            if (sts[i] != RKR_OK) errs[i] = g_err;
        });
        rkr_status bad = RKR_OK;
        for (int32_t i = 0; i < n && bad == RKR_OK; ++i)
            if (sts[i] != RKR_OK) {
                bad = sts[i];
                g_err = errs[i];
            }
        for (rkr_table* t : ts)
            if (t) b->tables.push_back(t);
        if (bad != RKR_OK && !(attempt == 0 && bad == RKR_ERR_INVALID)) {
            free_batch(b);
            return bad;
        }
        bool redo = bad != RKR_OK;  // a table does not fit K1t
        bool mixed = false;         // tables of both widths: all must run the wider one
        for (rkr_table* t : b->tables) mixed = mixed || t->width != b->tables[0]->width;
        if (attempt == 0 && !redo) {
            TilePlan& pr = b->proto;
            pr = b->tables[0]->tplan;
            for (rkr_table* t : b->tables) {
                pr.L = std::max(pr.L, t->tplan.L);
                pr.nq = std::max(pr.nq, t->tplan.nq);
                pr.ocap = std::max(pr.ocap, t->tplan.ocap);
                pr.cap = std::max(pr.cap, t->tplan.cap);
            }
            pr.comm = 1;  // every job is a latency-bound tile walk
            pr.stream = 0;  // batches stage their programs (else K1p)
            redo = tile_batch_smem(pr).total > 220 * 1024;
        }
        if (attempt == 1 && mixed && ex.width != RKR_WIDTH_64) {
            free_batch(b);  // the queue pass again, every table 64-bit
            b = nullptr;
            ex.width = RKR_WIDTH_64;
            --attempt;
            continue;
        }
        if (attempt == 0 && (redo || mixed)) {
            free_batch(b);
            b = nullptr;
            g_err.clear();
            if (mixed) ex.width = RKR_WIDTH_64;
            continue;
        }
        break;
    }
    pt0.mark("batch: prepare_table x n");
    DeviceGuard dg(b->device);
    PhaseTimer pt(exec);
    pt.st = b->tables[0]->stream;
    pt.mark("batch: host tables");
    rkr_status st = batch_tables_upload(b);
    pt.mark("batch: menus staged + H2D");
    if (st == RKR_OK) st = batch_layout(b);
    if (st == RKR_OK) st = batch_upload(b);
    pt.mark("batch: layout + descriptors");
    if (st == RKR_OK) {  // every table's cell programs and pads: one launch
        int64_t max_rows = 0;
        for (rkr_table* t : b->tables) max_rows = std::max(max_rows, t->g.rows);
        if (launch_prep_programs_batch(b->ddesc, n, max_rows, b->tables[0]->width, b->stream))
            st = cuda_fail(cudaGetLastError(), "batch program launch");
    }
    pt.mark("batch: programs");
    if (st == RKR_OK) st = batch_fill(b);
    pt.mark("batch: fill");
    if (st != RKR_OK) {
        free_batch(b);
        return st;
    }
    *out = b;
    return RKR_OK;
}

}  // namespace

extern "C" {

rkr_status rkr_batch_create(const rkr_menu* const* menus, const int64_t* units,
                            const int32_t* m_max, int32_t n, const rkr_exec* exec,
                            rkr_batch** out) {
    return batch_create_impl(menus, units, m_max, n, exec, out);
}

int32_t rkr_batch_size(const rkr_batch* b) { return b ? (int32_t)b->tables.size() : 0; }

rkr_table* rkr_batch_table(rkr_batch* b, int32_t i) {
    if (!b || i < 0 || i >= (int32_t)b->tables.size()) return nullptr;
    return b->tables[i];
}

rkr_status rkr_batch_refill(rkr_batch* b) {
    if (!b) return fail(RKR_ERR_ARGUMENT, "null batch");
    DeviceGuard dg(b->device);
    return batch_fill(b);
}

void* rkr_batch_stream(const rkr_batch* b) { return b ? (void*)b->stream : nullptr; }

rkr_status rkr_batch_sync(const rkr_batch* b) {
    if (!b) return fail(RKR_ERR_ARGUMENT, "null batch");
    DeviceGuard dg(b->device);
    CK(cudaStreamSynchronize(b->stream));
    return RKR_OK;
}

void rkr_batch_destroy(rkr_batch* b) { free_batch(b); }

// remat::solve_chain for many budgets of one chain (cmd_sweep's loop,
// remat.cpp:240-255) with every table in one batched fill, the top cells
// gathered in one launch, the schedules walked in one launch (a thread per
// budget) and the infeasible budgets' min-feasible search batched the same way.
// rkr_sweep over budgets whose chains may differ: mfor[i] is budget i's menu
// (one batch, one fill launch for all of them).
static rkr_status sweep_impl(const rkr_menu* const* mfor, const int64_t* budgets, int32_t n,
                             int32_t units, const rkr_exec* exec, int32_t* status,
                             int64_t* opt_time, int64_t* unit_out, int32_t* m_top_out,
                             int64_t* min_feasible, rkr_op* ops, int64_t ops_cap,
                             int64_t* ops_offsets) {
    if (!mfor || !budgets || !status || !opt_time || !unit_out || !m_top_out || !min_feasible ||
        !ops_offsets)
        return fail(RKR_ERR_ARGUMENT, "null argument");
    if (n < 1) return fail(RKR_ERR_ARGUMENT, "empty sweep");
    int Lmax = 0;
    for (int32_t i = 0; i < n; ++i) {
        if (!mfor[i]) return fail(RKR_ERR_ARGUMENT, "null menu");
        if (mfor[i]->n_blocks <= 0 || !mfor[i]->act_sizes)
            return fail(RKR_ERR_INVALID, "empty option menu");
        Lmax = std::max(Lmax, (int)mfor[i]->n_blocks);
    }
    std::vector<int64_t> unit(n), a0u(n);
    std::vector<int32_t> mtop(n, -1);
    std::vector<int32_t> idx;  // budgets with a table
    for (int32_t i = 0; i < n; ++i) {
        int64_t bu;
        rkr_status st = rkr_quantize(budgets[i], units, &unit[i], &bu);       // :257
        if (st) return st;
        a0u[i] = to_units(mfor[i]->act_sizes[0], unit[i]);                    // :258
        const int64_t mt = bu - a0u[i];                                        // :259
        status[i] = RKR_ERR_INFEASIBLE;
        opt_time[i] = 0;
        unit_out[i] = unit[i];
        m_top_out[i] = 0;
        min_feasible[i] = -1;
        if (mt < 0) continue;                                                  // :260-261
        if (mt > 0x7ffffffe) return fail(RKR_ERR_INVALID, "budget slots exceed int range");
        mtop[i] = (int32_t)mt;
        idx.push_back(i);
    }
    const int nb = (int)idx.size();
    std::vector<int64_t> top(nb, kInf64);
    std::vector<int64_t> walk_out(8 * (size_t)nb, 0);
    int64_t cap_each = 0;
    const int32_t* walk_ops = nullptr;  // pinned readback of every table's walk
    std::vector<std::vector<rkr_op>> big(nb);  // schedules that overflowed the batch slots
    if (nb > 0) {
        std::vector<const rkr_menu*> ms(nb);
        std::vector<int64_t> us(nb);
        std::vector<int32_t> mm(nb);
        for (int q = 0; q < nb; ++q) {
            ms[q] = mfor[idx[q]];
            us[q] = unit[idx[q]];
            mm[q] = mtop[idx[q]];
        }
        rkr_batch* b = nullptr;
        PhaseTimer spt(exec);
        rkr_status st = rkr_batch_create(ms.data(), us.data(), mm.data(), nb, exec, &b);
        if (st) return st;
        DeviceGuard dg(b->device);
        // scratch: m_at[nb] | active[nb] | tops[nb] | walk out[4 nb] | ops[nb * cap]
        cap_each = std::max<int64_t>(256, 16 * (int64_t)Lmax);
        const size_t bytes = (size_t)nb * (4 + 1 + 8 + 64) + 64 + (size_t)nb * cap_each * 12;
        void* scr = nullptr;
        cudaError_t e = cudaMallocAsync(&scr, bytes, b->stream);
        if (e != cudaSuccess) {
            rkr_batch_destroy(b);
            return cuda_fail(e, "sweep scratch");
        }
        unsigned char* p = static_cast<unsigned char*>(scr);
        int64_t* d_tops = reinterpret_cast<int64_t*>(p);
        int64_t* d_wout = d_tops + nb;
        int32_t* d_ops = reinterpret_cast<int32_t*>(d_wout + 8 * (size_t)nb);
        int32_t* d_mat = d_ops + (size_t)nb * cap_each * 3;
        uint8_t* d_act = reinterpret_cast<uint8_t*>(d_mat + nb);
        std::vector<uint8_t> act(nb, 1);
        // One round trip: every table walks from its top cell (a walk
        // reads opt(0, L-1, m_top) first and returns it, chain_dp.hpp:264;
        // an infinite top ends the walk at once), and the walk records and
        // op slots come back together through pinned memory.
        (void)d_tops;
        auto run = [&]() -> rkr_status {
            CK(cudaMemcpyAsync(d_mat, mm.data(), 4 * (size_t)nb, cudaMemcpyHostToDevice, b->stream));
            CK(cudaMemsetAsync(d_act, 1, nb, b->stream));
            if (launch_batch_walk(b->ddesc, d_mat, d_act, nb, b->width, d_ops, cap_each, d_wout,
                                  b->stream))
                return cuda_fail(cudaGetLastError(), "walk launch");
            const size_t rec = 64 * (size_t)nb, opsb = (size_t)nb * cap_each * 12;
            void* pin = nullptr;
            CK(t_sweep.get(rec + opsb, &pin));
            CK(cudaMemcpyAsync(pin, d_wout, rec, cudaMemcpyDeviceToHost, b->stream));
            CK(cudaMemcpyAsync(static_cast<char*>(pin) + rec, d_ops, opsb, cudaMemcpyDeviceToHost,
                               b->stream));
            CK(cudaStreamSynchronize(b->stream));
            std::memcpy(walk_out.data(), pin, rec);
            walk_ops = reinterpret_cast<const int32_t*>(static_cast<char*>(pin) + rec);
            for (int q = 0; q < nb; ++q) {
                top[q] = walk_out[8 * q + 4];
                act[q] = top[q] < kInf64 ? 1 : 0;   // :264-265
            }
            return RKR_OK;
        };
        spt.st = b->stream;
        spt.mark("sweep: create (incl fill)");
        st = run();
        spt.mark("sweep: tops + walks + D2H");
        cudaFreeAsync(scr, b->stream);
        // schedules longer than cap_each: walk those tables again on their own
        for (int q = 0; q < nb && st == RKR_OK; ++q) {
            if (!act[q] || walk_out[8 * q] <= cap_each) continue;
            big[q].resize((size_t)walk_out[8 * q]);
            int64_t nn = 0;
            st = rkr_backtrack(b->tables[q], 0, ms[q]->n_blocks - 1, mm[q], big[q].data(),
                               (int64_t)big[q].size(), &nn);
        }
        rkr_batch_destroy(b);
        spt.mark("sweep: destroy");
        if (st) return st;
    }
    // infeasible budgets with a table: the wide-table min-feasible search (:265-288)
    std::vector<int> inf_q;
    for (int q = 0; q < nb; ++q)
        if (top[q] >= kInf64) inf_q.push_back(q);
    if (!inf_q.empty()) {
        const int ni = (int)inf_q.size();
        std::vector<const rkr_menu*> ms(ni);
        std::vector<int64_t> us(ni);
        std::vector<int32_t> caps(ni);
        for (int r = 0; r < ni; ++r) {
            const int i = idx[inf_q[r]];
            const rkr_menu* menu = mfor[i];
            const int L = menu->n_blocks;
            ms[r] = menu;
            const int64_t u = unit[i];
            int64_t capu = 0;
            for (int bl = 0; bl < L; ++bl) {
                int64_t worst = 0;
                for (int o = menu->option_offsets[bl]; o < menu->option_offsets[bl + 1]; ++o)
                    worst = std::max({worst, to_units(menu->peak_fwd[o], u),
                                      to_units(menu->peak_bwd[o], u), to_units(menu->save_mem[o], u)});
                capu += worst;
            }
            for (int bl = 0; bl <= L; ++bl) capu += 2 * to_units(menu->act_sizes[bl], u);
            if (capu > 0x7ffffffe) return fail(RKR_ERR_INVALID, "feasibility cap exceeds int range");
            us[r] = u;
            caps[r] = (int32_t)capu;
        }
        rkr_batch* w = nullptr;
        rkr_status st = rkr_batch_create(ms.data(), us.data(), caps.data(), ni, exec, &w);
        if (st) return st;
        DeviceGuard dg(w->device);
        int32_t* d_ff = nullptr;
        std::vector<int32_t> ff(ni, -1);
        cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&d_ff), 4 * (size_t)ni, w->stream);
        if (e == cudaSuccess && launch_batch_first_feasible(w->ddesc, ni, w->width, d_ff, w->stream))
            e = cudaGetLastError();
        if (e == cudaSuccess)
            e = cudaMemcpyAsync(ff.data(), d_ff, 4 * (size_t)ni, cudaMemcpyDeviceToHost, w->stream);
        if (e == cudaSuccess) e = cudaStreamSynchronize(w->stream);
        if (d_ff) cudaFreeAsync(d_ff, w->stream);
        rkr_batch_destroy(w);
        if (e != cudaSuccess) return cuda_fail(e, "min-feasible search");
        for (int r = 0; r < ni; ++r) {
            const int i = idx[inf_q[r]];
            if (ff[r] >= 0) min_feasible[i] = (ff[r] + a0u[i]) * unit[i];       // :282
        }
    }
    // results and schedules, in budget order
    int64_t off = 0;
    ops_offsets[0] = 0;
    std::vector<int> qof(n, -1);
    for (int q = 0; q < nb; ++q) qof[idx[q]] = q;
    rkr_status result = RKR_OK;
    for (int32_t i = 0; i < n; ++i) {
        const int q = qof[i];
        int64_t cnt = 0;
        if (q >= 0 && top[q] < kInf64) {
            status[i] = RKR_OK;
            opt_time[i] = top[q];
            m_top_out[i] = mtop[i];
            cnt = walk_out[8 * q];
            if (walk_out[8 * q + 1] != 0) {
                result = fail(RKR_ERR_INFEASIBLE, "schedule walk failed for budget %d", i);
                cnt = 0;
            }
            for (int64_t o = 0; o < cnt; ++o)
                if (ops && off + o < ops_cap) {
                    if (!big[q].empty()) {
                        ops[off + o] = big[q][o];
                    } else {
                        const int32_t* src = &walk_ops[3 * ((size_t)q * cap_each + o)];
                        ops[off + o] = rkr_op{src[0], src[1], src[2]};
                    }
                }
        }
        off += cnt;
        ops_offsets[i + 1] = off;
    }
    if (result == RKR_OK && off > ops_cap)
        return fail(RKR_ERR_CAPACITY, "sweep schedules need %lld ops", (long long)off);
    return result;
}

rkr_status rkr_sweep(const rkr_menu* menu, const int64_t* budgets, int32_t n, int32_t units,
                     const rkr_exec* exec, int32_t* status, int64_t* opt_time, int64_t* unit_out,
                     int32_t* m_top_out, int64_t* min_feasible, rkr_op* ops, int64_t ops_cap,
                     int64_t* ops_offsets) {
    if (!menu) return fail(RKR_ERR_ARGUMENT, "null argument");
    if (n < 1) return fail(RKR_ERR_ARGUMENT, "empty sweep");
    std::vector<const rkr_menu*> mfor((size_t)n, menu);
    return sweep_impl(mfor.data(), budgets, n, units, exec, status, opt_time, unit_out, m_top_out,
                      min_feasible, ops, ops_cap, ops_offsets);
}

rkr_status rkr_sweep_chains(const rkr_menu* const* menus, const int32_t* n_budgets,
                            int32_t n_chains, const int64_t* budgets, int32_t units,
                            const rkr_exec* exec, int32_t* status, int64_t* opt_time,
                            int64_t* unit_out, int32_t* m_top_out, int64_t* min_feasible,
                            rkr_op* ops, int64_t ops_cap, int64_t* ops_offsets) {
    if (!menus || !n_budgets) return fail(RKR_ERR_ARGUMENT, "null argument");
    if (n_chains < 1) return fail(RKR_ERR_ARGUMENT, "no chains");
    std::vector<const rkr_menu*> mfor;
    for (int32_t c = 0; c < n_chains; ++c) {
        if (n_budgets[c] < 0) return fail(RKR_ERR_ARGUMENT, "negative budget count");
        mfor.insert(mfor.end(), (size_t)n_budgets[c], menus[c]);
    }
    if (mfor.size() > (size_t)INT32_MAX) return fail(RKR_ERR_ARGUMENT, "too many budgets");
    return sweep_impl(mfor.data(), budgets, (int32_t)mfor.size(), units, exec, status, opt_time,
                      unit_out, m_top_out, min_feasible, ops, ops_cap, ops_offsets);
}

}  // extern "C"

// ---------------------------------------------------------------------------
// Budget-axis sharding (config 5): one table split into contiguous budget
// ranges, each shard filled by the persistent kernel, halos pushed by the
// producing items straight into the next shard (peer memory across GPUs).
// ---------------------------------------------------------------------------
struct rkr_sharded {
    int n = 0, L = 0, M = 0, pad = 0, width = 32;
    std::vector<int32_t> lo, hi, dev;
    std::vector<rkr_table*> shards;
    std::vector<rkr_batch*> batches;   // one per device, shards in order
    ShardView* dview = nullptr;        // on shard 0's device
    int32_t* dops = nullptr;
    int64_t dops_cap = 0;
    int64_t* dout = nullptr;
    int32_t* dstack = nullptr;
};

namespace {

void free_sharded(rkr_sharded* sh) {
    if (!sh) return;
    for (rkr_batch* b : sh->batches) free_batch(b);
    for (rkr_table* t : sh->shards) free_table(t);
    if (!sh->shards.empty()) {
        DeviceGuard dg(sh->dev[0]);
        cudaDeviceSynchronize();
        cudaFree(sh->dview);
        cudaFree(sh->dops);
        cudaFree(sh->dout);
        cudaFree(sh->dstack);
    }
    delete sh;
}

rkr_status sharded_fill(rkr_sharded* sh) {
    for (rkr_batch* b : sh->batches) {
        DeviceGuard dg(b->device);
        rkr_status st = batch_zero(b);
        if (st) return st;
    }
    // every device's counters are zero before any shard can signal another
    for (rkr_batch* b : sh->batches) {
        DeviceGuard dg(b->device);
        CK(cudaStreamSynchronize(b->stream));
    }
    for (rkr_batch* b : sh->batches) {
        DeviceGuard dg(b->device);
        rkr_status st = batch_launch(b);
        if (st) return st;
    }
    return RKR_OK;
}

rkr_status sharded_create_impl(const rkr_menu* menu, int64_t unit, int32_t m_max, int32_t n,
                               const int32_t* devices, const rkr_exec* exec, rkr_sharded** out) {
    if (!out) return fail(RKR_ERR_ARGUMENT, "null output handle");
    *out = nullptr;
    if (n < 1 || n > 64) return fail(RKR_ERR_ARGUMENT, "n_shards must be in [1, 64]");
    if (m_max < 0) return fail(RKR_ERR_INVALID, "m_max must be >= 0");
    HostMenu h;
    rkr_status st = build_host_menu(menu, unit, h);
    if (st) return st;
    int64_t maxshift = 0;
    for (int64_t p : h.pack_chg) maxshift = std::max(maxshift, p);
    for (int32_t c = 1; c < h.L; ++c) maxshift = std::max(maxshift, h.act_u[c]);
    const int32_t pad = (int32_t)round_up(std::min<int64_t>(maxshift, (int64_t)m_max + 1), 8);
    const int32_t W = (m_max + 1) / n;
    if (n > 1 && W < std::max(pad, 1))
        return fail(RKR_ERR_INVALID,
                    "too many shards: each must own at least the halo of %d budget slots", pad);
    // Shards run as budget-tile jobs (K1t, one batch kernel per device) when
    // every shard qualifies; else the row-segment queue (K1p).
    const int R = persistent_choose_r(W - 1);
    rkr_sharded* sh = nullptr;
    bool tiles = !(exec && (exec->kernel == RKR_KERNEL_QUEUE || exec->kernel == RKR_KERNEL_DIAGONAL));
    for (int attempt = tiles ? 0 : 1; attempt < 2; ++attempt) {
        sh = new rkr_sharded();
        sh->n = n;
        sh->L = h.L;
        sh->M = m_max;
        sh->pad = pad;
        tiles = attempt == 0;
        int32_t jo = 0;
        bool redo = false;
        for (int r = 0; r < n; ++r) {
            const int32_t lo = r * W, hi = (r == n - 1) ? m_max + 1 : (r + 1) * W;
            rkr_exec ex{};
            if (exec) ex = *exec;
            ex.kernel = tiles ? RKR_KERNEL_TILES : RKR_KERNEL_QUEUE;
            if (devices) ex.device = devices[r];
            if (!ex.tile_rows) {  // every shard alike: from the slots one device runs
                int sms = 0;
                cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ex.device);
                int per_dev = devices ? 0 : n;
                for (int q = 0; devices && q < n; ++q) per_dev += devices[q] == devices[r];
                ex.tile_rows = tile_rows_for((int64_t)W * per_dev, sms, TileKnobs{ex.tune, 0});
            }
            if (devices && exec && exec->stream) ex.stream = nullptr;  // per-device library streams
            ShardSpec spec{lo, pad, jo};
            rkr_table* t = nullptr;
            st = prepare_table(menu, unit, hi - lo - 1, &ex, R, &t, &spec, /*batch_tiles=*/tiles);
            if (st == RKR_ERR_INVALID && tiles) {  // a shard does not fit K1t: all run K1p
                redo = true;
                break;
            }
            if (st) {
                free_sharded(sh);
                return st;
            }
            sh->shards.push_back(t);
            sh->lo.push_back(lo);
            sh->hi.push_back(hi);
            sh->dev.push_back(t->device);
            jo += t->plan.J;
        }
        if (redo) {
            free_sharded(sh);
            sh = nullptr;
            g_err.clear();
            continue;
        }
        break;
    }
    sh->width = sh->shards[0]->width;
    // peer access: producer shard -> next shard (halo stores), shard 0's
    // device -> every shard (the cross-shard walk)
    auto enable_peer = [&](int from, int to) -> rkr_status {
        if (from == to) return RKR_OK;
        int can = 0;
        cudaDeviceCanAccessPeer(&can, from, to);
        if (!can) return fail(RKR_ERR_CUDA, "GPU %d cannot access GPU %d (no peer path)", from, to);
        DeviceGuard dg(from);
        cudaError_t e = cudaDeviceEnablePeerAccess(to, 0);
        if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled)
            return cuda_fail(e, "cudaDeviceEnablePeerAccess");
        cudaGetLastError();
        return RKR_OK;
    };
    for (int r = 0; r < n && st == RKR_OK; ++r) {
        if (r + 1 < n) st = enable_peer(sh->dev[r], sh->dev[r + 1]);
        if (st == RKR_OK) st = enable_peer(sh->dev[0], sh->dev[r]);
    }
    if (st) {
        free_sharded(sh);
        return st;
    }
    // one batch per device (shards in chain order)
    std::vector<int> devs;
    for (int d : sh->dev)
        if (std::find(devs.begin(), devs.end(), d) == devs.end()) devs.push_back(d);
    std::vector<std::pair<int, int>> where(n);  // shard -> (batch, index)
    for (int d : devs) {
        rkr_batch* b = new rkr_batch();
        b->device = d;
        b->R = R;
        b->owns_tables = false;
        b->ordered = true;
        for (int r = 0; r < n; ++r)
            if (sh->dev[r] == d) {
                where[r] = {(int)sh->batches.size(), (int)b->tables.size()};
                b->tables.push_back(sh->shards[r]);
            }
        b->tiles = sh->shards[0]->tiles;
        if (b->tiles) {  // one shared-memory layout for every shard's jobs
            TilePlan& pr = b->proto;
            pr = b->tables[0]->tplan;
            for (rkr_table* t : b->tables) {
                pr.cap = std::max(pr.cap, t->tplan.cap);
                pr.stream = pr.stream || t->tplan.stream;
            }
            pr.comm = 1;
            pr.split = 0;
            pr.halo = 1;  // (one shard too: the kernel N shards run)
            pr.sm = tile_batch_smem(pr);
        }
        sh->batches.push_back(b);
        DeviceGuard dg(d);
        st = batch_layout(b);
        if (st) {
            free_sharded(sh);
            return st;
        }
    }
    for (int r = 0; r + 1 < n; ++r) {
        InstDesc& a = sh->batches[where[r].first]->hd[where[r].second];
        InstDesc& b2 = sh->batches[where[r + 1].first]->hd[where[r + 1].second];
        rkr_table* tn = sh->shards[r + 1];
        const PersistPlan& pr = sh->shards[r]->plan;
        const int32_t Wr = sh->hi[r] - sh->lo[r];
        a.next_opt = tn->opt;
        a.next_sr = tn->g.sr;
        a.next_halo = b2.halo;
        a.next_peer = sh->dev[r] != sh->dev[r + 1] ? 1 : 0;
        // producer tiles meeting the halo (K1t: 32-slot tiles; K1p: its segments)
        b2.halo_need = sh->shards[r]->tiles
                           ? sh->shards[r]->tplan.T - std::max(0, (Wr - pad) / sh->shards[r]->tplan.W)
                           : pr.J - std::max(0, (Wr - pad) / pr.TM);
    }
    for (rkr_batch* b : sh->batches) {
        DeviceGuard dg(b->device);
        st = batch_upload(b);
        if (st) {
            free_sharded(sh);
            return st;
        }
    }
    // walk views on shard 0's device
    {
        DeviceGuard dg(sh->dev[0]);
        std::vector<ShardView> v(n);
        for (int r = 0; r < n; ++r) {
            rkr_table* t = sh->shards[r];
            v[r] = ShardView{t->opt, t->arg, t->g.sr, t->g.sa, t->g.pad, sh->lo[r]};
        }
        CK(cudaMalloc(reinterpret_cast<void**>(&sh->dview), sizeof(ShardView) * n));
        CK(cudaMemcpy(sh->dview, v.data(), sizeof(ShardView) * n, cudaMemcpyHostToDevice));
        CK(cudaMalloc(reinterpret_cast<void**>(&sh->dout), 8 * sizeof(int64_t)));
        CK(cudaMalloc(reinterpret_cast<void**>(&sh->dstack), sizeof(int4) * (2 * (size_t)h.L + 16)));
    }
    for (rkr_batch* b : sh->batches) {
        DeviceGuard dg(b->device);
        CK(cudaStreamSynchronize(b->stream));  // programs, pads, descriptors in place
    }
    st = sharded_fill(sh);
    if (st) {
        free_sharded(sh);
        return st;
    }
    *out = sh;
    return RKR_OK;
}

int owner(const rkr_sharded* sh, int32_t m) {
    int q = 0;
    while (q + 1 < sh->n && m >= sh->lo[q + 1]) ++q;
    return q;
}

}  // namespace

extern "C" {

rkr_status rkr_sharded_create(const rkr_menu* menu, int64_t unit, int32_t m_max, int32_t n_shards,
                              const int32_t* devices, const rkr_exec* exec, rkr_sharded** out) {
    return sharded_create_impl(menu, unit, m_max, n_shards, devices, exec, out);
}

int32_t rkr_sharded_count(const rkr_sharded* sh) { return sh ? sh->n : 0; }

rkr_status rkr_sharded_range(const rkr_sharded* sh, int32_t i, int32_t* m_lo, int32_t* m_hi) {
    if (!sh || i < 0 || i >= sh->n || !m_lo || !m_hi) return fail(RKR_ERR_ARGUMENT, "bad shard");
    *m_lo = sh->lo[i];
    *m_hi = sh->hi[i];
    return RKR_OK;
}

rkr_table* rkr_sharded_shard(rkr_sharded* sh, int32_t i) {
    return (sh && i >= 0 && i < sh->n) ? sh->shards[i] : nullptr;
}

rkr_status rkr_sharded_refill(rkr_sharded* sh) {
    if (!sh) return fail(RKR_ERR_ARGUMENT, "null sharded table");
    return sharded_fill(sh);
}

rkr_status rkr_sharded_sync(const rkr_sharded* sh) {
    if (!sh) return fail(RKR_ERR_ARGUMENT, "null sharded table");
    for (rkr_batch* b : sh->batches) {
        DeviceGuard dg(b->device);
        CK(cudaStreamSynchronize(b->stream));
    }
    return RKR_OK;
}

rkr_status rkr_sharded_opt(const rkr_sharded* sh, int32_t s, int32_t t, int32_t m, int64_t* out) {
    if (!sh || !out) return fail(RKR_ERR_ARGUMENT, "null argument");
    if (m < 0) {
        *out = RKR_INF_TIME;
        return RKR_OK;
    }
    if (m > sh->M) m = sh->M;
    rkr_status st = rkr_sharded_sync(sh);
    if (st) return st;
    const int q = owner(sh, m);
    return rkr_table_opt(sh->shards[q], s, t, m - sh->lo[q], out);
}

rkr_status rkr_sharded_row(const rkr_sharded* sh, int32_t s, int32_t t, int64_t* opt, int8_t* kind,
                           int32_t* value) {
    if (!sh) return fail(RKR_ERR_ARGUMENT, "null sharded table");
    rkr_status st = rkr_sharded_sync(sh);
    if (st) return st;
    for (int q = 0; q < sh->n; ++q) {
        const int32_t lo = sh->lo[q];
        st = rkr_table_row(sh->shards[q], s, t, opt ? opt + lo : nullptr, kind ? kind + lo : nullptr,
                           value ? value + lo : nullptr);
        if (st) return st;
    }
    return RKR_OK;
}

rkr_status rkr_sharded_backtrack(rkr_sharded* sh, int32_t s, int32_t t, int32_t m, rkr_op* ops,
                                 int64_t cap, int64_t* n_ops) {
    if (!sh || !n_ops || (cap > 0 && !ops)) return fail(RKR_ERR_ARGUMENT, "null argument");
    if (s < 0 || t < s || t >= sh->L) return fail(RKR_ERR_ARGUMENT, "cell outside the table");
    rkr_status st = rkr_sharded_sync(sh);
    if (st) return st;
    DeviceGuard dg(sh->dev[0]);
    rkr_table* t0 = sh->shards[0];
    for (int attempt = 0; attempt < 2; ++attempt) {
        if (sh->dops_cap == 0) {
            sh->dops_cap = std::max<int64_t>(4096, 8 * (int64_t)sh->L + 64);
            CK(cudaMalloc(reinterpret_cast<void**>(&sh->dops), (size_t)sh->dops_cap * 12));
        }
        if (launch_walk_sharded(sh->dview, sh->n, t0->dm, sh->L, sh->M, sh->width, s, t, m,
                                sh->dops, sh->dops_cap, sh->dstack, sh->dout, t0->stream))
            return cuda_fail(cudaGetLastError(), "sharded walk launch");
        int64_t res[4];
        CK(cudaMemcpyAsync(res, sh->dout, sizeof res, cudaMemcpyDeviceToHost, t0->stream));
        CK(cudaStreamSynchronize(t0->stream));
        if (res[0] > sh->dops_cap) {
            cudaFree(sh->dops);
            sh->dops_cap = res[0];
            CK(cudaMalloc(reinterpret_cast<void**>(&sh->dops), (size_t)sh->dops_cap * 12));
            continue;
        }
        const int64_t ncopy = std::min(res[0], cap);
        if (ncopy > 0) CK(cudaMemcpy(ops, sh->dops, (size_t)ncopy * 12, cudaMemcpyDeviceToHost));
        *n_ops = res[0];
        if (res[1] == 2)
            return fail(RKR_ERR_INFEASIBLE, "no feasible schedule for blocks %lld..%lld",
                        (long long)res[2], (long long)res[3]);
        if (res[0] > cap) return fail(RKR_ERR_CAPACITY, "schedule needs %lld ops", (long long)res[0]);
        return RKR_OK;
    }
    return fail(RKR_ERR_CUDA, "sharded walk did not converge");
}

void rkr_sharded_destroy(rkr_sharded* sh) { free_sharded(sh); }

}  // extern "C"

// ---------------------------------------------------------------------------
// Multi-process budget sharding: one process per GPU (torchrun), shard r on
// rank r; the halo link to the next shard goes through CUDA IPC.
// ---------------------------------------------------------------------------
namespace {

struct ShardGeom {
    int32_t pad, W, R, TM;
    std::vector<int32_t> lo, hi, J, jo;
};

rkr_status shard_geometry(const rkr_menu* menu, int64_t unit, int32_t m_max, int32_t n,
                          ShardGeom& sg) {
    HostMenu h;
    rkr_status st = build_host_menu(menu, unit, h);
    if (st) return st;
    int64_t maxshift = 0;
    for (int64_t p : h.pack_chg) maxshift = std::max(maxshift, p);
    for (int32_t c = 1; c < h.L; ++c) maxshift = std::max(maxshift, h.act_u[c]);
    sg.pad = (int32_t)round_up(std::min<int64_t>(maxshift, (int64_t)m_max + 1), 8);
    sg.W = (m_max + 1) / n;
    if (n > 1 && sg.W < std::max(sg.pad, 1))
        return fail(RKR_ERR_INVALID,
                    "too many shards: each must own at least the halo of %d budget slots", sg.pad);
    sg.R = persistent_choose_r(sg.W - 1);
    sg.TM = 256 * sg.R;
    int32_t jo = 0;
    for (int r = 0; r < n; ++r) {
        const int32_t lo = r * sg.W, hi = (r == n - 1) ? m_max + 1 : (r + 1) * sg.W;
        sg.lo.push_back(lo);
        sg.hi.push_back(hi);
        sg.J.push_back((hi - lo + sg.TM - 1) / sg.TM);
        sg.jo.push_back(jo);
        jo += sg.J.back();
    }
    return RKR_OK;
}

}  // namespace

extern "C" {

rkr_status rkr_shard_create(const rkr_menu* menu, int64_t unit, int32_t m_max, int32_t n_shards,
                            int32_t shard, const rkr_exec* exec, rkr_table** out) {
    if (!out) return fail(RKR_ERR_ARGUMENT, "null output handle");
    *out = nullptr;
    if (n_shards < 1 || shard < 0 || shard >= n_shards)
        return fail(RKR_ERR_ARGUMENT, "shard %d of %d", shard, n_shards);
    if (m_max < 0) return fail(RKR_ERR_INVALID, "m_max must be >= 0");
    ShardGeom sg;
    rkr_status st = shard_geometry(menu, unit, m_max, n_shards, sg);
    if (st) return st;
    rkr_exec ex{};
    if (exec) ex = *exec;
    // budget tiles (K1t) when the shard qualifies -- every process decides
    // alike, from the same menu and geometry -- else the row-segment queue
    const bool want_tiles = !(exec && (exec->kernel == RKR_KERNEL_QUEUE || exec->kernel == RKR_KERNEL_DIAGONAL));
    if (!ex.tile_rows) {  // every process decides alike: from shard 0's width
        int sms = 0;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ex.device);
        ex.tile_rows = tile_rows_for((int64_t)sg.hi[0] - sg.lo[0], sms > 0 ? sms : 148,
                                     TileKnobs{ex.tune, 0});
    }
    ShardSpec spec{sg.lo[shard], sg.pad, sg.jo[shard]};
    spec.ipc = true;
    rkr_table* t = nullptr;
    st = RKR_ERR_INVALID;
    if (want_tiles) {
        ex.kernel = RKR_KERNEL_TILES;
        st = prepare_table(menu, unit, sg.hi[shard] - sg.lo[shard] - 1, &ex, sg.R, &t, &spec);
        if (st == RKR_ERR_INVALID) g_err.clear();
    }
    if (st == RKR_ERR_INVALID) {
        ex.kernel = RKR_KERNEL_QUEUE;
        st = prepare_table(menu, unit, sg.hi[shard] - sg.lo[shard] - 1, &ex, sg.R, &t, &spec);
    }
    if (st) return st;
    t->shard_lo = sg.lo[shard];
    t->shard_hi = sg.hi[shard];
    if (shard > 0) {  // tiles of the previous shard that meet this shard's halo
        const int32_t Wp = sg.hi[shard - 1] - sg.lo[shard - 1];
        t->hdesc.halo_need = t->tiles ? (Wp + t->tplan.W - 1) / t->tplan.W -
                                            std::max(0, (Wp - sg.pad) / t->tplan.W)
                                      : sg.J[shard - 1] - std::max(0, (Wp - sg.pad) / sg.TM);
    }
    DeviceGuard dg(t->device);
    CK(cudaMemcpyAsync(t->ddesc, &t->hdesc, sizeof(InstDesc), cudaMemcpyHostToDevice, t->stream));
    CK(cudaStreamSynchronize(t->stream));
    *out = t;
    return RKR_OK;
}

rkr_status rkr_shard_range(const rkr_table* t, int32_t* m_lo, int32_t* m_hi) {
    if (!t || !m_lo || !m_hi) return fail(RKR_ERR_ARGUMENT, "null argument");
    *m_lo = t->shard_lo;
    *m_hi = t->shard_hi;
    return RKR_OK;
}

rkr_status rkr_shard_export(const rkr_table* t, void* ipc_handle, int64_t* info) {
    if (!t || !ipc_handle || !info) return fail(RKR_ERR_ARGUMENT, "null argument");
    if (!t->ipc) return fail(RKR_ERR_ARGUMENT, "table was not created by rkr_shard_create");
    DeviceGuard dg(t->device);
    cudaIpcMemHandle_t hnd;
    CK(cudaIpcGetMemHandle(&hnd, t->block));
    std::memcpy(ipc_handle, &hnd, sizeof hnd);
    const unsigned char* b = static_cast<const unsigned char*>(t->block);
    info[0] = static_cast<const unsigned char*>(t->opt) - b;
    info[1] = t->g.sr;
    info[2] = reinterpret_cast<const unsigned char*>(t->hdesc.halo) - b;
    info[3] = reinterpret_cast<const unsigned char*>(t->arg) - b;
    info[4] = t->g.sa;
    info[5] = t->g.pad;
    info[6] = t->shard_lo;
    info[7] = t->shard_hi;
    return RKR_OK;
}

rkr_status rkr_shard_link(rkr_table* t, const void* next_ipc_handle, const int64_t* next_info) {
    if (!t || !next_ipc_handle || !next_info) return fail(RKR_ERR_ARGUMENT, "null argument");
    DeviceGuard dg(t->device);
    cudaIpcMemHandle_t hnd;
    std::memcpy(&hnd, next_ipc_handle, sizeof hnd);
    void* base = nullptr;
    CK(cudaIpcOpenMemHandle(&base, hnd, cudaIpcMemLazyEnablePeerAccess));
    t->ipc_open.push_back(base);
    unsigned char* b = static_cast<unsigned char*>(base);
    t->hdesc.next_opt = b + next_info[0];
    t->hdesc.next_sr = next_info[1];
    t->hdesc.next_halo = reinterpret_cast<int32_t*>(b + next_info[2]);
    t->hdesc.next_peer = 1;  // another process: system-scope fences
    CK(cudaMemcpyAsync(t->ddesc, &t->hdesc, sizeof(InstDesc), cudaMemcpyHostToDevice, t->stream));
    CK(cudaStreamSynchronize(t->stream));
    return RKR_OK;
}

rkr_status rkr_shard_zero(rkr_table* t) {
    if (!t) return fail(RKR_ERR_ARGUMENT, "null table");
    DeviceGuard dg(t->device);
    CK(cudaMemsetAsync(t->pdev.counter, 0, t->state_bytes, t->stream));
    CK(cudaStreamSynchronize(t->stream));
    return RKR_OK;
}

rkr_status rkr_shard_launch(rkr_table* t) {
    if (!t) return fail(RKR_ERR_ARGUMENT, "null table");
    DeviceGuard dg(t->device);
    if (t->tiles) {  // state zeroed by rkr_shard_zero
        TilePlan tp = t->tplan;
        if (tp.jobs) {
            if (launch_fill_tiles_batch(t->ddesc, t->dtp, t->djobs, tp.T,
                                        reinterpret_cast<unsigned int*>(t->pdev.counter), tp,
                                        t->stream, &tp))
                return cuda_fail(cudaGetLastError(), "shard launch");
        } else if (launch_fill_tiles(t->hdesc, tp, t->width, t->stream)) {
            return cuda_fail(cudaGetLastError(), "shard launch");
        }
        return RKR_OK;
    }
    if (launch_fill_batch(t->ddesc, &t->hdesc, t->lplan, t->width, t->plan.R,
                          std::max(t->g.L - 1, 1), std::max(t->hm.max_opts, 1), t->pdev.counter,
                          t->stream))
        return cuda_fail(cudaGetLastError(), "shard launch");
    return RKR_OK;
}

rkr_status rkr_shard_backtrack(rkr_table* t0, int32_t n, const void* const* ipc_handles,
                               const int64_t* infos, int32_t s, int32_t t, int32_t m, rkr_op* ops,
                               int64_t cap, int64_t* n_ops) {
    if (!t0 || n < 1 || !n_ops || (n > 1 && (!ipc_handles || !infos)))
        return fail(RKR_ERR_ARGUMENT, "null argument");
    DeviceGuard dg(t0->device);
    std::vector<ShardView> v(n);
    const int32_t m_glob = (int32_t)(n > 1 ? infos[8 * (n - 1) + 7] : t0->shard_hi) - 1;
    for (int r = 0; r < n; ++r) {
        const int64_t* in = infos + 8 * r;
        if (r == 0) {
            v[0] = ShardView{t0->opt, t0->arg, t0->g.sr, t0->g.sa, t0->g.pad, t0->shard_lo};
            continue;
        }
        cudaIpcMemHandle_t hnd;
        std::memcpy(&hnd, ipc_handles[r], sizeof hnd);
        void* base = nullptr;
        CK(cudaIpcOpenMemHandle(&base, hnd, cudaIpcMemLazyEnablePeerAccess));
        t0->ipc_open.push_back(base);
        unsigned char* b = static_cast<unsigned char*>(base);
        v[r] = ShardView{b + in[0], reinterpret_cast<const uint16_t*>(b + in[3]), in[1], in[4],
                         (int32_t)in[5], (int32_t)in[6]};
    }
    ShardView* dv = nullptr;
    int64_t* dout = nullptr;
    int32_t* dops = nullptr;
    int4* dstk = nullptr;
    const int64_t dcap = std::max<int64_t>(cap, 16);
    CK(cudaMalloc(reinterpret_cast<void**>(&dv), sizeof(ShardView) * n));
    CK(cudaMalloc(reinterpret_cast<void**>(&dout), 64));
    CK(cudaMalloc(reinterpret_cast<void**>(&dops), (size_t)dcap * 12));
    CK(cudaMalloc(reinterpret_cast<void**>(&dstk), sizeof(int4) * (2 * (size_t)t0->g.L + 16)));
    CK(cudaMemcpy(dv, v.data(), sizeof(ShardView) * n, cudaMemcpyHostToDevice));
    rkr_status st = RKR_OK;
    if (launch_walk_sharded(dv, n, t0->dm, t0->g.L, m_glob, t0->width, s, t, m,
                            dops, dcap, reinterpret_cast<int32_t*>(dstk), dout, t0->stream))
        st = cuda_fail(cudaGetLastError(), "shard walk launch");
    int64_t res[4] = {0, 0, -1, -1};
    if (st == RKR_OK) {
        cudaError_t e = cudaMemcpyAsync(res, dout, sizeof res, cudaMemcpyDeviceToHost, t0->stream);
        if (e == cudaSuccess) e = cudaStreamSynchronize(t0->stream);
        if (e == cudaSuccess && std::min(res[0], cap) > 0)
            e = cudaMemcpy(ops, dops, (size_t)std::min(res[0], cap) * 12, cudaMemcpyDeviceToHost);
        if (e != cudaSuccess) st = cuda_fail(e, "shard walk copy");
    }
    cudaFree(dv);
    cudaFree(dout);
    cudaFree(dops);
    cudaFree(dstk);
    if (st) return st;
    *n_ops = res[0];
    if (res[1] == 2)
        return fail(RKR_ERR_INFEASIBLE, "no feasible schedule for blocks %lld..%lld",
                    (long long)res[2], (long long)res[3]);
    if (res[0] > cap) return fail(RKR_ERR_CAPACITY, "schedule needs %lld ops", (long long)res[0]);
    return RKR_OK;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// Schedule validation gate (host): exact chain-level replay of a schedule in
// the block-atomic memory model the DP optimises over (the model of the
// reference's tests/test_helpers.hpp:249-322).  Returns the makespan and peak
// bytes, or RKR_ERR_INVALID with the offending op index.
// ---------------------------------------------------------------------------
extern "C" rkr_status rkr_replay(const rkr_menu* m, const rkr_op* ops, int64_t n, int64_t* peak_out,
                                 int64_t* time_out, int64_t* bad_op) {
    if (!m || (n > 0 && !ops) || !peak_out || !time_out) return fail(RKR_ERR_ARGUMENT, "null argument");
    const int L = m->n_blocks;
    if (L <= 0) return fail(RKR_ERR_INVALID, "empty option menu");
    const int64_t* a = m->act_sizes;
    std::vector<char> acts(L + 1, 0), grads(L + 1, 0);
    std::vector<int> packs(L, 0);
    acts[0] = 1;
    int64_t cur = a[0], peak = cur, elapsed = 0;
    auto find = [&](int b, int id) -> int {
        for (int o = m->option_offsets[b]; o < m->option_offsets[b + 1]; ++o)
            if (m->option_id[o] == id) return o;
        return -1;
    };
    for (int64_t i = 0; i < n; ++i) {
        const rkr_op& op = ops[i];
        const int b = op.block;
        auto bad = [&](const char* why) {
            if (bad_op) *bad_op = i;
            return fail(RKR_ERR_INVALID, "op %lld: %s", (long long)i, why);
        };
        if (op.kind != RKR_OP_COMPUTE && (b < 0 || b >= L)) return bad("block out of range");
        switch (op.kind) {
            case RKR_OP_BLOCK_FWD: {
                const int o = find(b, op.option);
                if (o < 0) return bad("unknown option");
                if (!acts[b]) return bad("forward without its input");
                const int64_t during = acts[b + 1] ? m->peak_fwd_pre[o] - a[b] - a[b + 1]
                                                   : m->peak_fwd[o] - a[b];
                peak = std::max(peak, cur + during);
                if (!acts[b + 1]) {
                    acts[b + 1] = 1;
                    cur += a[b + 1];
                }
                if (op.option != 0) {
                    if (packs[b]) return bad("second pack of a block");
                    packs[b] = op.option;
                    cur += m->save_mem[o] - a[b] - a[b + 1];
                }
                peak = std::max(peak, cur);
                elapsed += m->time_fwd[o];
                break;
            }
            case RKR_OP_COMPUTE:
                if (!acts[L] || grads[L]) return bad("loss without output or twice");
                grads[L] = 1;
                cur += a[L];
                peak = std::max(peak, cur);
                break;
            case RKR_OP_BLOCK_BWD: {
                const int o = find(b, op.option);
                if (o < 0 || !m->has_bwd[o]) return bad("unknown saved option");
                if (!acts[b] || !acts[b + 1] || packs[b] != op.option || !grads[b + 1])
                    return bad("backward without its pack, activations or gradient");
                peak = std::max(peak, cur - (m->save_mem[o] + a[b + 1]) + m->peak_bwd[o]);
                cur -= m->save_mem[o] - a[b] - a[b + 1];
                cur -= 2 * a[b + 1];
                packs[b] = 0;
                acts[b + 1] = 0;
                grads[b + 1] = 0;
                grads[b] = 1;
                cur += a[b];
                peak = std::max(peak, cur);
                elapsed += m->time_bwd[o];
                break;
            }
            case RKR_OP_FORGET:
                if (!acts[b]) return bad("forget of an absent activation");
                acts[b] = 0;
                cur -= a[b];
                break;
            default:
                return bad("unknown op kind");
        }
    }
    *peak_out = peak;
    *time_out = elapsed;
    if (bad_op) *bad_op = -1;
    return RKR_OK;
}
