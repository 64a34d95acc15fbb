// rkr_table.cu -- host half of librkr.so, single tables: the C ABI of
// include/rkr.h for create, accessors, walks, refills and solve_chain.
// Batches and sweeps, shards and the replay live in rkr_batch.cu,
// rkr_shard.cu and rkr_replay.cu; their shared internals in rkr_host.h.
//
// Host work here is exactly the reference's host-side bookkeeping (menu
// validation and the per-block unit precompute of the DpTable constructor,
// chain_dp.hpp:56-95; quantize/to_units :32-41; solve_chain's control flow
// :255-296).  Every table cell is computed on the device (rkr_kernels.cu);
// there is no CPU fallback.
#include "rkr_host.h"

namespace rkr {
namespace host {

thread_local std::string g_err;

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
        bool ascending = true;  // ids strictly ascending (the usual menu): every id is first
        for (int32_t o = o_lo + 1; o < o_hi && ascending; ++o)
            ascending = m->option_id[o - 1] < m->option_id[o];
        auto first_pos = [&](int32_t o) {
            if (ascending) return o;
            if (small) {
                for (int32_t q = o_lo; q < o; ++q)
                    if (m->option_id[q] == m->option_id[o]) return q;
                return o;
            }
            return std::lower_bound(first.begin(), first.end(),
                                    std::make_pair(m->option_id[o], INT32_MIN))->second;
        };
        if (!small && !ascending) {
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
    h.bounded64 = nonneg && ((long double)L * F + Bk) < (long double)kInf64;
    return RKR_OK;
}

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

thread_local Staging t_stage;
thread_local Staging t_back;   // pinned D2H staging (walk results)
thread_local Staging t_sweep;  // pinned D2H staging (a sweep's walks; outlives nested fetches)
thread_local Staging t_desc;   // pinned H2D staging of batch descriptors (overlaps the menu upload)


// Process-shard blocks (and shard 0's walk mirror) must come from
// cudaMalloc (cudaIpcGetMemHandle does not take pool memory); destroyed ones
// are kept, a few per device, and reused by the next request that fits --
// the pool's policy for ordinary tables, without a synchronous cudaMalloc +
// cudaFree of up to gigabytes per solve.
namespace {
constexpr int kIpcSlots = 4;
struct IpcBlockCache {
    std::mutex mu;
    void* p[64][kIpcSlots] = {};
    size_t bytes[64][kIpcSlots] = {};
} g_ipc_cache;
}  // namespace

void* ipc_block_take(int dev, size_t need, size_t* cap) {
    std::lock_guard<std::mutex> g(g_ipc_cache.mu);
    int best = -1;
    for (int i = 0; i < kIpcSlots; ++i) {
        const size_t have = g_ipc_cache.bytes[dev & 63][i];
        if (g_ipc_cache.p[dev & 63][i] && have >= need && have <= 2 * need &&
            (best < 0 || have < g_ipc_cache.bytes[dev & 63][best]))
            best = i;
    }
    if (best < 0) return nullptr;
    void* out = g_ipc_cache.p[dev & 63][best];
    g_ipc_cache.p[dev & 63][best] = nullptr;
    *cap = g_ipc_cache.bytes[dev & 63][best];
    return out;
}

void ipc_block_give(int dev, void* block, size_t bytes) {  // the device is current, the block idle
    void* old = nullptr;
    {
        std::lock_guard<std::mutex> g(g_ipc_cache.mu);
        int slot = 0;  // an empty slot, else the smallest block goes
        for (int i = 0; i < kIpcSlots; ++i) {
            if (!g_ipc_cache.p[dev & 63][i]) {
                slot = i;
                break;
            }
            if (g_ipc_cache.bytes[dev & 63][i] < g_ipc_cache.bytes[dev & 63][slot]) slot = i;
        }
        old = g_ipc_cache.p[dev & 63][slot];
        g_ipc_cache.p[dev & 63][slot] = block;
        g_ipc_cache.bytes[dev & 63][slot] = bytes;
    }
    if (old) cudaFree(old);
}

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
        ipc_block_give(t->device, t->block, t->block_cap);
        t->block = nullptr;
    }
    if (t->block && t->owns_block) cudaFreeAsync(t->block, t->stream);
    if (t->wrec) cudaFreeAsync(t->wrec, t->stream);
    if (t->mirror || t->walk_scratch) {
        cudaStreamSynchronize(t->stream);
        if (t->mirror) ipc_block_give(t->device, t->mirror, t->mirror_cap);
        if (t->walk_scratch) cudaFree(t->walk_scratch);
    }
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
    t->prog.ocap = t->tiles ? t->tplan.ocap  // (whole option batches of the plan's kernel)
                            : std::max<int32_t>(h.max_opts, 1);
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
        t->block_cap = t->block_bytes;
        t->block = ipc_block_take(t->device, t->block_bytes, &t->block_cap);
        if (!t->block) CK(cudaMalloc(&t->block, t->block_bytes));
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
            if (launch_fill_tiles_jobs1(t->hdesc, tp, reinterpret_cast<unsigned int*>(t->pdev.counter),
                                        t->stream))
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

// Everything rkr_table_create does except the fill: validation and unit
// precompute, geometry, plan, one pooled allocation + one H2D copy, pads,
// cell programs.  R = 0 lets the plan choose the per-thread slot count.
rkr_status prepare_table(const rkr_menu* menu, int64_t unit, int32_t m_max, const rkr_exec* exec,
                         int R, rkr_table** out, const ShardSpec* spec, bool batch_tiles,
                         bool defer) {
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
    // a multiple of 32 slots: a 32-slot budget tile of a row is then one
    // aligned 128-byte line (4 sectors per unshifted warp read, not 5)
    t->g.pad = (int32_t)round_up(t->g.pad, 32);
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
            kn.mixed = !spec && !batch_tiles;  // plain single tables only
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


rkr_status min_feasible_thresholds(const InstDesc* d, const std::vector<int32_t>& which,
                                   const std::vector<int32_t>& L, cudaStream_t st,
                                   std::vector<int64_t>& thr) {
    const int n = (int)which.size();
    thr.assign(n, kInf64);
    if (n == 0) return RKR_OK;
    std::vector<int64_t> off(n);
    int64_t tot = 0;
    for (int i = 0; i < n; ++i) {
        off[i] = tot;
        tot += (int64_t)L[i] * (L[i] + 1) / 2;
    }
    // one allocation: which[n] | off[n] | out[n] | scratch[tot]
    const size_t bytes = (size_t)n * (4 + 8 + 8) + 16 + (size_t)tot * 8;
    unsigned char* p = nullptr;
    CK(cudaMallocAsync(reinterpret_cast<void**>(&p), bytes, st));
    int64_t* d_off = reinterpret_cast<int64_t*>(p);
    int64_t* d_out = d_off + n;
    int32_t* d_which = reinterpret_cast<int32_t*>(d_out + n);
    int64_t* d_scr = reinterpret_cast<int64_t*>(p + (((size_t)n * 20 + 15) & ~(size_t)15));
    cudaError_t e = cudaMemcpyAsync(d_off, off.data(), 8 * (size_t)n, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(d_which, which.data(), 4 * (size_t)n, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess && launch_batch_thresholds(d, d_which, n, d_scr, d_off, d_out, st))
        e = cudaGetLastError();
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(thr.data(), d_out, 8 * (size_t)n, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    cudaFreeAsync(p, st);
    if (e != cudaSuccess) return cuda_fail(e, "min-feasible thresholds");
    return RKR_OK;
}

int64_t feasibility_cap(const rkr_menu* menu, int64_t unit) {
    const int L = menu->n_blocks;
    int64_t capu = 0;
    for (int i = 0; i < L; ++i) {
        int64_t worst = 0;
        for (int o = menu->option_offsets[i]; o < menu->option_offsets[i + 1]; ++o)
            worst = std::max({worst, to_units(menu->peak_fwd[o], unit), to_units(menu->peak_bwd[o], unit),
                              to_units(menu->save_mem[o], unit)});
        capu += worst;
    }
    for (int i = 0; i <= L; ++i) capu += 2 * to_units(menu->act_sizes[i], unit);
    return capu;
}

}  // namespace host
}  // namespace rkr


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
        const int64_t capu = feasibility_cap(menu, unit);
        if (t->hm.bounded64 && !(exec && (exec->tune & RKR_TUNE_WIDE_SEARCH))) {
            // the wide table's first finite m, by thresholds (no table fill)
            std::vector<int64_t> thr;
            DeviceGuard dg(t->device);
            st = min_feasible_thresholds(t->ddesc, {0}, {L}, t->stream, thr);
            rkr_table_destroy(t);
            if (st) return st;
            if (capu > 0x7ffffffe) return fail(RKR_ERR_INVALID, "feasibility cap exceeds int range");
            if (thr[0] <= capu) *min_feasible = (thr[0] + a0_u) * unit;
            return fail(RKR_ERR_INFEASIBLE, "budget of %lld bytes is infeasible for this chain",
                        (long long)budget_bytes);
        }
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

