// rkr_shard.cu -- host half of librkr.so, budget-axis shards (config 5):
// one table split into contiguous budget ranges, in one process over GPUs
// (rkr_sharded_*) or one process per GPU (rkr_shard_*, CUDA IPC).
#include "rkr_host.h"

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

rkr_status rkr_shard_mirror(rkr_table* t0, int32_t m_max, void* ipc_handle, int64_t* info) {
    if (!t0 || !ipc_handle || !info) return fail(RKR_ERR_ARGUMENT, "null argument");
    if (!t0->ipc || t0->shard_lo != 0) return fail(RKR_ERR_ARGUMENT, "not shard 0 of rkr_shard_create");
    if (m_max < t0->shard_hi - 1) return fail(RKR_ERR_ARGUMENT, "m_max below shard 0's range");
    DeviceGuard dg(t0->device);
    if (!t0->mirror) {
        const int64_t sa = round_up((int64_t)m_max + 1, 64);
        const size_t bytes = (size_t)t0->g.rows * sa * 2;
        t0->mirror_cap = bytes;
        t0->mirror = static_cast<uint16_t*>(ipc_block_take(t0->device, bytes, &t0->mirror_cap));
        if (!t0->mirror) CK(cudaMalloc(reinterpret_cast<void**>(&t0->mirror), bytes));
        t0->mirror_sa = sa;
        t0->mirror_M = m_max;
        t0->hdesc.arg_mirror = t0->mirror;
        t0->hdesc.mirror_sa = sa;
        t0->hdesc.mirror_base = 0;
        CK(cudaMemcpyAsync(t0->ddesc, &t0->hdesc, sizeof(InstDesc), cudaMemcpyHostToDevice, t0->stream));
        CK(cudaStreamSynchronize(t0->stream));
    }
    cudaIpcMemHandle_t hnd;
    CK(cudaIpcGetMemHandle(&hnd, t0->mirror));
    std::memcpy(ipc_handle, &hnd, sizeof hnd);
    info[0] = t0->mirror_sa;
    info[1] = t0->mirror_M;
    return RKR_OK;
}

rkr_status rkr_shard_attach_mirror(rkr_table* t, const void* ipc_handle, const int64_t* info) {
    if (!t || !ipc_handle || !info) return fail(RKR_ERR_ARGUMENT, "null argument");
    if (!t->ipc) return fail(RKR_ERR_ARGUMENT, "table was not created by rkr_shard_create");
    if (t->shard_lo == 0) return RKR_OK;  // shard 0 owns the mirror
    DeviceGuard dg(t->device);
    cudaIpcMemHandle_t hnd;
    std::memcpy(&hnd, ipc_handle, sizeof hnd);
    void* base = nullptr;
    CK(cudaIpcOpenMemHandle(&base, hnd, cudaIpcMemLazyEnablePeerAccess));
    t->ipc_open.push_back(base);
    t->hdesc.arg_mirror = static_cast<uint16_t*>(base);
    t->hdesc.mirror_sa = info[0];
    t->hdesc.mirror_base = t->shard_lo;
    CK(cudaMemcpyAsync(t->ddesc, &t->hdesc, sizeof(InstDesc), cudaMemcpyHostToDevice, t->stream));
    CK(cudaStreamSynchronize(t->stream));
    return RKR_OK;
}

rkr_status rkr_shard_backtrack(rkr_table* t0, int32_t n, const void* const* ipc_handles,
                               const int64_t* infos, int32_t s, int32_t t, int32_t m, rkr_op* ops,
                               int64_t cap, int64_t* n_ops) {
    if (!t0 || n < 1 || !n_ops || (n > 1 && (!ipc_handles || !infos)))
        return fail(RKR_ERR_ARGUMENT, "null argument");
    DeviceGuard dg(t0->device);
    const int32_t m_glob = (int32_t)(n > 1 ? infos[8 * (n - 1) + 7] : t0->shard_hi) - 1;
    // the views: shard 0's walk mirror (every shard stored its codes there:
    // local reads only), else every shard's rows through its IPC mapping,
    // opened once and cached with the scratch
    std::vector<unsigned char> key;
    for (int r = 1; r < n; ++r) {
        const unsigned char* h = static_cast<const unsigned char*>(ipc_handles[r]);
        key.insert(key.end(), h, h + sizeof(cudaIpcMemHandle_t));
    }
    const bool mirror = t0->mirror && t0->mirror_M == m_glob;
    const int nv = mirror ? 1 : n;
    const int64_t dcap = std::max<int64_t>(cap, 16);
    if (!t0->walk_scratch || t0->walk_key != key || t0->walk_n != nv || t0->walk_cap < dcap) {
        std::vector<ShardView> v(nv);
        if (mirror) {
            v[0] = ShardView{nullptr, t0->mirror, 0, t0->mirror_sa, 0, 0};
        } else {
            for (int r = 0; r < n; ++r) {
                const int64_t* in = infos + 8 * r;
                if (r == 0) {
                    v[0] = ShardView{t0->opt, t0->arg, t0->g.sr, t0->g.sa, t0->g.pad, t0->shard_lo};
                    continue;
                }
                cudaIpcMemHandle_t hnd;
                std::memcpy(&hnd, ipc_handles[r], sizeof hnd);
                void* base = nullptr;
                if (t0->walk_key != key || t0->walk_n != nv) {
                    CK(cudaIpcOpenMemHandle(&base, hnd, cudaIpcMemLazyEnablePeerAccess));
                    t0->ipc_open.push_back(base);
                } else {
                    base = t0->ipc_open[t0->ipc_open.size() - (n - 1) + (r - 1)];
                }
                unsigned char* b = static_cast<unsigned char*>(base);
                v[r] = ShardView{b + in[0], reinterpret_cast<const uint16_t*>(b + in[3]), in[1], in[4],
                                 (int32_t)in[5], (int32_t)in[6]};
            }
        }
        if (t0->walk_scratch) {
            cudaStreamSynchronize(t0->stream);
            cudaFree(t0->walk_scratch);
            t0->walk_scratch = nullptr;
        }
        const size_t stk = sizeof(int4) * (2 * (size_t)t0->g.L + 16);
        const size_t bytes = 256 + sizeof(ShardView) * nv + 64 + stk + (size_t)dcap * 12;
        CK(cudaMalloc(&t0->walk_scratch, bytes));
        CK(cudaMemcpy(t0->walk_scratch, v.data(), sizeof(ShardView) * nv, cudaMemcpyHostToDevice));
        t0->walk_key = key;
        t0->walk_n = nv;
        t0->walk_cap = dcap;
    }
    unsigned char* sp = static_cast<unsigned char*>(t0->walk_scratch);
    const ShardView* dv = reinterpret_cast<const ShardView*>(sp);
    int64_t* dout = reinterpret_cast<int64_t*>(sp + ((sizeof(ShardView) * nv + 255) & ~(size_t)255));
    int4* dstk = reinterpret_cast<int4*>(dout + 8);
    int32_t* dops = reinterpret_cast<int32_t*>(dstk + 2 * (size_t)t0->g.L + 16);
    rkr_status st = RKR_OK;
    if (launch_walk_sharded(dv, nv, t0->dm, t0->g.L, m_glob, t0->width, s, t, m, dops, t0->walk_cap,
                            reinterpret_cast<int32_t*>(dstk), dout, t0->stream))
        st = cuda_fail(cudaGetLastError(), "shard walk launch");
    int64_t res[4] = {0, 0, -1, -1};
    if (st == RKR_OK) {
        cudaError_t e = cudaMemcpyAsync(res, dout, sizeof res, cudaMemcpyDeviceToHost, t0->stream);
        if (e == cudaSuccess) e = cudaStreamSynchronize(t0->stream);
        if (e == cudaSuccess && std::min(res[0], cap) > 0)
            e = cudaMemcpy(ops, dops, (size_t)std::min(res[0], cap) * 12, cudaMemcpyDeviceToHost);
        if (e != cudaSuccess) st = cuda_fail(e, "shard walk copy");
    }
    if (st) return st;
    *n_ops = res[0];
    if (res[1] == 2)
        return fail(RKR_ERR_INFEASIBLE, "no feasible schedule for blocks %lld..%lld",
                    (long long)res[2], (long long)res[3]);
    if (res[0] > cap) return fail(RKR_ERR_CAPACITY, "schedule needs %lld ops", (long long)res[0]);
    return RKR_OK;
}

}  // extern "C"

