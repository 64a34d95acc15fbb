// rkr_batch.cu -- host half of librkr.so, batches: many independent tables
// in one persistent fill (rkr_batch_*), and the budget sweeps built on them
// (rkr_sweep / rkr_sweep_chains: cmd_sweep's loop, tools/remat.cpp:217-263).
#include "rkr_host.h"

namespace rkr {
namespace host {

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

}  // namespace host
}  // namespace rkr

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
    std::vector<uint8_t> top_done(nb, 0);      // infeasible budgets already searched
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
        // infeasible budgets whose menus pass the 64-bit overflow proof: the
        // min-feasible search by thresholds on the same tables (no wide fill)
        if (st == RKR_OK && !(exec && (exec->tune & RKR_TUNE_WIDE_SEARCH))) {
            std::vector<int32_t> which, Ls;
            for (int q = 0; q < nb; ++q)
                if (top[q] >= kInf64 && b->tables[q]->hm.bounded64) {
                    which.push_back(q);
                    Ls.push_back(b->tables[q]->g.L);
                }
            std::vector<int64_t> thr;
            st = min_feasible_thresholds(b->ddesc, which, Ls, b->stream, thr);
            for (size_t r = 0; st == RKR_OK && r < which.size(); ++r) {
                const int q = which[r], i = idx[q];
                const int64_t capu = feasibility_cap(mfor[i], unit[i]);
                if (capu > 0x7ffffffe) {
                    st = fail(RKR_ERR_INVALID, "feasibility cap exceeds int range");
                    break;
                }
                if (thr[r] <= capu) min_feasible[i] = (thr[r] + a0u[i]) * unit[i];   // :282
                top_done[q] = 1;
            }
            spt.mark("sweep: min-feasible thresholds");
        }
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
        if (top[q] >= kInf64 && !top_done[q]) inf_q.push_back(q);
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
            (void)L;
            const int64_t capu = feasibility_cap(menu, u);
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

