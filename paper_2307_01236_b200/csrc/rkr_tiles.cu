// rkr_tiles.cu -- K1t: the whole table fill as ONE co-resident launch in
// which every CTA owns a budget tile (sm_100a).
//
// Why budget tiles.  Every read of the fill goes to a strictly smaller span
// at a budget slot m' <= m (chain_dp.hpp:148, :166-167: shifts pack_chg,
// act_u >= 0; the left operand of a cut is unshifted).  So if CTA j owns the
// slots [jW, (j+1)W) of EVERY row, then diagonal k of its tile depends only
// on (a) its own tile's earlier diagonals -- a CTA barrier away -- and (b)
// the lower tiles j-d .. j-1 (d = ceil(pad / W)) up to diagonal k-1.  There
// is no work queue and no item holds an SM while it waits: each CTA walks
// the L diagonals of its tile in order, and the only cross-SM traffic is one
// done flag per (diagonal, tile).
//
// Warp roles.  Warps 0..26 compute; warp 27 communicates, so that no fence,
// flag poll or release ever stalls a compute warp:
//   compute, step k:  bulk(k) -> sync READY(k) -> tail(k) -> arrive DONE(k)
//   comm,    step k:  poll flags (k-1) of tiles j-d..j-1, acquire ->
//                     arrive READY(k) -> sync DONE(k) -> release flag (k, j)
//                     -> bulk-copy the programs of step k+2
// bulk(k)  cuts c in [s+2, t-1] of every row (s, t = s+k): they read
//          diagonals <= k-2 only (acquired before tail(k-1)), so they overlap
//          the lower tiles' progress on diagonal k-1.  When a diagonal has
//          fewer (row, warp slice) units than compute warps, the cut range is
//          split into P parts (late diagonals: few rows, many cuts).
// tail(k)  the options (row (s+1, t)) and cuts c = s+1 and c = t -- the only
//          candidates reading diagonal k-1 -- merged with the bulk parts in
//          the reference's scan order, then stored.
// Tie-break: options in menu order, then cuts ascending, each merged with a
// strict '<' in that order, so every cell keeps the reference's first
// minimum (chain_dp.hpp:139-174).
//
// Eligibility: 32-bit costs; T = ceil((M+1) / W) tiles co-resident (one
// 896-thread CTA per SM, cooperative launch); shared memory for the bulk
// partials and two steps of programs.  Otherwise the queue-scheduled K1p
// (rkr_persist.cu) runs.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <type_traits>

#include "rkr_internal.h"
#include "rkr_walk.cuh"

namespace rkr {

namespace {

constexpr uint32_t INF = kInf32;  // K1t runs the 32-bit cost path only

// timing experiments only (wrong results): skip the lower-tile wait / the
// release fence of the communication warp
#ifndef RKR_EXP_NOWAIT
#define RKR_EXP_NOWAIT 0
#endif
#ifndef RKR_EXP_RELAXED
#define RKR_EXP_RELAXED 0
#endif
#ifndef RKR_POLL_SLEEP
#define RKR_POLL_SLEEP 20
#endif
#ifndef RKR_POLL_RELAXED
#define RKR_POLL_RELAXED 1
#endif
// timing experiments: every compute warp waits for all tails of step k
// before bulk(k+1); RKR_TRACE_UNIT2 stamps warp 0's first tail unit in
// phases (scripts/trace_unit_phases.py)
#ifndef RKR_EXP_SYNCDONE
#define RKR_EXP_SYNCDONE 0
#endif
#ifndef RKR_EXP_DYNUNIT
#define RKR_EXP_DYNUNIT 0
#endif


__device__ __forceinline__ int t_ld_relaxed(const int* p) {
    int v;
    asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void t_fence_acq_rel() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
__device__ __forceinline__ void t_red_release_add(int* p, int v) {
    asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ int t_ld_relaxed_sys(const int* p) {
    int v;
    asm volatile("ld.relaxed.sys.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned long long t_gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* b, int count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* b) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
            "r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(b))
        : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
    asm volatile(
        "{\n .reg .pred p;\n"
        "W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra W;\n}" ::"r"(smem_u32(b)),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ int t_ld_acquire(const int* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
// 28 warps per CTA (27 compute + the communication warp), 72 registers per
// thread: against 32 warps / 64 registers, config 1 -7.5 %, configs 4-5
// -1-2 %, configs 2-3 unchanged; 24 warps / 80 registers loses 2-5 % on
// configs 2-3 (fewer warps to cover the gathers' latency)
constexpr int kNW = 28;        // warps per CTA
constexpr int kNT = kNW * 32;  // threads per CTA
// named barriers (0 is __syncthreads): compute warps arrive / sync, the
// communication warp syncs / arrives
constexpr int kBarReady = 1, kBarDone = 2, kBarSplit = 3;
__device__ __forceinline__ void nb_sync(int id) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(kNT) : "memory");
}
__device__ __forceinline__ void nb_sync_n(int id, int n) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void nb_arrive(int id) {
    asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(kNT) : "memory");
}


constexpr int kU = 8;          // cuts per load batch (2 kU loads in flight per lane)
#ifndef RKR_KUB
#define RKR_KUB 16
#endif
constexpr int kUB = RKR_KUB;   // (tile jobs) cuts per load batch, sweeps re-read
constexpr int kSlice = 64;          // STREAM: cut-program entries staged per warp at a time
template <int RPW>
constexpr int kOptBatch = RPW == 1 ? 16 : 8;  // options per load batch (ocap: a multiple)
constexpr int kPcap = 16;  // undominated options kept per block (more: the block is not pruned)

inline uint32_t al16(uint64_t x) { return (uint32_t)((x + 15) & ~15ull); }
inline int ceil_to(int x, int a) { return (x + a - 1) / a * a; }

// First budget slot of tile j and the tile holding slot x: W-slot tiles, or
// (mixed plans) j1 32-slot tiles followed by 16-slot ones.
__host__ __device__ __forceinline__ int tile_lo(const TilePlan& tp, int j) {
    return j < tp.j1 ? j * tp.W : tp.j1 * 32 + (j - tp.j1) * 16;
}
__host__ __device__ __forceinline__ int tile_of(const TilePlan& tp, int x) {
    return (tp.j1 == INT32_MAX || x < tp.j1 * 32) ? x / tp.W : tp.j1 + (x - tp.j1 * 32) / 16;
}
inline TileSmem tile_smem(const TilePlan& tp) {
    TileSmem m;
    const uint64_t L = tp.L;
    uint64_t pmax = 0;  // max over k of (L - k) k cut entries
    for (uint64_t k = 0; k < L; ++k) pmax = (L - k) * k > pmax ? (L - k) * k : pmax;
    m.prog_bytes = al16(pmax * 16);
    m.thr_bytes = al16(L * tp.ocap * 4);
    uint64_t b = 0;
    m.best = 0;
    // Bulk partials (values, then codes): [units 32] (>= kNT) for unsplit
    // steps and [kNT] for split steps (late diagonals, cut range over several
    // warps).  Without the communication warp the steps are barrier-aligned
    // and one [cap] region serves both.  With it, the bulk of step k+1 runs on
    // other warps than the tail of step k that reads step k's parts, so each
    // region is double-buffered by step parity: [2 cap | 2 kNT].  (Shared
    // memory is tight for config-3-sized co-resident tables: 12 KB more once
    // cost 30 % -- less L1 left for loads in flight.)  A dynamic split (bulk
    // items of 16-64 cuts taken from a shared counter by whichever warp is
    // free, merged with a 64-bit atomicMin on (value, code)) measured 5 %
    // slower on configs 3 and 2 at every item size.
    const uint64_t np = tp.comm ? 2ull * tp.cap + 2 * kNT : (uint64_t)tp.cap;
    b = al16(b + np * 4);
    m.code = (uint32_t)b;
    b = al16(b + np * 2);
    m.blk = (uint32_t)b;
    b = al16(b + (L + 2) * 4);  // block option offsets [L+1] + the last-CTA flag
    m.split = (uint32_t)b;      // per step: bulk parts and cuts per part; 2 unit counters
    b = al16(b + L * 8 + 8);
    m.thx = (uint32_t)b;  // per block: the terms of its largest option threshold
    b = al16(b + (tp.stream ? 0 : L * 24));
    m.opd = (uint32_t)b;
    m.pru = 0;
    if (tp.stream) {  // programs, thresholds and options from global memory;
        // per-warp program slices for the bulk
        m.prog_bytes = (uint32_t)(kNW * kSlice * 16 * tp.rpw);
        m.thr_bytes = 0;
        m.prog = (uint32_t)b;
        b += m.prog_bytes;
        // per-(warp, row) option slices: [kNW RPW][ocap] int2 | [kNW RPW][ocap] int
        m.thr = (uint32_t)b;
        b = al16(b + (uint64_t)kNW * tp.rpw * tp.ocap * 12);
    } else {
        b = al16(b + L * tp.ocap * 8);  // [block][ocap] {-pack shift, pass time}, padded
        if (tp.prune) {  // [block][kPcap] {-pack shift, pass time} | [block][kPcap] codes | [block] count
            m.pru = (uint32_t)b;
            b = al16(b + L * kPcap * 10 + L * 4);
        }
        m.prog = (uint32_t)b;
        b += 2ull * m.prog_bytes;
        m.thr = (uint32_t)b;
        b += 2ull * m.thr_bytes;
    }
    m.xch = (uint32_t)b;  // split-tail exchange: values [kNT] | codes [kNT] (comm only)
    b = al16(b + (tp.comm ? (uint64_t)kNT * 6 : 0));
    m.bar = (uint32_t)b;
    b += 16;
    m.total = (uint32_t)b;
    return m;
}

// One step's programs -> shared buffer (k & 1): the cut programs of diagonal
// k (contiguous, (L-k) k int4 entries) and its rows' option thresholds.
__device__ __forceinline__ void stage_step(const TilePlan& tp, const ProgDev& pq, const TileSmem& sm,
                                           unsigned char* smem, uint64_t* bars, int L, int k) {
    const int b = k & 1;
    const uint32_t pb = (uint32_t)(L - k) * (uint32_t)k * 16u;
    const uint32_t tb = (uint32_t)(L - k) * (uint32_t)tp.ocap * 4u;
    mbar_expect_tx(bars + b, pb + tb);
    if (pb)
        bulk_g2s(smem + sm.prog + b * sm.prog_bytes,
                 static_cast<const int4*>(pq.ptr) + diag_cut_off(L, k), pb, bars + b);
    bulk_g2s(smem + sm.thr + b * sm.thr_bytes, pq.thr + diag_off(L, k) * tp.ocap, tb, bars + b);
}

// Tail reads (the option windows of row (s+1, t) and the two tail cuts) go
// through L1: the windows of one row at the options' pack shifts overlap
// (config 3: 32 windows over ~10 lines), so most of them hit instead of
// paying an L2 round trip each, and the tail is a chain of dependent
// batches.  Coherent: every row is read only after the step that wrote it,
// its line holds no other row, and the acquisition of the lower tiles'
// diagonal k-1 before each tail (ld.acquire -> CCTL.IVALL) empties L1 of
// anything older; the bulk's reads, which never repeat, stay L2-only.
#ifndef RKR_PAIR_TAIL
#define RKR_PAIR_TAIL 1
#endif
#ifndef RKR_TAIL_L1
#define RKR_TAIL_L1 1
#endif
__device__ __forceinline__ uint32_t tail_ld(const uint32_t* p) {
    return RKR_TAIL_L1 ? __ldca(p) : __ldcg(p);
}

// The lane's table base opt + m as an opaque 64-bit register, so that a
// table address is ONE IMAD.WIDE.U32 (entry offset x 4 + base) instead of
// the compiler's re-associated 64-bit (m + offset) sum (four instructions).
__device__ __forceinline__ const uint32_t* lane_base(const uint32_t* opt, int m) {
    const uint32_t* p;
    asm("mov.b64 %0, %1;" : "=l"(p) : "l"(opt + m));
    return p;
}

// Eight ungated candidates c0 .. c0+7, in scan order, into (best, code) with
// the scan's strict '<'.  The sequential scan ends on the FIRST candidate
// holding the batch minimum when that minimum beats best, and changes
// nothing otherwise -- so: the minimum (three VIMNMX3 + one VIMNMX), one
// vote, and the position only when some lane improves.  Used for option
// batches (config 3: -2 %); on cut batches it measured neutral (late in a
// long scan most batches improve no lane, but the vote and the position
// search cost what the per-candidate compares save).
__device__ __forceinline__ void merge8(const uint32_t (&tot)[8], int c0, uint32_t& best, int& code) {
    const uint32_t x = __vimin3_u32(__vimin3_u32(tot[0], tot[1], tot[2]),
                                    __vimin3_u32(tot[3], tot[4], tot[5]), min(tot[6], tot[7]));
    if (__any_sync(0xffffffffu, x < best)) {
        int qf = 7;
#pragma unroll
        for (int q = 6; q >= 0; --q)
            if (tot[q] == x) qf = q;
        if (x < best) {
            best = x;
            code = c0 + qf;
        }
    }
}

// merge8 over a list whose position q holds code pcd[q] (the undominated
// options of a block, menu order)
__device__ __forceinline__ void merge8p(const uint32_t (&tot)[8], const uint16_t* pcd, uint32_t& best,
                                        int& code) {
    const uint32_t x = __vimin3_u32(__vimin3_u32(tot[0], tot[1], tot[2]),
                                    __vimin3_u32(tot[3], tot[4], tot[5]), min(tot[6], tot[7]));
    if (x < best) {
        int qf = 7;
#pragma unroll
        for (int q = 6; q >= 0; --q)
            if (tot[q] == x) qf = q;
        best = x;
        code = pcd[qf];
    }
}

// Cuts i in [ib, ie) of one cell slice, ascending, strict '<' into (best,
// code).  Program entry i of cell (s, s+k): element offsets of slot 0 of the
// left row (s, c-1) and of the right row (c, t) shifted by act_u[c]
// (:166-167), the option-0 sweep (:162) and the gate (:159, :164).
//
// Instruction budget per candidate (ncu, config 3: 57 % issue slots busy):
// one LDS.128 (program entry), two IMAD.WIDE (lane base + entry offset: the
// lane's `optm = opt + m` is formed once), two LDG, one IADD3 (sweep + left
// + right), VIMNMX + ISETP (DPX __vibmin_u32: min and "kept the old best";
// sm_100a has no fused predicate form) and one predicated code update --
// 10.4 per cut with the loop overhead, 13.5 before (profiles/r02_sass).
// The gate (:159, :164) is only tested per candidate in a batch where it
// splits the warp: it grows with i, so when every lane admits the batch's
// last cut, every lane admits every cut of the batch.  RPW = 1 (one row per
// warp, consecutive budgets): that is lane 0's test, warp-uniform, no vote.
// RPW = 2 (two rows per warp, 16 budgets each): a warp vote.
// U = cuts per load batch.  RR (tile jobs: configs 3, 4): the
// batch's addresses come from 8-byte program reads and the sweeps are read
// again after the loads, so a cut in flight holds two registers instead of
// four: batches of kUB cuts (2 kUB loads in flight per lane) at the cost of
// one more shared-memory read per cut -- the bulk is a chain of dependent
// round trips per warp.
template <int RPW, int U = kU, bool RR = false>
__device__ __forceinline__ bool scan_cuts(const uint32_t* __restrict__ opt, const int4* pe, int ib,
                                          int ie, int m, int cb, uint32_t& best, int& code) {
    const uint32_t* __restrict__ optm = lane_base(opt, m);
    const int m0 = m - (int)(threadIdx.x & 31);  // RPW = 1: warp-uniform, the smallest budget
    int i0 = ib;
    for (; i0 + U <= ie; i0 += U) {
        uint32_t lv[U], rv[U];
        int4 e[RR ? 1 : U];
#pragma unroll
        for (int q = 0; q < U; ++q) {
            int2 xy;
            if constexpr (RR) {
                xy = *reinterpret_cast<const int2*>(pe + i0 + q);
            } else {
                e[q] = pe[i0 + q];
                xy = make_int2(e[q].x, e[q].y);
            }
            // unconditional loads (every offset is inside the table); the
            // gate masks the candidate afterwards
            lv[q] = __ldcg(optm + (uint32_t)xy.x);
            rv[q] = __ldcg(optm + (uint32_t)xy.y);
        }
        int wl;
        if constexpr (RR)
            wl = pe[i0 + U - 1].w;
        else
            wl = e[U - 1].w;
        if (RPW == 1 ? wl <= m0 : __all_sync(0xffffffffu, wl <= m)) {
            // (warp-uniform) no lane gated in this batch
            uint32_t tot[U];
#pragma unroll
            for (int q = 0; q < U; ++q) {
                if constexpr (RR)
                    tot[q] = (uint32_t)pe[i0 + q].z + lv[q] + rv[q];
                else
                    tot[q] = (uint32_t)e[q].z + lv[q] + rv[q];
            }
#pragma unroll
            for (int q = 0; q < U; ++q) {
                bool keep;
                best = __vibmin_u32(best, tot[q], &keep);
                if (!keep) code = cb + i0 + q;  // strictly smaller: the scan's first minimum
            }
            continue;
        }
#pragma unroll
        for (int q = 0; q < U; ++q) {
            int2 zw;
            if constexpr (RR)
                zw = *reinterpret_cast<const int2*>(&pe[i0 + q].z);
            else
                zw = make_int2(e[q].z, e[q].w);
            const uint32_t tot = (uint32_t)zw.x + lv[q] + rv[q];
            if (zw.y <= m && tot < best) {
                best = tot;
                code = cb + i0 + q;
            }
        }
        // the gate only grows with i: stop once no lane admits the batch's
        // last cut (the `break` of :164)
        if (!__any_sync(0xffffffffu, wl <= m)) return true;
    }
    for (; i0 < ie; ++i0) {
        const int4 e = pe[i0];
        const uint32_t tot =
            (uint32_t)e.z + __ldcg(optm + (uint32_t)e.x) + __ldcg(optm + (uint32_t)e.y);
        if (e.w <= m && tot < best) {
            best = tot;
            code = cb + i0;
        }
    }
    return false;
}

// STREAM variant (long chains: a diagonal's programs do not fit shared
// memory): each warp stages its unit's program(s) kSlice entries at a time
// (RPW rows: one slice per row, staged by that row's lanes).
template <int RPW>
__device__ __forceinline__ void scan_cuts_streamed(const uint32_t* __restrict__ opt,
                                                   const int4* __restrict__ pe_g, int4* slice,
                                                   int ib, int ie, int m, int cb, uint32_t& best,
                                                   int& code) {
    constexpr int W = 32 / RPW;
    const int lane = threadIdx.x & 31, rw = lane / W, ml = lane % W;
    int4* mine = slice + rw * kSlice;
    for (int c0 = ib; c0 < ie; c0 += kSlice) {
        const int c1 = c0 + kSlice < ie ? c0 + kSlice : ie;
        __syncwarp();  // the previous chunk's readers are done
        for (int i = c0 + ml; i < c1; i += W) mine[i - c0] = __ldg(pe_g + i);
        __syncwarp();
        if (scan_cuts<RPW>(opt, mine - c0, c0, c1, m, cb, best, code)) return;
    }
}

// COMM: the last warp is the communication warp (latency-bound tables);
// otherwise all warps compute and warp 0 polls / thread 0 publishes inline, behind
// CTA barriers (throughput-bound tables, where the extra compute warp and
// barrier-aligned phases measured faster).
//
// tile_job: every diagonal of tile j of one table.  ph0/ph1 = completed
// phases of the two program mbarriers before this job (jobs of a batch
// reuse them).  The caller initialises the mbarriers once and separates
// jobs with a CTA barrier.
//
// RPW = rows per warp.  1: a warp computes 32 consecutive budget slots of
// one row (tile width W = 32).  2: lanes 0-15 and 16-31 take the same 16
// slots of two rows (W = 16), so a table has twice as many tiles, each half
// the work: the tile jobs of config 3 come out to 7 waves of 148 instead of
// 4 (the last one 46 % full), and a budget shard of 2048 slots occupies 128
// SMs instead of 64.  A unit is one warp's (row group, slots) share of a
// step; rows past the diagonal's last (an odd row count) are computed from a
// clamped row and not stored.
//
// OM (the plain single tables run as mixed-width jobs -- config 3): option
// batches whose thresholds no lane is below go ungated through merge8, and
// the padding of the last batch is not scanned (config 3 -2 %; configs 1, 2
// and 4 measured 3-7 % slower with it: their short option scans and low
// budgets gain nothing and pay the extra latency).
template <int RPW, bool COMM, bool SPLIT, bool STREAM, bool TABLE, bool HALO, bool OM = false>
__device__ __forceinline__ void tile_job(const InstDesc& D, const TilePlan& tp, const int j,
                                         unsigned char* smem_raw, uint32_t ph0, uint32_t ph1) {
    constexpr int W = 32 / RPW;
    constexpr int kNC = COMM ? kNW - 1 : kNW;  // compute warps
    // options per load batch: 16 with one row per warp (16 window reads in
    // flight per lane: config 3 -5 %, config 2 -3 % against 8; the plan pads
    // ocap to a multiple of 16), 8 with two rows per warp
    constexpr int kOB = kOptBatch<RPW>;

    const TileSmem& sm = tp.sm;
    int32_t* s_blk = reinterpret_cast<int32_t*>(smem_raw + sm.blk);
    int2* s_opd = reinterpret_cast<int2*>(smem_raw + sm.opd);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw + sm.bar);

    const Geometry& g = D.g;
    const DevMenu& dm = D.dm;
    const ProgDev& pq = D.prog;
    uint32_t* __restrict__ opt = static_cast<uint32_t*>(D.opt);
    uint16_t* __restrict__ arg = D.arg;
    const int L = g.L, M = g.M;
    const int sr = (int)g.sr;  // rows * sr < 2^31 (tile_plan)
    const int ocap = tp.ocap;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int rw = lane / W, ml = lane % W;  // row within the unit, slot within the tile
    const int m_lo = tile_lo(tp, j);

    // Table-independent data in shared memory: block option ranges, and per
    // (block, option slot) the pack shift (negated) clamped to pad (:148) and time_fwd
    // + time_bwd (:150), padded to ocap with options that never win (pass
    // time INF).  Cut programs and thresholds arrive per step by bulk copy,
    // two steps ahead (double buffer, one mbarrier per buffer).
    for (int c = tid; c <= L; c += kNT) s_blk[c] = __ldg(dm.blk_off + c);
    // per step: bulk parts P and cuts per part (late diagonals split the
    // cut range over warps; >= 8 cuts per part)
    int2* s_split = reinterpret_cast<int2*>(smem_raw + sm.split);
    for (int k = tid; TABLE && k < L; k += kNT) {
        const int units = (L - k + RPW - 1) / RPW, nb = k >= 3 ? k - 2 : 0;
        int P = 1, chunk = nb;
        if (nb > 0 && units < kNC) {
            P = kNC / units;
            const int pmax = (nb + 7) >> 3;
            if (P > pmax) P = pmax;
            chunk = (nb + P - 1) / P;
        }
        s_split[k] = make_int2(P, chunk);
    }
    int* s_ucnt = reinterpret_cast<int*>(smem_raw + sm.split) + 2 * L;  // bulk units taken, per step parity
    if (tid < 2) s_ucnt[tid] = 0;
    // (OM) per block, one warp (lanes over its options):
    // * s_opd: {-pack shift clamped to pad, pass time} per option slot;
    // * the terms of the largest option threshold of row (s, t),
    //   k > 0 (chain_dp.hpp:141-147, local slots): max(F[s] + seed[t], B[s])
    //   with F = max fwd_req, B = max(bwd_req, pack_chg) over block s's
    //   options and seed[t] = 2 act_u[t+1] (t < L-1); 64-bit (sizes are
    //   unbounded).  A row is *open* for a warp when that is <= the warp's
    //   smallest budget: every option admissible at every budget of the warp.
    // * (prune) dominance pruning for open rows: option x can never be the
    //   scan's first minimum if another option y of the block has a pack
    //   shift <= x's and a pass time <= x's (y before x in menu order) or <
    //   x's (y after x): opt(s+1, t) does not increase with the budget, so y's
    //   total is <= (before) / < (after) x's at every m (chain_dp.hpp:141-155;
    //   the reference's own option generator drops dominated options the same
    //   way, options.hpp:182-217, on more fields).  The undominated options
    //   (menu order, padded with options that never win) and their codes;
    //   blocks with more than kPcap of them scan everything.  (The shift is
    //   clamped to pad only for options whose threshold exceeds M, which no
    //   open row has.)
    int64_t* s_thx = reinterpret_cast<int64_t*>(smem_raw + sm.thx);
    int2* s_pru = reinterpret_cast<int2*>(smem_raw + sm.pru);
    uint16_t* s_pcd = reinterpret_cast<uint16_t*>(smem_raw + sm.pru + L * kPcap * 8);
    int32_t* s_pcnt = reinterpret_cast<int32_t*>(smem_raw + sm.pru + L * kPcap * 10);
    for (int q = tid; !OM && !STREAM && q < L * ocap; q += kNT) {
        const int b = q / ocap, i = q - b * ocap;
        const int o = __ldg(dm.blk_off + b) + i;
        s_opd[q] = o < __ldg(dm.blk_off + b + 1)
                       ? make_int2(-__ldg(pq.pc + o), (int)__ldg(static_cast<const uint32_t*>(pq.otot) + o))
                       : make_int2(0, (int)INF);
    }
    for (int b = warp; OM && !STREAM && b < L; b += kNW) {
        const int o0 = __ldg(dm.blk_off + b), own = __ldg(dm.blk_off + b + 1) - o0;
        int2* ob = s_opd + b * ocap;
        int64_t f = INT64_MIN / 4, bp = INT64_MIN / 4;
        for (int i = lane; i < ocap; i += 32) {
            int2 v = make_int2(0, (int)INF);
            if (i < own) {
                const int o = o0 + i;
                v = make_int2(-__ldg(pq.pc + o), (int)__ldg(static_cast<const uint32_t*>(pq.otot) + o));
                {
                    f = max(f, __ldg(dm.fwd_req + o) - g.m_base);
                    bp = max(bp, max(__ldg(dm.bwd_req + o), __ldg(dm.pack_chg + o)) - g.m_base);
                }
            }
            ob[i] = v;
        }
        {
#pragma unroll
            for (int d = 16; d; d >>= 1) {
                f = max(f, (int64_t)__shfl_xor_sync(0xffffffffu, (long long)f, d));
                bp = max(bp, (int64_t)__shfl_xor_sync(0xffffffffu, (long long)bp, d));
            }
            if (lane == 0) {
                s_thx[b] = f;
                s_thx[L + b] = bp;
                s_thx[2 * L + b] = b < L - 1 ? 2 * __ldg(dm.act_u + b + 1) : 0;
            }
        }
        if (!tp.prune) continue;
        __syncwarp();
        int cnt = 0;
        for (int i0 = 0; i0 < own; i0 += 32) {
            const int i = i0 + lane;
            bool keep = i < own;
            if (keep) {
                const int2 x = ob[i];
                for (int y = 0; y < own; ++y) {
                    const int2 v = ob[y];
                    if (y != i && v.x >= x.x &&
                        (y < i ? (uint32_t)v.y <= (uint32_t)x.y : (uint32_t)v.y < (uint32_t)x.y)) {
                        keep = false;
                        break;
                    }
                }
            }
            const unsigned bal = __ballot_sync(0xffffffffu, keep);
            const int pos = cnt + __popc(bal & ((1u << lane) - 1u));
            if (keep && pos < kPcap) {
                s_pru[b * kPcap + pos] = ob[i];
                s_pcd[b * kPcap + pos] = (uint16_t)(i + 1);
            }
            cnt += __popc(bal);
        }
        for (int q = cnt + lane; q < kPcap; q += 32) {
            s_pru[b * kPcap + q] = make_int2(0, (int)INF);
            s_pcd[b * kPcap + q] = 0;
        }
        if (lane == 0) s_pcnt[b] = cnt;
    }
    // lower tiles this one reads: those holding slots [m_lo - pad, m_lo)
    const int d_eff = j - tile_of(tp, m_lo - g.pad > 0 ? m_lo - g.pad : 0);
    // Budget shards (config 5).  Local slots [Wl - pad, Wl) of this shard are
    // the next shard's halo (its slots [-pad, 0)): tiles that compute them
    // also store them there (peer memory when the next shard is on another
    // GPU / in another process) and count L-k rows per diagonal into the
    // next shard's halo[k] after a (system-scope) fence; tiles whose reads
    // reach below local slot 0 wait for halo[k-1] >= (L-k+1) * halo_need.
    const int Wl = M + 1;
    const bool halo_in = HALO && D.halo_need > 0 && m_lo - g.pad < 0;
    const bool halo_out = HALO && D.next_opt != nullptr && m_lo + W > Wl - g.pad && m_lo < Wl;
    auto wait_halo = [&](int kk) {  // one thread
        const int need = (L - kk) * D.halo_need;
        while (t_ld_relaxed_sys(D.halo + kk) < need) __nanosleep(64);
        asm volatile("fence.acq_rel.sys;" ::: "memory");
    };
    auto push_halo = [&](int kk) {  // one thread, after the CTA stored diagonal kk
        if (D.next_peer)
            __threadfence_system();
        else
            __threadfence();
        atomicAdd(D.next_halo + kk, L - kk);
    };
    int* __restrict__ done = tp.done;
    __syncthreads();

    if (COMM && warp == kNC) {
        // ================= communication warp =================
        if (!STREAM && lane == 0) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            stage_step(tp, pq, sm, smem_raw, bars, L, 0);
            if (L > 1) stage_step(tp, pq, sm, smem_raw, bars, L, 1);
        }
        for (int k = 0; k < L; ++k) {
            if (k >= 1 && !RKR_EXP_NOWAIT) {  // diagonal k-1 of the lower tiles, acquired
                const int* row = done + (int64_t)(k - 1) * tp.T;
                // relaxed polls, then one acquiring load of the flag seen set:
                // an acquire (ld.acquire -> CCTL.IVALL) per poll would empty
                // the SM's L1 -- the compute warps' cached tail windows,
                // spills and plan reads -- every few tens of nanoseconds
                for (int q = lane; q < d_eff; q += 32) {
                    if (RKR_POLL_RELAXED) {
                        while (t_ld_relaxed(row + j - 1 - q) == 0)
                            if (RKR_POLL_SLEEP) __nanosleep(RKR_POLL_SLEEP);
                        (void)t_ld_acquire(row + j - 1 - q);
                    } else {
                        while (t_ld_acquire(row + j - 1 - q) == 0) __nanosleep(20);
                    }
                }
                // (tile 0 polls nothing: its own flag, for the L1 invalidation
                // the tail's cached reads rely on)
                if (d_eff == 0 && lane == 0) (void)t_ld_acquire(row + j);
                if (halo_in && lane == 0) wait_halo(k - 1);
                __syncwarp();
            }
            // trace: when the lower tiles' diagonal k-1 was acquired (the
            // compute warps pass READY at max(this, their last bulk))
#ifndef RKR_TRACE_UNIT2
            if (tp.trace && lane == 0) tp.trace[6 * ((int64_t)k * tp.T + j) + 3] = clock64();
#endif
            nb_arrive(kBarReady);
            nb_sync(kBarDone);  // the compute warps stored diagonal k
#ifdef RKR_TRACE_EXPERIMENT
            if (tp.trace && lane == 0) tp.trace[6 * ((int64_t)k * tp.T + j) + 0] = clock64();
#endif
            if (lane == 0) {
                // release-add: orders the CTA's stores (made visible to this
                // thread by the barrier) before the flag
                if (RKR_EXP_RELAXED)
                    atomicAdd(done + (int64_t)k * tp.T + j, 1);
                else
                    t_red_release_add(done + (int64_t)k * tp.T + j, 1);
                if (halo_out) push_halo(k);
                // buffer (k & 1) is free: every compute warp finished tail(k)
                if (!STREAM && k + 2 < L) {
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    stage_step(tp, pq, sm, smem_raw, bars, L, k + 2);
                }
            }
        }
    } else {
    // ================= compute warps =================
    if (!COMM && !STREAM && tid == 0) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        stage_step(tp, pq, sm, smem_raw, bars, L, 0);
        if (L > 1) stage_step(tp, pq, sm, smem_raw, bars, L, 1);
    }
    for (int k = 0; k < L; ++k) {
        // trace (per (diagonal, tile)): [0] globaltimer at the step start (the
        // cross-SM timeline); SM cycles: [1] step start, [2] warp 0's bulk
        // done, [3] the communication warp's acquisition of diagonal k-1
        // (COMM), [4] READY passed, [5] warp 0's tail done
        unsigned long long t0 = 0, c0 = 0, t1 = 0, t2 = 0, t3 = 0;
        if (tp.trace && tid == 0) {
            t0 = t_gtimer();
            c0 = clock64();
        }
        if (!STREAM) mbar_wait(bars + (k & 1), ((k & 1 ? ph1 : ph0) + (uint32_t)(k >> 1)) & 1u);
        // this step's cut programs and option thresholds: the staged copies,
        // or (STREAM) straight from global memory
        const int4* prog = STREAM ? static_cast<const int4*>(pq.ptr) + diag_cut_off(L, k)
                                  : reinterpret_cast<const int4*>(smem_raw + sm.prog + (k & 1) * sm.prog_bytes);
        const int32_t* thrs = STREAM ? pq.thr + diag_off(L, k) * ocap
                                     : reinterpret_cast<const int32_t*>(smem_raw + sm.thr + (k & 1) * sm.thr_bytes);

        const int rows = L - k;
        const int units = (rows + RPW - 1) / RPW;
        const int nb = k >= 3 ? k - 2 : 0;  // bulk cuts i = 1 .. k-2
        // late diagonals split the cut range into P parts of `chunk` cuts
        // (TABLE: precomputed per step, no integer division in the step loop
        // -- 5 % on configs 1-2; the tile-job kernels measured faster without)
        int P = 1, chunk = nb;
        if constexpr (TABLE) {
            const int2 pc2 = s_split[k];
            P = pc2.x;
            chunk = pc2.y;
        } else if (nb > 0 && units < kNC) {
            P = kNC / units;
            const int pmax = (nb + 7) >> 3;  // keep >= 8 cuts per part
            if (P > pmax) P = pmax;
            chunk = (nb + P - 1) / P;
        }
        const int TS = (COMM && SPLIT && 2 * units <= kNC) ? 2 : 1;
        // bulk partials (see tile_smem)
        const int poff = !COMM ? 0 : (P == 1 ? (k & 1) * tp.cap : 2 * tp.cap + (k & 1) * kNT);
        uint32_t* pbest = reinterpret_cast<uint32_t*>(smem_raw + sm.best) + poff;
        uint16_t* pcode = reinterpret_cast<uint16_t*>(smem_raw + sm.code) + poff;

        // ---- bulk: cuts i in [1, k-2] ahead of the wait -----------------------
        // (scanning them inside the tail instead, which frees the partials,
        // measured 3% slower on config 3)
        if (nb > 0) {
            // with the communication warp, bulk units go to the warps from the
            // top down: on late diagonals the tail of step k-1 occupies the
            // low warps, so the bulk of step k runs beside it
            const float rcp_units = TABLE ? __frcp_ru((float)units) : 0.f;  // it / units, exactly, it < 2^10
            const bool dyn = RKR_EXP_DYNUNIT && P == 1;
            auto grab = [&]() {
                int v = 0;
                if (lane == 0) v = atomicAdd(s_ucnt + (k & 1), 1);
                return __shfl_sync(0xffffffffu, v, 0);
            };
            for (int it = dyn ? grab() : (COMM ? kNC - 1 - warp : warp); it < units * P;
                 it = dyn ? grab() : it + kNC) {
                const int p = P == 1 ? 0 : (TABLE ? (int)((float)it * rcp_units) : it / units);
                const int u = it - p * units;
                const int s = min(u * RPW + rw, rows - 1);  // (a clamped row is not stored)
                const int m = m_lo + ml;
                const int ib = 1 + p * chunk;
                const int ie = ib + chunk < k - 1 ? ib + chunk : k - 1;
                uint32_t best = INF;
                int code = 0;
                if constexpr (STREAM)
                    scan_cuts_streamed<RPW>(opt, prog + s * k,
                                            reinterpret_cast<int4*>(smem_raw + sm.prog) + warp * RPW * kSlice,
                                            ib, ie, m, kCutBit | (s + 1), best, code);
                else
                    // tile jobs: batches of kUB cuts with the sweeps re-read
                    // (config 3 fill -4 %, config 4 -2.4 %); the co-resident
                    // tables keep kU (config 1 +8 % with kUB)
                    scan_cuts<RPW, TABLE ? kU : kUB, !TABLE>(opt, prog + s * k, ib, ie, m, kCutBit | (s + 1),
                                                           best, code);
                pbest[it * 32 + lane] = best;
                pcode[it * 32 + lane] = (uint16_t)code;
            }
        }
        if (tp.trace && tid == 0) t1 = clock64();
        // diagonal k-1 of the lower tiles acquired (and, with P > 1, every
        // bulk part of this step written)
        if constexpr (COMM) {
            nb_sync(kBarReady);
        } else {
            if (k >= 1 && warp == 0) {
                const int* row = done + (int64_t)(k - 1) * tp.T;
                for (int q = lane; q < d_eff; q += 32)
                    while (t_ld_relaxed(row + j - 1 - q) == 0) __nanosleep(20);
                __syncwarp();
                if (lane == 0) {
                    if (halo_in) wait_halo(k - 1);
                    t_fence_acq_rel();
                }
            }
            __syncthreads();
        }
        if (tp.trace && tid == 0) t2 = clock64();

        if (RKR_EXP_DYNUNIT && tid == 0) s_ucnt[k & 1] = 0;  // bulk(k) done: re-arm for k + 2

        // ---- tail -------------------------------------------------------------------
        // Candidates are merged in the reference's scan order -- options (menu
        // order), cut i = 0, the bulk parts (i = 1 .. k-2, part by part), cut
        // i = k-1 -- each with a strict '<', so the first minimum wins.
        const int rbase = (int)diag_off(L, k);
        // Late diagonals (at most half as many units as compute warps) split
        // each unit's tail over two warps: half h = 0 takes the first option
        // batches, half h = 1 the remaining options, cut i = 0, the bulk parts
        // and cut i = k-1.  All of h = 0's candidates precede h = 1's in the
        // scan, so the cell's first minimum is h0 if h0.value <= h1.value.
        uint32_t* xbest = reinterpret_cast<uint32_t*>(smem_raw + sm.xch);
        uint16_t* xcode = reinterpret_cast<uint16_t*>(xbest + kNT);
        // (OM) Two open units at once: when both rows of a warp's next two
        // units are open and have at most 8 undominated options, all their
        // reads (two tail cuts and 8 option windows each) go out together --
        // one memory round trip for the pair instead of one per unit (the
        // tail is a chain of dependent round trips per warp)
        auto tail_pair = [&](int vA, int vB) -> bool {
            const int sA = min(vA * RPW + rw, rows - 1), sB = min(vB * RPW + rw, rows - 1);
            const int64_t thA = max(s_thx[sA] + s_thx[2 * L + sA + k], s_thx[L + sA]);
            const int64_t thB = max(s_thx[sB] + s_thx[2 * L + sB + k], s_thx[L + sB]);
            if (!__all_sync(0xffffffffu, thA <= m_lo && thB <= m_lo && s_pcnt[sA] <= 8 && s_pcnt[sB] <= 8))
                return false;
            const int m = m_lo + ml;
            const int4 nil = make_int4(0, 0, 0, M + 2);
            const int4 a0 = prog[sA * k], b0 = prog[sB * k];
            const int4 a1 = k > 1 ? prog[sA * k + k - 1] : nil, b1 = k > 1 ? prog[sB * k + k - 1] : nil;
            uint32_t ca[4], cb[4];
            ca[0] = tail_ld(opt + (uint32_t)(a0.x + m));
            ca[1] = tail_ld(opt + (uint32_t)(a0.y + m));
            cb[0] = tail_ld(opt + (uint32_t)(b0.x + m));
            cb[1] = tail_ld(opt + (uint32_t)(b0.y + m));
            ca[2] = ca[3] = cb[2] = cb[3] = INF;
            if (k > 1) {
                ca[2] = tail_ld(opt + (uint32_t)(a1.x + m));
                ca[3] = tail_ld(opt + (uint32_t)(a1.y + m));
                cb[2] = tail_ld(opt + (uint32_t)(b1.x + m));
                cb[3] = tail_ld(opt + (uint32_t)(b1.y + m));
            }
            // row (s+1, t) of each unit: id rid - (L - k)
            const uint32_t* __restrict__ wA = lane_base(opt, (rbase + sA - (L - k)) * sr + g.pad + m);
            const uint32_t* __restrict__ wB = lane_base(opt, (rbase + sB - (L - k)) * sr + g.pad + m);
            const int4* pA = reinterpret_cast<const int4*>(s_pru + sA * kPcap);
            const int4* pB = reinterpret_cast<const int4*>(s_pru + sB * kPcap);
            uint32_t ta[8], tb[8];
#pragma unroll
            for (int q = 0; q < 8; q += 2) {
                const int4 x = pA[q >> 1], y = pB[q >> 1];
                ta[q] = (uint32_t)x.y + tail_ld(wA + x.x);
                ta[q + 1] = (uint32_t)x.w + tail_ld(wA + x.z);
                tb[q] = (uint32_t)y.y + tail_ld(wB + y.x);
                tb[q + 1] = (uint32_t)y.w + tail_ld(wB + y.z);
            }
            auto finish = [&](const uint32_t (&t)[8], const uint32_t (&c)[4], const int4& e0, const int4& e1,
                              int s, int u) {
                uint32_t best = INF;
                int code = 0;
                merge8p(t, s_pcd + s * kPcap, best, code);
                const int cbase = kCutBit | (s + 1);
                uint32_t tot = (uint32_t)e0.z + c[0] + c[1];
                if (e0.w <= m && tot < best) {
                    best = tot;
                    code = cbase;
                }
                for (int p = 0; nb > 0 && p < P; ++p) {
                    const int idx = (p * units + u) * 32 + lane;
                    const uint32_t vv = pbest[idx];
                    if (vv < best) {
                        best = vv;
                        code = pcode[idx];
                    }
                }
                tot = (uint32_t)e1.z + c[2] + c[3];
                if (e1.w <= m && tot < best) {
                    best = tot;
                    code = cbase + k - 1;
                }
                if (m <= M && (RPW == 1 || u * RPW + rw < rows)) {  // store (chain_dp.hpp:176-177)
                    const int rid = rbase + s;
                    opt[(int64_t)rid * sr + g.pad + m] = best;
                    arg[(int64_t)rid * g.sa + m] = (uint16_t)code;
                }
            };
            finish(ta, ca, a0, a1, sA, vA);
            finish(tb, cb, b0, b1, sB, vB);
            return true;
        };
        for (int v = warp; v < units * TS; v += kNC) {
            if constexpr (OM && !STREAM && !SPLIT && !HALO) {
                if (RKR_PAIR_TAIL && tp.prune && k > 0 && v + kNC < units && tail_pair(v, v + kNC)) {
                    v += kNC;
                    continue;
                }
            }
            const int h = TS == 1 ? -1 : (v >= units ? 1 : 0);  // -1: the whole tail
            const int u = TS == 1 ? v : v - h * units;
            const bool valid = RPW == 1 || u * RPW + rw < rows;  // stores only for real rows
            const int s = min(u * RPW + rw, rows - 1);
            const int m = m_lo + ml;
            const int rid = rbase + s;
            // options of the unit's rows, warp-uniform (the padded slots of a
            // shorter block never win: pass time INF, threshold M + 1)
            const int nopt = RPW == 1 ? s_blk[s + 1] - s_blk[s]
                                      : __reduce_max_sync(0xffffffffu, s_blk[s + 1] - s_blk[s]);
            // option batches of this half: [ia, ib)
            const int nb2 = (((nopt + kOB - 1) / kOB) + 1) / 2 * kOB;  // first half, whole batches
            const int ia = h == 1 ? nb2 : 0;
            const int ib = h == 0 ? (nb2 < nopt ? nb2 : nopt) : nopt;
            const bool cuts = h != 0;
            // tail cut operands: i = 0 (c = s+1) and i = k-1 (c = t); their
            // loads go out first
            uint32_t tl0 = INF, tr0 = INF, tl1 = INF, tr1 = INF;
            int4 e0 = make_int4(0, 0, 0, M + 2), e1 = e0;
            if (k > 0 && cuts) {
                e0 = STREAM ? __ldg(prog + s * k) : prog[s * k];
                tl0 = tail_ld(opt + (uint32_t)(e0.x + m));
                tr0 = tail_ld(opt + (uint32_t)(e0.y + m));
                if (k > 1) {
                    e1 = STREAM ? __ldg(prog + s * k + k - 1) : prog[s * k + k - 1];
                    tl1 = tail_ld(opt + (uint32_t)(e1.x + m));
                    tr1 = tail_ld(opt + (uint32_t)(e1.y + m));
                }
            }
            uint32_t best = INF;
            int code = 0;
            // Case 1 (chain_dp.hpp:139-156): options of block s in menu order;
            // windows of row (s+1, t) at m - pack_chg (row (s+1, t) is the next
            // row of diagonal k-1: id rid - (L - k))
            const int4* od4 = reinterpret_cast<const int4*>(s_opd + s * ocap);  // 2 options each
            const int4* th4 = reinterpret_cast<const int4*>(thrs + s * ocap);   // 4 options each
            if constexpr (STREAM) {
                // this unit's block options (shift, pass time) and row
                // thresholds into the warp's slice, coalesced, padded like
                // the staged layout (padding never wins: pass time INF,
                // threshold M+1)
                const int slot = warp * RPW + rw;
                int2* wo = reinterpret_cast<int2*>(smem_raw + sm.thr) + slot * ocap;
                int32_t* wt = reinterpret_cast<int32_t*>(smem_raw + sm.thr + (size_t)kNW * RPW * ocap * 8) +
                              slot * ocap;
                __syncwarp();  // the previous unit's readers are done
                const int o0 = s_blk[s], own = s_blk[s + 1] - o0;
                for (int i = ml; i < ocap; i += W) {
                    wo[i] = i < own ? make_int2(-__ldg(pq.pc + o0 + i),
                                                 (int)__ldg(static_cast<const uint32_t*>(pq.otot) + o0 + i))
                                     : make_int2(0, (int)INF);
                    wt[i] = __ldg(thrs + s * ocap + i);
                }
                __syncwarp();
                od4 = reinterpret_cast<const int4*>(wo);
                th4 = reinterpret_cast<const int4*>(wt);
            }
            // whole batches: the padding options never win.  Diagonal 0 has
            // no sub-row (chain_dp.hpp:146: s == t), so its loop is a separate
            // instantiation without loads; otherwise each window read is one
            // IMAD.WIDE off the lane's row base (shifts stored negated).
            // (OM) no option threshold of the row is above the warp's
            // smallest budget m_lo: the batches run ungated through merge8
            bool open = false, popen = false;
            int pbat = 0;  // (popen) batches of 8 undominated options
            if constexpr (OM && !STREAM) {
                const int64_t thx = max(s_thx[s] + s_thx[2 * L + s + k], s_thx[L + s]);
                open = __all_sync(0xffffffffu, thx <= m_lo);
                if (tp.prune && open && k > 0) {
                    const int pc = s_pcnt[s];
                    popen = __all_sync(0xffffffffu, pc <= kPcap);
                    pbat = (__reduce_max_sync(0xffffffffu, pc) + 7) >> 3;
                }
            }
            auto options = [&](auto has_sub) {
                constexpr bool SUB = decltype(has_sub)::value;
                const uint32_t* __restrict__ optw =
                    lane_base(opt, SUB ? (rid - (L - k)) * sr + g.pad + m : 0);
                auto sub_at = [&](int neg_shift) -> uint32_t {  // row (s+1, t) at m - shift
                    return SUB ? tail_ld(optw + neg_shift) : 0u;
                };
                // Whole batches [ia, ibf), then (OM) the options past them one
                // by one (the first one's read goes out with the first
                // batch's): OM scans no padding, the other kernels run the
                // last batch into it.  (Software-pipelining the batches -- the
                // next batch's reads in flight during this batch's compares --
                // spills at 64 registers per thread.)
                if constexpr (SUB && OM && !STREAM) {
                    if (popen) {  // open row: the block's undominated options only (h = 1: none)
                        if (h == 1) return;
                        const int4* pr4 = reinterpret_cast<const int4*>(s_pru + s * kPcap);
                        const uint16_t* pcd = s_pcd + s * kPcap;
                        for (int hb = 0; hb < pbat; ++hb) {
                            uint32_t tot[8];
#pragma unroll
                            for (int q = 0; q < 8; q += 2) {
                                const int4 o2 = pr4[(hb * 8 + q) >> 1];
                                tot[q] = (uint32_t)o2.y + sub_at(o2.x);
                                tot[q + 1] = (uint32_t)o2.w + sub_at(o2.z);
                            }
                            merge8p(tot, pcd + hb * 8, best, code);
                        }
                        return;
                    }
                }
                const int ibf = OM ? ia + (ib - ia) / kOB * kOB : ib;
                const int2* od2 = reinterpret_cast<const int2*>(od4);
                const int2 orem = ibf < ib ? od2[ibf] : make_int2(0, 0);
                const uint32_t srem = ibf < ib ? sub_at(orem.x) : 0u;
                for (int i0 = ia; i0 < ibf; i0 += kOB) {
                    uint32_t tot[kOB];
#pragma unroll
                    for (int q = 0; q < kOB; q += 2) {
                        const int4 o2 = od4[(i0 + q) >> 1];
                        tot[q] = (uint32_t)o2.y + sub_at(o2.x);
                        tot[q + 1] = (uint32_t)o2.w + sub_at(o2.z);
                    }
                    if (OM && SUB && open) {
#pragma unroll
                        for (int h = 0; h < kOB; h += 8)
                            merge8(*reinterpret_cast<uint32_t(*)[8]>(tot + h), i0 + h + 1, best, code);
                        continue;
                    }
                    int32_t th[kOB];
#pragma unroll
                    for (int q = 0; q < kOB; q += 4) {
                        const int4 t4 = th4[(i0 + q) >> 2];
                        th[q] = t4.x;
                        th[q + 1] = t4.y;
                        th[q + 2] = t4.z;
                        th[q + 3] = t4.w;
                    }
#pragma unroll
                    for (int q = 0; q < kOB; ++q) {
                        if (m >= th[q] && tot[q] < best) {
                            best = tot[q];
                            code = i0 + q + 1;
                        }
                    }
                }
                const int32_t* thr_row = reinterpret_cast<const int32_t*>(th4);
#pragma unroll 1
                for (int i = ibf; i < ib; ++i) {
                    const int2 o = i == ibf ? orem : od2[i];
                    const uint32_t tot = (uint32_t)o.y + (i == ibf ? srem : sub_at(o.x));
                    if (m >= thr_row[i] && tot < best) {
                        best = tot;
                        code = i + 1;
                    }
                }
            };
#ifdef RKR_TRACE_UNIT2
            unsigned long long xa = 0, xb = 0;
            if (tp.trace && tid == 0 && v == warp) xa = clock64();
#endif
            if (k > 0)
                options(std::true_type{});
            else
                options(std::false_type{});
#ifdef RKR_TRACE_UNIT2
            asm volatile("" ::"r"(best), "r"(code));
            if (tp.trace && tid == 0 && v == warp) {
                xb = clock64();
                unsigned long long* tr = tp.trace + 6 * ((int64_t)k * tp.T + j);
                tr[1] = xa;
                tr[2] = xb;
            }
#endif
            if (cuts) {
                // Case 2 (chain_dp.hpp:158-174): cut i = 0, bulk parts, cut i = k-1
                const int cb = kCutBit | (s + 1);
                {
                    const uint32_t tot = (uint32_t)e0.z + tl0 + tr0;
                    if (e0.w <= m && tot < best) {
                        best = tot;
                        code = cb;
                    }
                }
                if (nb > 0) {
                    for (int p = 0; p < P; ++p) {
                        const int idx = (p * units + u) * 32 + lane;
                        const uint32_t vv = pbest[idx];
                        if (vv < best) {
                            best = vv;
                            code = pcode[idx];
                        }
                    }
                }
                {
                    const uint32_t tot = (uint32_t)e1.z + tl1 + tr1;
                    if (e1.w <= m && tot < best) {
                        best = tot;
                        code = cb + k - 1;
                    }
                }
            }
#ifdef RKR_TRACE_UNIT2
            asm volatile("" ::"r"(best), "r"(code));
            if (tp.trace && tid == 0 && v == warp) tp.trace[6 * ((int64_t)k * tp.T + j) + 3] = clock64();
#endif
            if (h == 1) {  // hand the later half to the h = 0 warp
                xbest[u * 32 + lane] = best;
                xcode[u * 32 + lane] = (uint16_t)code;
            } else if (h == -1 && m <= M && valid) {  // store (chain_dp.hpp:176-177)
                opt[(int64_t)rid * sr + g.pad + m] = best;
                arg[(int64_t)rid * g.sa + m] = (uint16_t)code;
                if (HALO && D.arg_mirror)  // shard 0's walk mirror (peer store)
                    D.arg_mirror[(int64_t)rid * D.mirror_sa + D.mirror_base + m] = (uint16_t)code;
                if (halo_out && m >= Wl - g.pad)  // the next shard's halo slot m - Wl
                    static_cast<uint32_t*>(D.next_opt)[(int64_t)rid * D.next_sr + g.pad + (m - Wl)] = best;
            } else if (h == 0) {
                xbest[(kNT >> 1) + u * 32 + lane] = best;  // (merged below)
                xcode[(kNT >> 1) + u * 32 + lane] = (uint16_t)code;
            }
        }
        if (TS == 2 && warp < 2 * units) {
            // only the 2 * units tail warps meet here (warp w < 2 * units took
            // v = w): the others go straight on to bulk(k+1)
            nb_sync_n(kBarSplit, 2 * units * 32);
            for (int u = warp; u < units; u += kNC) {
                const bool valid = RPW == 1 || u * RPW + rw < rows;
                const int s = min(u * RPW + rw, rows - 1);
                const int m = m_lo + ml;
                const int rid = rbase + s;
                uint32_t best = xbest[(kNT >> 1) + u * 32 + lane];
                int code = xcode[(kNT >> 1) + u * 32 + lane];
                const uint32_t b1 = xbest[u * 32 + lane];
                if (b1 < best) {
                    best = b1;
                    code = xcode[u * 32 + lane];
                }
                if (m <= M && valid) {  // store (chain_dp.hpp:176-177)
                    opt[(int64_t)rid * sr + g.pad + m] = best;
                    arg[(int64_t)rid * g.sa + m] = (uint16_t)code;
                    if (halo_out && m >= Wl - g.pad)
                        static_cast<uint32_t*>(D.next_opt)[(int64_t)rid * D.next_sr + g.pad + (m - Wl)] = best;
                }
            }
        }
        if (tp.trace && tid == 0) {
            t3 = clock64();
            unsigned long long* tr = tp.trace + 6 * ((int64_t)k * tp.T + j);
#if !defined(RKR_TRACE_EXPERIMENT) && !defined(RKR_TRACE_UNIT2)
            tr[0] = t0;
#endif
#ifndef RKR_TRACE_UNIT2
            tr[1] = c0;
            tr[2] = t1;
            if (!COMM) tr[3] = t1;
#endif
            tr[4] = t2;
            tr[5] = t3;
        }
        if constexpr (COMM) {
#if RKR_EXP_SYNCDONE
            nb_sync(kBarDone);  // timing experiment: bulk(k+1) only after every tail(k)
#else
            nb_arrive(kBarDone);  // stores of diagonal k issued; go on to bulk(k+1)
#endif
        } else {
            __syncthreads();
            if (tid == 0) {
                t_red_release_add(done + (int64_t)k * tp.T + j, 1);
                if (halo_out) push_halo(k);
                if (!STREAM && k + 2 < L) {
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    stage_step(tp, pq, sm, smem_raw, bars, L, k + 2);
                }
            }
        }
    }
    }  // compute warps
}

// ---- fused K2: the last finisher walks the schedule -----------------------
// (build_schedule_rec, chain_dp.hpp:211-246).  Every CTA (every job) counts
// itself out with an acq_rel add after its last publish; the one that sees
// n_parts - 1 has acquired every other tile's stores.  Saves the walk's
// launch and reads a table that is still hot in L2.  Called by all threads
// of the CTA after its (last) tile job.
__device__ __forceinline__ void last_walk(const InstDesc& D, const TilePlan& tp, int n_parts,
                                       unsigned char* smem_raw) {
    const TileSmem& sm = tp.sm;
    const Geometry& g = D.g;
    const DevMenu& dm = D.dm;
    const uint32_t* __restrict__ opt = static_cast<const uint32_t*>(D.opt);
    const uint16_t* __restrict__ arg = D.arg;
    const int L = g.L;
    const int tid = threadIdx.x;
    __syncthreads();
    int* s_last = reinterpret_cast<int*>(smem_raw + sm.blk);  // s_blk is done with
    if (tid == 0) {
        int prev;
        asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], 1;"
                     : "=r"(prev)
                     : "l"(tp.fin)
                     : "memory");
        s_last[L + 1] = prev == n_parts - 1;
    }
    __syncthreads();
    if (!s_last[L + 1]) return;
    // menu lookups and the stack in shared memory (program and partial
    // buffers are free now); the global view when they do not fit
    int4* sstack = reinterpret_cast<int4*>(smem_raw + sm.best);
    int32_t* mb = reinterpret_cast<int32_t*>(smem_raw + sm.prog);
    // (the program region: two staged buffers, or one block of per-warp
    // slices when programs are streamed)
    const bool fit = 4ull * (2 * (L + 1) + 2 * (uint64_t)tp.nq) <=
                         (tp.stream ? 1ull : 2ull) * sm.prog_bytes &&
                     16ull * (2 * L + 16) <= (uint64_t)tp.cap * 4;
    if (fit) {
        int32_t *b = mb, *a = b + L + 1, *id = a + L + 1, *gq = id + tp.nq;
        for (int x = tid; x <= L; x += kNT) {
            b[x] = __ldg(dm.blk_off + x);
            a[x] = (int)__ldg(dm.act_u + x);
        }
        for (int x = tid; x < tp.nq; x += kNT) {
            id[x] = __ldg(dm.ids + x);
            gq[x] = (int)__ldg(dm.chg_bt + x);
        }
        __syncthreads();
        if (tid == 0)
            walk<uint32_t>(g, SharedMenuView{b, id, gq, a}, opt, arg, tp.ws, tp.wt, tp.wm, tp.wops,
                           tp.wcap, sstack, tp.wout);
    } else if (tid == 0) {
        walk<uint32_t>(g, GlobalMenuView{&dm}, opt, arg, tp.ws, tp.wt, tp.wm, tp.wops, tp.wcap,
                       tp.wstack, tp.wout);
    }
    __syncthreads();  // the walk's shared memory is free again
}

template <int RPW, bool COMM, bool SPLIT, bool STREAM, bool HALO>
__global__ void __launch_bounds__(kNT, 1) fill_tiles(const __grid_constant__ InstDesc D,
                                                    const __grid_constant__ TilePlan tp) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const TileSmem& sm = tp.sm;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw + sm.bar);
    const int tid = threadIdx.x;
    if (tid == 0) {
        mbar_init(bars + 0, 1);
        mbar_init(bars + 1, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    tile_job<RPW, COMM, SPLIT, STREAM, true, HALO>(D, tp, blockIdx.x, smem_raw, 0, 0);
    const Geometry& g = D.g;
    const DevMenu& dm = D.dm;
    uint32_t* __restrict__ opt = static_cast<uint32_t*>(D.opt);
    uint16_t* __restrict__ arg = D.arg;
    const int L = g.L;

    // ---- fused K2: the last CTA to finish walks the schedule ----------------
    // (inline here rather than last_walk(): measured 3 us faster on config 2)
    // (build_schedule_rec, chain_dp.hpp:211-246).  Every CTA counts itself
    // out with an acq_rel add after its last publish; the one that sees T-1
    // has acquired every other tile's stores.  Saves the walk's launch and
    // reads a table that is still hot in L2.  The last CTA also returns the
    // done flags and the counter to zero for the next launch (every CTA has
    // stopped polling by then), so a refill needs no memset first.
    __syncthreads();
    int* s_last = reinterpret_cast<int*>(smem_raw + sm.blk);  // s_blk is done with
    if (tid == 0) {
        int prev;
        asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], 1;"
                     : "=r"(prev)
                     : "l"(tp.fin)
                     : "memory");
        s_last[L + 1] = prev == tp.T - 1;
    }
    __syncthreads();
    if (!s_last[L + 1]) return;
    if (tid == 0) *tp.fin = 0;
    for (int i = tid - 32; i >= 0 && i < L * tp.T; i += kNT - 32) tp.done[i] = 0;  // warps 1..
    if (!tp.walk) return;
    // menu lookups and the stack in shared memory (program and partial
    // buffers are free now); the global view when they do not fit
    int4* sstack = reinterpret_cast<int4*>(smem_raw + sm.best);
    int32_t* mb = reinterpret_cast<int32_t*>(smem_raw + sm.prog);
    // (the program region: two staged buffers, or one block of per-warp
    // slices when programs are streamed)
    const bool fit = 4ull * (2 * (L + 1) + 2 * (uint64_t)tp.nq) <=
                         (tp.stream ? 1ull : 2ull) * sm.prog_bytes &&
                     16ull * (2 * L + 16) <= (uint64_t)tp.cap * 4;
    if (fit) {
        int32_t *b = mb, *a = b + L + 1, *id = a + L + 1, *gq = id + tp.nq;
        for (int x = tid; x <= L; x += kNT) {
            b[x] = __ldg(dm.blk_off + x);
            a[x] = (int)__ldg(dm.act_u + x);
        }
        for (int x = tid; x < tp.nq; x += kNT) {
            id[x] = __ldg(dm.ids + x);
            gq[x] = (int)__ldg(dm.chg_bt + x);
        }
        __syncthreads();
        if (tid == 0)
            walk<uint32_t>(g, SharedMenuView{b, id, gq, a}, opt, arg, tp.ws, tp.wt, tp.wm, tp.wops,
                           tp.wcap, sstack, tp.wout);
    } else if (tid == 0) {
        walk<uint32_t>(g, GlobalMenuView{&dm}, opt, arg, tp.ws, tp.wt, tp.wm, tp.wops, tp.wcap,
                       tp.wstack, tp.wout);
    }
}

// Batches (config 4 sweeps): persistent CTAs take (table, tile) jobs from a
// queue ordered table by table, tiles ascending.  A job only waits on lower
// tiles of its own table, which were dequeued earlier by CTAs that are
// running or done, so the queue cannot deadlock and tables need not be
// co-resident.
template <int RPW, bool COMM, bool SPLIT, bool STREAM, bool WALK, bool HALO>
__global__ void __launch_bounds__(kNT, 1) fill_tiles_batch(const InstDesc* __restrict__ descs,
                                                          const TilePlan* __restrict__ tps,
                                                          const int2* __restrict__ jobs, int njobs,
                                                          unsigned int* __restrict__ counter,
                                                          const __grid_constant__ TilePlan walkp) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    __shared__ int s_job;
    const TileSmem& sm = tps[0].sm;  // one layout for the whole batch
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw + sm.bar);
    const int tid = threadIdx.x;
    if (tid == 0) {
        mbar_init(bars + 0, 1);
        mbar_init(bars + 1, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    uint32_t ph0 = 0, ph1 = 0;
    for (;;) {
        if (tid == 0) s_job = (int)atomicAdd(counter, 1u);
        __syncthreads();
        const int q = s_job;
        if (q >= njobs) break;
        const int2 jb = jobs[q];
        const InstDesc& jd = descs[jb.x];
        const TilePlan& jp = tps[jb.x];
        tile_job<RPW, COMM, SPLIT, STREAM, false, HALO>(jd, jp, jb.y, smem_raw, ph0, ph1);
        const int L = jd.g.L;
        ph0 += (uint32_t)(L + 1) / 2;  // uses of mbarrier 0 (even steps) and 1
        ph1 += (uint32_t)L / 2;
        // a single table run as tile jobs: the last job to finish walks
        if constexpr (WALK) last_walk(descs[0], walkp, njobs, smem_raw);
        __syncthreads();  // shared memory and s_job are reused by the next job
    }
}

// One table as tile jobs (config 3: more tiles than SMs), tiles in budget
// order from a queue.  Like fill_tiles_batch on a one-table batch, but the
// descriptor and plan are kernel parameters (constant bank): as global reads
// they miss L1 after every acquisition of the lower tiles' flags (ld.acquire
// empties L1) and put L2 round trips on the tail's critical path, and
// constant-bank operands need no registers.
template <int RPW, bool COMM, bool SPLIT, bool STREAM, bool WALK, bool MIXED>
__global__ void __launch_bounds__(kNT, 1) fill_tiles_jobs1(const __grid_constant__ InstDesc D,
                                                          const __grid_constant__ TilePlan tp,
                                                          unsigned int* __restrict__ counter) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    __shared__ int s_job;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw + tp.sm.bar);
    const int tid = threadIdx.x;
    if (tid == 0) {
        mbar_init(bars + 0, 1);
        mbar_init(bars + 1, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    uint32_t ph0 = 0, ph1 = 0;
    for (;;) {
        if (tid == 0) s_job = (int)atomicAdd(counter, 1u);
        __syncthreads();
        const int j = s_job;
        if (j >= tp.T) break;
        if (MIXED && j >= tp.j1)  // a half tile of the last wave
            tile_job<2, COMM, SPLIT, STREAM, false, false, MIXED>(D, tp, j, smem_raw, ph0, ph1);
        else
            tile_job<RPW, COMM, SPLIT, STREAM, false, false, MIXED>(D, tp, j, smem_raw, ph0, ph1);
        ph0 += (uint32_t)(D.g.L + 1) / 2;
        ph1 += (uint32_t)D.g.L / 2;
        if constexpr (WALK) last_walk(D, tp, tp.T, smem_raw);
        __syncthreads();  // shared memory and s_job are reused by the next job
    }
}

template <int RPW, bool COMM, bool SPLIT, bool STREAM, bool HALO = false>
int launch_tiles_t(const InstDesc& d, const TilePlan& tp, cudaStream_t st) {
    auto kern = fill_tiles<RPW, COMM, SPLIT, STREAM, HALO>;
    const size_t smem = tp.sm.total;
    if (set_dyn_smem((const void*)kern, smem) != cudaSuccess)
        return 3;
    InstDesc dd = d;
    TilePlan pp = tp;
    void* args[] = {&dd, &pp};
    // cooperative: the CTAs wait on each other, so all T must be co-resident
    if (cudaLaunchCooperativeKernel((const void*)kern, dim3(tp.T), dim3(kNT), args, smem, st) !=
        cudaSuccess)
        return 3;
    return 0;
}

}  // namespace

// Tile width, warp roles and program staging of K1t for one table; 0 = not
// eligible (the queue-scheduled K1p runs instead).  kn: the caller's
// rkr_exec tuning fields (0 = the measured defaults below).
int tile_rows_for(int64_t slots, int sms, const TileKnobs& kn) {
    if (kn.rows == 1 || kn.rows == 2) return kn.rows;
    // RPW = 2 halves the tile (16 slots, two rows per warp): twice the tiles,
    // each with half the work but the same per-step costs (program staging,
    // flags, barriers) and twice the L1 wavefronts per load.  It only pays
    // where 32-slot tiles leave at least half the SMs idle: a co-resident
    // table of <= 74 tiles (config 1: fill 0.070 -> 0.064 ms; a budget shard
    // of config 3 on 8 GPUs: 64 tiles).  As tile jobs it loses even when it
    // evens out the waves (config 3: 1025 half jobs in 7 half waves, 4.96 ms,
    // against 513 jobs in 4 waves, 4.07 ms).
    const int64_t t1 = (slots + 31) / 32;
    return 2 * t1 <= sms ? 2 : 1;
}

int tile_plan(const Geometry& g, int width, int sms, int64_t nq, int ocap, const TileKnobs& kn,
              TilePlan& tp) {
    if (kn.tune & RKR_TUNE_NO_TILES) return 0;
    if (width != 32) return 0;
    // 32-bit element offsets inside the table (plus the tile over-read).
    // (A config-5 shard on 8 GPUs holds 4.4e9 elements: K1p, 64-bit row
    // pointers, runs it.)
    if ((double)g.rows * g.sr + 64.0 * 32 + g.pad >= 2147483647.0) return 0;
    // When the tiles do not all fit one CTA per SM the table runs as tile
    // jobs (fill_tiles_batch on one table): a dataflow queue needs no
    // co-residency, and walking the tiles in budget order keeps the rows
    // around the active band in L2 (config 3: 4.65 ms and 0.13 GB of DRAM
    // reads, against 5.14 ms and 13.3 GB with 129 co-resident 128-slot tiles)
    const int rpw = tile_rows_for((int64_t)g.M + 1, sms, kn);
    const int W = 32 / rpw;
    const int64_t T = ((int64_t)g.M + 1 + W - 1) / W;
    tp.jobs = (T > sms || (kn.tune & RKR_TUNE_JOBS)) ? 1 : 0;
    tp.rpw = rpw;
    tp.W = W;
    tp.T = (int32_t)T;
    tp.d = (g.pad + W - 1) / W;
    const int64_t units = ((int64_t)g.L + rpw - 1) / rpw;  // warp units of the widest step
    tp.cap = (int32_t)(units * 32 > kNT ? units * 32 : kNT);
    tp.L = g.L;
    tp.nq = (int32_t)nq;
    tp.ocap = (int32_t)ceil_to(ocap, rpw == 1 ? kOptBatch<1> : kOptBatch<2>);
    // the communication warp pays off where the fill is latency-bound
    // (per-step work of a few microseconds: configs 1-2), not where it is
    // throughput-bound (config 3: measured 5.36 ms without, 6.56 with)
    tp.comm = (tp.jobs || (double)g.rows * (g.M + 1) <= 16.0e6) ? 1 : 0;
    if (kn.tune & RKR_TUNE_COMM_OFF) tp.comm = 0;
    if (kn.tune & RKR_TUNE_COMM_ON) tp.comm = 1;
    // split tails on late diagonals: co-resident tables whose blocks have
    // two or more option batches (config 2: -3.5 %; measured slower with
    // one batch (config 1), as tile jobs (config 3: +7 %) and for batches
    // of tables (config 4))
    tp.split = tp.comm && !tp.jobs && tp.ocap >= 16 ? 1 : 0;
    if (kn.tune & RKR_TUNE_SPLIT_OFF) tp.split = 0;
    if (kn.tune & RKR_TUNE_SPLIT_ON) tp.split = tp.comm;
    tp.stream = 0;
    tp.prune = 0;
    tp.sm = tile_smem(tp);
    if (tp.sm.total > 220 * 1024 || (kn.tune & RKR_TUNE_STREAM)) {
        // long chains: a diagonal's programs do not fit shared memory.
        // The streamed variant reads them from global memory (each warp
        // stages its unit's program, options and thresholds into its own
        // slice); with the communication warp it beats the row-segment
        // queue (L=256, B=64, M=4096: 25.9 ms against K1p's 27.0 ms)
        tp.stream = 1;
        tp.split = 0;
        if (!(kn.tune & RKR_TUNE_COMM_OFF)) tp.comm = 1;
        tp.sm = tile_smem(tp);
    }
    // The last wave of tile jobs: 513 jobs of config 3 on 148 SMs run as 3
    // full waves and a fourth of 69 jobs (14 % of the SMs idle over the
    // fill).  When the jobs past the full waves cover at most half a wave,
    // they become 16-slot tiles (two rows per warp, measured 0.69 of a
    // 32-slot job): one wave of half jobs instead of a wave of whole ones.
    tp.j1 = INT32_MAX;
    if (kn.mixed && tp.jobs && rpw == 1 && tp.comm && !tp.stream && !tp.split &&
        !(kn.tune & RKR_TUNE_UNIFORM)) {
        const int64_t full = (T / sms) * sms;  // jobs in full waves
        const int64_t rest = (int64_t)g.M + 1 - 32 * full;
        const int64_t halves = (rest + 15) / 16;
        if (full > 0 && rest > 0 && halves <= sms) {
            tp.j1 = (int32_t)full;
            tp.T = (int32_t)(full + halves);
        }
    }
    if ((kn.tune & RKR_TUNE_MIXED) && kn.mixed && tp.jobs && rpw == 1 && tp.comm && !tp.stream &&
        !tp.split && T >= 2) {  // test knob: half the tiles 32-slot, the rest 16-slot
        const int64_t j1 = T / 2, rest = (int64_t)g.M + 1 - 32 * j1;
        tp.j1 = (int32_t)j1;
        tp.T = (int32_t)(j1 + (rest + 15) / 16);
    }
    // Dominance pruning of open rows (the mixed-width single-table jobs,
    // tile_job's OM): config 3 fill -8 %; the latency-bound co-resident
    // tables (configs 1-2) and batches (config 4) measured 2-10 % slower
    // with it (shorter scans, not shorter critical paths).
    if (tp.j1 != INT32_MAX && !(kn.tune & RKR_TUNE_NO_PRUNE)) {
        tp.prune = 1;
        tp.sm = tile_smem(tp);
        if (tp.sm.total > 220 * 1024) {  // the lists do not fit beside the staged programs
            tp.prune = 0;
            tp.sm = tile_smem(tp);
        }
    }
    return tp.sm.total <= 220 * 1024 ? 1 : 0;
}

namespace {

template <int RPW>
int launch_fill_tiles_r(const InstDesc& d, const TilePlan& tp, cudaStream_t st) {
    if (tp.halo) {  // budget shards: communication warp, no split tails
        if (!tp.comm || tp.split) return 3;
        return tp.stream ? launch_tiles_t<RPW, true, false, true, true>(d, tp, st)
                         : launch_tiles_t<RPW, true, false, false, true>(d, tp, st);
    }
    if (tp.stream) return tp.comm ? launch_tiles_t<RPW, true, false, true>(d, tp, st)
                                  : launch_tiles_t<RPW, false, false, true>(d, tp, st);
    if (tp.comm) return tp.split ? launch_tiles_t<RPW, true, true, false>(d, tp, st)
                                 : launch_tiles_t<RPW, true, false, false>(d, tp, st);
    return launch_tiles_t<RPW, false, false, false>(d, tp, st);
}

template <int RPW>
int launch_fill_tiles_batch_r(const InstDesc* descs, const TilePlan* tps, const int2* jobs,
                              int njobs, unsigned int* counter, const TilePlan& proto,
                              cudaStream_t st, const TilePlan* walk) {
    auto go = [&](auto kern) -> int {
        const size_t smem = proto.sm.total;
        if (set_dyn_smem((const void*)kern, smem) != cudaSuccess)
            return 3;
        int dev = 0, sms = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        const int grid = njobs < sms ? njobs : sms;  // persistent: one CTA per SM
        TilePlan wp{};
        if (walk) wp = *walk;  // a single table's plan with its walk request
        kern<<<grid, kNT, smem, st>>>(descs, tps, jobs, njobs, counter, wp);
        return cudaPeekAtLastError() == cudaSuccess ? 0 : 3;  // (the caller reports it)
    };
    if (proto.halo) {  // budget shards: communication warp, no split tails, no walk
        if (!proto.comm || proto.split || (walk && walk->walk)) return 3;
        return proto.stream ? go(fill_tiles_batch<RPW, true, false, true, false, true>)
                            : go(fill_tiles_batch<RPW, true, false, false, false, true>);
    }
    // the walk variant only for a single table with a walk request (no code
    // for it in the batch kernels)
    // (split tails only for a single table run as jobs, never for batches)
    const bool split = walk && proto.comm && proto.split;
    if (proto.j1 != INT32_MAX) return 3;  // mixed widths: single tables (fill_tiles_jobs1)
    if (walk && walk->walk) {
        if (proto.stream)
            return proto.comm ? go(fill_tiles_batch<RPW, true, false, true, true, false>)
                              : go(fill_tiles_batch<RPW, false, false, true, true, false>);
        if (split) return go(fill_tiles_batch<RPW, true, true, false, true, false>);
        return proto.comm ? go(fill_tiles_batch<RPW, true, false, false, true, false>)
                          : go(fill_tiles_batch<RPW, false, false, false, true, false>);
    }
    // (a single long table: the budget-shard instantiation, whose halo code
    // is inert here -- its register allocation spills 8 bytes where the
    // plain one spills 88)
    if (proto.stream)
        return proto.comm ? go(fill_tiles_batch<RPW, true, false, true, false, true>)
                          : go(fill_tiles_batch<RPW, false, false, true, false, false>);
    if (split) return go(fill_tiles_batch<RPW, true, true, false, false, false>);
    return proto.comm ? go(fill_tiles_batch<RPW, true, false, false, false, false>)
                      : go(fill_tiles_batch<RPW, false, false, false, false, false>);
}

}  // namespace

namespace {
template <int RPW>
int launch_jobs1_r(const InstDesc& d, const TilePlan& tp, unsigned int* counter, cudaStream_t st) {
    auto go = [&](auto kern) -> int {
        const size_t smem = tp.sm.total;
        if (set_dyn_smem((const void*)kern, smem) != cudaSuccess) return 3;
        int dev = 0, sms = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        const int grid = tp.T < sms ? tp.T : sms;  // persistent: one CTA per SM
        kern<<<grid, kNT, smem, st>>>(d, tp, counter);
        return cudaPeekAtLastError() == cudaSuccess ? 0 : 3;
    };
    if (tp.halo) return 3;
    if (RPW == 1 && tp.j1 != INT32_MAX) {  // mixed widths: staged programs, communication warp
        if (tp.stream || tp.split || !tp.comm) return 3;
        return tp.walk ? go(fill_tiles_jobs1<1, true, false, false, true, true>)
                       : go(fill_tiles_jobs1<1, true, false, false, false, true>);
    }
    if (tp.stream)
        return tp.comm ? (tp.walk ? go(fill_tiles_jobs1<RPW, true, false, true, true, false>)
                                  : go(fill_tiles_jobs1<RPW, true, false, true, false, false>))
                       : (tp.walk ? go(fill_tiles_jobs1<RPW, false, false, true, true, false>)
                                  : go(fill_tiles_jobs1<RPW, false, false, true, false, false>));
    if (tp.comm && tp.split)
        return tp.walk ? go(fill_tiles_jobs1<RPW, true, true, false, true, false>)
                       : go(fill_tiles_jobs1<RPW, true, true, false, false, false>);
    if (tp.comm)
        return tp.walk ? go(fill_tiles_jobs1<RPW, true, false, false, true, false>)
                       : go(fill_tiles_jobs1<RPW, true, false, false, false, false>);
    return tp.walk ? go(fill_tiles_jobs1<RPW, false, false, false, true, false>)
                   : go(fill_tiles_jobs1<RPW, false, false, false, false, false>);
}
}  // namespace

int launch_fill_tiles_jobs1(const InstDesc& d, const TilePlan& tp, unsigned int* counter, void* stream) {
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (tp.rpw == 1) return launch_jobs1_r<1>(d, tp, counter, st);
    if (tp.rpw == 2) return launch_jobs1_r<2>(d, tp, counter, st);
    return 3;
}

int launch_fill_tiles(const InstDesc& d, const TilePlan& tp, int width, void* stream) {
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (width != 32) return 3;  // 32-bit costs
    if (tp.rpw == 1) return launch_fill_tiles_r<1>(d, tp, st);
    if (tp.rpw == 2) return launch_fill_tiles_r<2>(d, tp, st);
    return 3;
}

TileSmem tile_batch_smem(const TilePlan& proto) { return tile_smem(proto); }

int launch_fill_tiles_batch(const InstDesc* descs, const TilePlan* tps, const int2* jobs,
                            int njobs, unsigned int* counter, const TilePlan& proto, void* stream,
                            const TilePlan* walk) {
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (njobs <= 0) return 0;
    if (proto.rpw == 1)
        return launch_fill_tiles_batch_r<1>(descs, tps, jobs, njobs, counter, proto, st, walk);
    if (proto.rpw == 2)
        return launch_fill_tiles_batch_r<2>(descs, tps, jobs, njobs, counter, proto, st, walk);
    return 3;
}

}  // namespace rkr
