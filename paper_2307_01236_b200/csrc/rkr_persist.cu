// rkr_persist.cu -- K1p: the whole table fill as ONE persistent, dataflow-
// scheduled launch (sm_100a), plus the per-table cell-program precompute.
//
// Work item = one row segment of one cell: (s, t = s + k, budget tile j of
// TM slots).  Items are dequeued from a global counter in the order of the
// host-built plan (PersistPlan: key lambda*j + k, then s).  An item of
// diagonal k may start once diagonal k-1 is complete on tiles [j - dj, j]
// (dj = halo tiles of the largest budget shift); by induction that covers
// every row the cell reads (chain_dp.hpp:148, :166-167 read only smaller
// spans at m' <= m).  Completion is published per (k, j) with a release
// fence + atomic add and observed with relaxed polls + one acquire fence --
// no grid barrier, no per-diagonal launch, no deadlock (items wait only on
// items dequeued earlier).
//
// Cell programs.  Everything about cell (s, t) that does not depend on the
// table -- the option thresholds of chain_dp.hpp:141-147, the row addresses
// of every cut, the option-0 sweep prefix sums (:162) and the `break` gate
// (:164) as a prefix maximum -- is computed once per table by prep_programs
// and copied into shared memory by each item before it waits.
//
// Two phases per item.  Only the options (row (s+1, t)), cut c = s+1 (right
// operand (s+1, t)) and cut c = t (left operand (s, t-1)) read diagonal k-1.
// The item first waits for diagonal k-2 and runs the other cuts ("bulk":
// each lane counts the cuts its slot admits by binary search on the
// monotone gate, then loads them in batches of U iterations so 2*U*R loads
// are in flight), then waits for k-1 and runs the short "tail": options
// through L1 (ld.ca; the acquire fence invalidated L1) and the two remaining
// cuts, merged with a lexicographic (value, code) minimum.  Completion is
// published with a release reduction (red.release.gpu).
// Tie-break: options in menu order, then cuts ascending -- the reference's
// first minimum (chain_dp.hpp:139-174).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <utility>
#include <vector>

#include "rkr_internal.h"

namespace rkr {

namespace {

template <typename V>
struct CostP;
template <>
struct CostP<uint32_t> {
    static constexpr uint32_t inf = kInf32;
    static constexpr bool checked = false;
};
template <>
struct CostP<int64_t> {
    static constexpr int64_t inf = kInf64;
    static constexpr bool checked = true;
};

__device__ __forceinline__ int32_t clampm(int64_t x, int32_t M) {
    return x < -1 ? -1 : (x > (int64_t)M + 1 ? M + 1 : (int32_t)x);
}

__device__ __forceinline__ int ld_relaxed(const int* p) {
    int v;
    asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void fence_acq_rel() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }

__device__ __forceinline__ void red_release_add(int* p, int v) {
    asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ int ld_relaxed_sys(const int* p) {
    int v;
    asm volatile("ld.relaxed.sys.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void fence_acq_rel_sys() {
    asm volatile("fence.acq_rel.sys;" ::: "memory");
}

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

template <typename V>
struct Programs {
    longlong2* ptr;   // per cut entry: {&L(s, c-1)[0], &R(c, t)[-act_u[c]]}
    V* sweep;         // per cut entry: sum_{j=s}^{c-1} time_fwd0[j]
    int32_t* gate;    // per cut entry: prefix-max gate, clamped to [-1, M+1]
    int32_t* thr;     // per (row, option): validity threshold, clamped
    int32_t* pc;      // per saved option: pack shift clamped to pad
    V* otot;          // per saved option: time_fwd + time_bwd
    int64_t nq;
    int32_t ocap;     // thr row stride
    int32_t tiles;    // 1: ptr holds K1t programs (int4 {off_l, off_r, sweep, gate}; width 32)
};


// ---------------------------------------------------------------------------
// prep_programs: one warp per cell (s, t); the option-0 sweep (:162) and the
// `break` gate (:164) are prefix sum / prefix max over the cuts, done 32 cuts
// at a time with warp shuffles.
// ---------------------------------------------------------------------------
template <typename V>
__device__ __forceinline__ void prep_body(const Geometry& g, const DevMenu& dm, const V* opt,
                                          const Programs<V>& pr, int64_t bx, int64_t nbx) {
    const int ocap = pr.ocap;
    const int L = g.L, M = g.M;
    const int lane = threadIdx.x & 31;
    const int64_t warps = nbx * (blockDim.x >> 5);
    for (int64_t rid = bx * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); rid < g.rows;
         rid += warps) {
        int lo = 0, hi = L - 1;  // rid -> (k, s): rows are diagonal-major
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (diag_off(L, mid) <= rid)
                lo = mid;
            else
                hi = mid - 1;
        }
        const int k = lo;
        const int s = (int)(rid - diag_off(L, k));
        const int t = s + k;
        const bool seeded = t < L - 1;                              // chain_dp.hpp:126
        const int64_t seed = seeded ? 2 * dm.act_u[t + 1] : 0;      // chain_dp.hpp:127
        const int o0 = dm.blk_off[s], nopt = dm.blk_off[s + 1] - o0;
        for (int i = nopt + lane; i < ocap; i += 32) pr.thr[rid * ocap + i] = M + 1;  // padding: never valid
        for (int i = lane; i < nopt; i += 32) {
            const int q = o0 + i;
            const int64_t need = (k == 0 && seeded) ? dm.fwd_req_pre[q] + dm.act_u[t + 1]
                                                    : dm.fwd_req[q] + seed;  // :141-143
            int64_t th = need > dm.bwd_req[q] ? need : dm.bwd_req[q];         // :144
            if (k > 0 && dm.pack_chg[q] > th) th = dm.pack_chg[q];            // :147
            pr.thr[rid * ocap + i] = clampm(th - g.m_base, M);  // local slots
        }
        if (k == 0) continue;
        const int64_t base = diag_cut_off(L, k) + (int64_t)s * k;
        V carry_sum = 0;
        long long carry_max = dm.fwd0_own[s] + seed;                          // :159
        for (int i0 = 0; i0 < k; i0 += 32) {
            const int i = i0 + lane;
            const int c = s + 1 + i;
            V inc = 0;
            long long gv = LLONG_MIN;
            if (i < k) {
                inc = (V)dm.tf0[c - 1];
                if (c - 1 > s) gv = dm.fwd0_full[c - 1] + seed;
            }
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {  // inclusive scans
                const V y = __shfl_up_sync(0xffffffffu, inc, off);
                const long long ym = __shfl_up_sync(0xffffffffu, gv, off);
                if (lane >= off) {
                    inc += y;
                    gv = ym > gv ? ym : gv;
                }
            }
            const V sweep = carry_sum + inc;
            const long long gmax = gv > carry_max ? gv : carry_max;
            if (i < k) {
                const int64_t a = dm.act_u[c];
                const int sh = a > g.pad ? g.pad : (int)a;
                if (pr.tiles) {
                    // K1t: element offsets of slot 0 (32-bit, tile_plan checks
                    // rows * sr < 2^31) and the sweep and gate in one entry
                    int4 q;
                    q.x = (int)(row_id(L, s, c - 1) * g.sr + g.pad);
                    q.y = (int)(row_id(L, c, t) * g.sr + g.pad - sh);
                    q.z = (int)sweep;
                    q.w = clampm(gmax - g.m_base, M);
                    reinterpret_cast<int4*>(pr.ptr)[base + i] = q;
                } else {
                    longlong2 p;
                    p.x = (long long)(opt + row_id(L, s, c - 1) * g.sr + g.pad);
                    p.y = (long long)(opt + row_id(L, c, t) * g.sr + g.pad - sh);
                    pr.ptr[base + i] = p;
                    pr.sweep[base + i] = sweep;
                    pr.gate[base + i] = clampm(gmax - g.m_base, M);
                }
            }
            carry_sum = __shfl_sync(0xffffffffu, sweep, 31);
            carry_max = __shfl_sync(0xffffffffu, gmax, 31);
        }
    }
    // the infinity pads of every opt row (init_pads, folded into this launch)
    {
        V* o = const_cast<V*>(opt);
        const int64_t n = g.rows * (int64_t)g.pad;
        for (int64_t i = bx * (int64_t)blockDim.x + threadIdx.x; i < n;
             i += nbx * blockDim.x) {
            const int64_t r = i / g.pad, p = i - r * g.pad;
            o[r * g.sr + p] = CostP<V>::inf;
        }
    }
    // per saved option: clamped pack shift and pass time
    for (int64_t q = bx * (int64_t)blockDim.x + threadIdx.x; q < pr.nq;
         q += nbx * blockDim.x) {
        const int64_t p = dm.pack_chg[q];
        pr.pc[q] = p > g.pad ? g.pad : (int)p;
        pr.otot[q] = (V)dm.tftb[q];
    }
}

template <typename V>
__global__ void prep_programs(Geometry g, DevMenu dm, const V* opt, Programs<V> pr,
                              uint32_t* __restrict__ zero, int64_t nzero) {
    prep_body<V>(g, dm, opt, pr, blockIdx.x, gridDim.x);
    // the fill state (item counter + done flags) of the first fill, so that
    // launch needs no memset of its own
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nzero;
         i += (int64_t)gridDim.x * blockDim.x)
        zero[i] = 0;
}

template <typename V>
__device__ inline Programs<V> programs_of(const ProgDev& q);

// Every table of a batch in one launch: blockIdx.y = table.
template <typename V>
__global__ void prep_programs_batch(const InstDesc* __restrict__ d) {
    const InstDesc& D = d[blockIdx.y];
    prep_body<V>(D.g, D.dm, static_cast<const V*>(D.opt), programs_of<V>(D.prog), blockIdx.x,
                 gridDim.x);
}

// ---------------------------------------------------------------------------
// fill_persistent
// ---------------------------------------------------------------------------
template <typename V>
struct PSmem {
    longlong2* ptr;   // [kcap]
    V* sweep;         // [kcap]
    int32_t* gate;    // [kcap]
    V* otot;          // [ocap]
    int32_t* thr;     // [ocap]
    int32_t* pc;      // [ocap]
    long long* item;  // [1]
};

struct Caps {
    int32_t kcap, ocap, TM;
};

template <typename V>
__host__ __device__ inline size_t psmem_bytes(const Caps& c) {
    size_t b = (size_t)c.kcap * 16;
    b += (size_t)c.kcap * sizeof(V);
    b = (b + 15) & ~size_t(15);
    b += (size_t)c.kcap * 4;
    b = (b + 15) & ~size_t(15);
    b += (size_t)c.ocap * sizeof(V);
    b = (b + 15) & ~size_t(15);
    b += (size_t)c.ocap * 8;
    b = (b + 15) & ~size_t(15);
    return b + 16;
}

template <typename V>
__device__ inline PSmem<V> pcarve(unsigned char* p, const Caps& c) {
    PSmem<V> s;
    size_t b = 0;
    s.ptr = reinterpret_cast<longlong2*>(p);
    b += (size_t)c.kcap * 16;
    s.sweep = reinterpret_cast<V*>(p + b);
    b += (size_t)c.kcap * sizeof(V);
    b = (b + 15) & ~size_t(15);
    s.gate = reinterpret_cast<int32_t*>(p + b);
    b += (size_t)c.kcap * 4;
    b = (b + 15) & ~size_t(15);
    s.otot = reinterpret_cast<V*>(p + b);
    b += (size_t)c.ocap * sizeof(V);
    b = (b + 15) & ~size_t(15);
    s.thr = reinterpret_cast<int32_t*>(p + b);
    s.pc = s.thr + c.ocap;
    b += (size_t)c.ocap * 8;
    b = (b + 15) & ~size_t(15);
    s.item = reinterpret_cast<long long*>(p + b);
    return s;
}

template <typename V>
__device__ inline Programs<V> programs_of(const ProgDev& q) {
    Programs<V> p;
    p.ptr = static_cast<longlong2*>(q.ptr);
    p.sweep = static_cast<V*>(q.sweep);
    p.gate = q.gate;
    p.thr = q.thr;
    p.pc = q.pc;
    p.otot = static_cast<V*>(q.otot);
    p.nq = q.nq;
    p.ocap = q.ocap;
    p.tiles = q.tiles;
    return p;
}

// SINGLE: one table whose descriptor travels as a kernel parameter (constant
// bank); batches read their descriptors from global memory (measured 22%
// slower per item on config 3, so the single-table path keeps the param).
constexpr int pl_sleep_ns = 32;  // poll back-off (ns; measured, profiles/r01_persist)

template <typename V, int NT, int R, int U, bool SINGLE, int MINB>
__global__ void __launch_bounds__(NT, MINB) fill_persistent(const InstDesc* __restrict__ inst,
                                                      const __grid_constant__ InstDesc d0,
                                                      LaunchPlan lp,
                                                      unsigned long long* __restrict__ counter,
                                                      Caps c) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    constexpr V INF = CostP<V>::inf;
    PSmem<V> sm = pcarve<V>(smem_raw, c);
    const int tid = threadIdx.x;
    long long next = 0;
    if (tid == 0) next = (long long)atomicAdd(counter, 1ull);

    for (;;) {
        if (tid == 0) sm.item[0] = next;
        __syncthreads();
        const int64_t gidx = sm.item[0];
        if (gidx >= lp.total) break;
        // prefetch the next item while this one runs (the earliest unfinished
        // item is always one being processed, so this cannot deadlock)
        if (tid == 0) next = (long long)atomicAdd(counter, 1ull);
        unsigned long long t0 = 0;
        // item -> (instance, diagonal, tile, s) through the launch plan
        int ea = 0, eb = lp.n - 1;
        while (ea < eb) {
            const int mid = (ea + eb + 1) >> 1;
            if (__ldg(lp.start + mid) <= gidx)
                ea = mid;
            else
                eb = mid - 1;
        }
        const int k = __ldg(lp.k + ea);
        const int j = __ldg(lp.j + ea);
        const int s = (int)(gidx - __ldg(lp.start + ea));
        const InstDesc& D = SINGLE ? d0 : inst[__ldg(lp.inst + ea)];
        // references, not copies: fields are re-read from the parameter bank
        // (single table) or L1 (batch) where used, instead of pinning ~40
        // registers for the whole item
        const Geometry& g = D.g;
        const DevMenu& dm = D.dm;
        const PlanDev& pl = D.plan;
        const ProgDev& pq = D.prog;
        V* __restrict__ opt = static_cast<V*>(D.opt);
        uint16_t* __restrict__ arg = D.arg;
        int* __restrict__ done = pl.done;
        const int64_t idx = gidx;  // trace slot (traced fills are single-table)
        const int L = g.L, M = g.M;
        if (pl.trace && tid == 0) t0 = gtimer();
        const int t = s + k;
        const int m0 = j * pl.TM;
        const int64_t rid = row_id(L, s, t);

        // ---- cell program -> smem (independent of the table: overlaps the wait)
        const int o0 = __ldg(dm.blk_off + s);
        const int nopt = __ldg(dm.blk_off + s + 1) - o0;
        for (int i = tid; i < nopt; i += NT) {
            sm.thr[i] = pq.thr[rid * pq.ocap + i];
            sm.pc[i] = pq.pc[o0 + i];
            sm.otot[i] = static_cast<const V*>(pq.otot)[o0 + i];
        }
        if (k > 0) {
            const int64_t base = diag_cut_off(L, k) + (int64_t)s * k;
            for (int i = tid; i < k; i += NT) {
                sm.ptr[i] = static_cast<const longlong2*>(pq.ptr)[base + i];
                sm.sweep[i] = static_cast<const V*>(pq.sweep)[base + i];
                sm.gate[i] = pq.gate[base + i];
            }
        }

        // Only three candidate groups of cell (s, t) read diagonal k-1: the
        // options (row (s+1, t)), cut c = s+1 (right operand (s+1, t)) and
        // cut c = t (left operand (s, t-1)).  Cuts c in [s+2, t-1] read
        // diagonals <= k-2, so they run first ("bulk", overlapping diagonal
        // k-1) and only the short "tail" sits on the critical path.
        // Thread 0 polls (relaxed) and fences once; the CTA barrier after it
        // orders every thread's table reads after the acquire.  (Per-warp
        // polling/publishing was measured 7x slower: 8x the pollers and
        // atomics on the same flag lines, profiles/r01_persist.)
        const bool need_halo = D.halo_need > 0 && j - pl.dj < 0;
        auto wait_diag = [&](int kk) {
            if (tid == 0) {
                const int need = L - kk;
                const int* row = done + (int64_t)kk * pl.J;
                for (int jj = (j - pl.dj > 0 ? j - pl.dj : 0); jj <= j; ++jj)
                    while (ld_relaxed(row + jj) < need) {
                        if (pl_sleep_ns) __nanosleep(pl_sleep_ns);
                    }
                if (need_halo) {  // slots below 0 come from the previous shard
                    const int* h = D.halo + kk;
                    while (ld_relaxed_sys(h) < need * D.halo_need) __nanosleep(64);
                    fence_acq_rel_sys();
                } else {
                    fence_acq_rel();
                }
            }
            __syncthreads();
        };
        if (k >= 3)
            wait_diag(k - 2);  // (its barrier also publishes the program in smem)
        else
            __syncthreads();
        unsigned long long ta = 0;
        if (pl.trace && tid == 0) ta = gtimer();

        const int mb = m0 + tid;
        V best[R];
        uint16_t code[R];
        int nlive[R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
            best[r] = INF;
            code[r] = 0;
            nlive[r] = 0;
        }
        const uint16_t cb = (uint16_t)(kCutBit | (s + 1));
        // ---- Case 2 bulk: cuts i in [1, k-2] ascending, strict '<' ------------
        if (k > 0) {
            int nmax = 0;
#pragma unroll
            for (int r = 0; r < R; ++r) {  // cuts admitted by the sweep gate and the `break`
                const int m = mb + NT * r;
                int lo = 0, hi = k;        // first i with gate[i] > m
                while (lo < hi) {
                    const int mid = (lo + hi) >> 1;
                    if (sm.gate[mid] <= m)
                        lo = mid + 1;
                    else
                        hi = mid;
                }
                nlive[r] = lo;
                nmax = lo > nmax ? lo : nmax;
            }
            const int iend = nmax < k - 1 ? nmax : k - 1;  // exclusive; i = k-1 is tail
            for (int i0 = 1; i0 < iend; i0 += U) {
                V lv[U][R], rv[U][R];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int i = i0 + u;
                    const longlong2 p = sm.ptr[i < iend ? i : 0];
                    const V* lp = reinterpret_cast<const V*>(p.x) + mb;
                    const V* rp = reinterpret_cast<const V*>(p.y) + mb;
#pragma unroll
                    for (int r = 0; r < R; ++r) {
                        if (i < iend && i < nlive[r]) {
                            lv[u][r] = __ldcg(lp + NT * r);
                            rv[u][r] = __ldcg(rp + NT * r);
                        } else {
                            lv[u][r] = INF;
                            rv[u][r] = INF;
                        }
                    }
                }
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int i = i0 + u;
                    const V sw = sm.sweep[i < iend ? i : 0];
#pragma unroll
                    for (int r = 0; r < R; ++r) {
                        const V tot = sw + lv[u][r] + rv[u][r];
                        bool ok = tot < best[r];
                        if constexpr (CostP<V>::checked) ok = ok && lv[u][r] < INF && rv[u][r] < INF;
                        if (ok) {
                            best[r] = tot;
                            code[r] = (uint16_t)(cb + i);
                        }
                    }
                }
            }
        }

        // ---- tail: wait for diagonal k-1 on tiles [j - dj, j] ------------------
        unsigned long long tb = 0;
        if (pl.trace && tid == 0) tb = gtimer();
        if (k >= 1) wait_diag(k - 1);
        unsigned long long t1 = 0;
        if (pl.trace && tid == 0) t1 = gtimer();
        const V* nxt = k > 0 ? opt + row_id(L, s + 1, t) * g.sr + g.pad : nullptr;
        // tail cut operands: i = 0 (c = s+1) and i = k-1 (c = t); issue the
        // loads together with the option-window staging
        V tl[2][R], tr[2][R];
        if (k > 0) {
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int i = e == 0 ? 0 : k - 1;
                const longlong2 p = sm.ptr[i];
                const V* lp = reinterpret_cast<const V*>(p.x) + mb;
                const V* rp = reinterpret_cast<const V*>(p.y) + mb;
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    if (i < nlive[r] && (e == 0 || k > 1)) {
                        tl[e][r] = __ldcg(lp + NT * r);
                        tr[e][r] = __ldcg(rp + NT * r);
                    } else {
                        tl[e][r] = INF;
                        tr[e][r] = INF;
                    }
                }
            }
        }
        // lexicographic (value, code) update: the reference's first minimum
        // in candidate order (options by menu position, then cuts ascending)
        auto offer = [&](int r, V tot, uint16_t cd, bool ok) {
            ok = ok && (tot < best[r] || (tot == best[r] && cd < code[r]));
            if (ok) {
                best[r] = tot;
                code[r] = cd;
            }
        };
        // Case 1 (chain_dp.hpp:139-156).  The option windows of row (s+1, t)
        // are loaded OB options at a time (OB*R loads in flight) before any
        // is consumed: this loop is on the diagonal's critical path, and a
        // load-use per option would serialise nopt L2 round trips.
        constexpr int OB = 8;
        for (int i0 = 0; i0 < nopt; i0 += OB) {
            V sub[OB][R];
            if (k > 0) {
#pragma unroll
                for (int u = 0; u < OB; ++u) {
                    const int i = i0 + u < nopt ? i0 + u : i0;
                    const int p = sm.pc[i];
#pragma unroll
                    for (int r = 0; r < R; ++r)
                        // L1-cached: the acquire fence above invalidated L1,
                        // so every line is fetched after the publish
                        sub[u][r] = __ldca(nxt + (mb + NT * r - p));
                }
            }
#pragma unroll
            for (int u = 0; u < OB; ++u) {
                const int i = i0 + u;
                if (i < nopt) {
                    const V tt = sm.otot[i];
                    const int th = sm.thr[i];
#pragma unroll
                    for (int r = 0; r < R; ++r) {
                        const int m = mb + NT * r;
                        V tot = tt;
                        bool ok = m >= th;
                        if (k > 0) {
                            if constexpr (CostP<V>::checked) ok = ok && sub[u][r] < INF;
                            tot = tt + sub[u][r];
                        }
                        if constexpr (!CostP<V>::checked) ok = ok && tot < INF;
                        offer(r, tot, (uint16_t)(i + 1), ok);
                    }
                }
            }
        }
        // Case 2 tail cuts (chain_dp.hpp:158-174)
        if (k > 0) {
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int i = e == 0 ? 0 : k - 1;
                const V sw = sm.sweep[i];
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    const V tot = sw + tl[e][r] + tr[e][r];
                    bool ok = tot < INF;
                    if constexpr (CostP<V>::checked) ok = tl[e][r] < INF && tr[e][r] < INF;
                    offer(r, tot, (uint16_t)(cb + i), ok && (e == 0 || k > 1));
                }
            }
        }
        unsigned long long t2 = 0;
        if (pl.trace && tid == 0) t2 = gtimer();
        // ---- store (chain_dp.hpp:176-177) and publish ---------------------------
        V* orow = opt + rid * g.sr + g.pad;
        uint16_t* arow = arg + rid * g.sa;
        // this tile's slots that are the next shard's halo: [W - pad, W)
        const int W = M + 1;
        const bool feeds_next = D.next_opt != nullptr && m0 + pl.TM > W - g.pad && m0 < W;
        V* nrow = feeds_next ? static_cast<V*>(D.next_opt) + rid * D.next_sr + g.pad - W : nullptr;
        // shard 0's walk mirror (process shards; peer memory)
        uint16_t* mrow = D.arg_mirror ? D.arg_mirror + rid * D.mirror_sa + D.mirror_base : nullptr;
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const int m = mb + NT * r;
            if (m <= M) {
                orow[m] = best[r];
                arow[m] = code[r];
                if (feeds_next && m >= W - g.pad) nrow[m] = best[r];
                if (mrow) mrow[m] = code[r];
            }
        }
        __syncthreads();
        if (tid == 0) {
            if (feeds_next) {
                if (D.next_peer)
                    __threadfence_system();
                else
                    __threadfence();
                atomicAdd(D.next_halo + k, 1);
            }
            // release-add: orders this CTA's stores (made visible to thread 0
            // by the barrier) before the count, without a separate fence
            red_release_add(done + (int64_t)k * pl.J + j, 1);
        }
        if (pl.trace && tid == 0) {
            unsigned long long* tr = pl.trace + 6 * idx;  // per-table item index
            tr[0] = t0;
            tr[1] = ta;
            tr[2] = tb;
            tr[3] = t1;
            tr[4] = t2;
            tr[5] = gtimer();
        }
    }
}

// Occupancy floor per R (registers: R=1 -> <=40, R=2 -> <=64, no spills);
// measured on config 3 (profiles/r01_persist/variants.txt).
template <int R>
constexpr int kMinBlocks = R == 1 ? 6 : 4;

template <typename V, int R, bool SINGLE, int U = 4, int MINB = kMinBlocks<R>>
int launch_t(const InstDesc* dev_desc, const InstDesc& d0, const LaunchPlan& lp, int kcap, int ocap,
             unsigned long long* counter, cudaStream_t st) {
    constexpr int NT = 256;
    Caps c;
    c.TM = NT * R;
    c.kcap = kcap > 0 ? kcap : 1;
    c.ocap = ocap > 0 ? ocap : 1;
    const size_t smem = psmem_bytes<V>(c);
    auto kern = fill_persistent<V, NT, R, U, SINGLE, MINB>;
    if (set_dyn_smem((const void*)kern, smem) != cudaSuccess)
        return 3;
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, NT, smem) != cudaSuccess ||
        per_sm < 1)
        return 3;
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    int64_t grid = (int64_t)per_sm * sms;
    if (grid > lp.total) grid = lp.total;
    if (grid < 1) return 0;
    kern<<<(unsigned)grid, NT, smem, st>>>(dev_desc, d0, lp, counter, c);
    return cudaPeekAtLastError() == cudaSuccess ? 0 : 3;  // (the caller reports it)
}

template <typename V>
Programs<V> host_programs_of(const LaunchCtx& cx) {
    Programs<V> p;
    p.ptr = static_cast<longlong2*>(cx.prog.ptr);
    p.sweep = static_cast<V*>(cx.prog.sweep);
    p.gate = cx.prog.gate;
    p.thr = cx.prog.thr;
    p.pc = cx.prog.pc;
    p.otot = static_cast<V*>(cx.prog.otot);
    p.nq = cx.prog.nq;
    p.ocap = cx.prog.ocap;
    p.tiles = cx.prog.tiles;
    return p;
}

template <typename V>
int prep_t(const LaunchCtx& cx) {
    cudaStream_t st = static_cast<cudaStream_t>(cx.stream);
    // one warp per cell; the option pass strides over threads
    const int64_t n = cx.g.rows * 32 > cx.prog.nq ? cx.g.rows * 32 : cx.prog.nq;
    int blocks = (int)((n + 127) / 128);
    if (blocks > 148 * 16) blocks = 148 * 16;
    if (blocks < 1) blocks = 1;
    prep_programs<V><<<blocks, 128, 0, st>>>(
        cx.g, cx.dm, static_cast<const V*>(cx.opt), host_programs_of<V>(cx),
        reinterpret_cast<uint32_t*>(cx.plan.counter),
        cx.prep_zero ? (int64_t)(cx.state_bytes / 4) : 0);
    return cudaPeekAtLastError() == cudaSuccess ? 0 : 3;  // (the caller reports it)
}

}  // namespace

int persistent_choose_r(int32_t M) {
    return (M + 1 >= 8192) ? 2 : 1;
}

void persistent_plan(const Geometry& g, int width, int R, PersistPlan& p) {
    const int L = g.L;
    const size_t vb = width == 32 ? 4 : 8;
    p.R = R;
    p.TM = 256 * p.R;
    p.J = (g.M + 1 + p.TM - 1) / p.TM;
    p.dj = (g.pad + p.TM - 1) / p.TM;
    // Order key lambda*j + k.  lambda = 1 is the 2D (tile, diagonal)
    // wavefront: critical path L + J - 1 item steps, every tile in flight.
    // lambda = 0 is diagonal-major (critical path L steps) and wins when the
    // whole table fits in L2.  Larger lambda trades parallelism for L2
    // locality (profiles/r01_persist: never paid off at this item latency).
    const double table_bytes = (double)g.rows * g.sr * vb;
    p.lambda = table_bytes <= 48.0 * (1 << 20) ? 0 : 1;
    std::vector<std::pair<int64_t, int64_t>> order;  // (key, j * L + k)
    order.reserve((size_t)p.J * L);
    for (int64_t jj = 0; jj < p.J; ++jj)
        for (int64_t k = 0; k < L; ++k) order.push_back({(int64_t)p.lambda * jj + k, jj * L + k});
    std::sort(order.begin(), order.end());
    p.start.clear();
    p.g.clear();
    p.k.clear();
    int64_t cur = 0;
    for (const auto& e : order) {
        const int64_t jj = e.second / L, k = e.second % L;
        p.start.push_back(cur);
        p.g.push_back((int32_t)jj);
        p.k.push_back((int32_t)k);
        cur += L - k;
    }
    p.total = cur;
}

size_t persistent_state_bytes(const Geometry& g, const PersistPlan& p) {
    // counter | done flags [L x J] | halo counters [L] (budget shards)
    return 8 + (size_t)g.L * p.J * sizeof(int) + (size_t)g.L * sizeof(int);
}

int64_t program_cut_entries(const Geometry& g) { return diag_cut_off(g.L, g.L); }

int launch_prep_programs(const LaunchCtx& c) {
    return c.width == 32 ? prep_t<uint32_t>(c) : prep_t<int64_t>(c);
}

int launch_prep_programs_batch(const InstDesc* d, int n, int64_t max_rows, int width, void* stream) {
    if (n <= 0) return 0;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    int bx = (int)((max_rows * 32 + 127) / 128);  // one warp per row of the largest table
    if (bx > 64) bx = 64;
    if (bx < 1) bx = 1;
    const dim3 grid(bx, n);
    if (width == 32)
        prep_programs_batch<uint32_t><<<grid, 128, 0, st>>>(d);
    else
        prep_programs_batch<int64_t><<<grid, 128, 0, st>>>(d);
    return cudaPeekAtLastError() == cudaSuccess ? 0 : 3;  // (the caller reports it)
}

int launch_fill_batch(const InstDesc* dev_desc, const InstDesc* single, const LaunchPlan& lp,
                      int width, int R, int kcap, int ocap, unsigned long long* counter,
                      void* stream) {
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    InstDesc d0{};
    if (single) d0 = *single;
    if (single) {
        if (width == 32)
            return R == 2 ? launch_t<uint32_t, 2, true>(dev_desc, d0, lp, kcap, ocap, counter, st)
                          : launch_t<uint32_t, 1, true>(dev_desc, d0, lp, kcap, ocap, counter, st);
        return R == 2 ? launch_t<int64_t, 2, true>(dev_desc, d0, lp, kcap, ocap, counter, st)
                      : launch_t<int64_t, 1, true>(dev_desc, d0, lp, kcap, ocap, counter, st);
    }
    if (width == 32)
        return R == 2 ? launch_t<uint32_t, 2, false>(dev_desc, d0, lp, kcap, ocap, counter, st)
                      : launch_t<uint32_t, 1, false>(dev_desc, d0, lp, kcap, ocap, counter, st);
    return R == 2 ? launch_t<int64_t, 2, false>(dev_desc, d0, lp, kcap, ocap, counter, st)
                  : launch_t<int64_t, 1, false>(dev_desc, d0, lp, kcap, ocap, counter, st);
}

void merge_plans(const std::vector<const PersistPlan*>& plans, const std::vector<int32_t>& L,
                 HostLaunchPlan& out) {
    struct E {
        int64_t key;
        int32_t inst, j, k;
    };
    std::vector<E> es;
    size_t n = 0;
    for (const PersistPlan* p : plans) n += p->start.size();
    es.reserve(n);
    for (size_t i = 0; i < plans.size(); ++i) {
        const PersistPlan& p = *plans[i];
        for (size_t e = 0; e < p.start.size(); ++e)
            es.push_back({(int64_t)p.lambda * (p.g[e] + p.j_offset) + p.k[e], (int32_t)i, p.g[e],
                          p.k[e]});
    }
    std::stable_sort(es.begin(), es.end(), [](const E& a, const E& b) {
        if (a.key != b.key) return a.key < b.key;
        if (a.inst != b.inst) return a.inst < b.inst;
        return a.j < b.j;
    });
    out.start.clear();
    out.inst.clear();
    out.k.clear();
    out.j.clear();
    int64_t cur = 0;
    for (const E& e : es) {
        out.start.push_back(cur);
        out.inst.push_back(e.inst);
        out.k.push_back(e.k);
        out.j.push_back(e.j);
        cur += L[e.inst] - e.k;
    }
    out.total = cur;
}

}  // namespace rkr
