// rkr_persist.cu -- K1p: the whole table fill as ONE persistent, dataflow-
// scheduled launch (sm_100a).
//
// Work item = one cell row segment (s, t = s + k, budget tile j of TM slots).
// Items are dequeued from a global counter in (column group, diagonal k,
// tile j, s) order.  An item of diagonal k may start once diagonal k-1 is
// complete on tiles [j - dj, j] (dj = halo tiles for the largest budget
// shift); by induction that covers every row the cell reads
// (chain_dp.hpp:148, :166-167 read only smaller spans at m' <= m).
// Completion is published per (k, j) with a release fence + atomic counter
// and observed with an acquire load -- no grid barrier, no per-diagonal launch.
//
// Column-group ordering keeps the working set of all rows restricted to a
// group of GW tiles (plus the halo) inside the 126 MB L2 while the wavefront
// sweeps all diagonals over it; the next group's early diagonals overlap
// this group's deep (low-parallelism) diagonals.
//
// Inside an item: the candidate parameters are staged in shared memory
// (sweep prefix sums and the `break` gate as a prefix maximum, computed with
// a block scan), each lane computes how many cuts its budget slot admits
// (binary search on the monotone gate), and the cut loop then runs without
// data-dependent exits so loads stay in flight.  The option window (row
// (s+1, t) at shifts m - pack_chg) is staged once in shared memory.
// Tie-break: options in menu order, then cuts ascending, strict '<' -- the
// reference's first-minimum (chain_dp.hpp:139-174).
#include <cuda_runtime.h>

#include <cstdint>

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

__device__ __forceinline__ int ld_acquire(const int* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

struct PCfg {
    int32_t TM;        // budget slots per item
    int32_t J;         // tiles per row
    int32_t GW;        // tiles per column group
    int32_t dj;        // halo tiles
    int32_t seg_cap;   // option-window slots staged in smem (0: read global)
    int32_t kcap;      // max cuts per cell staged (L - 1)
    int32_t ocap;      // max saved options per block
    int64_t total;     // items
};

template <typename V>
struct PSmem {
    long long* lptr;   // [kcap] address of L(s, c-1)[0]
    long long* rptr;   // [kcap] address of R(c, t)[-act_u[c]]
    V* sweep;          // [kcap] sum_{j=s}^{c-1} time_fwd0[j]
    int32_t* gate;     // [kcap] prefix-max gate (clamped to [-1, M+1])
    V* otot;           // [ocap]
    int32_t* thr;      // [ocap]
    int32_t* pc;       // [ocap]
    V* seg;            // [seg_cap + TM]
    V* wsum;           // [32]
    long long* wmax;   // [32]
    long long* item;   // [1]
};

template <typename V>
__host__ __device__ inline size_t psmem_bytes(int kcap, int ocap, int seg_cap, int TM) {
    size_t b = 0;
    b += (size_t)kcap * 16;
    b += (size_t)kcap * sizeof(V);
    b = (b + 7) & ~size_t(7);
    b += (size_t)kcap * 4;
    b = (b + 7) & ~size_t(7);
    b += (size_t)ocap * sizeof(V);
    b = (b + 7) & ~size_t(7);
    b += (size_t)ocap * 8;
    b = (b + 7) & ~size_t(7);
    b += (size_t)(seg_cap > 0 ? seg_cap + TM : 0) * sizeof(V);
    b = (b + 7) & ~size_t(7);
    b += 32 * sizeof(V) + 32 * 8 + 8;
    return b + 16;
}

template <typename V>
__device__ inline PSmem<V> pcarve(unsigned char* p, const PCfg& c) {
    PSmem<V> s;
    size_t b = 0;
    s.lptr = reinterpret_cast<long long*>(p);
    s.rptr = s.lptr + c.kcap;
    b += (size_t)c.kcap * 16;
    s.sweep = reinterpret_cast<V*>(p + b);
    b += (size_t)c.kcap * sizeof(V);
    b = (b + 7) & ~size_t(7);
    s.gate = reinterpret_cast<int32_t*>(p + b);
    b += (size_t)c.kcap * 4;
    b = (b + 7) & ~size_t(7);
    s.otot = reinterpret_cast<V*>(p + b);
    b += (size_t)c.ocap * sizeof(V);
    b = (b + 7) & ~size_t(7);
    s.thr = reinterpret_cast<int32_t*>(p + b);
    s.pc = s.thr + c.ocap;
    b += (size_t)c.ocap * 8;
    b = (b + 7) & ~size_t(7);
    s.seg = reinterpret_cast<V*>(p + b);
    b += (size_t)(c.seg_cap > 0 ? c.seg_cap + c.TM : 0) * sizeof(V);
    b = (b + 7) & ~size_t(7);
    s.wsum = reinterpret_cast<V*>(p + b);
    b += 32 * sizeof(V);
    s.wmax = reinterpret_cast<long long*>(p + b);
    b += 32 * 8;
    s.item = reinterpret_cast<long long*>(p + b);
    return s;
}

// item index -> (k, j, s); order: group, diagonal, tile, s.
__device__ inline void decode_item(int64_t idx, int L, int64_t rows, const PCfg& c, int& k, int& j,
                                   int& s) {
    const int64_t per_group = (int64_t)c.GW * rows;
    const int ng = (c.J + c.GW - 1) / c.GW;
    int g = (int)(idx / per_group);
    if (g > ng - 1) g = ng - 1;
    const int64_t ig = idx - (int64_t)g * per_group;
    const int gw = (g == ng - 1) ? c.J - g * c.GW : c.GW;
    const int64_t q = ig / gw;  // off(k) <= q < off(k+1)
    int lo = 0, hi = L - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (diag_off(L, mid) <= q)
            lo = mid;
        else
            hi = mid - 1;
    }
    k = lo;
    const int64_t rem = ig - (int64_t)gw * diag_off(L, k);
    const int n = L - k;
    j = g * c.GW + (int)(rem / n);
    s = (int)(rem % n);
}

template <typename V, int NT, int R>
__global__ void __launch_bounds__(NT) fill_persistent(Geometry g, DevMenu dm, V* __restrict__ opt,
                                                      uint16_t* __restrict__ arg,
                                                      int* __restrict__ done,
                                                      unsigned long long* __restrict__ counter,
                                                      PCfg c) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    constexpr V INF = CostP<V>::inf;
    constexpr int NW = NT / 32;
    PSmem<V> sm = pcarve<V>(smem_raw, c);
    const int L = g.L, M = g.M;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

    for (;;) {
        if (tid == 0) sm.item[0] = (long long)atomicAdd(counter, 1ull);
        __syncthreads();
        const int64_t idx = sm.item[0];
        if (idx >= c.total) break;
        int k, j, s;
        decode_item(idx, L, g.rows, c, k, j, s);
        const int t = s + k;
        const int m0 = j * c.TM;
        const bool seeded = t < L - 1;                              // chain_dp.hpp:126
        const int64_t seed = seeded ? 2 * dm.act_u[t + 1] : 0;      // chain_dp.hpp:127
        const int o0 = dm.blk_off[s];
        const int nopt = dm.blk_off[s + 1] - o0;

        // ---- stage menu-derived parameters (no table reads: overlaps the wait)
        for (int i = tid; i < nopt; i += NT) {
            const int q = o0 + i;
            int64_t need = (k == 0 && seeded) ? dm.fwd_req_pre[q] + dm.act_u[t + 1]
                                              : dm.fwd_req[q] + seed;  // :141-143
            int64_t th = need > dm.bwd_req[q] ? need : dm.bwd_req[q];   // :144
            if (k > 0 && dm.pack_chg[q] > th) th = dm.pack_chg[q];      // :147
            sm.thr[i] = clampm(th, M);
            const int64_t p = dm.pack_chg[q];
            sm.pc[i] = p > g.pad ? g.pad : (int)p;
            sm.otot[i] = (V)dm.tftb[q];
        }
        const int32_t gate0 = clampm(dm.fwd0_own[s] + seed, M);      // :159
        if (k > 0) {
            // pointers, then (sweep, gate) as a block-wide inclusive scan
            for (int i = tid; i < k; i += NT) {
                const int cc = s + 1 + i;
                sm.lptr[i] = (long long)(opt + row_id(L, s, cc - 1) * g.sr + g.pad);
                const int64_t a = dm.act_u[cc];
                const int sh = a > g.pad ? g.pad : (int)a;
                sm.rptr[i] = (long long)(opt + row_id(L, cc, t) * g.sr + g.pad - sh);
            }
            const int per = (k + NT - 1) / NT;
            const int b0 = tid * per, b1 = min(k, b0 + per);
            V acc = 0;
            long long mx = LLONG_MIN;
            for (int i = b0; i < b1; ++i) {
                acc += (V)dm.tf0[s + i];                               // :162
                if (i >= 1) {                                          // :164 (c-1 > s)
                    const long long gv = dm.fwd0_full[s + i] + seed;
                    mx = gv > mx ? gv : mx;
                }
            }
            V inc_acc = acc;
            long long inc_mx = mx;
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                const V y = __shfl_up_sync(0xffffffffu, inc_acc, off);
                const long long ym = __shfl_up_sync(0xffffffffu, inc_mx, off);
                if (lane >= off) {
                    inc_acc += y;
                    inc_mx = ym > inc_mx ? ym : inc_mx;
                }
            }
            if (lane == 31) {
                sm.wsum[warp] = inc_acc;
                sm.wmax[warp] = inc_mx;
            }
            __syncthreads();
            V ex = __shfl_up_sync(0xffffffffu, inc_acc, 1);
            long long exm = __shfl_up_sync(0xffffffffu, inc_mx, 1);
            if (lane == 0) {
                ex = 0;
                exm = LLONG_MIN;
            }
            for (int w = 0; w < warp; ++w) {
                ex += sm.wsum[w];
                exm = sm.wmax[w] > exm ? sm.wmax[w] : exm;
            }
            for (int i = b0; i < b1; ++i) {
                ex += (V)dm.tf0[s + i];
                if (i >= 1) {
                    const long long gv = dm.fwd0_full[s + i] + seed;
                    exm = gv > exm ? gv : exm;
                }
                sm.sweep[i] = ex;
                const long long gg = exm > (long long)gate0 ? exm : (long long)gate0;
                sm.gate[i] = clampm(gg, M);
            }
        }

        // ---- wait for diagonal k-1 on tiles [j - dj, j] ----------------------
        if (k > 0 && tid == 0) {
            const int need = L - k + 1;
            const int* row = done + (int64_t)(k - 1) * c.J;
            for (int jj = (j - c.dj > 0 ? j - c.dj : 0); jj <= j; ++jj)
                while (ld_acquire(row + jj) < need) __nanosleep(40);
        }
        __syncthreads();

        // ---- option window (row (s+1, t), slots [m0 - seg_cap, m0 + TM)) -----
        const bool use_seg = k > 0 && c.seg_cap > 0;
        const V* nxt = k > 0 ? opt + row_id(L, s + 1, t) * g.sr + g.pad : nullptr;
        if (use_seg) {
            const int n = c.seg_cap + c.TM;
            for (int i = tid; i < n; i += NT) sm.seg[i] = __ldcg(nxt + (m0 - c.seg_cap + i));
            __syncthreads();
        }

        // ---- lanes over budget slots mb + NT*jj -------------------------------
        const int mb = m0 + tid;
        V best[R];
        uint16_t code[R];
        int nlive[R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
            best[r] = INF;
            code[r] = 0;
        }
        // Case 1 (chain_dp.hpp:139-156)
        for (int i = 0; i < nopt; ++i) {
            const V tt = sm.otot[i];
            const int th = sm.thr[i];
            const int p = sm.pc[i];
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const int m = mb + NT * r;
                V tot = tt;
                bool ok = m >= th;
                if (k > 0) {
                    const V sub = use_seg ? sm.seg[m - m0 + c.seg_cap - p] : __ldcg(nxt + (m - p));
                    if constexpr (CostP<V>::checked) ok = ok && sub < INF;
                    tot = tt + sub;
                }
                if (ok && tot < best[r]) {
                    best[r] = tot;
                    code[r] = (uint16_t)(i + 1);
                }
            }
        }
        // Case 2 (chain_dp.hpp:158-174)
        if (k > 0) {
#pragma unroll
            for (int r = 0; r < R; ++r) {  // cuts admitted by the sweep gate / break
                const int m = mb + NT * r;
                int lo = 0, hi = k;  // first i with gate[i] > m
                while (lo < hi) {
                    const int mid = (lo + hi) >> 1;
                    if (sm.gate[mid] <= m)
                        lo = mid + 1;
                    else
                        hi = mid;
                }
                nlive[r] = lo;
            }
            int nmax = 0;
#pragma unroll
            for (int r = 0; r < R; ++r) nmax = nlive[r] > nmax ? nlive[r] : nmax;
            const uint16_t cb = (uint16_t)(kCutBit | (s + 1));
#pragma unroll 2
            for (int i = 0; i < nmax; ++i) {
                const V* lp = reinterpret_cast<const V*>(sm.lptr[i]) + mb;
                const V* rp = reinterpret_cast<const V*>(sm.rptr[i]) + mb;
                const V sw = sm.sweep[i];
                V lv[R], rv[R];
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    if (i < nlive[r]) {
                        lv[r] = __ldcg(lp + NT * r);
                        rv[r] = __ldcg(rp + NT * r);
                    } else {
                        lv[r] = INF;
                        rv[r] = INF;
                    }
                }
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    const V tot = sw + lv[r] + rv[r];
                    bool ok = tot < best[r];
                    if constexpr (CostP<V>::checked) ok = ok && lv[r] < INF && rv[r] < INF;
                    if (ok) {
                        best[r] = tot;
                        code[r] = (uint16_t)(cb + i);
                    }
                }
            }
        }
        // ---- store (chain_dp.hpp:176-177) and publish ---------------------------
        const int64_t rid = row_id(L, s, t);
        V* orow = opt + rid * g.sr + g.pad;
        uint16_t* arow = arg + rid * g.sa;
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const int m = mb + NT * r;
            if (m <= M) {
                orow[m] = best[r];
                arow[m] = code[r];
            }
        }
        __syncthreads();
        if (tid == 0) {
            __threadfence();
            atomicAdd(done + (int64_t)k * c.J + j, 1);
        }
    }
}

template <typename V, int R>
int launch_t(const LaunchCtx& cx) {
    constexpr int NT = 256;
    cudaStream_t st = static_cast<cudaStream_t>(cx.stream);
    const Geometry& g = cx.g;
    PCfg c;
    c.TM = NT * R;
    c.J = (g.M + 1 + c.TM - 1) / c.TM;
    c.dj = (g.pad + c.TM - 1) / c.TM;
    c.seg_cap = (g.pad + c.TM <= 4096) ? g.pad : 0;
    c.kcap = g.L > 1 ? g.L - 1 : 1;
    c.ocap = cx.max_opts > 0 ? cx.max_opts : 1;
    // column group: keep rows x (GW*TM + pad) cost values near 48 MB of L2
    const double budget = 48.0 * (1 << 20) / ((double)g.rows * sizeof(V));
    int gw = (int)((budget - g.pad) / c.TM);
    if (gw < 1) gw = 1;
    if (gw > c.J) gw = c.J;
    c.GW = gw;
    c.total = (int64_t)c.J * g.rows;
    const size_t smem = psmem_bytes<V>(c.kcap, c.ocap, c.seg_cap, c.TM);
    auto kern = fill_persistent<V, NT, R>;
    if (smem > 48 * 1024 &&
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
            cudaSuccess)
        return 3;
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, NT, smem) != cudaSuccess ||
        per_sm < 1)
        return 3;
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    int64_t grid = (int64_t)per_sm * sms;
    if (grid > c.total) grid = c.total;
    const size_t flag_bytes = (size_t)g.L * c.J * sizeof(int);
    if (cx.sched_bytes < flag_bytes + 8) return 3;
    int* done = reinterpret_cast<int*>(static_cast<unsigned char*>(cx.sched) + 8);
    unsigned long long* counter = static_cast<unsigned long long*>(cx.sched);
    if (cudaMemsetAsync(cx.sched, 0, flag_bytes + 8, st) != cudaSuccess) return 3;
    kern<<<(unsigned)grid, NT, smem, st>>>(g, cx.dm, static_cast<V*>(cx.opt), cx.arg, done, counter,
                                           c);
    return cudaGetLastError() == cudaSuccess ? 0 : 3;
}

}  // namespace

size_t persistent_sched_bytes(const Geometry& g) {
    // worst case over the R choices (smallest tile): flags for L x J tiles + counter
    const int TM = 256;
    const int64_t J = (g.M + 1 + TM - 1) / TM;
    return 8 + (size_t)g.L * J * sizeof(int);
}

int persistent_r(const Geometry& g) {
    if (g.M + 1 >= 8192) return 2;
    return 1;
}

int launch_fill_persistent(const LaunchCtx& c) {
    const int R = persistent_r(c.g);
    if (c.width == 32) return R == 2 ? launch_t<uint32_t, 2>(c) : launch_t<uint32_t, 1>(c);
    return R == 2 ? launch_t<int64_t, 2>(c) : launch_t<int64_t, 1>(c);
}

}  // namespace rkr
