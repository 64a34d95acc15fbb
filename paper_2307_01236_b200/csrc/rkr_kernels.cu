// rkr_kernels.cu -- sm_100a kernels of the rk-Rotor chain DP.
//
//   K1 fill_diag      one launch per anti-diagonal k = t - s; CTA = (s, tile of
//                     NT*R budget slots); lanes over consecutive m; the
//                     candidate loop (options in menu order, then cuts
//                     ascending) with a strict '<' reproduces the reference
//                     argmin exactly (chain_dp.hpp:125-183).
//   K2 backtrack      build_schedule_rec (chain_dp.hpp:211-246) as an explicit
//                     stack walk on one thread; only the ops go back to the host.
//   K3 first_feasible the min-feasible scan of solve_chain (chain_dp.hpp:280-284).
//   export_rows       converts packed rows (uint32/int64 cost + uint16 code) to
//                     the reference's (int64 Micros, DpArg) layout.
//
// Integer min-plus only: no tensor cores (there is no contraction to feed).
#include <cuda_runtime.h>

#include <cstdint>

#include "rkr_internal.h"
#include "rkr_walk.cuh"

namespace rkr {

namespace {

__device__ __forceinline__ int32_t clamp_thr(int64_t x, int32_t M) {
    return x < -1 ? -1 : (x > (int64_t)M + 1 ? M + 1 : (int32_t)x);
}

// Shared-memory image of one cell's candidates (uniform across the CTA).
template <typename V>
struct CellSmem {
    int64_t* lbase;  // [k] left row (s, c-1) base, element index of m = 0
    int64_t* rbase;  // [k] right row (c, t) base, pre-shifted by -act_u[c]
    V* inc;          // [k] time_fwd0[c-1]: sweep increment
    V* otot;         // [nopt] time_fwd + time_bwd
    int32_t* gate;   // [k] fwd0_full[c-1] + seed (clamped), -1 when c-1 == s
    int32_t* thr;    // [nopt] validity threshold of option oi (clamped)
    int32_t* pc;     // [nopt] pack_chg (clamped to pad)
};

template <typename V>
__host__ __device__ inline size_t cell_smem_bytes(int k, int nopt) {
    return (size_t)k * (8 + 8 + sizeof(V) + 4) + (size_t)nopt * (sizeof(V) + 4 + 4);
}

template <typename V>
__device__ inline CellSmem<V> carve(unsigned char* p, int k, int nopt) {
    CellSmem<V> c;
    c.lbase = reinterpret_cast<int64_t*>(p);
    c.rbase = c.lbase + k;
    c.inc = reinterpret_cast<V*>(c.rbase + k);
    c.otot = c.inc + k;
    c.gate = reinterpret_cast<int32_t*>(c.otot + nopt);
    c.thr = c.gate + k;
    c.pc = c.thr + nopt;
    return c;
}

// K1: fill every cell (s, s+k, m) of diagonal k.
template <typename V, int NT, int R>
__global__ void __launch_bounds__(NT) fill_diag(Geometry g, DevMenu dm, V* __restrict__ opt,
                                                uint16_t* __restrict__ arg, int k) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    constexpr V INF = Cost<V>::inf;
    const int L = g.L, M = g.M;
    const int s = blockIdx.y;
    const int t = s + k;
    const bool seeded = t < L - 1;                                    // chain_dp.hpp:126
    const int64_t seed = seeded ? 2 * dm.act_u[t + 1] : 0;            // chain_dp.hpp:127
    const int o0 = dm.blk_off[s];
    const int nopt = dm.blk_off[s + 1] - o0;
    CellSmem<V> cs = carve<V>(smem_raw, k, nopt);

    // ---- prologue: stage this cell's candidate parameters -------------------
    for (int i = threadIdx.x; i < k; i += NT) {
        const int c = s + 1 + i;
        cs.lbase[i] = row_id(L, s, c - 1) * g.sr + g.pad;
        const int64_t a = dm.act_u[c];
        const int sh = a > g.pad ? g.pad : (int)a;
        cs.rbase[i] = row_id(L, c, t) * g.sr + g.pad - sh;
        cs.inc[i] = (V)dm.tf0[c - 1];
        cs.gate[i] = (c - 1 > s) ? clamp_thr(dm.fwd0_full[c - 1] + seed, M) : -1;
    }
    for (int i = threadIdx.x; i < nopt; i += NT) {
        const int q = o0 + i;
        // chain_dp.hpp:141-147: fwd need, bwd need and (s < t) pack fit
        int64_t need = (k == 0 && seeded) ? dm.fwd_req_pre[q] + dm.act_u[t + 1]
                                          : dm.fwd_req[q] + seed;
        int64_t th = need > dm.bwd_req[q] ? need : dm.bwd_req[q];
        if (k > 0 && dm.pack_chg[q] > th) th = dm.pack_chg[q];
        cs.thr[i] = clamp_thr(th, M);
        const int64_t p = dm.pack_chg[q];
        cs.pc[i] = p > g.pad ? g.pad : (int)p;
        cs.otot[i] = (V)dm.tftb[q];
    }
    const int32_t gate0 = clamp_thr(dm.fwd0_own[s] + seed, M);       // chain_dp.hpp:159
    __syncthreads();

    // ---- lanes over consecutive budget slots ---------------------------------
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int mb = blockIdx.x * (NT * R) + warp * (32 * R) + lane;
    int mj[R];
    bool inr[R];
#pragma unroll
    for (int j = 0; j < R; ++j) {
        const int m = mb + 32 * j;
        inr[j] = m <= M;
        mj[j] = inr[j] ? m : M;
    }
    V best[R];
    uint16_t code[R];
#pragma unroll
    for (int j = 0; j < R; ++j) {
        best[j] = INF;
        code[j] = 0;
    }

    // ---- Case 1: saved options in menu order (chain_dp.hpp:139-156) ---------
    if (k == 0) {
        for (int i = 0; i < nopt; ++i) {
            const V tot = cs.otot[i];
            const int th = cs.thr[i];
#pragma unroll
            for (int j = 0; j < R; ++j)
                if (mj[j] >= th && tot < best[j]) {
                    best[j] = tot;
                    code[j] = (uint16_t)(i + 1);
                }
        }
    } else {
        const V* __restrict__ nxt = opt + row_id(L, s + 1, t) * g.sr + g.pad;
        for (int i = 0; i < nopt; ++i) {
            const V tt = cs.otot[i];
            const int th = cs.thr[i];
            const int p = cs.pc[i];
#pragma unroll
            for (int j = 0; j < R; ++j) {
                const V sub = __ldcg(nxt + (mj[j] - p));  // pad slots hold INF
                bool ok = mj[j] >= th;
                if constexpr (Cost<V>::checked) ok = ok && sub < INF;
                const V tot = tt + sub;
                if (ok && tot < best[j]) {
                    best[j] = tot;
                    code[j] = (uint16_t)(i + 1);
                }
            }
        }

        // ---- Case 2: cuts ascending with the option-0 sweep (chain_dp.hpp:158-174)
        bool alive[R];
#pragma unroll
        for (int j = 0; j < R; ++j) alive[j] = mj[j] >= gate0;
        V sweep = 0;
        for (int i = 0; i < k; ++i) {
            sweep += cs.inc[i];
            const int gt = cs.gate[i];
            bool any = false;
#pragma unroll
            for (int j = 0; j < R; ++j) {
                alive[j] = alive[j] && mj[j] >= gt;  // the reference's `break`
                any |= alive[j];
            }
            if (!any) break;
            const V* __restrict__ lrow = opt + cs.lbase[i];
            const V* __restrict__ rrow = opt + cs.rbase[i];
            const uint16_t cc = (uint16_t)(kCutBit | (s + 1 + i));
#pragma unroll
            for (int j = 0; j < R; ++j) {
                if (!alive[j]) continue;
                const V r = __ldcg(rrow + mj[j]);  // m - act_u[c] < 0 lands in the pad
                const V l = __ldcg(lrow + mj[j]);
                const V tot = sweep + r + l;
                bool ok = tot < best[j];
                if constexpr (Cost<V>::checked) ok = ok && r < INF && l < INF;
                if (ok) {
                    best[j] = tot;
                    code[j] = cc;
                }
            }
        }
    }

    // ---- store (chain_dp.hpp:176-177) ---------------------------------------
    const int64_t rid = row_id(L, s, t);
    V* __restrict__ orow = opt + rid * g.sr + g.pad;
    uint16_t* __restrict__ arow = arg + rid * g.sa;
#pragma unroll
    for (int j = 0; j < R; ++j)
        if (inr[j]) {
            orow[mj[j]] = best[j];
            arow[mj[j]] = code[j];
        }
}

template <typename V>
__global__ void init_pads(Geometry g, V* opt) {
    const int64_t n = g.rows * (int64_t)g.pad;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = i / g.pad, p = i - r * g.pad;
        opt[r * g.sr + p] = Cost<V>::inf;
    }
}

template <typename V>
__global__ void backtrack(Geometry g, DevMenu dm, const V* __restrict__ opt,
                          const uint16_t* __restrict__ arg, int s0, int t0, int m0,
                          int32_t* __restrict__ ops, int64_t cap, int4* __restrict__ stack,
                          int64_t* __restrict__ out, int smem_mode, int nq) {
    extern __shared__ int4 sbuf[];
    if (blockIdx.x != 0) return;
    const int L = g.L;
    if (smem_mode) {
        int4* sstack = sbuf;
        int32_t* b = reinterpret_cast<int32_t*>(sstack + 2 * L + 16);
        int32_t* a = b + L + 1;
        int32_t* i = a + L + 1;
        int32_t* gq = i + nq;
        for (int x = threadIdx.x; x <= L; x += blockDim.x) {
            b[x] = dm.blk_off[x];
            a[x] = (int)dm.act_u[x];
        }
        for (int x = threadIdx.x; x < nq; x += blockDim.x) {
            i[x] = dm.ids[x];
            gq[x] = (int)dm.chg_bt[x];
        }
        __syncthreads();
        if (threadIdx.x != 0) return;
        walk<V>(g, SharedMenuView{b, i, gq, a}, opt, arg, s0, t0, m0, ops, cap, sstack, out);
    } else {
        if (threadIdx.x != 0) return;
        walk<V>(g, GlobalMenuView{&dm}, opt, arg, s0, t0, m0, ops, cap, stack, out);
    }
}

// Batched K2: thread i walks table i from (0, L-1, m_at[i]) when active[i];
// ops of table i go to ops + 3 * cap * i (at most cap of them); its 8-word
// result record to out + 8 * i.
template <typename V>
__global__ void batch_walk(const InstDesc* __restrict__ d, const int32_t* __restrict__ m_at,
                           const uint8_t* __restrict__ active, int n, int32_t* __restrict__ ops,
                           int64_t cap, int64_t* __restrict__ out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    if (!active[i]) {
        out[8 * i] = 0;
        out[8 * i + 1] = -1;
        return;
    }
    const InstDesc& D = d[i];
    walk<V>(D.g, GlobalMenuView{&D.dm}, static_cast<const V*>(D.opt), D.arg, 0, D.g.L - 1,
            m_at[i], ops + 3 * cap * (int64_t)i, cap, static_cast<int4*>(D.stack), out + 8 * i);
}

// K2 across budget shards (config 5): identical walk, each cell read from the
// shard that owns its budget slot (peer memory when shards live on other GPUs).
template <typename V>
__global__ void walk_sharded(const ShardView* __restrict__ sv, int n_shards, DevMenu dm, int L,
                             int M, int s0, int t0, int m0, int32_t* __restrict__ ops, int64_t cap,
                             int4* __restrict__ stack, int64_t* __restrict__ out) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    int64_t n = 0;
    int sp = 0;
    int64_t status = 0, bad_s = -1, bad_t = -1;
    auto emit = [&](int kd, int b, int x) {
        if (n < cap) {
            ops[3 * n] = kd;
            ops[3 * n + 1] = b;
            ops[3 * n + 2] = x;
        }
        ++n;
    };
    stack[sp++] = make_int4(0, s0, t0, m0);
    while (sp > 0) {
        const int4 e = stack[--sp];
        if (e.x == 1) {
            emit(3, e.y, e.z);
            continue;
        }
        const int s = e.y, t = e.z, m = e.w;
        bool inf = m < 0;
        uint16_t code = 0;
        if (!inf) {
            const int mm = m > M ? M : m;
            int q = 0;
            while (q + 1 < n_shards && mm >= sv[q + 1].lo) ++q;
            const ShardView& v = sv[q];
            const int64_t rid = row_id(L, s, t);
            // one read per hop: a cell's code is 0 exactly when its value is
            // infinite (rkr_walk.cuh), so the owner's opt row is not read
            code = v.arg[rid * v.sa + (mm - v.lo)];
        }
        if (inf || code == 0) {
            status = 2;
            bad_s = s;
            bad_t = t;
            break;
        }
        if (!(code & kCutBit)) {
            const int q = dm.blk_off[s] + code - 1;
            const int val = dm.ids[q];
            emit(2, s, val);
            if (s == t) {
                if (t == L - 1) emit(0, t, -1);
                emit(3, s, val);
            } else {
                stack[sp++] = make_int4(1, s, val, 0);
                stack[sp++] = make_int4(0, s + 1, t, m - (int)dm.chg_bt[q]);
            }
        } else {
            const int c = code & 0x7fff;
            emit(2, s, 0);
            for (int j = s + 1; j < c; ++j) {
                emit(2, j, 0);
                emit(1, j, -1);
            }
            stack[sp++] = make_int4(0, s, c - 1, m);
            stack[sp++] = make_int4(0, c, t, m - (int)dm.act_u[c]);
        }
    }
    out[0] = n;
    out[1] = status;
    out[2] = bad_s;
    out[3] = bad_t;
}

// Batched top cells: out[i] = opt(0, L-1, min(m_at[i], M)) as int64 (kInf64 when infinite).
template <typename V>
__global__ void batch_tops(const InstDesc* __restrict__ d, const int32_t* __restrict__ m_at, int n,
                           int64_t* __restrict__ out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const InstDesc& D = d[i];
    int m = m_at[i];
    if (m < 0) {
        out[i] = kInf64;
        return;
    }
    if (m > D.g.M) m = D.g.M;
    const V v = static_cast<const V*>(D.opt)[row_id(D.g.L, 0, D.g.L - 1) * D.g.sr + D.g.pad + m];
    out[i] = v >= Cost<V>::inf ? kInf64 : (int64_t)v;
}

// Batched K3: block i finds the first finite m of table i's top row.
template <typename V>
__global__ void batch_first_feasible(const InstDesc* __restrict__ d, int n, int32_t* __restrict__ out) {
    const int i = blockIdx.x;
    if (i >= n) return;
    __shared__ int best;
    if (threadIdx.x == 0) best = 0x7fffffff;
    __syncthreads();
    const InstDesc& D = d[i];
    const V* row = static_cast<const V*>(D.opt) + row_id(D.g.L, 0, D.g.L - 1) * D.g.sr + D.g.pad;
    for (int m = threadIdx.x; m <= D.g.M; m += blockDim.x)
        if (row[m] < Cost<V>::inf) {
            atomicMin(&best, m);
            break;
        }
    __syncthreads();
    if (threadIdx.x == 0) out[i] = best == 0x7fffffff ? -1 : best;
}

// K3: first m with opt(s,t,m) < inf.
template <typename V>
__global__ void first_feasible(Geometry g, const V* __restrict__ opt, int s, int t, int* m_out) {
    const int64_t base = row_id(g.L, s, t) * g.sr + g.pad;
    for (int m = blockIdx.x * blockDim.x + threadIdx.x; m <= g.M; m += gridDim.x * blockDim.x)
        if (opt[base + m] < Cost<V>::inf) {
            atomicMin(m_out, m);
            return;
        }
}

// Packed rows -> reference layout for rows [r0, r1) of the s-major order.
template <typename V>
__global__ void export_rows(Geometry g, DevMenu dm, const V* __restrict__ opt,
                            const uint16_t* __restrict__ arg, int64_t r0, int64_t* __restrict__ o,
                            int8_t* __restrict__ kd, int32_t* __restrict__ val) {
    const int L = g.L;
    const int64_t r = r0 + blockIdx.y;
    int s = 0;
    int64_t first = 0;
    while (first + (L - s) <= r) {
        first += L - s;
        ++s;
    }
    const int t = s + (int)(r - first);
    const int64_t rid = row_id(L, s, t);
    const int64_t W = g.M + 1;
    const int64_t ob = (int64_t)blockIdx.y * W;
    for (int m = blockIdx.x * blockDim.x + threadIdx.x; m <= g.M; m += gridDim.x * blockDim.x) {
        const V v = opt[rid * g.sr + g.pad + m];
        const uint16_t c = arg[rid * g.sa + m];
        if (o) o[ob + m] = v >= Cost<V>::inf ? kInf64 : (int64_t)v;
        int8_t k = 0;
        int32_t x = -1;
        if (v < Cost<V>::inf && c != 0) {
            if (c & kCutBit) {
                k = 2;
                x = c & 0x7fff;
            } else {
                k = 1;
                x = dm.ids[dm.blk_off[s] + c - 1];
            }
        }
        if (kd) kd[ob + m] = k;
        if (val) val[ob + m] = x;
    }
}

template <typename V>
int fill_all_t(const LaunchCtx& c) {
    constexpr int NT = 128, R = 2;
    cudaStream_t st = static_cast<cudaStream_t>(c.stream);
    V* opt = static_cast<V*>(c.opt);
    const int tiles = (c.g.M + 1 + NT * R - 1) / (NT * R);
    const size_t max_smem = cell_smem_bytes<V>(c.g.L, c.max_opts);
    if (max_smem > 48 * 1024)
        cudaFuncSetAttribute(fill_diag<V, NT, R>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)max_smem);
    for (int k = 0; k < c.g.L; ++k) {
        dim3 grid(tiles, c.g.L - k);
        fill_diag<V, NT, R><<<grid, NT, cell_smem_bytes<V>(k, c.max_opts), st>>>(
            c.g, c.dm, opt, c.arg, k);
    }
    return cudaPeekAtLastError() == cudaSuccess ? 0 : 3;  // (the caller reports it)
}

}  // namespace

int launch_init_pads(const LaunchCtx& c) {
    if (c.g.pad == 0) return 0;
    cudaStream_t st = static_cast<cudaStream_t>(c.stream);
    const int64_t n = c.g.rows * (int64_t)c.g.pad;
    int blocks = (int)((n + 255) / 256);
    if (blocks > 148 * 16) blocks = 148 * 16;
    if (c.width == 32)
        init_pads<uint32_t><<<blocks, 256, 0, st>>>(c.g, static_cast<uint32_t*>(c.opt));
    else
        init_pads<int64_t><<<blocks, 256, 0, st>>>(c.g, static_cast<int64_t*>(c.opt));
    return cudaPeekAtLastError() == cudaSuccess ? 0 : 3;  // (the caller reports it)
}

int launch_fill_all(const LaunchCtx& c) {
    return c.width == 32 ? fill_all_t<uint32_t>(c) : fill_all_t<int64_t>(c);
}

int launch_backtrack(const LaunchCtx& c, int32_t s, int32_t t, int32_t m, int32_t* dev_ops,
                     int64_t cap, int32_t* dev_stack, int64_t* dev_out) {
    cudaStream_t st = static_cast<cudaStream_t>(c.stream);
    int4* stk = reinterpret_cast<int4*>(dev_stack);
    const int nq = c.nq;
    const size_t sbytes = sizeof(int4) * (2 * (size_t)c.g.L + 16) +
                          4 * (2 * ((size_t)c.g.L + 1) + 2 * (size_t)nq);
    const int use_smem = sbytes <= 48 * 1024 ? 1 : 0;
    const size_t dyn = use_smem ? sbytes : 0;
    if (c.width == 32)
        backtrack<uint32_t><<<1, 128, dyn, st>>>(c.g, c.dm, static_cast<const uint32_t*>(c.opt),
                                                 c.arg, s, t, m, dev_ops, cap, stk, dev_out,
                                                 use_smem, nq);
    else
        backtrack<int64_t><<<1, 128, dyn, st>>>(c.g, c.dm, static_cast<const int64_t*>(c.opt),
                                                c.arg, s, t, m, dev_ops, cap, stk, dev_out,
                                                use_smem, nq);
    return cudaPeekAtLastError() == cudaSuccess ? 0 : 3;  // (the caller reports it)
}

int launch_batch_walk(const InstDesc* d, const int32_t* m_at, const uint8_t* active, int n,
                      int width, int32_t* ops, int64_t cap, int64_t* out, void* stream) {
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int blocks = (n + 31) / 32;
    if (width == 32)
        batch_walk<uint32_t><<<blocks, 32, 0, st>>>(d, m_at, active, n, ops, cap, out);
    else
        batch_walk<int64_t><<<blocks, 32, 0, st>>>(d, m_at, active, n, ops, cap, out);
    return cudaPeekAtLastError() == cudaSuccess ? 0 : 3;  // (the caller reports it)
}

int launch_walk_sharded(const ShardView* sv, int n, const DevMenu& dm, int L, int M, int width,
                        int s, int t, int m, int32_t* ops, int64_t cap, int32_t* stack,
                        int64_t* out, void* stream) {
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    int4* stk = reinterpret_cast<int4*>(stack);
    if (width == 32)
        walk_sharded<uint32_t><<<1, 32, 0, st>>>(sv, n, dm, L, M, s, t, m, ops, cap, stk, out);
    else
        walk_sharded<int64_t><<<1, 32, 0, st>>>(sv, n, dm, L, M, s, t, m, ops, cap, stk, out);
    return cudaPeekAtLastError() == cudaSuccess ? 0 : 3;  // (the caller reports it)
}

int launch_batch_tops(const InstDesc* d, const int32_t* m_at, int n, int width, int64_t* out,
                      void* stream) {
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int blocks = (n + 127) / 128;
    if (width == 32)
        batch_tops<uint32_t><<<blocks, 128, 0, st>>>(d, m_at, n, out);
    else
        batch_tops<int64_t><<<blocks, 128, 0, st>>>(d, m_at, n, out);
    return cudaPeekAtLastError() == cudaSuccess ? 0 : 3;  // (the caller reports it)
}

// solve_chain's min-feasible search (chain_dp.hpp:265-288) without the wide
// table.  Whether opt(s, t, m) is finite does not depend on the times, and it
// is upward closed in m (every admission test of :141-174 is "requirement <=
// m" and every read of a smaller span is at m minus a shift >= 0), so it is
// the threshold thr(s, t) = the smallest feasible m, a min-max recurrence over
// the same candidates with no budget axis:
//   option oi (:141-151):  max(fwd_need, bwd_req [, pack_chg + thr(s+1, t)])
//   cut c (:158-171):      max(gate(s, c), act_u[c] + thr(c, t), thr(s, c-1))
// with gate(s, c) = the sweep gate (:159) and the prefix maximum behind the
// `break` (:164), and thr clamped at 0 (budgets are >= 0).  The wide table's
// first finite m is thr(0, L-1) when it is <= cap.  Exact as long as every
// finite candidate total stays below kInfTime (the host's 64-bit overflow
// proof; else the wide table runs).  One CTA per instance; the thresholds of
// a diagonal depend only on smaller spans, so a CTA barrier per diagonal.
__global__ void batch_thresholds(const InstDesc* __restrict__ d, const int32_t* __restrict__ which,
                                 int64_t* __restrict__ scratch, const int64_t* __restrict__ scr_off,
                                 int64_t* __restrict__ out) {
    const InstDesc& D = d[which[blockIdx.x]];
    const DevMenu& dm = D.dm;
    const int L = D.g.L;
    int64_t* thr = scratch + scr_off[blockIdx.x];  // [row_id(L, s, t)]
    for (int k = 0; k < L; ++k) {
        for (int s = threadIdx.x; s < L - k; s += blockDim.x) {
            const int t = s + k;
            const bool seeded = t < L - 1;                                     // :126-127
            const int64_t seed = seeded ? 2 * dm.act_u[t + 1] : 0;
            int64_t best = kInf64;
            const int64_t sub = s < t ? thr[row_id(L, s + 1, t)] : 0;
            for (int q = dm.blk_off[s]; q < dm.blk_off[s + 1]; ++q) {          // :139-156
                int64_t c = (s == t && seeded) ? dm.fwd_req_pre[q] + dm.act_u[t + 1]
                                               : dm.fwd_req[q] + seed;
                c = max(c, dm.bwd_req[q]);
                if (s < t) {
                    if (sub >= kInf64) continue;
                    c = max(c, dm.pack_chg[q] + sub);
                }
                best = min(best, c);
            }
            if (s < t) {                                                       // :158-174
                int64_t gate = dm.fwd0_own[s] + seed;
                for (int c = s + 1; c <= t; ++c) {
                    if (c - 1 > s) gate = max(gate, dm.fwd0_full[c - 1] + seed);
                    const int64_t r = thr[row_id(L, c, t)], l = thr[row_id(L, s, c - 1)];
                    if (r >= kInf64 || l >= kInf64) continue;
                    best = min(best, max(max(gate, dm.act_u[c] + r), l));
                }
            }
            thr[row_id(L, s, t)] = best >= kInf64 ? kInf64 : max(best, (int64_t)0);
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) out[blockIdx.x] = thr[row_id(L, 0, L - 1)];
}

int launch_batch_thresholds(const InstDesc* d, const int32_t* which, int n, int64_t* scratch,
                            const int64_t* scr_off, int64_t* out, void* stream) {
    if (n <= 0) return 0;
    batch_thresholds<<<n, 128, 0, static_cast<cudaStream_t>(stream)>>>(d, which, scratch, scr_off,
                                                                      out);
    return cudaPeekAtLastError() == cudaSuccess ? 0 : 3;  // (the caller reports it)
}

int launch_batch_first_feasible(const InstDesc* d, int n, int width, int32_t* out, void* stream) {
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (width == 32)
        batch_first_feasible<uint32_t><<<n, 256, 0, st>>>(d, n, out);
    else
        batch_first_feasible<int64_t><<<n, 256, 0, st>>>(d, n, out);
    return cudaPeekAtLastError() == cudaSuccess ? 0 : 3;  // (the caller reports it)
}

int launch_first_feasible(const LaunchCtx& c, int32_t s, int32_t t, int32_t* dev_m) {
    cudaStream_t st = static_cast<cudaStream_t>(c.stream);
    int blocks = (c.g.M + 1 + 255) / 256;
    if (blocks > 148 * 8) blocks = 148 * 8;
    if (c.width == 32)
        first_feasible<uint32_t><<<blocks, 256, 0, st>>>(
            c.g, static_cast<const uint32_t*>(c.opt), s, t, dev_m);
    else
        first_feasible<int64_t><<<blocks, 256, 0, st>>>(
            c.g, static_cast<const int64_t*>(c.opt), s, t, dev_m);
    return cudaPeekAtLastError() == cudaSuccess ? 0 : 3;  // (the caller reports it)
}

int launch_export(const LaunchCtx& c, int64_t r0, int64_t r1, int64_t* o, int8_t* kd,
                  int32_t* val) {
    cudaStream_t st = static_cast<cudaStream_t>(c.stream);
    if (r1 <= r0) return 0;
    int bx = (c.g.M + 1 + 255) / 256;
    if (bx > 64) bx = 64;
    dim3 grid(bx, (unsigned)(r1 - r0));
    if (c.width == 32)
        export_rows<uint32_t><<<grid, 256, 0, st>>>(
            c.g, c.dm, static_cast<const uint32_t*>(c.opt), c.arg, r0, o, kd, val);
    else
        export_rows<int64_t><<<grid, 256, 0, st>>>(
            c.g, c.dm, static_cast<const int64_t*>(c.opt), c.arg, r0, o, kd, val);
    return cudaPeekAtLastError() == cudaSuccess ? 0 : 3;  // (the caller reports it)
}

}  // namespace rkr
