// rkr_walk.cuh -- K2, build_schedule_rec (chain_dp.hpp:211-246) as an
// explicit-stack walk on one thread, shared by the stand-alone backtrack
// kernels (rkr_kernels.cu) and the walk fused into the K1t fill (rkr_tiles.cu).
#pragma once

#include <cuda_runtime.h>

#include <climits>
#include <cstdint>

#include "rkr_internal.h"

namespace rkr {
namespace {

template <typename V>
struct Cost;
template <>
struct Cost<uint32_t> {
    static constexpr uint32_t inf = kInf32;
    static constexpr bool checked = false;  // bounded by the host overflow proof
};
template <>
struct Cost<int64_t> {
    static constexpr int64_t inf = kInf64;
    static constexpr bool checked = true;   // arbitrary int64: explicit inf tests
};

// Menu lookups the walk needs, straight from the device menu or from a
// shared-memory copy (the walk is a chain of dependent loads, so every hop
// it takes off global memory shortens it).  chg/act are cast to int exactly
// as build_schedule_rec does (chain_dp.hpp:229, :240).
struct GlobalMenuView {
    const DevMenu* dm;
    __device__ int blk(int s) const { return dm->blk_off[s]; }
    __device__ int id(int q) const { return dm->ids[q]; }
    __device__ int chg(int q) const { return (int)dm->chg_bt[q]; }
    __device__ int act(int c) const { return (int)dm->act_u[c]; }
};
struct SharedMenuView {
    const int32_t *b, *i, *g, *a;
    __device__ int blk(int s) const { return b[s]; }
    __device__ int id(int q) const { return i[q]; }
    __device__ int chg(int q) const { return g[q]; }
    __device__ int act(int c) const { return a[c]; }
};

// K2: build_schedule_rec as an explicit stack walk on one thread.  Stack
// entries are int4 {type, s, t, m}: type 0 = cell to expand, type 1 =
// pending BlockBwd(s, t = option).  out = {n_ops, status, bad_s, bad_t, top};
// status 2 = infinite cell (bad_s, bad_t), 3 = the menu lacks the option
// (bad_s = block, bad_t = option id).
template <typename V, typename MV>
__device__ void walk(const Geometry& g, const MV& mv, const V* __restrict__ opt,
                     const uint16_t* __restrict__ arg, int s0, int t0, int m0,
                     int32_t* __restrict__ ops, int64_t cap, int4* __restrict__ stack,
                     int64_t* __restrict__ out) {
    const int L = g.L, M = g.M;
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
    {  // the root cell's value (solve_chain's opt_time / feasibility test)
        int64_t top = kInf64;
        if (m0 >= 0) {
            const V v = opt[row_id(L, s0, t0) * g.sr + g.pad + (m0 > M ? M : m0)];
            top = v >= Cost<V>::inf ? kInf64 : (int64_t)v;
        }
        out[4] = top;
    }
    // the cell expanded next stays in registers (the child an expansion
    // would push and pop at once); the stack keeps the deferred BlockBwds
    // and the left children of cuts
    int cs = s0, ct = t0, cm = m0;
    bool have = true;
    for (;;) {
        if (!have) {
            bool found = false;
            while (sp > 0) {
                const int4 e = stack[--sp];
                if (e.x == 1) {  // deferred BlockBwd of an option turn (chain_dp.hpp:230)
                    emit(3, e.y, e.z);
                    continue;
                }
                cs = e.y;
                ct = e.z;
                cm = e.w;
                found = true;
                break;
            }
            if (!found) break;
        }
        const int s = cs, t = ct, m = cm;
        // table.opt(s,t,m) >= kInfTime -> InfeasibleBudget (chain_dp.hpp:213-215)
        const int64_t rid = row_id(L, s, t);
        const bool inf = m < 0;
        const int mm = m > M ? M : (m < 0 ? 0 : m);
        // One table read per hop: a cell's code is 0 exactly when its value
        // is infinite (every fill updates value and code together, with a
        // strict '<' from infinity), so the code alone decides.  L1-cached
        // load (the walk runs in its own launch, or after the fill's acquire
        // fence, so L1 holds no stale line).
        const uint16_t code = __ldca(arg + rid * g.sa + mm);
        if (inf || code == 0) {  // infinite (or undecided) cell
            status = 2;
            bad_s = s;
            bad_t = t;
            break;
        }
        if (!(code & kCutBit)) {  // Option (chain_dp.hpp:217-232)
            const int q = mv.blk(s) + code - 1;
            const int val = mv.id(q);
            const int chg = mv.chg(q);
            if (chg == kMissingShift) {  // (rkr_backtrack_menu)  // menu_option throws (chain_dp.hpp:203)
                status = 3;
                bad_s = s;
                bad_t = val;
                break;
            }
            emit(2, s, val);
            if (s == t) {
                if (t == L - 1) emit(0, t, -1);
                emit(3, s, val);
                have = false;
            } else {
                stack[sp++] = make_int4(1, s, val, 0);
                cs = s + 1;  // (s + 1, t, m - chg) next
                cm = m - chg;
                have = true;
            }
        } else {  // Cut (chain_dp.hpp:233-244)
            const int c = code & 0x7fff;
            emit(2, s, 0);
            for (int j = s + 1; j < c; ++j) {
                emit(2, j, 0);
                emit(1, j, -1);
            }
            stack[sp++] = make_int4(0, s, c - 1, m);  // left, after
            cs = c;                                   // right, next
            cm = m - mv.act(c);
            have = true;
            // the left child is expanded after the whole right subtree: pull
            // its cell into L1 now so that hop costs an L1 hit
            if (m >= 0) {
                const int64_t lr = row_id(L, s, c - 1);
                const int mm = m > M ? M : m;
                asm volatile("prefetch.global.L1 [%0];" ::"l"(arg + lr * g.sa + mm));
            }
        }
    }
    out[0] = n;
    out[1] = status;
    out[2] = bad_s;
    out[3] = bad_t;
}

// The walk is a chain of dependent loads (code -> next cell); one warp stages
// the stack and the menu lookups in shared memory when they fit, so each hop
// costs one table read.
}  // namespace
}  // namespace rkr
