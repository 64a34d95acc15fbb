// l2probe.cu -- L2 read-bandwidth micro-benchmark (measurement infrastructure
// for bench.py's roofline; not part of the solver).
//
// The budget-tile fill reads earlier-diagonal rows that stay resident in L2
// (ncu: 97 % L2 hit rate, ~0.5 GB of DRAM traffic against ~35 GB of L2 traffic
// per config-3 fill), so its memory roof is the L2, not HBM.  MEASURED_PEAKS.json
// holds no L2 figure, so this kernel measures one: every SM streams an
// L2-resident buffer with the fill's own load flavour (ld.global.cg = L2 only,
// SASS LDG.E.STRONG.GPU), either 16 B per lane (the peak) or 4 B per lane (the
// fill's access: one 128-byte row segment per warp instruction).
//
//   extern "C" int l2probe_run(int device, int64_t bytes, int reps, int vec16,
//                              double* gbs)
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -shared -Xcompiler -fPIC
#include <cuda_runtime.h>

#include <cstdint>

namespace {

__global__ void __launch_bounds__(1024) read16(const int4* __restrict__ p, int64_t n, int reps,
                                               int* __restrict__ sink) {
    int acc = 0;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int r = 0; r < reps; ++r) {
        // rotate the start so consecutive passes hit different L2 slices first
        const int64_t base = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x + (int64_t)r * 4096) % stride;
        int64_t i = base;
        for (; i + 3 * stride < n; i += 4 * stride) {
            const int4 a = __ldcg(p + i), b = __ldcg(p + i + stride);
            const int4 c = __ldcg(p + i + 2 * stride), d = __ldcg(p + i + 3 * stride);
            acc ^= a.x ^ a.y ^ a.z ^ a.w ^ b.x ^ b.y ^ b.z ^ b.w ^ c.x ^ c.y ^ c.z ^ c.w ^ d.x ^ d.y ^
                   d.z ^ d.w;
        }
        for (; i < n; i += stride) {
            const int4 a = __ldcg(p + i);
            acc ^= a.x ^ a.y ^ a.z ^ a.w;
        }
    }
    if (acc == 0x7fffffff) sink[0] = acc;
}

__global__ void __launch_bounds__(1024) read4(const int* __restrict__ p, int64_t n, int reps,
                                              int* __restrict__ sink) {
    int acc = 0;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int r = 0; r < reps; ++r) {
        const int64_t base = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x + (int64_t)r * 4096) % stride;
        int64_t i = base;
        for (; i + 7 * stride < n; i += 8 * stride) {
            int v[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) v[q] = __ldcg(p + i + q * stride);
#pragma unroll
            for (int q = 0; q < 8; ++q) acc ^= v[q];
        }
        for (; i < n; i += stride) acc ^= __ldcg(p + i);
    }
    if (acc == 0x7fffffff) sink[0] = acc;
}

}  // namespace

extern "C" int l2probe_run(int device, int64_t bytes, int reps, int vec16, double* gbs) {
    if (cudaSetDevice(device) != cudaSuccess) return 1;
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    void* buf = nullptr;
    int* sink = nullptr;
    if (cudaMalloc(&buf, bytes) != cudaSuccess) return 2;
    if (cudaMalloc(&sink, 64) != cudaSuccess) return 2;
    cudaMemset(buf, 1, bytes);
    cudaStream_t st;
    cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const dim3 grid(sms * 2), block(1024);
    auto launch = [&]() {
        if (vec16)
            read16<<<grid, block, 0, st>>>(static_cast<const int4*>(buf), bytes / 16, reps, sink);
        else
            read4<<<grid, block, 0, st>>>(static_cast<const int*>(buf), bytes / 4, reps, sink);
    };
    for (int w = 0; w < 3; ++w) launch();  // warm: the buffer is now L2-resident
    float best = 1e30f;
    for (int it = 0; it < 10; ++it) {
        cudaEventRecord(e0, st);
        launch();
        cudaEventRecord(e1, st);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    const int rc = cudaGetLastError() == cudaSuccess ? 0 : 3;
    *gbs = (double)bytes * reps / (best * 1e-3) / 1e9;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaStreamDestroy(st);
    cudaFree(buf);
    cudaFree(sink);
    return rc;
}
