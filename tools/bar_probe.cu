// Probe: do named-barrier arrivals of a warp that first diverges (lane 0
// polls / stamps) hold bar.sync of the other warps?  And are clock64 stamps
// of different warps of one SM comparable?  (tools/, measurement only)
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void nb_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void nb_arrive(int id, int n) { asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__global__ void probe(long long* out, int spin, int diverge) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int it = 0; it < 8; ++it) {
        if (warp == 31) {
            long long t = clock64();
            if (diverge) {
                if (lane == 0) while (clock64() - t < spin) {}
                __syncwarp();
            } else {
                while (clock64() - t < spin) {}
            }
            if (lane == 0) out[it * 4 + 0] = clock64();  // comm stamp
            nb_arrive(1, 1024);
        } else {
            if (warp == 0 && lane == 0) out[it * 4 + 1] = clock64();
            nb_sync(1, 1024);
            if (warp == 0 && lane == 0) out[it * 4 + 2] = clock64();  // passed
        }
        __syncthreads();
    }
}
int main() {
    long long* d; cudaMalloc(&d, 8 * 32 * 8);
    long long h[32];
    for (int dv = 0; dv < 2; ++dv) {
        probe<<<1, 1024>>>(d, 4000, dv);
        cudaMemcpy(h, d, 8 * 32, cudaMemcpyDeviceToHost);
        for (int it = 1; it < 8; ++it)
            printf("diverge=%d it=%d: comm_stamp - warp0_before = %lld, warp0_after - comm_stamp = %lld\n", dv, it,
                   h[it * 4 + 0] - h[it * 4 + 1], h[it * 4 + 2] - h[it * 4 + 0]);
    }
    return 0;
}
