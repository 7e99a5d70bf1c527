// Microbenchmark: the k_blocksum inner loop (128B-swizzled rows, 8 parts x 16 adds per
// 1 KB chunk per lane) with the data already in shared memory -- separates the add-chain
// cost from the TMA ring. nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false
#include <cstdio>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(32) loop_only(double* out, long long* cyc, int chunks, int desc) {
    __shared__ __align__(1024) unsigned char st[32 * 1024];
    const int lane = threadIdx.x;
    for (int i = lane; i < 32 * 1024 / 8; i += 32) reinterpret_cast<double*>(st)[i] = 1e-3 * (i & 255);
    __syncwarp();
    const unsigned sw = static_cast<unsigned>(lane & 7);
    double acc = 0.0;
    long long t0 = clock64();
    for (int c = 0; c < chunks; ++c) {
        if (!desc) {
#pragma unroll
            for (int p = 0; p < 8; ++p) {
                const double2* row = reinterpret_cast<const double2*>(st + (p * 32 + lane) * 128);
                double2 v[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) v[u] = row[u ^ sw];
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    acc = __dadd_rn(acc, v[u].x);
                    acc = __dadd_rn(acc, v[u].y);
                }
            }
        } else {
#pragma unroll
            for (int p = 7; p >= 0; --p) {
                const double2* row = reinterpret_cast<const double2*>(st + (p * 32 + lane) * 128);
                double2 v[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) v[u] = row[(7 - u) ^ sw];
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    acc = __dadd_rn(acc, v[u].y);
                    acc = __dadd_rn(acc, v[u].x);
                }
            }
        }
        __syncwarp();
    }
    long long t1 = clock64();
    out[blockIdx.x * 32 + lane] = acc;
    if (lane == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
    double* d;
    long long* c;
    cudaMalloc(&d, 1 << 20);
    cudaMalloc(&c, 1 << 16);
    long long h[256];
    for (int desc = 0; desc < 2; ++desc)
        for (int blocks : {1, 148, 296}) {
            loop_only<<<blocks, 32>>>(d, c, 32, desc);
            loop_only<<<blocks, 32>>>(d, c, 32, desc);
            cudaMemcpy(h, c, 8, cudaMemcpyDeviceToHost);
            printf("blocksum loop (%s), %3d warps: %.2f cycles/add\n", desc ? "desc" : "asc", blocks,
                   double(h[0]) / (32 * 128));
        }
    return 0;
}
