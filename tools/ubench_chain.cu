// Microbenchmark: dependent DADD chain fed from shared memory (the k_blocksum pattern).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench_chain tools/ubench_chain.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void chain_lds(double* out, long long* cyc, int reps) {
    __shared__ double2 row[32 * 66];
    const int lane = threadIdx.x;
    for (int i = lane; i < 32 * 66; i += 32) row[i] = make_double2(1e-3 * i, 2e-3 * i);
    __syncwarp();
    const double2* r = row + lane * 65;
    double acc = 0.0;
    long long t0 = clock64();
    for (int rep = 0; rep < reps; ++rep) {
        double2 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) v[u] = r[u];
#pragma unroll
        for (int k = 0; k < 64; k += 4) {
            double2 nv[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) nv[u] = r[(k + 4 + u) & 63];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                acc = __dadd_rn(acc, v[u].x);
                acc = __dadd_rn(acc, v[u].y);
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) v[u] = nv[u];
        }
    }
    long long t1 = clock64();
    out[blockIdx.x * 32 + lane] = acc;
    if (lane == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void chain_reg(double* out, long long* cyc, int n) {
    const int lane = threadIdx.x;
    double a = 1e-3 * lane, acc = 0.0;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) acc = __dadd_rn(acc, a);
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
    const int reps = 64;  // 64 x 128 adds = 8192 adds
    for (int blocks : {1, 148}) {
        chain_lds<<<blocks, 32>>>(d, c, reps);
        chain_lds<<<blocks, 32>>>(d, c, reps);
        cudaDeviceSynchronize();
        cudaMemcpy(h, c, 8 * blocks, cudaMemcpyDeviceToHost);
        printf("LDS-fed chain, %3d warps (1/SM): %.2f cycles/add\n", blocks, double(h[0]) / (reps * 128));
        chain_reg<<<blocks, 32>>>(d, c, 8192);
        cudaDeviceSynchronize();
        cudaMemcpy(h, c, 8 * blocks, cudaMemcpyDeviceToHost);
        printf("register chain, %3d warps (1/SM): %.2f cycles/add\n", blocks, double(h[0]) / 8192);
    }
    return 0;
}
