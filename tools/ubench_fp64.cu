// Microbenchmark: FP64 dependent latency and throughput on the current GPU (B200).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench_fp64 tools/ubench_fp64.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void chain_dadd(double* out, long long* cyc, int n, double x) {
    double acc = 0.0;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) acc = __dadd_rn(acc, x);
    long long t1 = clock64();
    out[0] = acc;
    cyc[0] = t1 - t0;
}
__global__ void chain_dmul(double* out, long long* cyc, int n, double x) {
    double acc = 1.0;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) acc = __dmul_rn(acc, x);
    long long t1 = clock64();
    out[0] = acc;
    cyc[0] = t1 - t0;
}
__global__ void chain_fadd(float* out, long long* cyc, int n, float x) {
    float acc = 0.0f;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) acc = __fadd_rn(acc, x);
    long long t1 = clock64();
    out[0] = acc;
    cyc[0] = t1 - t0;
}
// 8 independent chains per thread: throughput
__global__ void tput_dadd(double* out, int n, double x) {
    double a[8] = {0, 1, 2, 3, 4, 5, 6, 7};
    for (int i = 0; i < n; ++i)
#pragma unroll
        for (int k = 0; k < 8; ++k) a[k] = __dadd_rn(a[k], x);
    double s = 0;
    for (int k = 0; k < 8; ++k) s += a[k];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void tput_dmul(double* out, int n, double x) {
    double a[8] = {1, 1, 2, 3, 4, 5, 6, 7};
    for (int i = 0; i < n; ++i)
#pragma unroll
        for (int k = 0; k < 8; ++k) a[k] = __dmul_rn(a[k], x);
    double s = 0;
    for (int k = 0; k < 8; ++k) s += a[k];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
// the mixer_pair pattern: 8 DMUL + 4 DADD per pair, 4 independent pairs per thread
__global__ void tput_rx(double* out, int n, double c, double s) {
    double2 a[8];
    for (int k = 0; k < 8; ++k) a[k] = make_double2(k * 0.1, 1.0 - k * 0.1);
    for (int i = 0; i < n; ++i)
#pragma unroll
        for (int k = 0; k < 8; k += 2) {
            const double2 t0 = a[k], t1 = a[k + 1];
            a[k].x = __dadd_rn(__dmul_rn(c, t0.x), __dmul_rn(s, t1.y));
            a[k].y = __dsub_rn(__dmul_rn(c, t0.y), __dmul_rn(s, t1.x));
            a[k + 1].x = __dadd_rn(__dmul_rn(s, t0.y), __dmul_rn(c, t1.x));
            a[k + 1].y = __dsub_rn(__dmul_rn(c, t1.y), __dmul_rn(s, t0.x));
        }
    double r = 0;
    for (int k = 0; k < 8; ++k) r += a[k].x + a[k].y;
    out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}

// pass-A-like register round: 16 amps/thread, RX on 4 local bits (ascending)
__global__ void __launch_bounds__(512, 1) tput_rx16(double* out, int n, double c, double s) {
    double2 a[16];
    for (int k = 0; k < 16; ++k) a[k] = make_double2(k * 0.1 + threadIdx.x, 1.0 - k * 0.1);
    for (int i = 0; i < n; ++i) {
#pragma unroll
        for (int b = 0; b < 4; ++b)
#pragma unroll
            for (int j = 0; j < 16; ++j)
                if (!(j & (1 << b))) {
                    double2& x0 = a[j];
                    double2& x1 = a[j | (1 << b)];
                    const double2 t0 = x0, t1 = x1;
                    x0.x = __dadd_rn(__dmul_rn(c, t0.x), __dmul_rn(s, t1.y));
                    x0.y = __dsub_rn(__dmul_rn(c, t0.y), __dmul_rn(s, t1.x));
                    x1.x = __dadd_rn(__dmul_rn(s, t0.y), __dmul_rn(c, t1.x));
                    x1.y = __dsub_rn(__dmul_rn(c, t1.y), __dmul_rn(s, t0.x));
                }
    }
    double r = 0;
    for (int k = 0; k < 16; ++k) r += a[k].x + a[k].y;
    out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}

int main() {
    double* d;
    float* f;
    long long* c;
    cudaMalloc(&d, 1 << 26);
    cudaMalloc(&f, 64);
    cudaMalloc(&c, 64);
    long long cyc;
    const int n = 1 << 16;
    chain_dadd<<<1, 1>>>(d, c, n, 1e-3);
    chain_dadd<<<1, 1>>>(d, c, n, 1e-3);
    cudaMemcpy(&cyc, c, 8, cudaMemcpyDeviceToHost);
    printf("dependent DADD latency: %.2f cycles\n", double(cyc) / n);
    chain_dmul<<<1, 1>>>(d, c, n, 1.0000001);
    cudaMemcpy(&cyc, c, 8, cudaMemcpyDeviceToHost);
    printf("dependent DMUL latency: %.2f cycles\n", double(cyc) / n);
    chain_fadd<<<1, 1>>>(f, c, n, 1e-3f);
    cudaMemcpy(&cyc, c, 8, cudaMemcpyDeviceToHost);
    printf("dependent FADD latency: %.2f cycles\n", double(cyc) / n);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int clk = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int it = 4096;
    tput_dadd<<<sms * 8, 256>>>(d, it, 1e-3);
    cudaEventRecord(e0);
    tput_dadd<<<sms * 8, 256>>>(d, it, 1e-3);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double ops = double(sms) * 8 * 256 * it * 8;
    printf("DADD throughput: %.2f Tops/s (%d SMs, clock %d MHz) = %.1f per SM per cycle at max clock\n",
           ops / ms / 1e9, sms, clk / 1000, ops / (ms * 1e-3) / sms / (clk * 1e3));
    tput_dmul<<<sms * 8, 256>>>(d, it, 1.0000001);
    cudaEventRecord(e0);
    tput_dmul<<<sms * 8, 256>>>(d, it, 1.0000001);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("DMUL throughput: %.2f Tops/s = %.1f per SM per cycle at max clock\n", ops / ms / 1e9,
           ops / (ms * 1e-3) / sms / (clk * 1e3));
    const int itr = 1024;
    tput_rx<<<sms * 8, 256>>>(d, itr, 0.6, 0.8);
    cudaEventRecord(e0);
    tput_rx<<<sms * 8, 256>>>(d, itr, 0.6, 0.8);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    const double ops_rx = double(sms) * 8 * 256 * itr * 4 * 12;
    printf("mixer_pair pattern (8 DMUL + 4 DADD): %.2f Tops/s = %.1f ops per SM per cycle; "
           "%.3g amp-targets/s\n", ops_rx / ms / 1e9, ops_rx / (ms * 1e-3) / sms / (clk * 1e3),
           ops_rx / 6 / (ms * 1e-3));
    for (int thr : {128, 256, 512}) {
        const int it16 = 256;
        tput_rx16<<<sms, thr>>>(d, it16, 0.6, 0.8);
        cudaEventRecord(e0);
        tput_rx16<<<sms, thr>>>(d, it16, 0.6, 0.8);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        const double o = double(sms) * thr * it16 * 4 * 8 * 12;
        printf("rx16 (16 amps/thread, 4 targets/round), %d threads/SM: %.2f Tops/s = %.1f ops/SM/clk\n",
               thr, o / ms / 1e9, o / (ms * 1e-3) / sms / (clk * 1e3));
    }
    return 0;
}
