// Read-bandwidth microbenchmark: 1-D TMA bulk copies (cp.async.bulk, mbarrier ring) vs
// plain 16-byte vector loads, streaming a buffer larger than L2 with no compute. Tells
// whether the TMA read path has a per-SM ceiling below HBM bandwidth (k_blocksum question).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench_tma_read tools/ubench_tma_read.cu
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdint>

__device__ __forceinline__ unsigned su32(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}

// each warp-CTA streams its contiguous share in `chunk`-byte bulk copies, `stages` deep
__global__ void k_tma(const char* __restrict__ src, size_t bytes_per_cta, unsigned chunk, int stages,
                      double* sink) {
    extern __shared__ __align__(1024) unsigned char sm[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(sm + stages * chunk);
    const int lane = threadIdx.x;
    if (lane < stages) asm volatile("mbarrier.init.shared.b64 [%0], 1;\n" ::"r"(su32(bar + lane)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    __syncwarp();
    const char* base = src + blockIdx.x * bytes_per_cta;
    const int n = static_cast<int>(bytes_per_cta / chunk);
    auto issue = [&](int c) {
        if (c >= n || lane != 0) return;
        const int s = c % stages;
        asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;\n" ::"r"(su32(bar + s)), "r"(chunk) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                         su32(sm + s * chunk)),
                     "l"(base + static_cast<size_t>(c) * chunk), "r"(chunk), "r"(su32(bar + s))
                     : "memory");
    };
    for (int c = 0; c < stages - 1; ++c) issue(c);
    double acc = 0;
    for (int c = 0; c < n; ++c) {
        issue(c + stages - 1);
        const unsigned addr = su32(bar + c % stages), par = (c / stages) & 1;
        unsigned done = 0;
        while (!done)
            asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                         : "=r"(done)
                         : "r"(addr), "r"(par)
                         : "memory");
        acc += reinterpret_cast<const double*>(sm + (c % stages) * chunk)[lane];
        __syncwarp();
    }
    if (acc == 1.2345) *sink = acc;
}

__global__ void k_ldg(const uint4* __restrict__ src, size_t n16, double* sink) {
    uint32_t acc = 0;
    for (size_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += size_t(gridDim.x) * blockDim.x) {
        const uint4 v = __ldcs(src + i);
        acc ^= v.x ^ v.y ^ v.z ^ v.w;
    }
    if (acc == 0x12345678u) *sink = acc;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const size_t total = size_t{1} << 30;  // 1 GiB
    char* buf;
    double* sink;
    cudaMalloc(&buf, total);
    cudaMalloc(&sink, 8);
    cudaMemset(buf, 1, total);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    auto run_ldg = [&]() {
        k_ldg<<<sms * 4, 512>>>(reinterpret_cast<const uint4*>(buf), total / 16, sink);
        cudaEventRecord(a);
        for (int r = 0; r < 5; ++r) k_ldg<<<sms * 4, 512>>>(reinterpret_cast<const uint4*>(buf), total / 16, sink);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        printf("LDG.128 stream (4 x 512 threads per SM): %.0f GB/s\n", 5.0 * total / (ms * 1e-3) / 1e9);
    };
    run_ldg();
    const unsigned chunks[] = {8192, 32768};
    const int stage_list[] = {2, 3, 4, 6};
    const int per_sm_list[] = {1, 2, 4, 8};
    for (unsigned chunk : chunks)
        for (int stages : stage_list)
            for (int per_sm : per_sm_list) {
                const size_t smem = stages * chunk + 64;
                if (smem * per_sm > 220 * 1024) continue;
                cudaFuncSetAttribute(k_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
                const int ctas = sms * per_sm;
                size_t per = (total / ctas) / chunk * chunk;
                k_tma<<<ctas, 32, smem>>>(buf, per, chunk, stages, sink);
                cudaEventRecord(a);
                for (int r = 0; r < 5; ++r) k_tma<<<ctas, 32, smem>>>(buf, per, chunk, stages, sink);
                cudaEventRecord(b);
                cudaEventSynchronize(b);
                float ms = 0;
                cudaEventElapsedTime(&ms, a, b);
                const cudaError_t e = cudaGetLastError();
                printf("TMA bulk: chunk %5u B, %d stages, %d warp-CTAs/SM: %.0f GB/s%s\n", chunk, stages, per_sm,
                       5.0 * per * ctas / (ms * 1e-3) / 1e9, e == cudaSuccess ? "" : cudaGetErrorString(e));
            }
    return 0;
}
