// Read-bandwidth microbenchmark: 1-D TMA bulk copies (cp.async.bulk, mbarrier ring) vs
// plain 16-byte vector loads, streaming a buffer larger than L2 with no compute. Tells
// whether the TMA read path has a per-SM ceiling below HBM bandwidth (k_blocksum question).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench_tma_read tools/ubench_tma_read.cu
#include <cuda.h>
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


// k_blocksum's access: per stage, 32 blocks (32 KB apart) x 1 KB each. (a) one 3-D tensor
// box {16 doubles, 32 blocks, 8 parts} with the 128-byte swizzle; (b) 32 per-lane 1-D bulk
// copies of 1 KB. Each warp-CTA walks its 32 blocks (a 1 MB region) chunk by chunk.
__global__ void k_box(const __grid_constant__ CUtensorMap tmap, int stages, int per_warp_groups, double* sink) {
    extern __shared__ __align__(1024) unsigned char sm[];
    constexpr unsigned kStage = 32768;
    uint64_t* bar = reinterpret_cast<uint64_t*>(sm + stages * kStage);
    const int lane = threadIdx.x;
    if (lane < stages) asm volatile("mbarrier.init.shared.b64 [%0], 1;\n" ::"r"(su32(bar + lane)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    __syncwarp();
    const int n = 32 * per_warp_groups;  // chunks: 32 per 32-block group
    auto issue = [&](int c) {
        if (c >= n || lane != 0) return;
        const int s = c % stages, grp = blockIdx.x * per_warp_groups + c / 32, part0 = (c % 32) * 8;
        asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;\n" ::"r"(su32(bar + s)), "r"(kStage) : "memory");
        asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes "
                     "[%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(su32(sm + s * kStage)),
                     "l"(reinterpret_cast<uint64_t>(&tmap)), "r"(0), "r"(grp * 32), "r"(part0), "r"(su32(bar + s))
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
                         : "=r"(done) : "r"(addr), "r"(par) : "memory");
        acc += reinterpret_cast<const double*>(sm + (c % stages) * kStage)[lane];
        __syncwarp();
    }
    if (acc == 1.2345) *sink = acc;
}

__global__ void k_lanes(const char* __restrict__ src, int stages, int per_warp_groups, double* sink) {
    extern __shared__ __align__(1024) unsigned char sm[];
    constexpr unsigned kStage = 32768;
    uint64_t* bar = reinterpret_cast<uint64_t*>(sm + stages * kStage);
    const int lane = threadIdx.x;
    if (lane < stages) asm volatile("mbarrier.init.shared.b64 [%0], 32;\n" ::"r"(su32(bar + lane)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    __syncwarp();
    const int n = 32 * per_warp_groups;
    auto issue = [&](int c) {
        if (c >= n) return;
        const int s = c % stages, grp = blockIdx.x * per_warp_groups + c / 32, part = c % 32;
        const char* g = src + (static_cast<size_t>(grp * 32 + lane) * 32768) + part * 1024;
        asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;\n" ::"r"(su32(bar + s)), "r"(1024) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 1024, [%2];\n" ::"r"(
                         su32(sm + s * kStage + lane * 1024)), "l"(g), "r"(su32(bar + s)) : "memory");
    };
    for (int c = 0; c < stages - 1; ++c) issue(c);
    double acc = 0;
    for (int c = 0; c < n; ++c) {
        __syncwarp();
        issue(c + stages - 1);
        const unsigned addr = su32(bar + c % stages), par = (c / stages) & 1;
        unsigned done = 0;
        while (!done)
            asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                         : "=r"(done) : "r"(addr), "r"(par) : "memory");
        acc += reinterpret_cast<const double*>(sm + (c % stages) * kStage)[lane];
    }
    if (acc == 1.2345) *sink = acc;
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
    // k_blocksum's access pattern: f as {16 doubles, blocks (32 KB stride), parts (128 B)}
    using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q{};
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    const uint64_t blocks = total / 32768;
    CUtensorMap tm;
    const cuuint64_t dims[3] = {16, blocks, 256};
    const cuuint64_t strides[2] = {32768, 128};
    const cuuint32_t box[3] = {16, 32, 8};
    const cuuint32_t es[3] = {1, 1, 1};
    reinterpret_cast<EncodeFn>(fn)(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, buf, dims, strides, box, es,
                                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                   CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    const int groups = static_cast<int>(blocks / 32);
    for (int stages : {2, 3, 6})
        for (int per_sm : {1, 2, 3}) {
            const size_t smem = stages * 32768 + 64;
            if (smem * per_sm > 220 * 1024) continue;
            const int ctas = sms * per_sm;
            const int pwg = groups / ctas;
            for (int kind = 0; kind < 2; ++kind) {
                if (kind == 0) {
                    cudaFuncSetAttribute(k_box, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
                    k_box<<<ctas, 32, smem>>>(tm, stages, pwg, sink);
                    cudaEventRecord(a);
                    for (int r = 0; r < 5; ++r) k_box<<<ctas, 32, smem>>>(tm, stages, pwg, sink);
                    cudaEventRecord(b);
                } else {
                    cudaFuncSetAttribute(k_lanes, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
                    k_lanes<<<ctas, 32, smem>>>(buf, stages, pwg, sink);
                    cudaEventRecord(a);
                    for (int r = 0; r < 5; ++r) k_lanes<<<ctas, 32, smem>>>(buf, stages, pwg, sink);
                    cudaEventRecord(b);
                }
                cudaEventSynchronize(b);
                float ms = 0;
                cudaEventElapsedTime(&ms, a, b);
                const cudaError_t e = cudaGetLastError();
                printf("blocksum pattern, %s: %d stages, %d warp-CTAs/SM: %.0f GB/s%s\n",
                       kind == 0 ? "3-D box {16,32,8}" : "32 x 1 KB per-lane bulk", stages, per_sm,
                       5.0 * 32768.0 * 32 * pwg * ctas / (ms * 1e-3) / 1e9, e == cudaSuccess ? "" : cudaGetErrorString(e));
            }
        }
    return 0;
}
