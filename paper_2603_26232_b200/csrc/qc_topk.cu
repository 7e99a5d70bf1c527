// Top-K measurement outcomes of one state (qaoa.hpp:158-193 top_candidates), sm_100a.
//
// Classes: folded -> even z with prob norm(a_z) + norm(a_{z^full}) (qaoa.hpp:169-173);
// unfolded -> every z with norm(a_z). In SYM storage (half state, a_{~z} == a_z bit for
// bit) stored index i is class i (i even) or class ~i (i odd), prob norm + norm.
// Order (qaoa.hpp:179-182): probability descending, then lex_less_mask ascending
// (graph.hpp:167-171), which is ascending bit-reversed z. Both fit one 96-bit key:
// (double bits of prob — monotone for p >= +0, ~brev(z)), maximised.
//
// Selection: CTAs bitonic-sort 2048-key chunks in shared memory and keep their top K;
// the survivors are re-chunked until one chunk remains. K > 1024 (every class of a
// large state) uses a global bitonic sort instead.
#include <cuda_runtime.h>

#include <cstdint>

#include "qc_internal.hpp"

namespace qcg {

namespace {

constexpr int kChunk = 2048;
constexpr int kSortThreads = 1024;

struct Key {
    uint64_t p;    // prob bits
    uint32_t nl;   // ~brev(bits)
    uint32_t pad;
};

__device__ __forceinline__ bool key_gt(const Key& a, const Key& b) {
    return a.p > b.p || (a.p == b.p && a.nl > b.nl);
}

__device__ __forceinline__ double norm_rn2(double2 a) {
    return __dadd_rn(__dmul_rn(a.x, a.x), __dmul_rn(a.y, a.y));
}

// class c -> key
__device__ __forceinline__ Key class_key(const double2* __restrict__ st, uint64_t c, int q,
                                         bool sym, bool fold) {
    const uint32_t full = (q == 32) ? ~0u : ((1u << q) - 1u);
    uint32_t bits;
    double prob;
    if (sym) {
        const uint32_t half = 1u << (q - 1);
        if (fold) {
            const uint32_t i = static_cast<uint32_t>(c);
            bits = (i & 1u) ? (full ^ i) : i;
            const double n = norm_rn2(st[i]);
            prob = __dadd_rn(n, n);
        } else {
            bits = static_cast<uint32_t>(c);
            const uint32_t i = bits < half ? bits : (full ^ bits);
            prob = norm_rn2(st[i]);
        }
    } else if (fold) {
        bits = static_cast<uint32_t>(c) << 1;
        prob = __dadd_rn(norm_rn2(st[bits]), norm_rn2(st[bits ^ full]));
    } else {
        bits = static_cast<uint32_t>(c);
        prob = norm_rn2(st[bits]);
    }
    Key k;
    k.p = static_cast<uint64_t>(__double_as_longlong(prob));
    k.nl = ~__brev(bits);
    k.pad = 0;
    return k;
}

// Sort a kChunk-key shared array descending (best first).
__device__ void bitonic_desc(Key* s) {
    for (int size = 2; size <= kChunk; size <<= 1) {
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            __syncthreads();
            for (int t = threadIdx.x; t < kChunk / 2; t += kSortThreads) {
                const int i = 2 * t - (t & (stride - 1));
                const int j = i + stride;
                const bool desc = ((i & size) == 0);
                const Key a = s[i], b = s[j];
                const bool swap = desc ? key_gt(b, a) : key_gt(a, b);
                if (swap) {
                    s[i] = b;
                    s[j] = a;
                }
            }
        }
    }
    __syncthreads();
}

// Stage 1: keys from the state, chunk top-k -> out (k per chunk).
__global__ void __launch_bounds__(kSortThreads) k_topk_state(const double2* __restrict__ st, int q,
                                                           int sym, int fold, uint64_t classes,
                                                           int k, Key* __restrict__ out) {
    __shared__ Key s[kChunk];
    const uint64_t base = static_cast<uint64_t>(blockIdx.x) * kChunk;
    for (int t = threadIdx.x; t < kChunk; t += kSortThreads) {
        const uint64_t c = base + t;
        if (c < classes) {
            s[t] = class_key(st, c, q, sym != 0, fold != 0);
        } else {
            s[t].p = 0;
            s[t].nl = 0;
            s[t].pad = 0;
        }
    }
    bitonic_desc(s);
    for (int t = threadIdx.x; t < k; t += kSortThreads) out[(size_t)blockIdx.x * k + t] = s[t];
}

// Stage 2: chunks of survivor keys -> chunk top-k.
__global__ void __launch_bounds__(kSortThreads) k_topk_keys(const Key* __restrict__ in,
                                                          uint64_t count, int k,
                                                          Key* __restrict__ out) {
    __shared__ Key s[kChunk];
    const uint64_t base = static_cast<uint64_t>(blockIdx.x) * kChunk;
    for (int t = threadIdx.x; t < kChunk; t += kSortThreads) {
        const uint64_t c = base + t;
        if (c < count) {
            s[t] = in[c];
        } else {
            s[t].p = 0;
            s[t].nl = 0;
            s[t].pad = 0;
        }
    }
    bitonic_desc(s);
    for (int t = threadIdx.x; t < k; t += kSortThreads) out[(size_t)blockIdx.x * k + t] = s[t];
}

// Global bitonic sort (descending) for K > kChunk/2.
__global__ void k_fill_keys(const double2* __restrict__ st, int q, int sym, int fold,
                            uint64_t classes, uint64_t padded, Key* __restrict__ keys) {
    const uint64_t c = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (c >= padded) return;
    if (c < classes) {
        keys[c] = class_key(st, c, q, sym != 0, fold != 0);
    } else {
        Key z;
        z.p = 0;
        z.nl = 0;
        z.pad = 0;
        keys[c] = z;
    }
}

__global__ void k_bitonic_step(Key* __restrict__ keys, uint64_t n, uint64_t size,
                               uint64_t stride) {
    const uint64_t t = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= n / 2) return;
    const uint64_t i = 2 * t - (t & (stride - 1));
    const uint64_t j = i + stride;
    const bool desc = ((i & size) == 0);
    const Key a = keys[i], b = keys[j];
    if (desc ? key_gt(b, a) : key_gt(a, b)) {
        keys[i] = b;
        keys[j] = a;
    }
}

__global__ void k_emit(const Key* __restrict__ keys, int k, uint32_t* __restrict__ bits,
                       double* __restrict__ probs) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= k) return;
    bits[t] = __brev(~keys[t].nl);
    probs[t] = __longlong_as_double(static_cast<long long>(keys[t].p));
}

uint64_t class_count(int q, bool fold) {
    return fold ? (uint64_t{1} << (q - 1)) : (uint64_t{1} << q);
}

uint64_t pow2_ceil(uint64_t x) {
    uint64_t p = 1;
    while (p < x) p <<= 1;
    return p;
}

}  // namespace

size_t topk_scratch_bytes(int q, bool fold, int k) {
    const uint64_t classes = class_count(q, fold);
    if (k > kChunk / 2) return pow2_ceil(classes) * sizeof(Key);
    const uint64_t chunks = (classes + kChunk - 1) / kChunk;
    return 2 * chunks * static_cast<uint64_t>(k) * sizeof(Key) + sizeof(Key);
}

int launch_topk(const double2* d_state, int q, bool sym, bool fold, int k, void* d_scratch,
                uint32_t* d_bits, double* d_probs, cudaStream_t stream, Prof* prof) {
    const uint64_t classes = class_count(q, fold);
    const double sbytes = static_cast<double>(sym ? (uint64_t{1} << (q - 1)) : (uint64_t{1} << q)) * 16.0;
    if (prof) prof->begin(K_TOPK, sbytes, stream);
    struct End {
        Prof* p;
        cudaStream_t s;
        ~End() {
            if (p) p->end(s);
        }
    } end_guard{prof, stream};
    Key* keys = static_cast<Key*>(d_scratch);
    int launches = 0;
    if (k > kChunk / 2) {
        const uint64_t n = pow2_ceil(classes);
        k_fill_keys<<<static_cast<unsigned>((n + 255) / 256), 256, 0, stream>>>(
            d_state, q, sym, fold, classes, n, keys);
        ++launches;
        for (uint64_t size = 2; size <= n; size <<= 1)
            for (uint64_t stride = size >> 1; stride > 0; stride >>= 1) {
                k_bitonic_step<<<static_cast<unsigned>((n / 2 + 255) / 256), 256, 0, stream>>>(
                    keys, n, size, stride);
                ++launches;
            }
        k_emit<<<(k + 255) / 256, 256, 0, stream>>>(keys, k, d_bits, d_probs);
        QC_CUDA(cudaGetLastError());
        return launches + 1;
    }
    uint64_t chunks = (classes + kChunk - 1) / kChunk;
    Key* a = keys;
    Key* b = keys + chunks * static_cast<uint64_t>(k);
    k_topk_state<<<static_cast<unsigned>(chunks), kSortThreads, 0, stream>>>(
        d_state, q, sym, fold, classes, k, a);
    ++launches;
    uint64_t count = chunks * static_cast<uint64_t>(k);
    if (classes < static_cast<uint64_t>(k)) count = classes;
    while (chunks > 1) {
        const uint64_t next = (count + kChunk - 1) / kChunk;
        k_topk_keys<<<static_cast<unsigned>(next), kSortThreads, 0, stream>>>(a, count, k, b);
        ++launches;
        count = next * static_cast<uint64_t>(k);
        chunks = next;
        Key* t = a;
        a = b;
        b = t;
    }
    k_emit<<<(k + 255) / 256, 256, 0, stream>>>(a, k, d_bits, d_probs);
    QC_CUDA(cudaGetLastError());
    return launches + 1;
}

}  // namespace qcg
