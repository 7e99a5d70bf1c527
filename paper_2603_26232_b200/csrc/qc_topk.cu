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

#include <algorithm>
#include <cstdint>
#include <cstdlib>

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
__device__ __forceinline__ double norm_rn2(float2 a) {  // fp32 mode: exact products in double
    return norm_rn2(make_double2(a.x, a.y));
}

// class c -> key
template <typename V>
__device__ __forceinline__ Key class_key(const V* __restrict__ st, uint64_t c, int q, bool sym,
                                         bool fold) {
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
template <typename V>
__global__ void __launch_bounds__(kSortThreads) k_topk_state(const V* __restrict__ st, int q,
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
template <typename V>
__global__ void k_fill_keys(const V* __restrict__ st, int q, int sym, int fold,
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

// ---------------------------------------------------------------------------
// K <= 32 (every configuration of the paper: K in {1,2,4,8}): one pass over the classes,
// each thread keeping its best KT keys in registers (KT = K rounded up to a power of
// two), then KT rounds of block-wide argmax; stage 2 merges the CTAs' lists the same
// way. Keys are unique (bits are distinct), so the selection is exactly the reference's
// total order (qaoa.hpp:179-186).
// ---------------------------------------------------------------------------
constexpr int kSmallThreads = 256;

__device__ __forceinline__ bool kgt(uint64_t ap, uint32_t an, uint64_t bp, uint32_t bn) {
    return ap > bp || (ap == bp && an > bn);
}

template <int KT>
struct TopList {
    uint64_t p[KT];
    uint32_t n[KT];
    __device__ __forceinline__ void clear() {
#pragma unroll
        for (int i = 0; i < KT; ++i) {
            p[i] = 0;
            n[i] = 0;
        }
    }
    // insert (descending); keys with p == 0 && n == 0 are "empty"
    __device__ __forceinline__ void push(uint64_t xp, uint32_t xn) {
#pragma unroll
        for (int i = 0; i < KT; ++i) {
            const bool gt = kgt(xp, xn, p[i], n[i]);
            const uint64_t tp = p[i];
            const uint32_t tn = n[i];
            p[i] = gt ? xp : tp;
            n[i] = gt ? xn : tn;
            xp = gt ? tp : xp;
            xn = gt ? tn : xn;
        }
    }
    __device__ __forceinline__ void pop() {
#pragma unroll
        for (int i = 0; i + 1 < KT; ++i) {
            p[i] = p[i + 1];
            n[i] = n[i + 1];
        }
        p[KT - 1] = 0;
        n[KT - 1] = 0;
    }
};

// KT rounds of block argmax over the threads' list heads -> out[0..k)
template <int KT>
__device__ __forceinline__ void block_select(TopList<KT>& L, int k, Key* __restrict__ out) {
    __shared__ uint64_t wp[kSmallThreads / 32];
    __shared__ uint32_t wn[kSmallThreads / 32];
    __shared__ uint32_t wt[kSmallThreads / 32];
    __shared__ uint32_t win;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int r = 0; r < k; ++r) {
        uint64_t bp = L.p[0];
        uint32_t bn = L.n[0];
        uint32_t bt = threadIdx.x;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const uint64_t op = __shfl_xor_sync(0xffffffffu, bp, o);
            const uint32_t on = __shfl_xor_sync(0xffffffffu, bn, o);
            const uint32_t ot = __shfl_xor_sync(0xffffffffu, bt, o);
            if (kgt(op, on, bp, bn)) {
                bp = op;
                bn = on;
                bt = ot;
            }
        }
        if (lane == 0) {
            wp[warp] = bp;
            wn[warp] = bn;
            wt[warp] = bt;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            int b = 0;
            for (int w = 1; w < kSmallThreads / 32; ++w)
                if (kgt(wp[w], wn[w], wp[b], wn[b])) b = w;
            Key key;
            key.p = wp[b];
            key.nl = wn[b];
            key.pad = 0;
            out[r] = key;
            win = wt[b];
        }
        __syncthreads();
        if (threadIdx.x == win) L.pop();
    }
}

template <int KT, typename V>
__global__ void __launch_bounds__(kSmallThreads) k_topk_small_state(const V* __restrict__ st,
                                                                  int q, int sym, int fold,
                                                                  uint64_t classes, int k,
                                                                  Key* __restrict__ out) {
    TopList<KT> L;
    L.clear();
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * kSmallThreads;
    for (uint64_t c = static_cast<uint64_t>(blockIdx.x) * kSmallThreads + threadIdx.x; c < classes;
         c += stride) {
        const Key x = class_key(st, c, q, sym != 0, fold != 0);
        L.push(x.p, x.nl);
    }
    block_select<KT>(L, k, out + static_cast<size_t>(blockIdx.x) * k);
}

template <int KT>
__global__ void __launch_bounds__(kSmallThreads) k_topk_small_keys(const Key* __restrict__ in,
                                                                 uint64_t count, int k,
                                                                 Key* __restrict__ out) {
    TopList<KT> L;
    L.clear();
    for (uint64_t c = threadIdx.x; c < count; c += kSmallThreads) L.push(in[c].p, in[c].nl);
    block_select<KT>(L, k, out);
}

template <int KT, typename V>
int launch_small(const V* d_state, int q, bool sym, bool fold, uint64_t classes, int k,
                 Key* keys, cudaStream_t stream) {
    const int sms = device_sm_count();
    const uint64_t want = (classes + 8 * kSmallThreads - 1) / (8 * kSmallThreads);  // >= 8 per thread
    const unsigned grid = static_cast<unsigned>(std::max<uint64_t>(1, std::min<uint64_t>(want, 2u * sms)));
    Key* part = keys + 1024;  // stage-1 lists (grid * k keys), final list at keys[0..k)
    k_topk_small_state<KT, V><<<grid, kSmallThreads, 0, stream>>>(d_state, q, sym, fold, classes, k,
                                                              grid == 1 ? keys : part);
    if (grid > 1)
        k_topk_small_keys<KT><<<1, kSmallThreads, 0, stream>>>(part, static_cast<uint64_t>(grid) * k,
                                                              k, keys);
    return grid > 1 ? 2 : 1;
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
    if (k <= 32) return (1024 + 2 * 148 * 32 + 64) * sizeof(Key) + 4096 * sizeof(Key);
    if (k > kChunk / 2) return pow2_ceil(classes) * sizeof(Key);
    const uint64_t chunks = (classes + kChunk - 1) / kChunk;
    return 2 * chunks * static_cast<uint64_t>(k) * sizeof(Key) + sizeof(Key);
}

template <typename V>
int launch_topk_t(const V* d_state, int q, bool sym, bool fold, int k, void* d_scratch,
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
    if (k <= 32 && !std::getenv("QCG_TOPK_SORT")) {
        const int kk = static_cast<int>(std::min<uint64_t>(static_cast<uint64_t>(k), classes));
        if (k <= 1)
            launches = launch_small<1, V>(d_state, q, sym, fold, classes, kk, keys, stream);
        else if (k <= 2)
            launches = launch_small<2, V>(d_state, q, sym, fold, classes, kk, keys, stream);
        else if (k <= 4)
            launches = launch_small<4, V>(d_state, q, sym, fold, classes, kk, keys, stream);
        else if (k <= 8)
            launches = launch_small<8, V>(d_state, q, sym, fold, classes, kk, keys, stream);
        else if (k <= 16)
            launches = launch_small<16, V>(d_state, q, sym, fold, classes, kk, keys, stream);
        else
            launches = launch_small<32, V>(d_state, q, sym, fold, classes, kk, keys, stream);
        k_emit<<<1, 32, 0, stream>>>(keys, k, d_bits, d_probs);
        QC_CUDA(cudaGetLastError());
        return launches + 1;
    }
    if (k > kChunk / 2) {
        const uint64_t n = pow2_ceil(classes);
        k_fill_keys<V><<<static_cast<unsigned>((n + 255) / 256), 256, 0, stream>>>(
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
    k_topk_state<V><<<static_cast<unsigned>(chunks), kSortThreads, 0, stream>>>(
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

int launch_topk(const double2* d_state, int q, bool sym, bool fold, int k, void* d_scratch,
                uint32_t* d_bits, double* d_probs, cudaStream_t stream, Prof* prof, bool fp32) {
    if (fp32)
        return launch_topk_t(reinterpret_cast<const float2*>(d_state), q, sym, fold, k, d_scratch,
                             d_bits, d_probs, stream, prof);
    return launch_topk_t(d_state, q, sym, fold, k, d_scratch, d_bits, d_probs, stream, prof);
}

}  // namespace qcg
