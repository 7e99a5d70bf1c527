// Amplitude arithmetic shared by the statevector kernels (qc_pass.cu, qc_kernels.cu,
// qc_topk.cu). Device-only; include from .cu files.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace qcg {

// Kernel span trace (tool-only -DQCG_TRACE build, tools/trace_spans.py): every CTA group /
// warp leader appends {kind, block, sm | group << 16, entry ns, exit ns} (globaltimer). One
// buffer per translation unit (no -rdc), read by qc_span_read_<tu>.
#ifdef QCG_TRACE
struct SpanRec {
    uint32_t kind, block, smg, pad;
    unsigned long long t0, t1;
};
constexpr uint32_t kSpanCap = 1u << 20;
static __device__ SpanRec g_span[kSpanCap];
static __device__ unsigned int g_span_n;
__device__ __forceinline__ unsigned long long span_now() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ void span_end(uint32_t kind, uint32_t grp, unsigned long long t0) {
    const unsigned i = atomicAdd(&g_span_n, 1u);
    if (i < kSpanCap) {
        uint32_t smid;
        asm volatile("mov.u32 %0, %smid;" : "=r"(smid));
        g_span[i] = SpanRec{kind, blockIdx.x, smid | (grp << 16), 0u, t0, span_now()};
    }
}
#define QCG_SPAN_BEGIN() const unsigned long long qcg_span_t0_ = ::qcg::span_now()
#define QCG_SPAN_END(kind, grp, who)                                   \
    do {                                                               \
        if (who) ::qcg::span_end((kind), (grp), qcg_span_t0_);         \
    } while (0)
#define QCG_SPAN_READER(name)                                                                 \
    extern "C" int name(void* out, int cap, int* n) {                                         \
        unsigned cnt = 0;                                                                     \
        if (cudaMemcpyFromSymbol(&cnt, ::qcg::g_span_n, sizeof(cnt)) != cudaSuccess) return 4; \
        cnt = cnt < ::qcg::kSpanCap ? cnt : ::qcg::kSpanCap;                                  \
        const unsigned m = cnt < static_cast<unsigned>(cap) ? cnt : static_cast<unsigned>(cap); \
        if (m && cudaMemcpyFromSymbol(out, ::qcg::g_span, m * sizeof(::qcg::SpanRec)) != cudaSuccess) return 4; \
        *n = static_cast<int>(m);                                                             \
        const unsigned z = 0;                                                                 \
        cudaMemcpyToSymbol(::qcg::g_span_n, &z, sizeof(z));                                   \
        return 0;                                                                             \
    }
#else
#define QCG_SPAN_BEGIN() \
    do {                 \
    } while (0)
#define QCG_SPAN_END(kind, grp, who) \
    do {                             \
    } while (0)
#endif

__device__ __forceinline__ void cpa16(uint32_t s, const void* g) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(g) : "memory");
}

// Amplitude arithmetic. fp64 (the parity path): every product/sum explicitly rounded
// (__dmul_rn/__dadd_rn/__dsub_rn), no FMA, in statevector.hpp:176-180's order. fp32 (the
// optional 1e-4 mode): FMA-contracted single precision, 8-byte amplitudes.
template <typename V>
struct Amp;
template <>
struct Amp<double2> {
    using S = double;
    static constexpr uint32_t kBytes = 16, kSwMask = 7;
    __device__ static __forceinline__ double2 mk(double x, double y) { return make_double2(x, y); }
    __device__ static __forceinline__ double2 cmul(double2 a, double2 l) {
        // std::complex<double> *= : (ac - bd, ad + bc)
        return make_double2(__dsub_rn(__dmul_rn(a.x, l.x), __dmul_rn(a.y, l.y)),
                            __dadd_rn(__dmul_rn(a.x, l.y), __dmul_rn(a.y, l.x)));
    }
    // statevector.hpp:176-180 mixer_pair
    __device__ static __forceinline__ void rx(double2& a0, double2& a1, double c, double s) {
        const double2 t0 = a0, t1 = a1;
        a0.x = __dadd_rn(__dmul_rn(c, t0.x), __dmul_rn(s, t1.y));
        a0.y = __dsub_rn(__dmul_rn(c, t0.y), __dmul_rn(s, t1.x));
        a1.x = __dadd_rn(__dmul_rn(s, t0.y), __dmul_rn(c, t1.x));
        a1.y = __dsub_rn(__dmul_rn(c, t1.y), __dmul_rn(s, t0.x));
    }
    __device__ static __forceinline__ double nrm(double2 a) {  // std::norm
        return __dadd_rn(__dmul_rn(a.x, a.x), __dmul_rn(a.y, a.y));
    }
    __device__ static __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
    __device__ static __forceinline__ void cpa(uint32_t s, const void* g) { cpa16(s, g); }
};
template <>
struct Amp<float2> {
    using S = float;
    static constexpr uint32_t kBytes = 8, kSwMask = 15;
    __device__ static __forceinline__ float2 mk(float x, float y) { return make_float2(x, y); }
    __device__ static __forceinline__ float2 cmul(float2 a, float2 l) {
        return make_float2(fmaf(a.x, l.x, -a.y * l.y), fmaf(a.x, l.y, a.y * l.x));
    }
    __device__ static __forceinline__ void rx(float2& a0, float2& a1, float c, float s) {
        const float2 t0 = a0, t1 = a1;
        a0.x = fmaf(c, t0.x, s * t1.y);
        a0.y = fmaf(c, t0.y, -s * t1.x);
        a1.x = fmaf(s, t0.y, c * t1.x);
        a1.y = fmaf(c, t1.y, -s * t0.x);
    }
    __device__ static __forceinline__ float nrm(float2 a) { return fmaf(a.x, a.x, a.y * a.y); }
    __device__ static __forceinline__ float mul(float a, float b) { return a * b; }
    __device__ static __forceinline__ void cpa(uint32_t s, const void* g) {
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(g) : "memory");
    }
};
// conflict-free XOR swizzle (pass kernels) of the tile index for 16-byte (fp64) / 8-byte (fp32) amplitudes
template <typename V>
__device__ __forceinline__ uint32_t sw(uint32_t e) { return e ^ ((e >> 4) & Amp<V>::kSwMask); }

// fractional weights: std::polar(1, -gamma*val) (device sincos), out of line so the
// integral path keeps its registers
template <typename V>
__device__ __noinline__ V phase_frac(V v, double gamma, double val) {
    double sn, cs;
    sincos(__dmul_rn(-gamma, val), &sn, &cs);
    return Amp<V>::cmul(v, Amp<V>::mk(static_cast<typename Amp<V>::S>(cs),
                                      static_cast<typename Amp<V>::S>(sn)));
}

// RX on local bits [B0, B0+NB) of a[16] (ascending)
template <typename V, int B0, int NB>
__device__ __forceinline__ void rx_local(V (&a)[16], typename Amp<V>::S c, typename Amp<V>::S s) {
#pragma unroll
    for (int b = B0; b < B0 + NB; ++b) {
#pragma unroll
        for (int j = 0; j < 16; ++j)
            if (!(j & (1 << b))) Amp<V>::rx(a[j], a[j | (1 << b)], c, s);
    }
}

// Walsh–Hadamard mixer variant (fp32 mode only, F_WHT). statevector.hpp's
// mixer_pair is RX(β) = e^{-iβX} = cos β·I − i sin β·X, and X = H Z H, so on any set T of
// n register bits RX^{⊗T} = H^{⊗T} · diag_k(2^{-n} e^{-iβ(n − 2|k|)}) · H^{⊗T}, |k| the
// popcount of k on T, H the unnormalised (+,−) butterfly: two add/sub-only transforms and
// one complex scale per amplitude instead of n rotations. d[w] = 2^{-n} E^{n−2w} with
// E = e^{-iβ} = (c, −s).
__device__ __forceinline__ void wht_diag(float2 (&d)[5], int n, float c, float s) {
    const float2 E = make_float2(c, -s);
    const float2 up = make_float2(c * c - s * s, 2.f * c * s);  // E^{-2} = e^{2iβ}
    float2 x = make_float2(ldexpf(1.f, -n), 0.f);
#pragma unroll
    for (int i = 0; i < 4; ++i)
        if (i < n) x = Amp<float2>::cmul(x, E);
    d[0] = x;
#pragma unroll
    for (int w = 1; w < 5; ++w) d[w] = Amp<float2>::cmul(d[w - 1], up);
}
__device__ __forceinline__ void hbfly(float2& x, float2& y) {
    const float2 t = x;
    x = make_float2(t.x + y.x, t.y + y.y);
    y = make_float2(t.x - y.x, t.y - y.y);
}
// RX^{⊗T} on the register bits of `opmask` (bits < NB) of a[16]
template <int NB>
__device__ __forceinline__ void wht_local(float2 (&a)[16], uint32_t opmask, float c, float s) {
    float2 d[5];
    wht_diag(d, __popc(opmask), c, s);
#pragma unroll
    for (int b = 0; b < NB; ++b) {
        if (!(opmask & (1u << b))) continue;
#pragma unroll
        for (int j = 0; j < 16; ++j)
            if (!(j & (1 << b))) hbfly(a[j], a[j | (1 << b)]);
    }
#pragma unroll
    for (int j = 0; j < 16; ++j) {
        const int w = __popc(static_cast<uint32_t>(j) & opmask & ((1u << NB) - 1u));
        const float2 dj = w == 0 ? d[0] : w == 1 ? d[1] : w == 2 ? d[2] : w == 3 ? d[3] : d[4];
        a[j] = Amp<float2>::cmul(a[j], dj);
    }
#pragma unroll
    for (int b = 0; b < NB; ++b) {
        if (!(opmask & (1u << b))) continue;
#pragma unroll
        for (int j = 0; j < 16; ++j)
            if (!(j & (1 << b))) hbfly(a[j], a[j | (1 << b)]);
    }
}
// the 4-bit register round of the pass kernels: RX butterflies, or (fp32, F_WHT) the
// Walsh–Hadamard form
template <typename V>
__device__ __forceinline__ void mix4(V (&a)[16], typename Amp<V>::S c, typename Amp<V>::S s,
                                     bool wht) {
    if constexpr (sizeof(V) == 8) {
        if (wht) {
            wht_local<4>(a, 0xFu, c, s);
            return;
        }
    }
    rx_local<V, 0, 4>(a, c, s);
}


}  // namespace qcg
