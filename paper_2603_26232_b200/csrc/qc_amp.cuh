// Amplitude arithmetic shared by the statevector kernels (qc_pass.cu, qc_kernels.cu,
// qc_topk.cu). Device-only; include from .cu files.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace qcg {

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


}  // namespace qcg
