// Statevector kernels for the batched QAOA objective (qaoa.hpp:59-68 run_ansatz +
// statevector.hpp:224-235 expectation), sm_100a.
//
// Storage. A QAOA state of a Max-Cut instance is exactly complement-symmetric:
// C(z) = C(~z), |+> is symmetric and mixer_pair (statevector.hpp:176-180) maps a
// mirrored pair to a mirrored pair with the same floating-point operations (IEEE
// addition commutes). So a_{~z} == a_z bit for bit through every layer, and the
// engine stores only the half z < 2^(q-1) ("SYM" mode, Q = q-1 stored index bits).
// RX on qubit q-1 pairs z with z + 2^(q-1) = ~(~z mod 2^(q-1)), i.e. stored i with
// stored ~i: it becomes the "mirror" op rx(a_i, a_~i). FULL mode (Q = q) serves the
// API calls on arbitrary states (statevector.hpp lower-level functions).
//
// Exactness. Every product/sum is an explicitly rounded __dmul_rn/__dadd_rn/__dsub_rn
// (no FMA contraction, like the reference's -O3 x86-64 build), RX targets are applied
// in ascending order per amplitude (tiling only reorders independent pairs), the
// phase LUT is the host's std::polar table, and the expectation reproduces
// blocked_sum's association: sequential within 4096-blocks, partials in block order.
//
// Passes (Q > 12), one HBM round trip each:
//   pass A  (k_pass_low):  2^12 contiguous amps per CTA, [init |+>] + phase + RX 0..11
//   pass Bk (k_pass_high): 8 gather bits x 8-amp columns per CTA, RX on bits >= 12,
//                          mirror op last; the final one emits f(z)=|a|^2 C(z)
//   k_blocksum: the blocked sequential expectation over f (+ the in-order block sum).
// Q <= 12 (k_onchip): the whole state lives in one CTA's shared memory for all layers.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "qc_internal.hpp"

namespace qcg {

// ---------------------------------------------------------------------------
// exact fp64 building blocks
// ---------------------------------------------------------------------------
__device__ __forceinline__ double2 cmul_rn(double2 a, double2 l) {
    // std::complex<double> *= : (ac - bd, ad + bc)
    return make_double2(__dsub_rn(__dmul_rn(a.x, l.x), __dmul_rn(a.y, l.y)),
                        __dadd_rn(__dmul_rn(a.x, l.y), __dmul_rn(a.y, l.x)));
}

// statevector.hpp:176-180 mixer_pair
__device__ __forceinline__ void rx_rn(double2& a0, double2& a1, double c, double s) {
    const double2 t0 = a0, t1 = a1;
    a0.x = __dadd_rn(__dmul_rn(c, t0.x), __dmul_rn(s, t1.y));
    a0.y = __dsub_rn(__dmul_rn(c, t0.y), __dmul_rn(s, t1.x));
    a1.x = __dadd_rn(__dmul_rn(s, t0.y), __dmul_rn(c, t1.x));
    a1.y = __dsub_rn(__dmul_rn(c, t1.y), __dmul_rn(s, t0.x));
}

// std::norm = x*x + y*y
__device__ __forceinline__ double norm_rn(double2 a) {
    return __dadd_rn(__dmul_rn(a.x, a.x), __dmul_rn(a.y, a.y));
}

__device__ __forceinline__ double cost_of(const SlotDesc& S, uint32_t g) {
    if (S.lev) return static_cast<double>(S.lev[g]);
    return S.val ? S.val[g] : 1.0;  // unit cost: norm_sq (statevector.hpp:237-241)
}

// statevector.hpp:154-164: lut[lev] (integral) or std::polar(1, -gamma*val) (fractional)
__device__ __forceinline__ double2 phase_rn(double2 a, const SlotDesc& S, const LayerParam& L,
                                            uint32_t g) {
    if (S.lev) return cmul_rn(a, L.lut[S.lev[g]]);
    double sn, cs;
    sincos(__dmul_rn(-L.gamma, S.val[g]), &sn, &cs);
    return cmul_rn(a, make_double2(cs, sn));
}

__device__ __forceinline__ uint32_t deposit(uint32_t v, uint32_t mask) {
    uint32_t x = 0;
    while (mask) {
        const uint32_t low = mask & (~mask + 1u);
        if (v & 1u) x |= low;
        v >>= 1;
        mask &= mask - 1u;
    }
    return x;
}

// ---------------------------------------------------------------------------
// cut-level / cut-value tables (statevector.hpp:75-111), one entry per stored index
// ---------------------------------------------------------------------------
constexpr int kLevThreads = 256;
constexpr int kLevPerThread = 8;
constexpr int kEdgeChunk = 1024;

__global__ void __launch_bounds__(kLevThreads) k_levels(const uint32_t* __restrict__ eu,
                                                      const uint32_t* __restrict__ ev,
                                                      const double* __restrict__ ew, int m,
                                                      uint32_t N, int integral,
                                                      uint16_t* __restrict__ lev,
                                                      double* __restrict__ val) {
    __shared__ uint32_t su[kEdgeChunk], sv[kEdgeChunk];
    __shared__ double sw[kEdgeChunk];
    const uint32_t z0 = (blockIdx.x * kLevThreads) * kLevPerThread + threadIdx.x;
    uint32_t acc_i[kLevPerThread];
    double acc_d[kLevPerThread];
#pragma unroll
    for (int r = 0; r < kLevPerThread; ++r) {
        acc_i[r] = 0;
        acc_d[r] = 0.0;
    }
    for (int base = 0; base < m; base += kEdgeChunk) {
        const int cnt = min(kEdgeChunk, m - base);
        __syncthreads();
        for (int k = threadIdx.x; k < cnt; k += kLevThreads) {
            su[k] = eu[base + k];
            sv[k] = ev[base + k];
            sw[k] = ew[base + k];
        }
        __syncthreads();
#pragma unroll
        for (int r = 0; r < kLevPerThread; ++r) {
            const uint32_t z = z0 + r * kLevThreads;
            for (int k = 0; k < cnt; ++k) {
                const uint32_t cut = ((z >> su[k]) ^ (z >> sv[k])) & 1u;
                if (integral)
                    acc_i[r] += cut * static_cast<uint32_t>(sw[k]);
                else if (cut)
                    acc_d[r] = __dadd_rn(acc_d[r], sw[k]);  // values_[z] += e.w, edge order
            }
        }
    }
#pragma unroll
    for (int r = 0; r < kLevPerThread; ++r) {
        const uint32_t z = z0 + r * kLevThreads;
        if (z < N) {
            if (integral)
                lev[z] = static_cast<uint16_t>(acc_i[r]);
            else
                val[z] = acc_d[r];
        }
    }
}

int launch_levels(const uint32_t* d_eu, const uint32_t* d_ev, const double* d_ew, int m, int Q,
                  bool integral, uint16_t* d_lev, double* d_val, cudaStream_t stream) {
    const uint32_t N = 1u << Q;
    const uint32_t per_block = kLevThreads * kLevPerThread;
    const uint32_t blocks = (N + per_block - 1) / per_block;
    k_levels<<<blocks, kLevThreads, 0, stream>>>(d_eu, d_ev, d_ew, m, N, integral ? 1 : 0, d_lev,
                                                 d_val);
    QC_CUDA(cudaGetLastError());
    return 1;
}

// ---------------------------------------------------------------------------
// k_onchip: Q <= 12. One CTA per slot, whole stored state in shared memory.
// ---------------------------------------------------------------------------
constexpr int kOnchipThreads = 256;

__global__ void __launch_bounds__(kOnchipThreads) k_onchip(const SlotDesc* __restrict__ slots,
                                                         const LayerParam* __restrict__ lp,
                                                         int p, int Q, uint32_t flags,
                                                         double* __restrict__ out) {
    extern __shared__ double2 smem[];
    const uint32_t N = 1u << Q;
    double2* sa = smem;
    double* sf = reinterpret_cast<double*>(smem + N);
    const SlotDesc S = slots[blockIdx.x];
    const bool sym = flags & F_SYM;
    const uint32_t tid = threadIdx.x;

    for (uint32_t e = tid; e < N; e += kOnchipThreads)
        sa[e] = (flags & F_INIT) ? make_double2(S.amp0, 0.0) : S.state[e];

    for (int l = 0; l < p; ++l) {
        const LayerParam L = lp[S.layer_base + l];
        if (L.phase)
            for (uint32_t e = tid; e < N; e += kOnchipThreads) sa[e] = phase_rn(sa[e], S, L, e);
        __syncthreads();
        if (!L.mix) continue;
        for (int t = 0; t < Q; ++t) {
            const uint32_t half = 1u << t, lo = half - 1u;
            for (uint32_t k = tid; k < N / 2; k += kOnchipThreads) {
                const uint32_t i = ((k & ~lo) << 1) | (k & lo);
                rx_rn(sa[i], sa[i | half], L.c, L.s);
            }
            __syncthreads();
        }
        if (sym) {  // RX on qubit q-1: stored i pairs with stored ~i
            for (uint32_t k = tid; k < N / 2; k += kOnchipThreads)
                rx_rn(sa[k], sa[(N - 1u) ^ k], L.c, L.s);
            __syncthreads();
        }
    }

    if (flags & F_EXPECT) {
        for (uint32_t e = tid; e < N; e += kOnchipThreads)
            sf[e] = __dmul_rn(norm_rn(sa[e]), cost_of(S, e));
        __syncthreads();
        const int q = sym ? Q + 1 : Q;
        if (q <= 12) {
            // one block covering all 2^q basis states; the upper half mirrors the
            // stored half in descending order
            if (tid == 0) {
                double acc = 0.0;
                for (uint32_t e = 0; e < N; ++e) acc = __dadd_rn(acc, sf[e]);
                if (sym)
                    for (uint32_t e = N; e-- > 0;) acc = __dadd_rn(acc, sf[e]);
                out[blockIdx.x] = __dadd_rn(0.0, acc);
            }
        } else {  // sym, q == 13: blocks {stored ascending}, {stored descending}
            __shared__ double part[2];
            if (tid < 2) {
                double acc = 0.0;
                if (tid == 0)
                    for (uint32_t e = 0; e < N; ++e) acc = __dadd_rn(acc, sf[e]);
                else
                    for (uint32_t e = N; e-- > 0;) acc = __dadd_rn(acc, sf[e]);
                part[tid] = acc;
            }
            __syncthreads();
            if (tid == 0) out[blockIdx.x] = __dadd_rn(__dadd_rn(0.0, part[0]), part[1]);
        }
    }
    if (flags & F_STATE_OUT)
        for (uint32_t e = tid; e < N; e += kOnchipThreads) S.state[e] = sa[e];
}

// ---------------------------------------------------------------------------
// cp.async (LDGSTS) helpers: 16-byte global->shared copies that bypass registers, so a
// persistent CTA streams its next tile in while it computes the current one.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_wait1() { asm volatile("cp.async.wait_group 1;\n" ::: "memory"); }
__device__ __forceinline__ void bar_named(int id, int n) {
    asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(n) : "memory");
}

// ---------------------------------------------------------------------------
// k_pass_low: pass A, 4096 contiguous stored amplitudes per tile, targets 0..11.
// Persistent: one 256-thread CTA per SM walks tiles blockIdx.x, +gridDim.x, ...;
// tile k+1 (amplitudes + cut levels) is prefetched with cp.async into the other
// stage while tile k runs three register rounds of 4 targets (16 amps/thread)
// exchanged through an XOR-swizzled stage (conflict-free 16-byte accesses).
// ---------------------------------------------------------------------------
constexpr int kLowThreads = 256;
constexpr size_t kLowSmem = 2 * 4096 * sizeof(double2) + 2 * 4096 * sizeof(uint16_t);

__device__ __forceinline__ uint32_t swz(uint32_t e) { return e ^ ((e >> 4) & 7u); }

// Apply RX on the 4 thread-local bits (ascending) of a[16].
__device__ __forceinline__ void rx_local4(double2 (&a)[16], double c, double s) {
#pragma unroll
    for (int b = 0; b < 4; ++b) {
#pragma unroll
        for (int j = 0; j < 16; ++j)
            if (!(j & (1 << b))) rx_rn(a[j], a[j | (1 << b)], c, s);
    }
}

__global__ void __launch_bounds__(kLowThreads, 1) k_pass_low(const SlotDesc* __restrict__ slots,
                                                           const LayerParam* __restrict__ lp,
                                                           int layer, int Q, uint32_t flags,
                                                           uint32_t total_tiles) {
    extern __shared__ __align__(16) unsigned char smraw[];
    double2* buf = reinterpret_cast<double2*>(smraw);                       // [2][4096]
    uint16_t* levs = reinterpret_cast<uint16_t*>(smraw + 2 * 4096 * sizeof(double2));  // [2][4096]
    const int tshift = Q - 12;
    const uint32_t tmask = (1u << tshift) - 1u;
    const bool init = flags & F_INIT;
    const uint32_t tid = threadIdx.x;

    auto issue = [&](uint32_t t, int stage) {
        if (t < total_tiles) {
            const SlotDesc& S = slots[t >> tshift];
            const LayerParam& L = lp[S.layer_base + layer];
            if (init || L.phase || L.mix) {
                const uint32_t base = (t & tmask) << 12;
                if (!init) {
                    const double2* src = S.state + base;
                    double2* dst = buf + stage * 4096;
#pragma unroll
                    for (int k = 0; k < 16; ++k)
                        cp_async16(dst + swz(k * kLowThreads + tid), src + k * kLowThreads + tid);
                }
                if (L.phase && S.lev) {
                    const uint16_t* src = S.lev + base;
                    uint16_t* dst = levs + stage * 4096;
                    cp_async16(dst + tid * 8, src + tid * 8);
                    cp_async16(dst + (tid + 256) * 8, src + (tid + 256) * 8);
                }
            }
        }
        cp_commit();
    };

    uint32_t t = blockIdx.x;
    issue(t, 0);
    for (int k = 0; t < total_tiles; ++k, t += gridDim.x) {
        const int stage = k & 1;
        issue(t + gridDim.x, stage ^ 1);
        cp_wait1();
        __syncthreads();
        const SlotDesc S = slots[t >> tshift];
        const LayerParam L = lp[S.layer_base + layer];
        if (init || L.phase || L.mix) {  // else: identity layer, memory already holds it
            const uint32_t base = (t & tmask) << 12;
            double2* sm = buf + stage * 4096;
            const uint16_t* lv = levs + stage * 4096;
            double2 a[16];
            // round 0: bits 0..3 thread-local (e = tid*16 + j), phase first
#pragma unroll
            for (int j = 0; j < 16; ++j) {
                const uint32_t e = tid * 16u + j;
                double2 v = init ? make_double2(S.amp0, 0.0) : sm[swz(e)];
                if (L.phase) {
                    if (S.lev)
                        v = cmul_rn(v, L.lut[lv[e]]);
                    else
                        v = phase_rn(v, S, L, base + e);
                }
                a[j] = v;
            }
            if (L.mix) rx_local4(a, L.c, L.s);
#pragma unroll
            for (int j = 0; j < 16; ++j) sm[swz(tid * 16u + j)] = a[j];
            __syncthreads();
            // round 1: bits 4..7 (e = (tid>>4)<<8 | j<<4 | tid&15)
            const uint32_t r1 = ((tid >> 4) << 8) | (tid & 15u);
#pragma unroll
            for (int j = 0; j < 16; ++j) a[j] = sm[swz(r1 | (j << 4))];
            if (L.mix) rx_local4(a, L.c, L.s);
#pragma unroll
            for (int j = 0; j < 16; ++j) sm[swz(r1 | (j << 4))] = a[j];
            __syncthreads();
            // round 2: bits 8..11 (e = j<<8 | tid), stored straight back (coalesced)
#pragma unroll
            for (int j = 0; j < 16; ++j) a[j] = sm[swz((j << 8) | tid)];
            if (L.mix) rx_local4(a, L.c, L.s);
            double2* st = S.state + base;
#pragma unroll
            for (int j = 0; j < 16; ++j) st[(j << 8) | tid] = a[j];
        }
        __syncthreads();  // this stage is refilled by the next iteration's prefetch
    }
}

// ---------------------------------------------------------------------------
// k_pass_high: 3 column bits (8 contiguous amps) x 8 tile bits per tile.
// Tile bit kinds: 1 RX target (mask = one stored bit), 2 mirror (mask = all Q bits,
// RX on qubit q-1), 0 batch (no op). Targets precede the mirror in tile-bit order.
// In the mirror half of a tile (mirror bit set) every stored bit is complemented, so
// the RX roles (a0 = bit clear) of target pairs swap.
// Persistent: each 256-thread CTA runs two independent 128-thread tile streams
// (named barriers), each double-buffering its next tile's 128-byte column segments
// with cp.async.
// ---------------------------------------------------------------------------
constexpr int kHighThreads = 256;
constexpr size_t kHighSmem = 2 * 2 * 2048 * sizeof(double2);

template <int OFF>
__device__ __forceinline__ void high_round(double2 (&a)[16], const HighPass& hp, int mir_local,
                                           bool mir_thread, double c, double s) {
#pragma unroll
    for (int b = 0; b < 4; ++b) {
        const int kind = hp.kind[OFF + b];
        if (kind == 0) continue;
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            if (j & (1 << b)) continue;
            if (kind == 2) {
                rx_rn(a[j], a[j | (1 << b)], c, s);  // mirror: role order is immaterial
            } else {
                const bool mir = mir_thread ^ (mir_local >= 0 && ((j >> mir_local) & 1));
                if (mir)
                    rx_rn(a[j | (1 << b)], a[j], c, s);
                else
                    rx_rn(a[j], a[j | (1 << b)], c, s);
            }
        }
    }
}

__global__ void __launch_bounds__(kHighThreads, 1) k_pass_high(const SlotDesc* __restrict__ slots,
                                                             const LayerParam* __restrict__ lp,
                                                             int layer, int Q, HighPass hp,
                                                             uint32_t flags, uint32_t total_tiles) {
    extern __shared__ __align__(16) unsigned char smraw[];
    const int half = threadIdx.x >> 7;
    double2* hbuf = reinterpret_cast<double2*>(smraw) + half * 2 * 2048;  // [2][2048]
    const int tshift = Q - 11;
    const uint32_t tmask = (1u << tshift) - 1u;
    const bool fout = flags & F_EXPECT;
    const bool sout = !fout || (flags & F_STATE_OUT);
    const uint32_t ht = threadIdx.x & 127u;
    const uint32_t w = ht & 7u;
    const uint32_t hb = ht >> 3;  // round 0: tile bits 4..7; round 1: tile bits 0..3
    int mpos = -1;                // tile-bit index of the mirror pseudo-bit
#pragma unroll
    for (int k = 0; k < 8; ++k)
        if (hp.kind[k] == 2) mpos = k;
    // XOR of the thread's own tile-bit masks
    uint32_t thr_hi = 0, thr_lo = 0;
#pragma unroll
    for (int b = 0; b < 4; ++b) {
        if ((hb >> b) & 1u) thr_hi ^= hp.mask[4 + b];
        if ((hb >> b) & 1u) thr_lo ^= hp.mask[b];
    }
    const uint32_t streams = 2 * gridDim.x;

    auto issue = [&](uint32_t t, int stage) {
        if (t < total_tiles) {
            const SlotDesc& S = slots[t >> tshift];
            const LayerParam& L = lp[S.layer_base + layer];
            if (L.mix || fout) {
                const uint32_t gt = deposit(t & tmask, hp.freemask) | w;
                double2* dst = hbuf + stage * 2048;
#pragma unroll
                for (int j = 0; j < 16; ++j) {
                    uint32_t g = gt ^ thr_hi;
#pragma unroll
                    for (int b = 0; b < 4; ++b)
                        if ((j >> b) & 1) g ^= hp.mask[b];
                    cp_async16(dst + (w | (j << 3) | (hb << 7)), S.state + g);
                }
            }
        }
        cp_commit();
    };

    uint32_t t = blockIdx.x * 2 + half;
    issue(t, 0);
    for (int k = 0; t < total_tiles; ++k, t += streams) {
        const int stage = k & 1;
        issue(t + streams, stage ^ 1);
        cp_wait1();
        const SlotDesc S = slots[t >> tshift];
        const LayerParam L = lp[S.layer_base + layer];
        if (L.mix || fout) {
            const bool mix = L.mix;
            const uint32_t gt = deposit(t & tmask, hp.freemask) | w;
            double2* sm = hbuf + stage * 2048;
            double2 a[16];
            // round 0: tile bits 0..3 local; the thread reads exactly what it copied
            {
                const bool mir_t = mpos >= 4 && ((hb >> (mpos - 4)) & 1u);
#pragma unroll
                for (int j = 0; j < 16; ++j) a[j] = sm[w | (j << 3) | (hb << 7)];
                if (mix) high_round<0>(a, hp, mpos < 4 ? mpos : -1, mir_t, L.c, L.s);
#pragma unroll
                for (int j = 0; j < 16; ++j) sm[w | (j << 3) | (hb << 7)] = a[j];
            }
            bar_named(1 + half, 128);
            // round 1: tile bits 4..7 local; thread = (w, tile bits 0..3 = hb)
            {
                const bool mir_t = mpos >= 0 && mpos < 4 && ((hb >> mpos) & 1u);
#pragma unroll
                for (int j = 0; j < 16; ++j) a[j] = sm[w | (hb << 3) | (j << 7)];
                if (mix) high_round<4>(a, hp, mpos >= 4 ? mpos - 4 : -1, mir_t, L.c, L.s);
                const uint32_t g0 = gt ^ thr_lo;
#pragma unroll
                for (int j = 0; j < 16; ++j) {
                    uint32_t g = g0;
#pragma unroll
                    for (int b = 0; b < 4; ++b)
                        if ((j >> b) & 1) g ^= hp.mask[4 + b];
                    if (sout) S.state[g] = a[j];
                    if (fout) S.fbuf[g] = __dmul_rn(norm_rn(a[j]), cost_of(S, g));
                }
            }
        }
        bar_named(1 + half, 128);  // this stage is refilled by the next prefetch
    }
}

// ---------------------------------------------------------------------------
// blocked expectation over f (statevector.hpp:48-65). One warp per stored 4096-block:
// the warp streams the block through shared memory (coalesced 16-byte loads, double
// buffered) while lane 0 runs the ascending chain (the block itself) and, in SYM mode,
// lane 1 the descending chain (its mirror block in the upper half, 2nbl-1-b). Partials
// land in full-index block order; the last warp of a slot (atomic ticket) sums them in
// block order from 0.0 and writes the expectation.
// ---------------------------------------------------------------------------
constexpr int kSumWarps = 4;
constexpr int kSumChunk = 512;  // doubles per chunk

__global__ void __launch_bounds__(kSumWarps * 32) k_blocksum(const SlotDesc* __restrict__ slots,
                                                          int n_slots, int Q, int sym,
                                                          double* __restrict__ partials,
                                                          unsigned* __restrict__ tickets,
                                                          double* __restrict__ out) {
    extern __shared__ double sbuf[];  // [warp][2 stages][fwd, bwd][kSumChunk]
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nbl = 1 << (Q - 12);
    const int chains = sym ? 2 * nbl : nbl;
    const int gw = blockIdx.x * kSumWarps + warp;
    const int slot = gw / nbl;
    if (slot >= n_slots) return;
    const int b = gw - slot * nbl;
    const double2* f2 = reinterpret_cast<const double2*>(slots[slot].fbuf + (size_t)b * kBlock);
    double* wb = sbuf + (size_t)warp * 2 * 2 * kSumChunk;
    constexpr int kPer = kSumChunk / 2 / 32;  // double2 per lane per chunk
    constexpr int kChunks = kBlock / kSumChunk;
    double2 rf[kPer], rb[kPer];
    auto load = [&](int c) {
#pragma unroll
        for (int u = 0; u < kPer; ++u) rf[u] = f2[c * (kSumChunk / 2) + u * 32 + lane];
        if (sym)
#pragma unroll
            for (int u = 0; u < kPer; ++u) rb[u] = f2[(kChunks - 1 - c) * (kSumChunk / 2) + u * 32 + lane];
    };
    auto stash = [&](int stage) {
        double2* d = reinterpret_cast<double2*>(wb + stage * 2 * kSumChunk);
#pragma unroll
        for (int u = 0; u < kPer; ++u) d[u * 32 + lane] = rf[u];
        if (sym)
#pragma unroll
            for (int u = 0; u < kPer; ++u) d[kSumChunk / 2 + u * 32 + lane] = rb[u];
    };
    load(0);
    stash(0);
    __syncwarp();
    double acc = 0.0;
    for (int c = 0; c < kChunks; ++c) {
        if (c + 1 < kChunks) load(c + 1);  // in flight while the chains run
        const double* cur = wb + (c & 1) * 2 * kSumChunk;
        if (lane == 0) {
#pragma unroll 16
            for (int k = 0; k < kSumChunk; ++k) acc = __dadd_rn(acc, cur[k]);
        } else if (lane == 1 && sym) {
#pragma unroll 16
            for (int k = kSumChunk - 1; k >= 0; --k) acc = __dadd_rn(acc, cur[kSumChunk + k]);
        }
        __syncwarp();
        if (c + 1 < kChunks) stash((c + 1) & 1);
        __syncwarp();
    }
    double* pp = partials + (size_t)slot * chains;
    if (lane == 0) pp[b] = acc;
    if (lane == 1 && sym) pp[2 * nbl - 1 - b] = acc;
    __syncwarp();
    if (lane == 0) {
        __threadfence();
        const unsigned ticket = atomicAdd(&tickets[slot], 1u);
        if (ticket == static_cast<unsigned>(nbl - 1)) {  // last block of this slot
            __threadfence();
            double total = 0.0;
            for (int k = 0; k < chains; ++k) total = __dadd_rn(total, __ldcg(pp + k));
            out[slot] = total;
            tickets[slot] = 0u;
        }
    }
}

// ---------------------------------------------------------------------------
// host-side planning + launch
// ---------------------------------------------------------------------------
ChainPlan plan_chain(int q, bool sym) {
    ChainPlan plan;
    plan.sym = sym;
    plan.Q = sym ? q - 1 : q;
    plan.onchip = plan.Q <= 12;
    if (plan.onchip) return plan;
    const int Q = plan.Q;
    std::vector<int> items;  // stored-bit targets, -1 = mirror
    for (int b = 12; b < Q; ++b) items.push_back(b);
    if (sym) items.push_back(-1);
    const uint32_t all = (Q == 32) ? ~0u : ((1u << Q) - 1u);
    for (size_t i = 0; i < items.size(); i += 8) {
        HighPass hp{};
        uint32_t single = 0x7u;  // column bits 0..2
        bool mirror = false;
        int k = 0;
        for (; k < 8 && i + k < items.size(); ++k) {
            const int it = items[i + k];
            if (it < 0) {
                hp.mask[k] = all;
                hp.kind[k] = 2;
                mirror = true;
            } else {
                hp.mask[k] = 1u << it;
                hp.kind[k] = 1;
                single |= 1u << it;
            }
        }
        for (int pad = 3; k < 8; ++pad) {  // batch bits: widen the contiguous columns
            hp.mask[k] = 1u << pad;
            hp.kind[k] = 0;
            single |= 1u << pad;
            ++k;
        }
        uint32_t freem = all & ~single;
        if (mirror) {  // one representative per {x, ~x}: pin the highest free bit to 0
            int top = 31;
            while (top >= 0 && !((freem >> top) & 1u)) --top;
            freem &= ~(1u << top);
        }
        hp.freemask = freem;
        plan.high.push_back(hp);
    }
    return plan;
}

size_t partials_per_slot(const ChainPlan& plan) {
    if (plan.onchip) return 0;
    const size_t nbl = size_t{1} << (plan.Q - 12);
    return plan.sym ? 2 * nbl : nbl;
}

int launch_chain(const ChainPlan& plan, const SlotDesc* d_slots, const LayerParam* d_lp,
                 int n_slots, int p, uint32_t flags, double* d_partials, unsigned* d_tickets,
                 double* d_out, cudaStream_t stream, const ChainStats* stats, Prof* prof) {
    if (n_slots <= 0) return 0;
    const int Q = plan.Q;
    const double N = static_cast<double>(size_t{1} << Q);
    const uint32_t symf = plan.sym ? F_SYM : 0u;
    auto cnt = [&](const std::vector<int>* v, int l) {
        return (stats && v && l < static_cast<int>(v->size())) ? (*v)[static_cast<size_t>(l)] : n_slots;
    };
    if (plan.onchip) {
        const size_t Ns = size_t{1} << Q;
        const size_t smem = Ns * sizeof(double2) + ((flags & F_EXPECT) ? Ns * sizeof(double) : 0);
        static bool attr_done = false;
        if (!attr_done) {
            QC_CUDA(cudaFuncSetAttribute(k_onchip, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (1 << 12) * 24));
            attr_done = true;
        }
        const double b = n_slots * N * (((flags & F_INIT) ? 0.0 : 16.0) + ((flags & F_STATE_OUT) ? 16.0 : 0.0));
        if (prof) prof->begin(K_ONCHIP, b, stream);
        k_onchip<<<n_slots, kOnchipThreads, smem, stream>>>(d_slots, d_lp, p, Q, flags | symf,
                                                            d_out);
        if (prof) prof->end(stream);
        QC_CUDA(cudaGetLastError());
        return 1;
    }
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        QC_CUDA(cudaGetDevice(&dev));
        QC_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        QC_CUDA(cudaFuncSetAttribute(k_pass_low, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(kLowSmem)));
        QC_CUDA(cudaFuncSetAttribute(k_pass_high, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(kHighSmem)));
    }
    int launches = 0;
    const uint32_t low_tiles = static_cast<uint32_t>(n_slots) << (Q - 12);
    const uint32_t high_tiles = static_cast<uint32_t>(n_slots) << (Q - 11);
    const unsigned low_grid = std::min<uint32_t>(low_tiles, static_cast<uint32_t>(sms));
    const unsigned high_grid = std::min<uint32_t>((high_tiles + 1) / 2, static_cast<uint32_t>(sms));
    for (int l = 0; l < p; ++l) {
        const uint32_t fa = (l == 0 && (flags & F_INIT)) ? F_INIT : 0u;
        const int nph = cnt(stats ? &stats->phase : nullptr, l);
        const int nmix = cnt(stats ? &stats->mix : nullptr, l);
        // pass A moves a slot if it initialises, phases or mixes it; levels read when phased
        const int active = fa ? n_slots : std::max(nph, nmix);
        const double ba = (fa ? n_slots * 16.0 : active * 32.0) * N + nph * 2.0 * N;
        if (prof) prof->begin(K_PASS_LOW, ba, stream);
        k_pass_low<<<low_grid, kLowThreads, kLowSmem, stream>>>(d_slots, d_lp, l, Q, fa, low_tiles);
        if (prof) prof->end(stream);
        ++launches;
        for (size_t h = 0; h < plan.high.size(); ++h) {
            const bool last = (l == p - 1) && (h + 1 == plan.high.size());
            uint32_t fh = 0;
            if (last && (flags & F_EXPECT)) fh |= F_EXPECT;
            if (last && (flags & F_STATE_OUT)) fh |= F_STATE_OUT;
            double bh;
            if (fh & F_EXPECT)  // read state, write f (+ state), read levels
                bh = n_slots * N * (16.0 + 8.0 + 2.0 + ((fh & F_STATE_OUT) ? 16.0 : 0.0));
            else
                bh = nmix * 32.0 * N;
            if (prof) prof->begin(K_PASS_HIGH, bh, stream);
            k_pass_high<<<high_grid, kHighThreads, kHighSmem, stream>>>(d_slots, d_lp, l, Q,
                                                                        plan.high[h], fh,
                                                                        high_tiles);
            if (prof) prof->end(stream);
            ++launches;
        }
    }
    QC_CUDA(cudaGetLastError());
    if (flags & F_EXPECT) {
        const int nbl = 1 << (Q - 12);
        const int warps = nbl * n_slots;
        const size_t smem = static_cast<size_t>(kSumWarps) * 2 * 2 * kSumChunk * sizeof(double);
        static bool sum_attr = false;
        if (!sum_attr) {
            QC_CUDA(cudaFuncSetAttribute(k_blocksum, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem)));
            sum_attr = true;
        }
        if (prof) prof->begin(K_BLOCKSUM, n_slots * N * 8.0, stream);
        k_blocksum<<<(warps + kSumWarps - 1) / kSumWarps, kSumWarps * 32, smem, stream>>>(
            d_slots, n_slots, Q, plan.sym ? 1 : 0, d_partials, d_tickets, d_out);
        if (prof) prof->end(stream);
        launches += 1;
        QC_CUDA(cudaGetLastError());
    }
    return launches;
}

}  // namespace qcg
