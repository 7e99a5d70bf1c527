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
// Passes (Q > 12), one HBM round trip each (qc_pass.cu):
//   pass A:  2^12 contiguous amps per tile, [init |+>] + phase + RX 0..11
//   pass B:  9 gather bits x 8-amp columns per tile, RX on bits >= 12, mirror op last;
//            the final one emits f(z)=|a|^2 C(z)
//   k_blocksum: the blocked sequential expectation over f (+ the in-order block sum).
// Q <= 12 (k_onchip): the whole state lives in one CTA's shared memory for all layers.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <string>
#include <cstdint>

#include "qc_amp.cuh"
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
    if (S.plev) return cmul_rn(a, L.lut[S.plev[g]]);
    double sn, cs;
    sincos(__dmul_rn(-L.gamma, S.val[g]), &sn, &cs);
    return cmul_rn(a, make_double2(cs, sn));
}

__device__ __forceinline__ unsigned smem_u32_any(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
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
    QCG_SPAN_BEGIN();
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
    QCG_SPAN_END(6, 0, threadIdx.x == 0);
}

// ---------------------------------------------------------------------------
// Optional fp32 mode (F_FP32, 1e-4): float2 amplitudes, float f(z). Same schedule as the
// fp64 kernels (phase, RX targets ascending, mirror last); sums accumulate in double.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kOnchipThreads) k_onchip_f32(const SlotDesc* __restrict__ slots,
                                                             const LayerParam* __restrict__ lp,
                                                             int p, int Q, uint32_t flags,
                                                             double* __restrict__ out) {
    extern __shared__ float2 smemf[];
    using A = Amp<float2>;
    const uint32_t N = 1u << Q;
    float2* sa = smemf;
    __shared__ double red[kOnchipThreads / 32];
    __shared__ float2 dtab[16];  // F_WHT: diagonal by popcount
    const SlotDesc S = slots[blockIdx.x];
    float2* gst = reinterpret_cast<float2*>(S.state);
    const bool sym = flags & F_SYM;
    const uint32_t tid = threadIdx.x;
    for (uint32_t e = tid; e < N; e += kOnchipThreads)
        sa[e] = (flags & F_INIT) ? make_float2(static_cast<float>(S.amp0), 0.f) : gst[e];
    for (int l = 0; l < p; ++l) {
        const LayerParam L = lp[S.layer_base + l];
        const float c = static_cast<float>(L.c), sn = static_cast<float>(L.s);
        if (L.phase) {
            const float2* lut = reinterpret_cast<const float2*>(L.lut);
            for (uint32_t e = tid; e < N; e += kOnchipThreads) {
                if (S.plev) {
                    sa[e] = A::cmul(sa[e], lut[S.plev[e]]);
                } else {
                    double s_, c_;
                    sincos(-L.gamma * S.val[e], &s_, &c_);
                    sa[e] = A::cmul(sa[e], make_float2(static_cast<float>(c_), static_cast<float>(s_)));
                }
            }
        }
        __syncthreads();
        if (!L.mix) continue;
        if (flags & F_WHT) {
            // Walsh–Hadamard form over the whole stored state (qc_amp.cuh wht_local): the RX
            // layer on the Q stored bits and the mirror op (cI - isP, P = the complement = X
            // on every stored bit, eigenvalue (-1)^|k|) are diagonal after H^{(x)Q}:
            // d(|k| = w) = 2^-Q E^{Q - 2w + (sym ? (-1)^w : 0)}, E = e^{-iβ} = (c, -s)
            if (tid <= static_cast<uint32_t>(Q)) {
                const int w = static_cast<int>(tid);
                const int m = Q - 2 * w + (sym ? ((w & 1) ? -1 : 1) : 0);
                double xr = 1.0, xi = 0.0;
                const double er = L.c, ei = m >= 0 ? -L.s : L.s;
                for (int i = 0; i < (m >= 0 ? m : -m); ++i) {
                    const double t = xr * er - xi * ei;
                    xi = xr * ei + xi * er;
                    xr = t;
                }
                const double sc = ldexp(1.0, -Q);
                dtab[w] = make_float2(static_cast<float>(xr * sc), static_cast<float>(xi * sc));
            }
            for (int pass = 0; pass < 2; ++pass) {
                for (int t = 0; t < Q; ++t) {
                    const uint32_t half = 1u << t, lo = half - 1u;
                    for (uint32_t k = tid; k < N / 2; k += kOnchipThreads) {
                        const uint32_t i = ((k & ~lo) << 1) | (k & lo);
                        hbfly(sa[i], sa[i | half]);
                    }
                    __syncthreads();
                }
                if (pass == 0) {
                    for (uint32_t k = tid; k < N; k += kOnchipThreads) sa[k] = A::cmul(sa[k], dtab[__popc(k)]);
                    __syncthreads();
                }
            }
            continue;
        }
        for (int t = 0; t < Q; ++t) {
            const uint32_t half = 1u << t, lo = half - 1u;
            for (uint32_t k = tid; k < N / 2; k += kOnchipThreads) {
                const uint32_t i = ((k & ~lo) << 1) | (k & lo);
                A::rx(sa[i], sa[i | half], c, sn);
            }
            __syncthreads();
        }
        if (sym) {
            for (uint32_t k = tid; k < N / 2; k += kOnchipThreads) A::rx(sa[k], sa[(N - 1u) ^ k], c, sn);
            __syncthreads();
        }
    }
    if (flags & F_EXPECT) {
        double acc = 0.0;
        for (uint32_t e = tid; e < N; e += kOnchipThreads) {
            const double cst = S.lev ? static_cast<double>(S.lev[e]) : (S.val ? S.val[e] : 1.0);
            acc += static_cast<double>(A::nrm(sa[e])) * cst;
        }
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if ((tid & 31) == 0) red[tid >> 5] = acc;
        __syncthreads();
        if (tid == 0) {
            double t = 0.0;
            for (int w = 0; w < kOnchipThreads / 32; ++w) t += red[w];
            out[blockIdx.x] = sym ? 2.0 * t : t;
        }
    }
    if (flags & F_STATE_OUT)
        for (uint32_t e = tid; e < N; e += kOnchipThreads) gst[e] = sa[e];
}

// fp32 expectation: one CTA per stored 4096-block sums float f in double; the last CTA of
// a slot adds the partials in block order (x2 for the mirror half in SYM storage).
constexpr int kFsumThreads = 256;
__global__ void __launch_bounds__(kFsumThreads) k_fsum_f32(const float* __restrict__ f, int Q, int sym,
                                                         double* __restrict__ partials,
                                                         unsigned* __restrict__ tickets,
                                                         double* __restrict__ out) {
    __shared__ double red[kFsumThreads / 32];
    const int nbl = 1 << (Q - 12);
    const int slot = blockIdx.x / nbl, b = blockIdx.x % nbl;
    const float4* src = reinterpret_cast<const float4*>(f + (static_cast<size_t>(slot) << Q) +
                                                        static_cast<size_t>(b) * kBlock);
    double acc = 0.0;
    for (int i = threadIdx.x; i < kBlock / 4; i += kFsumThreads) {
        const float4 v = __ldcg(src + i);
        acc += (static_cast<double>(v.x) + v.y) + (static_cast<double>(v.z) + v.w);
    }
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
    __syncthreads();
    __shared__ unsigned last;
    double* pp = partials + static_cast<size_t>(slot) * nbl;
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < kFsumThreads / 32; ++w) t += red[w];
        pp[b] = t;
        __threadfence();
        last = atomicAdd(&tickets[slot], 1u) == static_cast<unsigned>(nbl - 1);
    }
    __syncthreads();
    if (!last) return;
    // the slot's last CTA: every thread adds a strided share of the partials (fp32 mode
    // has no summation-order contract; up to 2^14 partials at 26 qubits)
    __threadfence();
    double t = 0.0;
    for (int k = threadIdx.x; k < nbl; k += kFsumThreads) t += __ldcg(pp + k);
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    __syncthreads();  // red[] reuse
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = t;
    __syncthreads();
    if (threadIdx.x == 0) {
        double total = 0.0;
        for (int w = 0; w < kFsumThreads / 32; ++w) total += red[w];
        out[slot] = sym ? 2.0 * total : total;
        tickets[slot] = 0u;
    }
}


// ---------------------------------------------------------------------------
// blocked expectation over f (statevector.hpp:48-65). Every 4096-block partial is a
// chain of 4096 dependent adds (8.3-cycle DADD latency on B200 => >= 17 us), so the
// kernel maximises concurrent chains: each LANE owns one chain. A warp covers up to 32
// stored blocks in one direction: ascending warps produce the blocks' own partials,
// descending warps (SYM) those of the mirror blocks 2nbl-1-b in the upper half. Each
// lane's next 1 KB chunk arrives by a TMA bulk copy (cp.async.bulk, mbarrier ring of 3
// stages) into its own shared-memory row. Partials land in full-index block order; the last warp of a slot (atomic
// ticket) sums them in block order from 0.0 and writes the expectation.
// ---------------------------------------------------------------------------
// a stage holds kParts 16-double parts (128 B each) of each lane's chain: 4 KB per part
template <int kParts>
__host__ __device__ constexpr size_t sum_stage_bytes() { return size_t{32} * 16 * kParts * sizeof(double); }
// stages in flight: 3 lets two warp-CTAs share an SM (launches of more warps than SMs);
// a launch that fits one warp per SM uses 6 (each 32 KB tensor copy takes ~1 us in the
// SM's TMA unit, so deeper lookahead hides it)
// W warps per CTA (each with its own ring and chains, exactly one 1-warp CTA's work)
template <int STAGES, int PARTS, int W = 1>
constexpr size_t sum_smem() { return W * (STAGES * sum_stage_bytes<PARTS>() + STAGES * 8) + 1024; }

__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}

// tmap: the f buffer of the launch as a 3-D tensor {16 doubles, block (32 KB stride),
// part (128 B stride)}, box {16, 32, kSumParts}, 128-byte swizzle: the shared box is
// [part][block][16 doubles] and 16-byte unit u of row r sits at unit u ^ (r & 7), so the
// 32 lanes (one block each) read one part conflict-free.
template <int kSumStages, int kSumParts, int kW = 1>
__global__ void __launch_bounds__(32 * kW) k_blocksum(const __grid_constant__ CUtensorMap tmap,
                                                int n_slots, int Q, int sym, int mode,
                                                double* __restrict__ partials,
                                                unsigned* __restrict__ tickets,
                                                double* __restrict__ out) {
    QCG_SPAN_BEGIN();
    constexpr int kSumChunk = 16 * kSumParts;  // doubles per chunk per chain
    constexpr size_t kSumStageBytes = sum_stage_bytes<kSumParts>();
    extern __shared__ unsigned char sraw[];
    // 1024-byte aligned base by pointer arithmetic, so the compiler keeps the shared
    // address space (LDS instead of generic LD on the chain's operand path)
    unsigned char* const abase = sraw + ((1024u - (smem_u32(sraw) & 1023u)) & 1023u);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int vb = blockIdx.x * kW + wid;            // this warp's work unit
    unsigned char* sbase = abase + wid * (kSumStages * kSumStageBytes);
    uint64_t* mbar = reinterpret_cast<uint64_t*>(abase + kW * kSumStages * kSumStageBytes) + wid * kSumStages;
    const int nbl = 1 << (Q - 12);                   // stored blocks per slot
    const int chains = sym ? 2 * nbl : nbl;
    // direction-uniform warps: each covers up to 32 stored blocks in ONE direction (SYM:
    // ascending warps then descending warps), so every lane of a warp runs the same code
    const int bpw = min(32, nbl);                    // blocks per warp
    const int wpd = nbl / bpw;                       // warps per direction per slot
    const int wps = sym ? 2 * wpd : wpd;             // warps per slot
    const int slot = vb / wps;
    if (slot >= n_slots) return;
    const int wis = vb - slot * wps;
    // SYM: the ascending and the descending warp of a block group are adjacent CTAs, so
    // they run together and the second read of each stored block can hit L2 (at 24+ qubits
    // f does not fit in L2 and the sum is bound by its read stream)
    const bool pair_dirs = mode & 1;
    const bool desc = sym && pair_dirs ? (wis & 1) : wis >= wpd;
    const int grp = sym && pair_dirs ? (wis >> 1) : (desc ? wis - wpd : wis);
    const int b0 = grp * bpw;                         // first block (within the slot)
    const int gb0 = slot * nbl + b0;                 // first block (tensor coordinate)
    constexpr int kChunks = kBlock / kSumChunk;
    if (lane < kSumStages)
        asm volatile("mbarrier.init.shared.b64 [%0], 1;\n" ::"r"(smem_u32(mbar + lane)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    __syncwarp();
    asm volatile("griddepcontrol.wait;\n" ::: "memory");  // f is written by the previous pass
    // lane 0 issues, by predication rather than a branch, so the (uniform) issue code can
    // be scheduled into the gaps of the dependent add chain
    // SYM with mode bit 1: L2 hints for the two reads of every stored part (the ascending
    // chain of its block and the descending chain of the mirror block). Whichever warp of
    // the pair reads a part first (c < kChunks/2) keeps it (evict_last) for the other; the
    // second read (c >= kChunks/2) marks it evict_first.
    const bool hint = sym && (mode & 2);
    uint64_t pol_keep = 0, pol_drop = 0;
    if (hint) {
        asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(pol_keep));
        if (mode & 4)
            asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;\n" : "=l"(pol_drop));
        else
            asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(pol_drop));
    }
    auto issue = [&](int c) {
        if (c >= kChunks) return;
        const int st = c % kSumStages;
        const int part0 = (desc ? kChunks - 1 - c : c) * kSumParts;
        if (hint) {
            const uint64_t pol = 2 * c < kChunks ? pol_keep : pol_drop;
            asm volatile(
                "{\n .reg .pred p;\n setp.eq.u32 p, %6, 0;\n"
                " @p mbarrier.arrive.expect_tx.shared.b64 _, [%5], %7;\n"
                " @p cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint "
                "[%0], [%1, {%2, %3, %4}], [%5], %8;\n}\n" ::"r"(smem_u32(sbase + st * kSumStageBytes)),
                "l"(reinterpret_cast<uint64_t>(&tmap)), "r"(0), "r"(gb0), "r"(part0), "r"(smem_u32(mbar + st)),
                "r"(lane), "r"(static_cast<unsigned>(kSumStageBytes)), "l"(pol)
                : "memory");
            return;
        }
        asm volatile(
            "{\n .reg .pred p;\n setp.eq.u32 p, %6, 0;\n"
            " @p mbarrier.arrive.expect_tx.shared.b64 _, [%5], %7;\n"
            " @p cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes "
            "[%0], [%1, {%2, %3, %4}], [%5];\n}\n" ::"r"(smem_u32(sbase + st * kSumStageBytes)),
            "l"(reinterpret_cast<uint64_t>(&tmap)), "r"(0), "r"(gb0), "r"(part0), "r"(smem_u32(mbar + st)),
            "r"(lane), "r"(static_cast<unsigned>(kSumStageBytes))
            : "memory");
    };
    auto wait = [&](int c) {
        const unsigned addr = smem_u32(mbar + c % kSumStages);
        const unsigned parity = static_cast<unsigned>((c / kSumStages) & 1);
        unsigned done = 0;
        while (!done) {
            asm volatile(
                "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                : "=r"(done)
                : "r"(addr), "r"(parity)
                : "memory");
        }
    };
    for (int c = 0; c + 1 < kSumStages; ++c) issue(c);
    double acc = 0.0;
    const unsigned sw = static_cast<unsigned>(lane & 7);
    for (int c = 0; c < kChunks; ++c) {
        issue(c + kSumStages - 1);
        wait(c);
        const unsigned char* st = sbase + (c % kSumStages) * kSumStageBytes;
        if (!desc) {
#pragma unroll
            for (int p = 0; p < kSumParts; ++p) {
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
            for (int p = kSumParts - 1; p >= 0; --p) {
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
        __syncwarp();  // every lane is done with this stage before it is refilled
    }
    double* pp = partials + (size_t)slot * chains;
    if (lane < bpw) pp[desc ? 2 * nbl - 1 - (b0 + lane) : (b0 + lane)] = acc;
    __threadfence();
    __syncwarp();
    unsigned ticket = 0;
    if (lane == 0) ticket = atomicAdd(&tickets[slot], 1u);
    ticket = __shfl_sync(0xffffffffu, ticket, 0);
    if (ticket == static_cast<unsigned>(wps - 1)) {  // last warp of this slot
        __threadfence();
        // the whole warp stages the partials (coalesced, one L2 round trip) into the
        // chain stage it no longer needs; lane 0 then adds them in block order
        double* sp = reinterpret_cast<double*>(sbase);
        constexpr int kBatch = static_cast<int>(kSumStages * kSumStageBytes / sizeof(double));
        double total = 0.0;
        for (int k0 = 0; k0 < chains; k0 += kBatch) {  // 26 qubits: 16,384 partials
            const int kn = min(kBatch, chains - k0);
            for (int k = lane; k < kn; k += 32) sp[k] = __ldcg(pp + k0 + k);
            __syncwarp();
            if (lane == 0)
                for (int k = 0; k < kn; ++k) total = __dadd_rn(total, sp[k]);
            __syncwarp();
        }
        if (lane == 0) {
            out[slot] = total;
            tickets[slot] = 0u;
        }
    }
    QCG_SPAN_END(5, 0, lane == 0);
}

// Encode the f-buffer tensor map (driver entry point resolved once through the runtime).
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static CUtensorMap fbuf_tensor_map(double* fbuf, uint64_t total_blocks, int parts) {
    static EncodeTiledFn encode = nullptr;
    if (!encode) {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q{};
        QC_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
        if (!fn || q != cudaDriverEntryPointSuccess) internal_error("cuTensorMapEncodeTiled unavailable");
        encode = reinterpret_cast<EncodeTiledFn>(fn);
    }
    CUtensorMap m;
    const cuuint64_t dims[3] = {16, total_blocks, kBlock / 16};
    const cuuint64_t strides[2] = {kBlock * sizeof(double), 16 * sizeof(double)};
    const cuuint32_t box[3] = {16, 32, static_cast<cuuint32_t>(parts)};
    const cuuint32_t estr[3] = {1, 1, 1};
    const CUresult r = encode(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, fbuf, dims, strides, box, estr,
                              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) internal_error("cuTensorMapEncodeTiled failed: " + std::to_string(static_cast<int>(r)));
    return m;
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
    // As few passes as the 9 gather bits allow, with the items spread evenly over them
    // (e.g. 7 + 7 at 26 qubits rather than 9 + 5): a pass with <= 8 items needs 2
    // register rounds instead of 3, and its free gather bits become pads that lengthen
    // the contiguous runs each tile reads (measured: 9-target pass 4.4 TB/s vs a padded
    // pass 5.6 TB/s at 24 qubits).
    const size_t npass = (items.size() + kHighBits - 1) / kHighBits;
    for (size_t i = 0, pi = 0; i < items.size(); ++pi) {
        const size_t left = items.size() - i, passes_left = npass - pi;
        const size_t take = (left + passes_left - 1) / passes_left;
        HighPass hp{};
        hp.mpos = -1;
        uint32_t single = 0x7u;  // column bits 0..2
        bool mirror = false;
        int k = 0;
        for (; k < static_cast<int>(take); ++k) {
            const int it = items[i + k];
            if (it < 0) {
                hp.mask[k] = all;
                hp.kind[k] = 2;
                hp.mpos = k;
                mirror = true;
            } else {
                hp.mask[k] = 1u << it;
                hp.kind[k] = 1;
                single |= 1u << it;
            }
        }
        for (int pad = 3; k < kHighBits; ++pad) {  // batch bits: widen the contiguous columns
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
        i += take;
    }
    return plan;
}

size_t partials_per_slot(const ChainPlan& plan) {
    if (plan.onchip) return 0;
    const size_t nbl = size_t{1} << (plan.Q - 12);
    return plan.sym ? 2 * nbl : nbl;
}

int launch_chain(const ChainPlan& plan, const SlotDesc* d_slots, const LayerParam* d_lp,
                 int n_slots, int p, uint32_t flags, double* d_fbuf, double* d_partials,
                 unsigned* d_tickets, double* d_out, cudaStream_t stream, const ChainStats* stats,
                 Prof* prof, const void* state_base, cudaEvent_t passes_done) {
    if (n_slots <= 0) return 0;
    const int Q = plan.Q;
    const double N = static_cast<double>(size_t{1} << Q);
    const uint32_t symf = plan.sym ? F_SYM : 0u;
    auto cnt = [&](const std::vector<int>* v, int l) {
        return (stats && v && l < static_cast<int>(v->size())) ? (*v)[static_cast<size_t>(l)] : n_slots;
    };
    const bool fp32 = flags & F_FP32;
    if (plan.onchip && fp32) {
        const size_t smem = (size_t{1} << Q) * sizeof(float2);
        static PerDeviceOnce attr32;
        attr32.run([] {
            QC_CUDA(cudaFuncSetAttribute(k_onchip_f32, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (1 << 12) * 8));
        });
        if (prof) prof->begin(K_ONCHIP, 0.0, stream);
        k_onchip_f32<<<n_slots, kOnchipThreads, smem, stream>>>(d_slots, d_lp, p, Q, flags | symf, d_out);
        if (prof) prof->end(stream);
        QC_CUDA(cudaGetLastError());
        if (passes_done) QC_CUDA(cudaEventRecord(passes_done, stream));
        return 1;
    }
    if (plan.onchip) {
        const size_t Ns = size_t{1} << Q;
        const size_t smem = Ns * sizeof(double2) + ((flags & F_EXPECT) ? Ns * sizeof(double) : 0);
        static PerDeviceOnce attr_done;
        attr_done.run([] {
            QC_CUDA(cudaFuncSetAttribute(k_onchip, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (1 << 12) * 24));
        });
        const double b = n_slots * N * (((flags & F_INIT) ? 0.0 : 16.0) + ((flags & F_STATE_OUT) ? 16.0 : 0.0));
        // no HBM stream: the ceiling is the FP64 pipe (explicit DMUL/DADD) and latency.
        // Per stored amplitude and layer: phase 6 + RX 6 per target (Q stored bits, + the
        // mirror op with half-state storage); expectation |a|^2 C(z) 4 + the ordered sum 1
        const double tq = Q + (plan.sym ? 1.0 : 0.0);
        const double ops = n_slots * N * (p * (6.0 + 6.0 * tq) + ((flags & F_EXPECT) ? 5.0 : 0.0));
        if (prof) prof->begin(K_ONCHIP, b, stream, ops);
        k_onchip<<<n_slots, kOnchipThreads, smem, stream>>>(d_slots, d_lp, p, Q, flags | symf,
                                                            d_out);
        if (prof) prof->end(stream);
        QC_CUDA(cudaGetLastError());
        if (passes_done) QC_CUDA(cudaEventRecord(passes_done, stream));
        return 1;
    }
    int launches = 0;
    // Programmatic dependent launch for every kernel whose stream predecessor is a kernel
    // of this chain (the first one follows the staging copy). Off by default: with two
    // chunk streams the early-scheduled dependent CTAs hold SMs the other stream's kernels
    // need (C2: 82.8 ms/solve with PDL vs 75.6 without). QCG_PDL=1 enables it.
    static const bool pdl_ok = [] {
        const char* e = std::getenv("QCG_PDL");
        return e && e[0] == '1';
    }();
    for (int l = 0; l < p; ++l) {
        const uint32_t fa = (l == 0 && (flags & F_INIT)) ? F_INIT : 0u;
        const int nph = cnt(stats ? &stats->phase : nullptr, l);
        const int nmix = cnt(stats ? &stats->mix : nullptr, l);
        // pass A moves a slot if it initialises, phases or mixes it; levels read when phased
        const int active = fa ? n_slots : std::max(nph, nmix);
        // amplitude bytes: 16 (fp64 complex) or 8 (fp32 mode); f(z) 8 or 4
        const double ab = fp32 ? 8.0 : 16.0, fb = fp32 ? 4.0 : 8.0;
        const double ba = (fa ? n_slots * ab : active * 2.0 * ab) * N + nph * 2.0 * N;
        // FP64: 6 per amplitude for the phase, 6 per amplitude per RX target (12 targets)
        const double oa = (nph * 6.0 + nmix * 72.0) * N;
        if (prof) prof->begin(K_PASS_LOW, ba, stream, oa);
        launch_pass_a4(d_slots, d_lp, l, Q, fa | (flags & (F_FP32 | F_WHT | F_BALGRID)), n_slots, stream, pdl_ok && l > 0,
                       state_base);
        if (prof) prof->end(stream);
        ++launches;
        for (size_t h = 0; h < plan.high.size(); ++h) {
            const bool last = (l == p - 1) && (h + 1 == plan.high.size());
            uint32_t fh = 0;
            if (last && (flags & F_EXPECT)) fh |= F_EXPECT;
            if (last && (flags & F_STATE_OUT)) fh |= F_STATE_OUT;
            double bh;
            if (fh & F_EXPECT)  // read state, write f (+ state), read levels
                bh = n_slots * N * (ab + fb + 2.0 + ((fh & F_STATE_OUT) ? ab : 0.0));
            else
                bh = nmix * 2.0 * ab * N;
            int items = 0;
            for (int b = 0; b < kHighBits; ++b) items += plan.high[h].kind[b] != 0 ? 1 : 0;
            // 6 per amplitude per pair op (RX target or mirror), + |a|^2 C(z) (4) when f is emitted
            const double oh = nmix * 6.0 * items * N + ((fh & F_EXPECT) ? n_slots * 4.0 * N : 0.0);
            if (prof) prof->begin(K_PASS_HIGH, bh, stream, oh);
            launch_pass_b4(d_slots, d_lp, l, Q, plan.high[h], fh | (flags & (F_FP32 | F_WHT | F_BALGRID)), n_slots, stream, pdl_ok,
                           state_base);
            if (prof) prof->end(stream);
            ++launches;
        }
    }
    QC_CUDA(cudaGetLastError());
    // every pass of the chain is queued: a chunk queued behind this one may start its
    // passes now (lockstep ping-pong, qc_engine.cpp optimize_batch)
    if (passes_done) QC_CUDA(cudaEventRecord(passes_done, stream));
    if ((flags & F_EXPECT) && fp32) {
        const int nbl = 1 << (Q - 12);
        if (prof) prof->begin(K_BLOCKSUM, n_slots * N * 4.0, stream);
        k_fsum_f32<<<static_cast<unsigned>(n_slots * nbl), kFsumThreads, 0, stream>>>(
            reinterpret_cast<const float*>(d_fbuf), Q, plan.sym ? 1 : 0, d_partials, d_tickets, d_out);
        if (prof) prof->end(stream);
        QC_CUDA(cudaGetLastError());
        return launches + 1;
    }
    if (flags & F_EXPECT) {
        const int nbl = 1 << (Q - 12);
        const int bpw = std::min(32, nbl);
        const int warps = (nbl / bpw) * (plan.sym ? 2 : 1) * n_slots;
        const int sms = device_sm_count();
        static PerDeviceOnce sum_attrs;
        sum_attrs.run([] {
            QC_CUDA(cudaFuncSetAttribute(k_blocksum<3, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(sum_smem<3, 8>())));
            QC_CUDA(cudaFuncSetAttribute(k_blocksum<6, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(sum_smem<6, 8>())));
            QC_CUDA(cudaFuncSetAttribute(k_blocksum<3, 8, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(sum_smem<3, 8, 2>())));
            QC_CUDA(cudaFuncSetAttribute(k_blocksum<3, 4, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(sum_smem<3, 4, 4>())));
            QC_CUDA(cudaFuncSetAttribute(k_blocksum<3, 2, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(sum_smem<3, 2, 8>())));
        });
        // Warps per CTA (QCG_SUM_WARPS = 1 | 2 | 4 | 8; stages of 8 / 8 / 4 / 2 parts): packs
        // a launch's chains onto fewer SMs, leaving the rest to the other chunk's passes.
        static const int sum_warps = [] {
            const char* e = std::getenv("QCG_SUM_WARPS");
            const int w = e ? std::atoi(e) : 1;
            return (w == 2 || w == 4 || w == 8) ? w : 1;
        }();
        const int sum_parts = sum_warps == 4 ? 4 : sum_warps == 8 ? 2 : 8;
        // stages x 1 KB-per-lane chunks: 6 deep when every warp has an SM to itself, else
        // 3 (two warp-CTAs per SM). Smaller stages measured slower at every size
        // (profiles/r1_blocksum_stages.txt).
        const CUtensorMap tmap = fbuf_tensor_map(d_fbuf, static_cast<uint64_t>(n_slots) * nbl, sum_parts);
        if (prof) prof->begin(K_BLOCKSUM, n_slots * N * 8.0, stream, n_slots * N * (plan.sym ? 2.0 : 1.0));
        // Ring depth: 3 stages (two warp-CTAs per SM) by default. With two chunk streams the
        // two chunks' block sums often run at once (C2: 80 + 88 warps > 148 SMs), and 6-stage
        // warp-CTAs (one per SM) then serialise on 20 SMs: C2 69.6 -> 69.0 ms per solve with
        // 3. QCG_SUM_STAGES=6 restores the deeper ring whenever every warp has an SM.
        static const int pair_dirs = [] {  // QCG_SUM_PAIR=0: ascending warps, then descending
            const char* e = std::getenv("QCG_SUM_PAIR");
            return e ? std::atoi(e) : 1;
        }();
        // L2 keep/drop hints on the two reads of each stored part (SYM): block sum at q = 22 /
        // 24 / 26 118.6 -> 115.2, 176.8 -> 169.8, 261.4 -> 250.6 us per launch; at q = 20 x 21
        // slots (88 MB of f, L2-resident) 38.5 -> 39.5, so on when the launch's f exceeds
        // 96 MB. QCG_SUM_HINT=0/1 forces.
        static const int sum_hint_env = [] {
            const char* e = std::getenv("QCG_SUM_HINT");
            return e ? std::atoi(e) : -1;
        }();
        const double f_bytes = static_cast<double>(n_slots) * N * 8.0;
        const int sum_hint = sum_hint_env >= 0 ? sum_hint_env : (f_bytes > 96.0 * (1 << 20) ? 1 : 0);
        const int sum_mode = (pair_dirs ? 1 : 0) | (sum_hint ? 2 : 0) | (sum_hint == 2 ? 4 : 0);
        static const int sum_stages = [] {
            const char* e = std::getenv("QCG_SUM_STAGES");
            return e ? std::atoi(e) : 3;
        }();
        const unsigned wgrid = static_cast<unsigned>((warps + sum_warps - 1) / sum_warps);
        if (sum_warps == 2)
            launch_ex(k_blocksum<3, 8, 2>, dim3(wgrid), dim3(64), sum_smem<3, 8, 2>(), stream, pdl_ok, tmap,
                      n_slots, Q, plan.sym ? 1 : 0, sum_mode, d_partials, d_tickets, d_out);
        else if (sum_warps == 4)
            launch_ex(k_blocksum<3, 4, 4>, dim3(wgrid), dim3(128), sum_smem<3, 4, 4>(), stream, pdl_ok, tmap,
                      n_slots, Q, plan.sym ? 1 : 0, sum_mode, d_partials, d_tickets, d_out);
        else if (sum_warps == 8)
            launch_ex(k_blocksum<3, 2, 8>, dim3(wgrid), dim3(256), sum_smem<3, 2, 8>(), stream, pdl_ok, tmap,
                      n_slots, Q, plan.sym ? 1 : 0, sum_mode, d_partials, d_tickets, d_out);
        else if (sum_stages == 7 || (sum_stages == 6 && warps <= sms))
            launch_ex(k_blocksum<6, 8>, dim3(warps), dim3(32), sum_smem<6, 8>(), stream, pdl_ok, tmap, n_slots,
                      Q, plan.sym ? 1 : 0, sum_mode, d_partials, d_tickets, d_out);
        else
            launch_ex(k_blocksum<3, 8>, dim3(warps), dim3(32), sum_smem<3, 8>(), stream, pdl_ok, tmap, n_slots,
                      Q, plan.sym ? 1 : 0, sum_mode, d_partials, d_tickets, d_out);
        if (prof) prof->end(stream);
        launches += 1;
        QC_CUDA(cudaGetLastError());
    }
    return launches;
}

}  // namespace qcg
#ifdef QCG_TRACE
QCG_SPAN_READER(qc_span_read_kernels)
#endif
