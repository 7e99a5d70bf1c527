// Streaming pass kernels v4 (sm_100a): persistent CTAs, two consumer groups per CTA and
// a three-stage cp.async ring in shared memory.
//
// Why this shape. A pass moves every stored amplitude HBM -> SM -> HBM once and applies
// 6 FP64 ops per amplitude per RX target (no FMA: statevector.hpp:176-180 is replayed
// with explicit __dmul_rn/__dadd_rn). On B200 the per-SM share of HBM is ~23 B/clk, so a
// 4096-amplitude tile (64 KB in + 64 KB out) costs ~5.7k clk of bandwidth, while pass A's
// 78 FP64 ops/amp cost ~5.0k clk of the 64-lane FP64 pipe and the shared-memory rounds
// ~3.5k clk. All three must overlap. v3 (one tile per CTA, 2 CTAs/SM) serialised "load ->
// compute" inside each CTA and left HBM idle whenever both CTAs computed. Here:
//   * loads of tiles k+1, k+2 are in flight (cp.async -> mbarrier) while tile k computes;
//   * two 256-thread groups work on alternate tiles, so one group's FP64 rounds overlap
//     the other's shared-memory traffic (group-local named barriers, no CTA barrier);
//   * 16 amplitudes per thread: 4 targets per register round, 3 rounds for 12 bits
//     (v3: 8 amps, 4 rounds), i.e. fewer shared-memory round trips per tile.
//
// Ring protocol. Local tile k of a CTA lives in stage k % 3 and is computed by group
// k % 2. The group that finishes reading tile k from its stage immediately refills the
// stage with tile k + 3 (which the OTHER group computes). Each stage has a "full"
// mbarrier (256 arrivals: every issuing thread's cp.async.mbarrier.arrive.noinc) and a
// tag word = the local tile index it was last filled with; a consumer first waits for the
// tag (so it never tests the parity of a phase two generations ahead), then the parity.
//
// Exactness is unchanged from v3: per amplitude the phase precedes RX targets in
// ascending order, the mirror op (RX on qubit q-1 in half-state storage) comes last, and
// mixer_pair is bitwise symmetric in its two operands (IEEE add/mul commute), so the
// order of a pair's roles is immaterial.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstdint>
#include <string>
#include <type_traits>

#include "qc_amp.cuh"
#include "qc_internal.hpp"

namespace qcg {
namespace v4 {

constexpr int kGT = 256;             // threads per consumer group
constexpr int kThreads = 2 * kGT;    // two groups
constexpr int kStages = 3;
constexpr int kLutCap = 224;         // LUT entries kept per group in shared memory
constexpr int kDescCap = 24;         // slot descriptors cached per CTA
constexpr uint32_t kStageAmpBytes = 4096u * 16u;
constexpr uint32_t kOffLev = kStages * kStageAmpBytes;             // levels per stage (8 KB)
constexpr uint32_t kOffLut = kOffLev + kStages * 4096u * 2u;       // per-group LUT
constexpr uint32_t kOffBar = kOffLut + 2u * kLutCap * 16u;         // full barriers
constexpr uint32_t kOffTag = kOffBar + kStages * 8u;               // tags + per-stage words
constexpr uint32_t kOffDesc = kOffTag + 32u;

// Per-slot view of (SlotDesc, LayerParam[layer]) cached in shared memory at kernel start,
// so a tile's first instructions do not wait on two dependent global loads.
struct PD {
    double2* state;
    double* fbuf;
    const uint16_t* lev;
    const double* val;
    const double2* lut;
    double amp0, c, s, gamma;
    int32_t phase, mix, lut_len, key;
};
constexpr uint32_t kSmem = kOffDesc + kDescCap * sizeof(PD);
static_assert(kSmem + 1024 <= 232448, "shared memory budget (+1 KB alignment slack for TMA)");

__device__ __forceinline__ uint32_t su32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void cpa_arrive(uint32_t bar) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void bar_arrive(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void bar_wait(uint32_t bar, uint32_t parity) {
    uint32_t done = 0;
    while (!done) {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
            " selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(done)
            : "r"(bar), "r"(parity)
            : "memory");
    }
}
// Programmatic dependent launch: let the next kernel of the chain be scheduled now (its
// CTAs land as ours exit), and wait for the previous kernel's completion before any
// state access (no-ops when the launch did not set the attribute).
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }

// Phase trace of the pass A tile loop (tools/trace_pass.py; built only with -DQCG_TRACE
// into a separate tool library): CTAs < kTraceCtas, per group, per local tile, kTraceEv
// clock64 stamps taken by the group's lane 0.
#ifdef QCG_TRACE
constexpr int kTraceCtas = 4, kTraceTiles = 40, kTraceEv = 8;
__device__ long long g_trace[kTraceCtas * 2 * kTraceTiles * kTraceEv];
// every CTA (globaltimer ns): entry, after the prologue, group 0 done, group 1 done
constexpr int kTraceMaxCtas = 1024;
__device__ unsigned long long g_cta[kTraceMaxCtas * 4];
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#define QCG_CTA(ev, cond)                                                  \
    do {                                                                   \
        if ((cond) && blockIdx.x < kTraceMaxCtas) g_cta[blockIdx.x * 4 + (ev)] = gtimer(); \
    } while (0)
#define QCG_TR(k, ev)                                                                          \
    do {                                                                                       \
        if (gt == 0 && blockIdx.x < kTraceCtas && (k) / 2 < kTraceTiles)                       \
            g_trace[((blockIdx.x * 2 + g) * kTraceTiles + (k) / 2) * kTraceEv + (ev)] = clock64(); \
    } while (0)
#else
#define QCG_TR(k, ev) \
    do {              \
    } while (0)
#define QCG_CTA(ev, cond) \
    do {                  \
    } while (0)
#endif

__device__ __forceinline__ void grp_sync(uint32_t g) {
    asm volatile("bar.sync %0, %1;\n" ::"r"(g + 1u), "n"(kGT) : "memory");
}

__device__ __forceinline__ void tile_range(uint32_t total, uint32_t& t0, int& cnt) {
    const uint64_t b = blockIdx.x, G = gridDim.x;
    t0 = static_cast<uint32_t>(b * total / G);
    cnt = static_cast<int>(static_cast<uint32_t>((b + 1) * total / G) - t0);
}

// Slot range of this CTA's tiles -> descriptor cache (caller guarantees it fits).
// PHASE: the phase passes (pass A) read the phase-LUT index levels (SlotDesc::plev), the
// f passes (pass B) the cost levels (SlotDesc::lev)
template <bool PHASE = false>
__device__ __forceinline__ void load_descs(PD* pd, const SlotDesc* __restrict__ slots,
                                           const LayerParam* __restrict__ lp, int layer,
                                           uint32_t sa, uint32_t n) {
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
        const SlotDesc S = slots[sa + i];
        const LayerParam L = lp[S.layer_base + layer];
        PD d;
        d.state = S.state;
        d.fbuf = S.fbuf;
        d.lev = PHASE ? S.plev : S.lev;
        d.val = S.val;
        d.lut = L.lut;
        d.amp0 = S.amp0;
        d.c = L.c;
        d.s = L.s;
        d.gamma = L.gamma;
        d.phase = L.phase;
        d.mix = L.mix;
        d.lut_len = L.lut_len;
        d.key = static_cast<int32_t>(sa + i);
        pd[i] = d;
    }
}

__device__ __forceinline__ void ring_init(unsigned char* sm) {
    if (threadIdx.x < kStages) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(su32(sm + kOffBar) + threadIdx.x * 8u),
                     "r"(kGT)
                     : "memory");
        reinterpret_cast<volatile int*>(sm + kOffTag)[threadIdx.x] = -1;
    }
}

// ---------------------------------------------------------------------------
// pass A: tile = 4096 contiguous stored amplitudes; [|+> init] + phase + RX 0..11.
// Rounds: bits 0-3 (e = gt*16 + j), bits 4-7, bits 8-11 (e = j*256 + gt, coalesced store).
// ---------------------------------------------------------------------------
template <typename V>
__global__ void __launch_bounds__(kThreads, 1)
    k_pass_a(const SlotDesc* __restrict__ slots, const LayerParam* __restrict__ lp, int layer,
             int Q, uint32_t flags, uint32_t total_tiles) {
    QCG_SPAN_BEGIN();
    extern __shared__ __align__(1024) unsigned char sm[];
    const uint32_t tid = threadIdx.x, g = tid / kGT, gt = tid % kGT;
    const int tshift = Q - 12;
    const uint32_t tmask = (1u << tshift) - 1u;
    using S = typename Amp<V>::S;
    const bool init = flags & F_INIT;
    const bool wht = flags & F_WHT;
    uint32_t t0;
    int cnt;
    tile_range(total_tiles, t0, cnt);
    if (cnt <= 0) return;
    const uint32_t sa = t0 >> tshift;
    PD* pd = reinterpret_cast<PD*>(sm + kOffDesc);
    load_descs<true>(pd, slots, lp, layer, sa, ((t0 + cnt - 1) >> tshift) - sa + 1);
    ring_init(sm);
    __syncthreads();
    pdl_trigger();
    pdl_wait();
    const uint32_t bar0 = su32(sm + kOffBar);
    volatile int* tag = reinterpret_cast<volatile int*>(sm + kOffTag);

    // the calling group fills stage k%3 with local tile k
    auto issue = [&](int k) {
        if (k >= cnt) return;
        const int s = k % kStages;
        const uint32_t t = t0 + static_cast<uint32_t>(k);
        const PD& d = pd[(t >> tshift) - sa];
        const uint32_t base = (t & tmask) << 12;
        bool any = false;
        if (init || d.phase || d.mix) {
            if (!init) {
                const uint32_t sb = su32(sm + s * kStageAmpBytes);
                const V* src = reinterpret_cast<const V*>(d.state) + base + gt;
                const uint32_t d0 = sb + sw<V>(gt) * Amp<V>::kBytes;  // sw(gt + 256 i) = sw(gt) + 256 i
#pragma unroll
                for (int i = 0; i < 16; ++i) Amp<V>::cpa(d0 + i * (kGT * Amp<V>::kBytes), src + kGT * i);
                any = true;
            }
            if (d.phase && d.lev) {
                const uint32_t lb = su32(sm + kOffLev + s * 8192u);
#pragma unroll
                for (int i = 0; i < 2; ++i) {
                    const uint32_t u = gt + kGT * i;  // 16-byte unit = 8 levels
                    cpa16(lb + u * 16u, d.lev + base + u * 8u);
                }
                any = true;
            }
        }
        if (gt == 0) tag[s] = k;
        if (any)
            cpa_arrive(bar0 + s * 8u);
        else
            bar_arrive(bar0 + s * 8u);
    };
    if (g == 0) {
        issue(0);
        issue(2);
    } else {
        issue(1);
    }

    V* slut = reinterpret_cast<V*>(sm + kOffLut) + g * kLutCap;
    int lut_owner = -1;  // slot whose LUT slut holds
    for (int k = static_cast<int>(g); k < cnt; k += 2) {
        const int s = k % kStages;
        const uint32_t t = t0 + static_cast<uint32_t>(k);
        const PD& d = pd[(t >> tshift) - sa];
        const bool act = init || d.phase || d.mix;
        const bool use_lev = d.phase && d.lev;
        const bool lut_sm = use_lev && d.lut_len <= kLutCap;
        if (lut_sm && lut_owner != d.key) {
            // every thread of the group is past the previous tile's phase (round-0) reads
            const V* lsrc = reinterpret_cast<const V*>(d.lut);  // host-staged V entries
            for (int i = static_cast<int>(gt); i < d.lut_len; i += kGT) slut[i] = lsrc[i];
            lut_owner = d.key;
            grp_sync(g);
        }
        while (tag[s] != k) {
        }
        bar_wait(bar0 + s * 8u, static_cast<uint32_t>((k / kStages) & 1));
        if (!act) {
            grp_sync(g);  // every thread has seen tag k before the refill overwrites it
            issue(k + kStages);
            continue;  // identity layer: memory already holds the result
        }
        const uint32_t base = (t & tmask) << 12;
        V* st = reinterpret_cast<V*>(sm + s * kStageAmpBytes);
        const S c = static_cast<S>(d.c), sn = static_cast<S>(d.s);
        const bool mix = d.mix;
        V a[16];
        // round 0: bits 0-3, phase first. Two instantiations (staged LUT: LDS; global LUT:
        // LDG) so the lookups do not compile to generic loads, as in k_pass_a5/a7.
        {
            const uint4* lv = reinterpret_cast<const uint4*>(sm + kOffLev + s * 8192u) + gt * 2u;
            const bool phase = d.phase;
            const S amp0 = static_cast<S>(d.amp0);
            auto round0 = [&](const V* __restrict__ lutp) {
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const uint4 l4 = use_lev ? lv[h] : make_uint4(0, 0, 0, 0);
#pragma unroll
                    for (int jj = 0; jj < 8; ++jj) {
                        const int j = h * 8 + jj;
                        const uint32_t e = gt * 16u + j;
                        V v = init ? Amp<V>::mk(amp0, S(0)) : st[sw<V>(e)];
                        if (phase) {
                            if (use_lev) {
                                const uint32_t word = (jj >> 1) == 0 ? l4.x : (jj >> 1) == 1 ? l4.y
                                                    : (jj >> 1) == 2 ? l4.z : l4.w;
                                v = Amp<V>::cmul(v, lutp[(word >> ((jj & 1) * 16)) & 0xffffu]);
                            } else {
                                v = phase_frac<V>(v, d.gamma, d.val[base + e]);
                            }
                        }
                        a[j] = v;
                    }
                }
            };
            if (lut_sm)
                round0(slut);
            else
                round0(reinterpret_cast<const V*>(d.lut));
            if (mix) mix4<V>(a, c, sn, wht);
#pragma unroll
            for (int j = 0; j < 16; ++j) st[sw<V>(gt * 16u + j)] = a[j];
        }
        // round 1 reads only what its own half-warp wrote in round 0 (e>>8 = gt>>4)
        __syncwarp();
        // round 1: bits 4-7, e = (gt>>4)<<8 | j<<4 | gt&15
        {
            const uint32_t r = ((gt >> 4) << 8) | (gt & 15u);
#pragma unroll
            for (int j = 0; j < 16; ++j) a[j] = st[sw<V>(r | (j << 4))];
            if (mix) mix4<V>(a, c, sn, wht);
#pragma unroll
            for (int j = 0; j < 16; ++j) st[sw<V>(r | (j << 4))] = a[j];
        }
        grp_sync(g);
        // round 2: bits 8-11, e = j<<8 | gt
        const V* st2 = st + sw<V>(gt);  // sw(j<<8 | gt) = j<<8 | sw(gt)
#pragma unroll
        for (int j = 0; j < 16; ++j) a[j] = st2[j << 8];
        V* __restrict__ dst = reinterpret_cast<V*>(d.state) + base;
        grp_sync(g);  // the whole group is done with this stage: refill it
        issue(k + kStages);
        // last target (bit 11 = local bit 3) pair by pair, each pair stored as soon as it
        // is final: spreads the 64 KB of stores over the round instead of one burst
        if (sizeof(V) == 8 && wht) {
            if (mix) mix4<V>(a, c, sn, true);
#pragma unroll
            for (int j = 0; j < 16; ++j) dst[(j << 8) | gt] = a[j];
            continue;
        }
        if (mix) rx_local<V, 0, 3>(a, c, sn);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            if (mix) Amp<V>::rx(a[j], a[j + 8], c, sn);
            dst[(j << 8) | gt] = a[j];
            dst[((j + 8) << 8) | gt] = a[j + 8];
        }
    }
    QCG_SPAN_END(2, g, gt == 0);
}

// ---------------------------------------------------------------------------
// pass A, TMA variant (fp64 default; QCG_PASS_A=v4 for the cp.async/STG kernel above): the
// compute warps issue no global memory
// instructions. One elected lane per group moves the data: a 3-D tensor copy brings the
// 64 KB tile in ({16 doubles, 256 sixteen-amp groups (stride 256 B), 2 halves (stride
// 128 B)}, 128-byte swizzle: row r = m + 256*half, so rounds R0/R1/R2 read conflict-free),
// a 1-D bulk copy the levels; results are staged linearly in the same stage and leave by
// one 64 KB bulk store, after which the lane refills the stage.
// ---------------------------------------------------------------------------
// tile index -> amplitude slot in the stage. fp64: 128-byte rows r = m + 256*half, 128-byte
// swizzle (16-byte unit u at u ^ (r & 7)); fp32: 64-byte rows, 64-byte swizzle (16-byte
// unit = two amplitudes, at unit ^ ((r >> 1) & 3)).
template <typename V>
__device__ __forceinline__ uint32_t ph5(uint32_t e) {
    const uint32_t m = e >> 4, half = (e >> 3) & 1u, u = e & 7u;
    const uint32_t r = m + (half << 8);
    if constexpr (sizeof(V) == 16)
        return (r << 3) | (u ^ (m & 7u));
    else
        return (r << 3) | ((((u >> 1) ^ (r >> 1)) & 3u) << 1) | (u & 1u);
}

template <typename V, bool INIT>
__global__ void __launch_bounds__(kThreads, 1)
    k_pass_a5(const SlotDesc* __restrict__ slots, const LayerParam* __restrict__ lp, int layer,
              int Q, uint32_t flags, uint32_t total_tiles, const __grid_constant__ CUtensorMap tmap) {
    QCG_SPAN_BEGIN();
    using A = Amp<V>;
    using S = typename A::S;
    constexpr uint32_t kTileBytes = 4096u * sizeof(V);
    extern __shared__ __align__(1024) unsigned char sm_raw[];
    unsigned char* sm = sm_raw + ((1024u - (su32(sm_raw) & 1023u)) & 1023u);  // TMA 128B swizzle
    const uint32_t tid = threadIdx.x, g = tid / kGT, gt = tid % kGT;
    const int tshift = Q - 12;
    const uint32_t tmask = (1u << tshift) - 1u;
    QCG_CTA(0, tid == 0);
    constexpr bool init = INIT;  // first layer: |+> (no state read)
    const bool wht = flags & F_WHT;
    uint32_t t0;
    int cnt;
    tile_range(total_tiles, t0, cnt);
    if (cnt <= 0) return;
    const uint32_t sa = t0 >> tshift;
    PD* pd = reinterpret_cast<PD*>(sm + kOffDesc);
    load_descs<true>(pd, slots, lp, layer, sa, ((t0 + cnt - 1) >> tshift) - sa + 1);
    const uint32_t bar0 = su32(sm + kOffBar);
    volatile int* tag = reinterpret_cast<volatile int*>(sm + kOffTag);
    if (tid < kStages) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(bar0 + tid * 8u) : "memory");
        tag[tid] = -1;
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    __syncthreads();
    pdl_trigger();
    pdl_wait();

    // elected lane of the calling group: fill stage k%3 with local tile k
    auto issue = [&](int k) {
        if (k >= cnt || gt != 0) return;
        const int s = k % kStages;
        const uint32_t t = t0 + static_cast<uint32_t>(k);
        const PD& d = pd[(t >> tshift) - sa];
        const uint32_t base = (t & tmask) << 12;
        const uint32_t bar = bar0 + s * 8u;
        tag[s] = k;
        const bool lv = d.phase && d.lev;
        if (init || d.phase || d.mix) {
            const uint32_t bytes = (init ? 0u : kTileBytes) + (lv ? 8192u : 0u);
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes)
                         : "memory");
            if (!init)
                asm volatile(
                    "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes "
                    "[%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(su32(sm + s * kStageAmpBytes)),
                    "l"(reinterpret_cast<uint64_t>(&tmap)), "r"(0), "r"(t << 8), "r"(0), "r"(bar)
                    : "memory");
            if (lv)
                asm volatile(
                    "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 8192, [%2];\n" ::"r"(
                        su32(sm + kOffLev + s * 8192u)),
                    "l"(d.lev + base), "r"(bar)
                    : "memory");
        } else {
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(bar) : "memory");
        }
    };
    if (g == 0) {
        issue(0);
        issue(2);
    } else {
        issue(1);
    }

    QCG_CTA(1, tid == 0);
    V* slut = reinterpret_cast<V*>(sm + kOffLut) + g * kLutCap;
    int lut_owner = -1;
    int pending = -1;  // local tile whose refill waits on this group's last bulk store
    for (int k = static_cast<int>(g); k < cnt; k += 2) {
        QCG_TR(k, 0);
        // refill the stage of this group's previous tile as soon as its bulk store has read
        // it, before waiting for this tile's data
        if (pending >= 0) {
            if (gt == 0) asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
            issue(pending);
            pending = -1;
        }
        const int s = k % kStages;
        const uint32_t t = t0 + static_cast<uint32_t>(k);
        // tile-constant descriptor fields, read once (pd lives in shared memory next to the
        // stages the rounds write)
        const PD& d = pd[(t >> tshift) - sa];
        const bool phase = d.phase, mix = d.mix;
        const bool act = init || phase || mix;
        const bool use_lev = phase && d.lev;
        const int lut_len = d.lut_len;
        const bool lut_sm = use_lev && lut_len <= kLutCap;
        const V* const glut = reinterpret_cast<const V*>(d.lut);
        const S amp0 = static_cast<S>(d.amp0);
        if (lut_sm && lut_owner != d.key) {
            // the init layer stages amp0 * lut (the same cmul each amplitude would do)
            for (int i = static_cast<int>(gt); i < lut_len; i += kGT) {
                const V l = glut[i];
                slut[i] = init ? A::cmul(A::mk(amp0, S(0)), l) : l;
            }
            lut_owner = d.key;
            grp_sync(g);
        }
        QCG_TR(k, 1);
        while (tag[s] != k) {
        }
        bar_wait(bar0 + s * 8u, static_cast<uint32_t>((k / kStages) & 1));
        QCG_TR(k, 2);
        if (!act) {
            grp_sync(g);
            issue(k + kStages);
            continue;
        }
        const uint32_t base = (t & tmask) << 12;
        V* st = reinterpret_cast<V*>(sm + s * kStageAmpBytes);
        const double c = d.c, sn = d.s;
        V a[16];
        // round 0: phase + bits 0-3. Two instantiations so the staged-LUT reads compile to
        // LDS (a pointer that may be shared or global compiles to generic loads, which wait
        // on the long scoreboard); `pre`: the staged LUT already holds amp0 * lut.
        auto round0 = [&](const V* __restrict__ lutp, bool pre) {
            const uint4* lv = reinterpret_cast<const uint4*>(sm + kOffLev + s * 8192u) + gt * 2u;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const uint4 l4 = use_lev ? lv[h] : make_uint4(0, 0, 0, 0);
#pragma unroll
                for (int jj = 0; jj < 8; ++jj) {
                    const int j = h * 8 + jj;
                    const uint32_t e = gt * 16u + j;
                    V v;
                    if (use_lev) {
                        const uint32_t word = (jj >> 1) == 0 ? l4.x : (jj >> 1) == 1 ? l4.y
                                            : (jj >> 1) == 2 ? l4.z : l4.w;
                        const V l = lutp[(word >> ((jj & 1) * 16)) & 0xffffu];
                        v = init ? (pre ? l : A::cmul(A::mk(amp0, S(0)), l)) : A::cmul(st[ph5<V>(e)], l);
                    } else {
                        v = init ? A::mk(amp0, S(0)) : st[ph5<V>(e)];
                        if (phase) v = phase_frac<V>(v, d.gamma, d.val[base + e]);
                    }
                    a[j] = v;
                }
            }
            if (mix) mix4<V>(a, c, sn, wht);
#pragma unroll
            for (int j = 0; j < 16; ++j) st[ph5<V>(gt * 16u + j)] = a[j];
        };
        if (lut_sm)
            round0(slut, init);
        else
            round0(glut, false);
        QCG_TR(k, 3);
        __syncwarp();  // round 1 reads only what its own half-warp wrote (e>>8 = gt>>4)
        {
            const uint32_t r = ((gt >> 4) << 8) | (gt & 15u);
#pragma unroll
            for (int j = 0; j < 16; ++j) a[j] = st[ph5<V>(r | (j << 4))];
            if (mix) mix4<V>(a, c, sn, wht);
#pragma unroll
            for (int j = 0; j < 16; ++j) st[ph5<V>(r | (j << 4))] = a[j];
        }
        QCG_TR(k, 4);
        grp_sync(g);
#pragma unroll
        for (int j = 0; j < 16; ++j) a[j] = st[ph5<V>((j << 8) | gt)];
        grp_sync(g);  // the stage's tile is in registers: it becomes the output staging
        QCG_TR(k, 5);
        if (mix) mix4<V>(a, c, sn, wht);
#pragma unroll
        for (int j = 0; j < 16; ++j) st[(j << 8) | gt] = a[j];  // linear, conflict-free
        QCG_TR(k, 6);
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        grp_sync(g);
        QCG_TR(k, 7);
        if (gt == 0) {
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(
                             reinterpret_cast<V*>(d.state) + base),
                         "r"(su32(st)), "r"(kTileBytes)
                         : "memory");
            asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
        }
        // the refill of this stage waits for the store to have read it: done by the elected
        // lane after its next wait (the read is long finished by then), not stalling here
        pending = k + kStages;
    }
    if (pending >= 0) {
        if (gt == 0) asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
        issue(pending);
    }
    if (gt == 0) asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
    QCG_CTA(2 + g, gt == 0);
    QCG_SPAN_END(1, g, gt == 0);
}

// ---------------------------------------------------------------------------
// pass A, split-buffer variant (fp64 default): one input stage PER GROUP plus one output
// buffer SHARED by the two groups, instead of a three-stage in/out ring.
//
// Why. In k_pass_a5 the tile's stage is also its output staging, so the stage can be
// refilled only after the 64 KB bulk store has read it (~2.9k clk at the SM's share of
// HBM), and only the thread that issued a bulk store can wait for it: the group's elected
// lane blocked ~2.7k clk per tile at the top of its next tile and the whole group then
// waited for that warp at the round-2 barrier (tools/trace_pass.py). Here a group's input
// stage is free as soon as round 2 has loaded it into registers, so the elected lane
// refills it with the group's next tile right then, with nothing to wait for. The results
// go to OUT, which the two groups use alternately (tile n, n+1, ... in local order): the
// writer of tile n waits on `out_free` for the release of tile n-1, and a group releases
// its last write after round 0 of its next tile, when the store has long read OUT (its
// wait_group.read returns at once). Shared memory: 2 x 64 KB in + 64 KB out + 2 x 8 KB of
// cut levels + two 480-entry phase LUTs (C3's weighted LUTs fit) + descriptors.
// ---------------------------------------------------------------------------
constexpr int kLutCap7 = 480;
constexpr uint32_t kA7OffOut = 2u * kStageAmpBytes;
constexpr uint32_t kA7OffLev = 3u * kStageAmpBytes;
constexpr uint32_t kA7OffLut = kA7OffLev + 2u * 8192u;
constexpr uint32_t kA7OffBar = kA7OffLut + 2u * kLutCap7 * 16u;  // full[2], out_free
constexpr uint32_t kA7OffDesc = kA7OffBar + 32u;
constexpr uint32_t kA7Smem = kA7OffDesc + kDescCap * sizeof(PD);
static_assert(kA7Smem + 1024 <= 232448, "a7 shared memory budget");

template <typename V, bool INIT>
__global__ void __launch_bounds__(kThreads, 1)
    k_pass_a7(const SlotDesc* __restrict__ slots, const LayerParam* __restrict__ lp, int layer,
              int Q, uint32_t flags, uint32_t total_tiles, const __grid_constant__ CUtensorMap tmap) {
    QCG_SPAN_BEGIN();
    using A = Amp<V>;
    using S = typename A::S;
    constexpr uint32_t kTileBytes = 4096u * sizeof(V);
    extern __shared__ __align__(1024) unsigned char sm_raw[];
    unsigned char* sm = sm_raw + ((1024u - (su32(sm_raw) & 1023u)) & 1023u);  // TMA 128B swizzle
    const uint32_t tid = threadIdx.x, g = tid / kGT, gt = tid % kGT;
    const int tshift = Q - 12;
    const uint32_t tmask = (1u << tshift) - 1u;
    QCG_CTA(0, tid == 0);
    constexpr bool init = INIT;
    const bool wht = flags & F_WHT;
    const bool early_release = flags & F_A7EARLY;
    uint32_t t0;
    int cnt;
    tile_range(total_tiles, t0, cnt);
    if (cnt <= 0) return;
    const uint32_t sa = t0 >> tshift;
    PD* pd = reinterpret_cast<PD*>(sm + kA7OffDesc);
    load_descs<true>(pd, slots, lp, layer, sa, ((t0 + cnt - 1) >> tshift) - sa + 1);
    const uint32_t full = su32(sm + kA7OffBar) + g * 8u;  // this group's input barrier
    const uint32_t ofree = su32(sm + kA7OffBar) + 16u;
    if (tid < 2) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(su32(sm + kA7OffBar) + tid * 8u) : "memory");
    if (tid == 2) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(su32(sm + kA7OffBar) + 16u) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    __syncthreads();
    pdl_trigger();
    pdl_wait();

    unsigned char* in = sm + g * kStageAmpBytes;
    unsigned char* lev = sm + kA7OffLev + g * 8192u;
    // elected lane: load local tile k (one of this group's) into the group's stage
    auto issue = [&](int k) {
        if (k >= cnt || gt != 0) return;
        const uint32_t t = t0 + static_cast<uint32_t>(k);
        const PD& d = pd[(t >> tshift) - sa];
        const bool lv = d.phase && d.lev;
        if (init || d.phase || d.mix) {
            const uint32_t bytes = (init ? 0u : kTileBytes) + (lv ? 8192u : 0u);
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(full), "r"(bytes)
                         : "memory");
            if (!init)
                asm volatile(
                    "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes "
                    "[%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(su32(in)),
                    "l"(reinterpret_cast<uint64_t>(&tmap)), "r"(0), "r"(t << 8), "r"(0), "r"(full)
                    : "memory");
            if (lv)
                asm volatile(
                    "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 8192, [%2];\n" ::"r"(
                        su32(lev)),
                    "l"(d.lev + ((t & tmask) << 12)), "r"(full)
                    : "memory");
        } else {
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(full) : "memory");
        }
    };
    // release this group's last OUT write (its store has read OUT by now)
    bool pending = false;
    auto release = [&] {
        if (pending) {
            if (gt == 0) {
                asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
                bar_arrive(ofree);
            }
            pending = false;
        }
    };
    issue(static_cast<int>(g));

    QCG_CTA(1, tid == 0);
    V* slut = reinterpret_cast<V*>(sm + kA7OffLut) + g * kLutCap7;
    V* out = reinterpret_cast<V*>(sm + kA7OffOut);
    int lut_owner = -1;
    uint32_t it = 0;  // this group's tile count (input barrier phase)
    for (int k = static_cast<int>(g); k < cnt; k += 2, ++it) {
        QCG_TR(k, 0);
        const uint32_t t = t0 + static_cast<uint32_t>(k);
        const PD& d = pd[(t >> tshift) - sa];
        const bool phase = d.phase, mix = d.mix;
        const bool act = init || phase || mix;
        const bool use_lev = phase && d.lev;
        const int lut_len = d.lut_len;
        const bool lut_sm = use_lev && lut_len <= kLutCap7;
        const V* const glut = reinterpret_cast<const V*>(d.lut);
        const S amp0 = static_cast<S>(d.amp0);
        if (lut_sm && lut_owner != d.key) {
            for (int i = static_cast<int>(gt); i < lut_len; i += kGT) {
                const V l = glut[i];
                slut[i] = init ? A::cmul(A::mk(amp0, S(0)), l) : l;
            }
            lut_owner = d.key;
            grp_sync(g);
        }
        QCG_TR(k, 1);
        bar_wait(full, it & 1u);
        QCG_TR(k, 2);
        if (!act) {  // identity layer: memory already holds the result; keep OUT's turn order
            release();
            if (k > 0) bar_wait(ofree, static_cast<uint32_t>((k - 1) & 1));
            grp_sync(g);
            if (gt == 0) bar_arrive(ofree);
            issue(k + 2);
            continue;
        }
        const uint32_t base = (t & tmask) << 12;
        V* st = reinterpret_cast<V*>(in);
        const double c = d.c, sn = d.s;
        V a[16];
        auto round0 = [&](const V* __restrict__ lutp, bool pre) {
            const uint4* lv = reinterpret_cast<const uint4*>(lev) + gt * 2u;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const uint4 l4 = use_lev ? lv[h] : make_uint4(0, 0, 0, 0);
#pragma unroll
                for (int jj = 0; jj < 8; ++jj) {
                    const int j = h * 8 + jj;
                    const uint32_t e = gt * 16u + j;
                    V v;
                    if (use_lev) {
                        const uint32_t word = (jj >> 1) == 0 ? l4.x : (jj >> 1) == 1 ? l4.y
                                            : (jj >> 1) == 2 ? l4.z : l4.w;
                        const V l = lutp[(word >> ((jj & 1) * 16)) & 0xffffu];
                        v = init ? (pre ? l : A::cmul(A::mk(amp0, S(0)), l)) : A::cmul(st[ph5<V>(e)], l);
                    } else {
                        v = init ? A::mk(amp0, S(0)) : st[ph5<V>(e)];
                        if (phase) v = phase_frac<V>(v, d.gamma, d.val[base + e]);
                    }
                    a[j] = v;
                }
            }
            if (mix) mix4<V>(a, c, sn, wht);
#pragma unroll
            for (int j = 0; j < 16; ++j) st[ph5<V>(gt * 16u + j)] = a[j];
        };
        if (lut_sm)
            round0(slut, init);
        else
            round0(glut, false);
        QCG_TR(k, 3);
        release();     // the previous write's store has read OUT long ago
        __syncwarp();  // round 1 reads only what its own half-warp wrote (e>>8 = gt>>4)
        {
            const uint32_t r = ((gt >> 4) << 8) | (gt & 15u);
#pragma unroll
            for (int j = 0; j < 16; ++j) a[j] = st[ph5<V>(r | (j << 4))];
            if (mix) mix4<V>(a, c, sn, wht);
#pragma unroll
            for (int j = 0; j < 16; ++j) st[ph5<V>(r | (j << 4))] = a[j];
        }
        QCG_TR(k, 4);
        grp_sync(g);
#pragma unroll
        for (int j = 0; j < 16; ++j) a[j] = st[ph5<V>((j << 8) | gt)];
        grp_sync(g);   // the group's stage and levels are consumed: load its next tile now
        issue(k + 2);
        QCG_TR(k, 5);
        if (mix) mix4<V>(a, c, sn, wht);
        // OUT's turn: tile k-1 (the other group) must have released it
        if (k > 0) bar_wait(ofree, static_cast<uint32_t>((k - 1) & 1));
#pragma unroll
        for (int j = 0; j < 16; ++j) out[(j << 8) | gt] = a[j];  // linear, conflict-free
        QCG_TR(k, 6);
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        grp_sync(g);
        QCG_TR(k, 7);
        if (gt == 0) {
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(
                             reinterpret_cast<V*>(d.state) + base),
                         "r"(su32(out)), "r"(kTileBytes)
                         : "memory");
            asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
        }
        pending = true;
        if (early_release) release();  // F_A7EARLY: hand OUT over as soon as the store read it
    }
    release();
    if (gt == 0) asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
    QCG_CTA(2 + g, gt == 0);
    QCG_SPAN_END(1, g, gt == 0);
}

// ---------------------------------------------------------------------------
// pass B: tile = 8 contiguous amps (column bits 0-2) x 9 gathered tile bits (RX targets
// >= 12, then the mirror pseudo-bit whose mask is every stored bit, then no-op pads).
// Tile index e = w | gb << 3 (gb: 9 gather bits); global index = x ^ hx(gb) where
// x = deposit(tile, freemask) | w and hx() folds the gather-bit masks (kernel parameters:
// the XORs of compile-time bit subsets compile to LOP3s on constant-bank operands).
// Rounds: gather bits 0-3, 4-7, 8 (each only if it holds an op); the last round writes
// the state and/or f(z) = |a|^2 C(z) straight from registers.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t hx(const HighPass& hp, uint32_t bits) {
    uint32_t x = 0;
#pragma unroll
    for (int b = 0; b < kHighBits; ++b)
        if ((bits >> b) & 1u) x ^= hp.mask[b];
    return x;
}

__device__ __forceinline__ uint32_t deposit4(uint32_t v, uint32_t mask) {
    uint32_t x = 0;
    while (mask) {
        const uint32_t low = mask & (~mask + 1u);
        if (v & 1u) x |= low;
        v >>= 1;
        mask &= mask - 1u;
    }
    return x;
}

// pair ops on local bits of a[16]: local bit b -> gather bit G0 + b (kind != 0 => op)
template <typename V, int G0, int NB>
__device__ __forceinline__ void ops_local(V (&a)[16], const HighPass& hp, typename Amp<V>::S c,
                                          typename Amp<V>::S s, bool wht) {
    if constexpr (sizeof(V) == 8) {  // fp32 mode, F_WHT: Walsh–Hadamard form over the op bits
        if (wht) {
            uint32_t opmask = 0;
#pragma unroll
            for (int b = 0; b < NB; ++b) opmask |= (hp.kind[G0 + b] != 0 ? 1u : 0u) << b;
            wht_local<NB>(a, opmask, c, s);
            return;
        }
    }
#pragma unroll
    for (int b = 0; b < NB; ++b) {
        if (hp.kind[G0 + b] == 0) continue;
#pragma unroll
        for (int j = 0; j < 16; ++j)
            if (!(j & (1 << b))) Amp<V>::rx(a[j], a[j | (1 << b)], c, s);
    }
}

// gather bits of amp j in round R (the j-dependent part; compile-time after unrolling)
template <int R>
__device__ __forceinline__ uint32_t gb_local(int j) {
    if (R == 0) return static_cast<uint32_t>(j);
    if (R == 1) return static_cast<uint32_t>(j) << 4;
    return (static_cast<uint32_t>(j >> 1) & 7u) | (static_cast<uint32_t>(j & 1) << 8);
}

template <typename V>
__global__ void __launch_bounds__(kThreads, 1)
    k_pass_b(const SlotDesc* __restrict__ slots, const LayerParam* __restrict__ lp, int layer,
             int Q, const __grid_constant__ HighPass hp, uint32_t flags, uint32_t total_tiles) {
    QCG_SPAN_BEGIN();
    extern __shared__ __align__(1024) unsigned char sm[];
    const uint32_t tid = threadIdx.x, g = tid / kGT, gt = tid % kGT;
    const int tshift = Q - 12;
    const uint32_t tmask = (1u << tshift) - 1u;
    using S = typename Amp<V>::S;
    const bool fout = flags & F_EXPECT;
    const bool sout = !fout || (flags & F_STATE_OUT);
    const bool wht = flags & F_WHT;
    uint32_t t0;
    int cnt;
    tile_range(total_tiles, t0, cnt);
    if (cnt <= 0) return;
    const uint32_t sa = t0 >> tshift;
    PD* pd = reinterpret_cast<PD*>(sm + kOffDesc);
    load_descs(pd, slots, lp, layer, sa, ((t0 + cnt - 1) >> tshift) - sa + 1);
    ring_init(sm);
    __syncthreads();
    pdl_trigger();
    pdl_wait();
    const uint32_t bar0 = su32(sm + kOffBar);
    volatile int* tag = reinterpret_cast<volatile int*>(sm + kOffTag);
    volatile uint32_t* sxb = reinterpret_cast<volatile uint32_t*>(sm + kOffTag + 16);  // per stage
    const int nr = (hp.kind[8] != 0) ? 3 : ((hp.kind[4] != 0) ? 2 : 1);  // rounds with ops
    const uint32_t w = gt & 7u;
    const uint32_t tx_issue = hx(hp, gt >> 3);             // gather bits 0-4 of issue units
    const uint32_t tx_lev = hx(hp, gt & 255u);             // levels: column gb = gt (+256)

    auto issue = [&](int k) {
        if (k >= cnt) return;
        const int s = k % kStages;
        const uint32_t t = t0 + static_cast<uint32_t>(k);
        const PD& d = pd[(t >> tshift) - sa];
        bool any = false;
        if (d.mix || fout) {
            const uint32_t xb = deposit4(t & tmask, hp.freemask);
            const uint32_t sb = su32(sm + s * kStageAmpBytes) + sw<V>(gt) * Amp<V>::kBytes;
            const uint32_t x = (xb | w) ^ tx_issue;
            const V* gs = reinterpret_cast<const V*>(d.state);
#pragma unroll
            for (int i = 0; i < 16; ++i)  // unit e = gt + 256 i: gb = gt>>3 | i<<5
                Amp<V>::cpa(sb + i * (kGT * Amp<V>::kBytes), gs + (x ^ hx(hp, static_cast<uint32_t>(i) << 5)));
            if (fout && d.lev) {
                const uint32_t lb = su32(sm + kOffLev + s * 8192u);
#pragma unroll
                for (int i = 0; i < 2; ++i) {
                    const uint32_t col = gt + kGT * i;
                    const uint32_t gx = (xb ^ tx_lev ^ (i ? hp.mask[8] : 0u)) & ~7u;
                    cpa16(lb + col * 16u, d.lev + gx);
                }
            }
            if (gt == 0) sxb[s] = xb;
            any = true;
        }
        if (gt == 0) tag[s] = k;
        if (any)
            cpa_arrive(bar0 + s * 8u);
        else
            bar_arrive(bar0 + s * 8u);
    };
    if (g == 0) {
        issue(0);
        issue(2);
    } else {
        issue(1);
    }

    for (int k = static_cast<int>(g); k < cnt; k += 2) {
        const int s = k % kStages;
        const uint32_t t = t0 + static_cast<uint32_t>(k);
        const PD& d = pd[(t >> tshift) - sa];
        const bool mix = d.mix;
        while (tag[s] != k) {
        }
        bar_wait(bar0 + s * 8u, static_cast<uint32_t>((k / kStages) & 1));
        if (!mix && !fout) {
            grp_sync(g);  // every thread has seen tag k before the refill overwrites it
            issue(k + kStages);
            continue;
        }
        const int nrr = mix ? nr : 1;  // no mixer: only f(z) to emit
        const uint32_t xb = sxb[s] | w;
        const S c = static_cast<S>(d.c), sn = static_cast<S>(d.s);
        V* st = reinterpret_cast<V*>(sm + s * kStageAmpBytes);
        const uint16_t* slev = reinterpret_cast<const uint16_t*>(sm + kOffLev + s * 8192u);
        V* const gstate = reinterpret_cast<V*>(d.state);
        S* const gf = reinterpret_cast<S*>(d.fbuf);  // f(z) in the amplitude precision
        const uint16_t* const glev = d.lev;
        const double* const gval = d.val;
        V a[16];
        // tile index of amp j in round R
        auto e_of = [&](auto R, int j) -> uint32_t {
            if constexpr (decltype(R)::value == 0)
                return w | (static_cast<uint32_t>(j) << 3) | ((gt >> 3) << 7);
            else if constexpr (decltype(R)::value == 1)
                return w | (((gt >> 3) & 15u) << 3) | (static_cast<uint32_t>(j) << 7) | ((gt >> 7) << 11);
            else
                return w | ((static_cast<uint32_t>(j >> 1) & 7u) << 3) | ((gt >> 3) << 6) |
                       (static_cast<uint32_t>(j & 1) << 11);
        };
        // final round: write out (state and/or f) at xb ^ hx(gb)
        auto emit = [&](auto R) {
            constexpr int r = decltype(R)::value;
            const uint32_t txt = r == 0 ? hx(hp, (gt >> 3) << 4)
                               : r == 1 ? hx(hp, ((gt >> 3) & 15u) | ((gt >> 7) << 8))
                                        : hx(hp, (gt >> 3) << 3);
            const uint32_t xt = xb ^ txt;
#pragma unroll
            for (int j = 0; j < 16; ++j) {
                const uint32_t gidx = xt ^ hx(hp, gb_local<r>(j));
                if (sout) __stcs(gstate + gidx, a[j]);
                if (fout) {
                    S cst;
                    if (glev)
                        cst = static_cast<S>(slev[(e_of(R, j) >> 3) * 8u + (gidx & 7u)]);
                    else
                        cst = static_cast<S>(gval ? gval[gidx] : 1.0);
                    gf[gidx] = Amp<V>::mul(Amp<V>::nrm(a[j]), cst);  // stays in L2 for k_blocksum
                }
            }
        };
        auto finish = [&](auto R) {
            if (fout && glev && !(flags & F_NOLEVREG)) {
                // f pass: take this thread's 16 cut levels into registers (two per word)
                // so the stage can be refilled before the f(z) stores, like the other passes
                constexpr int r = decltype(R)::value;
                const uint32_t txt = r == 0 ? hx(hp, (gt >> 3) << 4)
                                   : r == 1 ? hx(hp, ((gt >> 3) & 15u) | ((gt >> 7) << 8))
                                            : hx(hp, (gt >> 3) << 3);
                const uint32_t xt = xb ^ txt;
                uint32_t lvp[8];
#pragma unroll
                for (int j = 0; j < 16; j += 2) {
                    const uint32_t g0 = xt ^ hx(hp, gb_local<r>(j));
                    const uint32_t g1 = xt ^ hx(hp, gb_local<r>(j + 1));
                    lvp[j >> 1] = static_cast<uint32_t>(slev[(e_of(R, j) >> 3) * 8u + (g0 & 7u)]) |
                                  (static_cast<uint32_t>(slev[(e_of(R, j + 1) >> 3) * 8u + (g1 & 7u)]) << 16);
                }
                grp_sync(g);
                issue(k + kStages);
#pragma unroll
                for (int j = 0; j < 16; ++j) {
                    const uint32_t gidx = xt ^ hx(hp, gb_local<r>(j));
                    if (sout) __stcs(gstate + gidx, a[j]);
                    const S cst = static_cast<S>((lvp[j >> 1] >> ((j & 1) * 16)) & 0xffffu);
                    gf[gidx] = Amp<V>::mul(Amp<V>::nrm(a[j]), cst);
                }
                return;
            }
            grp_sync(g);
            if (!fout) issue(k + kStages);  // f reads the stage's levels: refill after
            emit(R);
            if (fout) {
                grp_sync(g);
                issue(k + kStages);
            }
        };
        using R0 = std::integral_constant<int, 0>;
        using R1 = std::integral_constant<int, 1>;
        using R2 = std::integral_constant<int, 2>;
        // round 0: gather bits 0-3 local
#pragma unroll
        for (int j = 0; j < 16; ++j) a[j] = st[sw<V>(e_of(R0{}, j))];
        if (mix) ops_local<V, 0, 4>(a, hp, c, sn, wht);
        if (nrr == 1) {
            finish(R0{});
            continue;
        }
#pragma unroll
        for (int j = 0; j < 16; ++j) st[sw<V>(e_of(R0{}, j))] = a[j];
        grp_sync(g);
        // round 1: gather bits 4-7 local
#pragma unroll
        for (int j = 0; j < 16; ++j) a[j] = st[sw<V>(e_of(R1{}, j))];
        ops_local<V, 4, 4>(a, hp, c, sn, wht);
        if (nrr == 2) {
            finish(R1{});
            continue;
        }
#pragma unroll
        for (int j = 0; j < 16; ++j) st[sw<V>(e_of(R1{}, j))] = a[j];
        grp_sync(g);
        // round 2: gather bit 8 local (j bit 0); j bits 1-3 carry gather bits 0-2
#pragma unroll
        for (int j = 0; j < 16; ++j) a[j] = st[sw<V>(e_of(R2{}, j))];
        ops_local<V, 8, 1>(a, hp, c, sn, wht);
        finish(R2{});
    }
    QCG_SPAN_END(3, g, gt == 0);
}

// ---------------------------------------------------------------------------
// pass B, TMA variant (fp64 at Q >= 21 and fp32 by default; QCG_PASS_B=v4|tma forces a
// kernel). fp32 boxes have 64-byte rows (8 float2) under the 64-byte swizzle.
// The 9 gather bits of a HighPass are [NT RX targets (one contiguous run of stored bits)]
// [mirror, if HM] [pads: bits 3.. (contiguous)], so a tile is one box of a 5-D tensor view
// of the launch's states: {16 doubles (column bits 0-2), targets, pads, low free run, high
// free run x slots}; the mirror partners (x -> ~x) are a second 32 KB box at the
// complemented free coordinates, whose elements sit in the box in reversed order. Box row
// r0 = pads | targets << NP (pads innermost: the copy walks the contiguous runs first;
// 128 bytes per row, 128-byte swizzle: unit u at u ^ (r & 7)). Under the complement both
// the row and the column reverse, so the swizzled unit is unchanged:
//   byte(e) = m << 15 | (r0 ^ (m ? 255 : 0)) << 7 | ((w ^ r0) & 7) << 4.
// Compute rounds are v4's; results go back to the same box positions and leave by tensor
// stores of the same boxes (F_TSTORE), or straight from registers. Levels (f passes) still
// arrive by per-thread cp.async, so a stage's barrier then expects 256 + 1 arrivals.
// ---------------------------------------------------------------------------
struct B5Geo {
    uint32_t lo_shift, lo_mask;   // low free run of stored bits (incl. a pinned mirror bit)
    uint32_t hi_shift, hi_mask;   // high free run (merged with the slot index)
    uint32_t hi_bits, allq;       // allq: the Q stored-bit mask (mirror complement)
};

template <typename V, int NT, int HM>
__device__ __forceinline__ uint32_t pb5(uint32_t e) {
    constexpr int NP = kHighBits - NT - HM;  // pads (the box's innermost row dimension)
    const uint32_t w = e & 7u, gb = e >> 3;
    const uint32_t targets = gb & ((1u << NT) - 1u);
    const uint32_t pads = gb >> (NT + HM);
    const uint32_t r0 = pads | (targets << NP);
    if constexpr (sizeof(V) == 16) {  // fp64: 128-byte rows, one amplitude per 16-byte unit
        if constexpr (HM == 0) {
            return (r0 << 7) | (((w ^ r0) & 7u) << 4);
        } else {
            const uint32_t m = (gb >> NT) & 1u;
            return (m << 15) | ((r0 ^ (0u - m)) & 255u) << 7 | (((w ^ r0) & 7u) << 4);
        }
    } else {  // fp32: 64-byte rows, 64-byte swizzle (unit ^= row bits 1-2), two amps per unit
        const uint32_t unit = ((w >> 1) ^ (r0 >> 1)) & 3u;
        if constexpr (HM == 0) {
            return (r0 << 6) | (unit << 4) | ((w & 1u) << 3);
        } else {
            // complement: row and column reverse; the swizzled unit is unchanged and only
            // the amplitude inside the unit flips
            const uint32_t m = (gb >> NT) & 1u;
            return (m << 14) | ((r0 ^ (0u - m)) & 255u) << 6 | (unit << 4) | (((w & 1u) ^ m) << 3);
        }
    }
}

template <typename V, int NT, int HM>
__global__ void __launch_bounds__(kThreads, 1)
    k_pass_b5(const SlotDesc* __restrict__ slots, const LayerParam* __restrict__ lp, int layer,
              int Q, const __grid_constant__ HighPass hp, uint32_t flags, uint32_t total_tiles,
              const __grid_constant__ B5Geo geo, const __grid_constant__ CUtensorMap tmap) {
    QCG_SPAN_BEGIN();
    using A = Amp<V>;
    using S = typename A::S;
    constexpr uint32_t kHalf = sizeof(V) == 16 ? 32768u : 16384u;  // bytes of a mirror box
    extern __shared__ __align__(1024) unsigned char sm_raw[];
    unsigned char* sm = sm_raw + ((1024u - (su32(sm_raw) & 1023u)) & 1023u);  // swizzle atoms
    const uint32_t tid = threadIdx.x, g = tid / kGT, gt = tid % kGT;
    const int tshift = Q - 12;
    const uint32_t tmask = (1u << tshift) - 1u;
    const bool fout = flags & F_EXPECT;
    const bool sout = !fout || (flags & F_STATE_OUT);
    const bool wht = flags & F_WHT;
    const bool tstore = flags & F_TSTORE;  // results leave by tensor stores of the boxes
    const bool early = flags & F_B5EARLY;  // experiment: refill before the next tile's wait
    uint32_t t0;
    int cnt;
    tile_range(total_tiles, t0, cnt);
    if (cnt <= 0) return;
    const uint32_t sa = t0 >> tshift;
    PD* pd = reinterpret_cast<PD*>(sm + kOffDesc);
    load_descs(pd, slots, lp, layer, sa, ((t0 + cnt - 1) >> tshift) - sa + 1);
    const uint32_t bar0 = su32(sm + kOffBar);
    volatile int* tag = reinterpret_cast<volatile int*>(sm + kOffTag);
    volatile uint32_t* sxb = reinterpret_cast<volatile uint32_t*>(sm + kOffTag + 16);
    if (tid < kStages) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bar0 + tid * 8u),
                     "r"(fout ? kGT + 1 : 1)
                     : "memory");
        tag[tid] = -1;
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    __syncthreads();
    pdl_trigger();
    pdl_wait();
    const int nr = (hp.kind[8] != 0) ? 3 : ((hp.kind[4] != 0) ? 2 : 1);
    const uint32_t w = gt & 7u;
    const uint32_t tx_lev = hx(hp, gt & 255u);

    auto tma = [&](bool store, uint32_t sdst, uint32_t x, uint32_t slot, uint32_t bar) {
        const int c3 = static_cast<int>((x >> geo.lo_shift) & geo.lo_mask);
        const int c4 = static_cast<int>(((x >> geo.hi_shift) & geo.hi_mask) | (slot << geo.hi_bits));
        if (store)
            asm volatile(
                "cp.async.bulk.tensor.5d.global.shared::cta.bulk_group [%0, {%1, %2, %3, %4, %5}], [%6];\n" ::"l"(
                    reinterpret_cast<uint64_t>(&tmap)),
                "r"(0), "r"(0), "r"(0), "r"(c3), "r"(c4), "r"(sdst)
                : "memory");
        else
            asm volatile(
                "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes "
                "[%0], [%1, {%2, %3, %4, %5, %6}], [%7];\n" ::"r"(sdst),
                "l"(reinterpret_cast<uint64_t>(&tmap)), "r"(0), "r"(0), "r"(0), "r"(c3), "r"(c4), "r"(bar)
                : "memory");
    };
    // whole group: fill stage k%3 with local tile k (box loads by the elected lane, levels
    // by every thread on f passes)
    auto issue = [&](int k) {
        if (k >= cnt) return;
        const int s = k % kStages;
        const uint32_t t = t0 + static_cast<uint32_t>(k);
        const PD& d = pd[(t >> tshift) - sa];
        const uint32_t bar = bar0 + s * 8u;
        const bool act = d.mix || fout;
        const bool lead = gt == 0;
        if (!lead && !fout) return;
        const uint32_t xb = deposit4(t & tmask, hp.freemask);
        if (lead) {
            sxb[s] = xb;
            tag[s] = k;
            if (act) {
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(2u * kHalf)
                             : "memory");
                const uint32_t sdst = su32(sm + s * kStageAmpBytes);
                tma(false, sdst, xb, t >> tshift, bar);
                if (HM) tma(false, sdst + kHalf, xb ^ geo.allq, t >> tshift, bar);
            } else {
                bar_arrive(bar);
            }
        }
        if (fout) {
            if (d.lev) {
                const uint32_t lb = su32(sm + kOffLev + s * 8192u);
#pragma unroll
                for (int i = 0; i < 2; ++i) {
                    const uint32_t gx = (xb ^ tx_lev ^ (i ? hp.mask[8] : 0u)) & ~7u;
                    cpa16(lb + (gt + kGT * i) * 16u, d.lev + gx);
                }
                cpa_arrive(bar);
            } else {
                bar_arrive(bar);
            }
        }
    };
    if (g == 0) {
        issue(0);
        issue(2);
    } else {
        issue(1);
    }

    int pending = -1;  // local tile whose refill waits on this group's last tensor store
    for (int k = static_cast<int>(g); k < cnt; k += 2) {
        const int s = k % kStages;
        const uint32_t t = t0 + static_cast<uint32_t>(k);
        const PD& d = pd[(t >> tshift) - sa];
        const bool mix = d.mix;
        if (pending >= 0 && early) {  // refill the previous tile's stage once its store has read it
            if (gt == 0) asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
            issue(pending);
            pending = -1;
        }
        while (tag[s] != k) {
        }
        bar_wait(bar0 + s * 8u, static_cast<uint32_t>((k / kStages) & 1));
        if (pending >= 0) {
            if (gt == 0) asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
            issue(pending);
            pending = -1;
        }
        if (!mix && !fout) {
            grp_sync(g);
            issue(k + kStages);
            continue;
        }
        const int nrr = mix ? nr : 1;
        const uint32_t xs = sxb[s];
        const uint32_t xb = xs | w;
        const S c = static_cast<S>(d.c), sn = static_cast<S>(d.s);
        unsigned char* stb = sm + s * kStageAmpBytes;
        const uint16_t* slev = reinterpret_cast<const uint16_t*>(sm + kOffLev + s * 8192u);
        S* const gf = reinterpret_cast<S*>(d.fbuf);  // f(z) in the amplitude precision
        const uint16_t* const glev = d.lev;
        const double* const gval = d.val;
        V a[16];
        auto at = [&](uint32_t e) -> V& { return *reinterpret_cast<V*>(stb + pb5<V, NT, HM>(e)); };
        auto e_of = [&](auto R, int j) -> uint32_t {
            if constexpr (decltype(R)::value == 0)
                return w | (static_cast<uint32_t>(j) << 3) | ((gt >> 3) << 7);
            else if constexpr (decltype(R)::value == 1)
                return w | (((gt >> 3) & 15u) << 3) | (static_cast<uint32_t>(j) << 7) | ((gt >> 7) << 11);
            else
                return w | ((static_cast<uint32_t>(j >> 1) & 7u) << 3) | ((gt >> 3) << 6) |
                       (static_cast<uint32_t>(j & 1) << 11);
        };
        auto finish = [&](auto R) {
            constexpr int r = decltype(R)::value;
            const uint32_t txt = r == 0 ? hx(hp, (gt >> 3) << 4)
                               : r == 1 ? hx(hp, ((gt >> 3) & 15u) | ((gt >> 7) << 8))
                                        : hx(hp, (gt >> 3) << 3);
            const uint32_t xt = xb ^ txt;
            if (!tstore) {  // registers -> global; the stage refills once every thread read it
                if (!fout) {
                    grp_sync(g);
                    issue(k + kStages);
                }
                V* const gstate = reinterpret_cast<V*>(d.state);
#pragma unroll
                for (int j = 0; j < 16; ++j) {
                    const uint32_t gidx = xt ^ hx(hp, gb_local<r>(j));
                    if (sout) __stcs(gstate + gidx, a[j]);
                    if (fout) {
                        S cst;
                        if (glev)
                            cst = static_cast<S>(slev[(e_of(R, j) >> 3) * 8u + (gidx & 7u)]);
                        else
                            cst = static_cast<S>(gval ? gval[gidx] : 1.0);
                        gf[gidx] = A::mul(A::nrm(a[j]), cst);
                    }
                }
                if (fout) {
                    grp_sync(g);  // levels of the stage read
                    issue(k + kStages);
                }
                return;
            }
            if (fout) {
#pragma unroll
                for (int j = 0; j < 16; ++j) {
                    const uint32_t gidx = xt ^ hx(hp, gb_local<r>(j));
                    S cst;
                    if (glev)
                        cst = static_cast<S>(slev[(e_of(R, j) >> 3) * 8u + (gidx & 7u)]);
                    else
                        cst = static_cast<S>(gval ? gval[gidx] : 1.0);
                    gf[gidx] = A::mul(A::nrm(a[j]), cst);  // stays in L2 for k_blocksum
                }
            }
            if (sout) {
#pragma unroll
                for (int j = 0; j < 16; ++j) at(e_of(R, j)) = a[j];
                asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
                grp_sync(g);
                if (gt == 0) {
                    const uint32_t sb = su32(stb);
                    tma(true, sb, xs, t >> tshift, 0);
                    if (HM) tma(true, sb + kHalf, xs ^ geo.allq, t >> tshift, 0);
                    asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
                }
                pending = k + kStages;
            } else {
                grp_sync(g);  // levels of the stage read
                issue(k + kStages);
            }
        };
        using R0 = std::integral_constant<int, 0>;
        using R1 = std::integral_constant<int, 1>;
        using R2 = std::integral_constant<int, 2>;
#pragma unroll
        for (int j = 0; j < 16; ++j) a[j] = at(e_of(R0{}, j));
        if (mix) ops_local<V, 0, 4>(a, hp, c, sn, wht);
        if (nrr == 1) {
            finish(R0{});
            continue;
        }
#pragma unroll
        for (int j = 0; j < 16; ++j) at(e_of(R0{}, j)) = a[j];
        grp_sync(g);
#pragma unroll
        for (int j = 0; j < 16; ++j) a[j] = at(e_of(R1{}, j));
        ops_local<V, 4, 4>(a, hp, c, sn, wht);
        if (nrr == 2) {
            finish(R1{});
            continue;
        }
#pragma unroll
        for (int j = 0; j < 16; ++j) at(e_of(R1{}, j)) = a[j];
        grp_sync(g);
#pragma unroll
        for (int j = 0; j < 16; ++j) a[j] = at(e_of(R2{}, j));
        ops_local<V, 8, 1>(a, hp, c, sn, wht);
        finish(R2{});
    }
    if (pending >= 0) {
        if (gt == 0) asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
        issue(pending);
    }
    if (gt == 0) asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
    QCG_SPAN_END(4, g, gt == 0);
}

}  // namespace v4


namespace {
template <typename V>
void set_attrs() {
    QC_CUDA(cudaFuncSetAttribute(v4::k_pass_a<V>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(v4::kSmem)));
    QC_CUDA(cudaFuncSetAttribute(v4::k_pass_b<V>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(v4::kSmem)));
}
int sm_count() {
    static PerDeviceOnce attrs;
    attrs.run([] {
        set_attrs<double2>();
        set_attrs<float2>();
    });
    return device_sm_count();
}
// Slots per launch such that every CTA's contiguous tile range spans <= kDescCap slots
// (a CTA spans at most slots/grid + 3).
int slots_per_launch(int sms) { return (v4::kDescCap - 3) * sms; }
// Persistent grid for `tiles` tiles of n slots. Full grid: min(tiles, SMs). Balanced: the
// smallest grid with the same number of group-tile rounds (two groups per CTA take
// alternate tiles), leaving the other SMs to a concurrently queued chunk. Each launch alone
// is slower with fewer SMs (C2 shape pass A 81 -> 85 us), but with two chunk streams the
// other chunk's kernels start on the freed SMs at once: C2 67.6 -> 66.6 ms per solve
// (tools/grid_bal.sh). So the engine asks for it (F_BALGRID) only when chunks share the
// GPU. QCG_GRID=full|bal forces one; x2|x3: 2 or 3 CTA waves (measured slower, §4a (18)).
uint32_t pass_grid(uint32_t tiles, int n, int sms, uint32_t flags) {
    static const int gmode = [] {  // -1 auto, 0 full, 1 bal, k >= 2: k waves
        const char* e = std::getenv("QCG_GRID");
        if (e && std::string(e) == "bal") return 1;
        if (e && std::string(e) == "full") return 0;
        if (e && e[0] == 'x') return std::max(2, std::atoi(e + 1));
        return -1;
    }();
    const bool full = gmode == 0 || (gmode == -1 && !(flags & F_BALGRID));
    if (gmode >= 2) {
        const uint32_t g = std::min<uint32_t>(tiles, static_cast<uint32_t>(gmode * sms));
        if (static_cast<uint32_t>(n) / std::max<uint32_t>(g, 1) + 3 <= static_cast<uint32_t>(v4::kDescCap)) return g;
    }
    const uint32_t g0 = std::min<uint32_t>(tiles, static_cast<uint32_t>(sms));
    if (full || g0 == 0) return g0;
    const uint32_t rounds = (tiles + 2 * g0 - 1) / (2 * g0);
    const uint32_t g = (tiles + 2 * rounds - 1) / (2 * rounds);
    // the descriptor cache bounds the slots one CTA's tile range may span
    return (static_cast<uint32_t>(n) / g + 3 <= static_cast<uint32_t>(v4::kDescCap)) ? g : g0;
}
}  // namespace

size_t pass4_smem() { return v4::kSmem; }

namespace {
using EncodeTiledFn5 = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                    const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                    const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                    CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
// the launch's contiguous stored states as {16 doubles, 16-amp groups, 2 halves}
EncodeTiledFn5 tensor_encoder() {
    static EncodeTiledFn5 encode = nullptr;
    if (!encode) {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q{};
        QC_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
        if (!fn || q != cudaDriverEntryPointSuccess) internal_error("cuTensorMapEncodeTiled unavailable");
        encode = reinterpret_cast<EncodeTiledFn5>(fn);
    }
    return encode;
}
// {16 scalars (8 amplitudes), 16-amplitude groups, 2 halves}; fp32 rows are 64 bytes
CUtensorMap state_tensor_map(const void* base, uint64_t amps, bool fp32 = false) {
    const EncodeTiledFn5 encode = tensor_encoder();
    CUtensorMap m;
    const cuuint64_t ab = fp32 ? 8 : 16;
    const cuuint64_t dims[3] = {16, amps / 16, 2};
    const cuuint64_t strides[2] = {16 * ab, 8 * ab};
    const cuuint32_t box[3] = {16, 256, 2};
    const cuuint32_t es[3] = {1, 1, 1};
    const CUresult r = encode(&m, fp32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3,
                              const_cast<void*>(base), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                              fp32 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) internal_error("state tensor map: " + std::to_string(static_cast<int>(r)));
    return m;
}
// TMA pass A: default for fp64, and for fp32 at Q >= 21 (fp32 per launch with 2-4 slots:
// q=24 161.9 -> 146.1 us, q=26 313 -> 276; q=20 60.6 -> 58.8 but the C2 bench is 1% slower;
// the C3/C5 fp32 solves are unchanged); QCG_PASS_A=v4|tma forces one kernel
// fp64 TMA pass A kernel: the split-buffer a7 (default) or the ring a5 (QCG_PASS_A=a5)
bool use_a7() {
    static const bool a7 = [] {
        const char* e = std::getenv("QCG_PASS_A");
        return !(e && std::string(e) == "a5");
    }();
    return a7;
}
bool tma_pass_a(bool fp32, int Q) {
    static const int mode = [] {
        const char* e = std::getenv("QCG_PASS_A");
        if (e && std::string(e) == "v4") return 0;
        if (e && std::string(e) == "tma") return 1;
        return 2;
    }();
    return mode == 1 || (mode == 2 && (!fp32 || Q >= 21));
}
template <typename V>
void a5_attr() {
    static PerDeviceOnce attr;
    attr.run([] {
        QC_CUDA(cudaFuncSetAttribute(v4::k_pass_a5<V, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(v4::kSmem + 1024)));
        QC_CUDA(cudaFuncSetAttribute(v4::k_pass_a5<V, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(v4::kSmem + 1024)));
        QC_CUDA(cudaFuncSetAttribute(v4::k_pass_a7<V, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(v4::kA7Smem + 1024)));
        QC_CUDA(cudaFuncSetAttribute(v4::k_pass_a7<V, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(v4::kA7Smem + 1024)));
    });
}
}  // namespace

int launch_pass_a4(const SlotDesc* d_slots, const LayerParam* d_lp, int layer, int Q, uint32_t flags,
                   int n_slots, cudaStream_t stream, bool pdl, const void* state_base) {
    const int sms = sm_count();
    const bool fp32 = flags & F_FP32;
    if (tma_pass_a(fp32, Q) && state_base) {
        if (fp32)
            a5_attr<float2>();
        else
            a5_attr<double2>();
        int launches = 0;
        for (int s0 = 0; s0 < n_slots; s0 += slots_per_launch(sms)) {
            const int n = std::min(n_slots - s0, slots_per_launch(sms));
            const uint32_t tiles = static_cast<uint32_t>(n) << (Q - 12);
            const uint32_t grid = pass_grid(tiles, n, sms, flags);
            const CUtensorMap tm = state_tensor_map(
                static_cast<const char*>(state_base) + (static_cast<size_t>(s0) << Q) * (fp32 ? 8 : 16),
                static_cast<uint64_t>(n) << Q, fp32);
            const bool init = flags & F_INIT;
            auto* kern = fp32 ? (init ? v4::k_pass_a5<float2, true> : v4::k_pass_a5<float2, false>)
                              : nullptr;
            auto* kern64 = init ? v4::k_pass_a5<double2, true> : v4::k_pass_a5<double2, false>;
            if (fp32)
                launch_ex(kern, dim3(grid), dim3(v4::kThreads), v4::kSmem + 1024, stream,
                          pdl || s0 > 0, d_slots + s0, d_lp, layer, Q, flags, tiles, tm);
            else if (use_a7()) {
                // When a group hands the output buffer back: right after its store has read it
                // (default; the elected lane waits ~0.5-1.5k clk) or after round 0 of its next
                // tile (QCG_A7_RELEASE=late; =init: early only on the first layer). Measured:
                // q=20 x 21 pass A 84.5 -> 83.1 us, C2 68.95 -> 68.77 ms per solve.
                static const int rel = [] {
                    const char* e = std::getenv("QCG_A7_RELEASE");
                    if (e && std::string(e) == "late") return 0;
                    if (e && std::string(e) == "init") return 1;
                    return 2;
                }();
                const uint32_t ef = (rel == 2 || (rel == 1 && init)) ? static_cast<uint32_t>(F_A7EARLY) : 0u;
                launch_ex(init ? v4::k_pass_a7<double2, true> : v4::k_pass_a7<double2, false>, dim3(grid),
                          dim3(v4::kThreads), v4::kA7Smem + 1024, stream, pdl || s0 > 0, d_slots + s0, d_lp,
                          layer, Q, flags | ef, tiles, tm);
            }
            else
                launch_ex(kern64, dim3(grid), dim3(v4::kThreads), v4::kSmem + 1024, stream,
                          pdl || s0 > 0, d_slots + s0, d_lp, layer, Q, flags, tiles, tm);
            ++launches;
        }
        return launches;
    }
    int launches = 0;
    for (int s0 = 0; s0 < n_slots; s0 += slots_per_launch(sms)) {
        const int n = std::min(n_slots - s0, slots_per_launch(sms));
        const uint32_t tiles = static_cast<uint32_t>(n) << (Q - 12);
        const uint32_t grid = pass_grid(tiles, n, sms, flags);
        if (fp32)
            launch_ex(v4::k_pass_a<float2>, dim3(grid), dim3(v4::kThreads), v4::kSmem, stream,
                      pdl || s0 > 0, d_slots + s0, d_lp, layer, Q, flags, tiles);
        else
            launch_ex(v4::k_pass_a<double2>, dim3(grid), dim3(v4::kThreads), v4::kSmem, stream,
                      pdl || s0 > 0, d_slots + s0, d_lp, layer, Q, flags, tiles);
        ++launches;
    }
    return launches;
}

namespace {
using B5Kernel = void (*)(const SlotDesc*, const LayerParam*, int, int, HighPass, uint32_t, uint32_t,
                          v4::B5Geo, CUtensorMap);
template <typename V, int NT, int HM>
B5Kernel b5_kernel() {
    static PerDeviceOnce attr;
    attr.run([] {
        QC_CUDA(cudaFuncSetAttribute(v4::k_pass_b5<V, NT, HM>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(v4::kSmem + 1024)));
    });
    return v4::k_pass_b5<V, NT, HM>;
}
template <typename V>
B5Kernel b5_lookup_t(int nt, int hm) {
    switch (nt * 2 + hm) {
        case 1: return b5_kernel<V, 0, 1>();
        case 2: return b5_kernel<V, 1, 0>();
        case 3: return b5_kernel<V, 1, 1>();
        case 4: return b5_kernel<V, 2, 0>();
        case 5: return b5_kernel<V, 2, 1>();
        case 6: return b5_kernel<V, 3, 0>();
        case 7: return b5_kernel<V, 3, 1>();
        case 8: return b5_kernel<V, 4, 0>();
        case 9: return b5_kernel<V, 4, 1>();
        case 10: return b5_kernel<V, 5, 0>();
        case 11: return b5_kernel<V, 5, 1>();
        case 12: return b5_kernel<V, 6, 0>();
        case 13: return b5_kernel<V, 6, 1>();
        case 14: return b5_kernel<V, 7, 0>();
        case 15: return b5_kernel<V, 7, 1>();
        case 16: return b5_kernel<V, 8, 0>();
        case 17: return b5_kernel<V, 8, 1>();
        case 18: return b5_kernel<V, 9, 0>();
        default: return nullptr;
    }
}
B5Kernel b5_lookup(int nt, int hm, bool fp32) {
    return fp32 ? b5_lookup_t<float2>(nt, hm) : b5_lookup_t<double2>(nt, hm);
}

// HighPass -> 5-D box geometry of k_pass_b5 over a launch's contiguous states. False if
// the pass lacks the [targets][mirror][pads] run structure (then v4 runs it).
struct B5Plan {
    int nt = 0, hm = 0;
    v4::B5Geo geo{};
    cuuint64_t dims[5];
    cuuint64_t strides[4];
    cuuint32_t box[5];
};
bool b5_plan(const HighPass& hp, int Q, bool fp32, B5Plan& P) {
    const cuuint64_t ab = fp32 ? 8 : 16;  // bytes per amplitude
    int nt = 0, npad = 0, tstart = -1;
    uint32_t tmask = 0, pmask = 0;
    for (int b = 0; b < kHighBits; ++b) {
        if (hp.kind[b] == 1) {
            if (npad || P.hm) return false;  // targets come first
            const int bit = __builtin_ctz(hp.mask[b]);
            if (tstart < 0) tstart = bit;
            if (bit != tstart + nt) return false;  // one contiguous run
            tmask |= hp.mask[b];
            ++nt;
        } else if (hp.kind[b] == 2) {
            if (npad || b != nt) return false;
            P.hm = 1;
        } else {
            if (hp.mask[b] != (1u << (3 + npad))) return false;  // pads: bits 3, 4, ...
            pmask |= hp.mask[b];
            ++npad;
        }
    }
    P.nt = nt;
    const uint32_t allq = (Q == 32) ? ~0u : ((1u << Q) - 1u);
    const uint32_t fr = allq & ~(7u | tmask | pmask);  // free bits incl. a pinned mirror bit
    if (!fr) return false;
    const int lo = __builtin_ctz(fr);
    int lo_bits = 0;
    while (lo + lo_bits < Q && ((fr >> (lo + lo_bits)) & 1u)) ++lo_bits;
    const uint32_t rest = fr & ~(((1u << lo_bits) - 1u) << lo);
    int hi = Q, hi_bits = 0;
    if (rest) {
        hi = __builtin_ctz(rest);
        hi_bits = Q - hi;
        if ((rest >> hi) != (1u << hi_bits) - 1u) return false;  // must run up to Q-1
    }
    if (P.hm && hi_bits) return false;  // a mirror pass ends at the top stored bit
    P.geo = v4::B5Geo{static_cast<uint32_t>(lo), (1u << lo_bits) - 1u, static_cast<uint32_t>(hi),
                      (1u << hi_bits) - 1u, static_cast<uint32_t>(hi_bits), allq};
    // dims: 0 columns, 1 pads (or the targets' low 8 when there are no pads), 2 targets
    // (or the 9th target, or size 1), 3 low free run, 4 high free run x slots (size set
    // per launch); row order = pb5's r0 = pads | targets << npad
    P.dims[0] = P.box[0] = 16;
    if (npad) {
        P.dims[1] = P.box[1] = 1u << npad;
        P.strides[0] = 8 * ab;
        P.dims[2] = P.box[2] = 1u << nt;
        P.strides[1] = nt ? (ab << tstart) : 16ull;
    } else {
        P.dims[1] = P.box[1] = 1u << std::min(nt, 8);
        P.strides[0] = ab << tstart;
        P.dims[2] = P.box[2] = nt == 9 ? 2u : 1u;
        P.strides[1] = nt == 9 ? (ab << (tstart + 8)) : 16ull;
    }
    P.dims[3] = 1ull << lo_bits;
    P.box[3] = 1;
    P.strides[2] = ab << lo;
    P.box[4] = 1;
    P.strides[3] = ab << hi;
    return (nt + P.hm + npad) == kHighBits && b5_lookup(nt, P.hm, fp32) != nullptr;
}
// Pass B kernel: the TMA kernel (tensor stores) where it measured faster: fp64 at Q >= 25
// (q=26: 8 slots 1687 -> 1505 us with its early stage refill; at q = 20..25 v4's
// per-thread gathers are 3-7% faster in round 2: q=24 x 12 slots 544 vs 527 us, C3
// 1311 -> 1275 ms per solve), fp32 at every size (v4 moves fp32 in 8-byte cp.async / STG
// per amplitude: q=20 65 -> 54 us, q=26 372 -> 255 us) (profiles/r1_pass_b_tma.txt).
// QCG_PASS_B=v4|tma forces one.
bool tma_pass_b(int Q, bool fp32) {
    static const int mode = [] {
        const char* e = std::getenv("QCG_PASS_B");
        if (e && std::string(e) == "v4") return 0;
        if (e && std::string(e) == "tma") return 1;
        return 2;
    }();
    return mode == 1 || (mode == 2 && (fp32 || Q >= 25));
}
}  // namespace

int launch_pass_b4(const SlotDesc* d_slots, const LayerParam* d_lp, int layer, int Q,
                   const HighPass& hp, uint32_t flags, int n_slots, cudaStream_t stream, bool pdl,
                   const void* state_base) {
    const int sms = sm_count();
    const bool fp32 = flags & F_FP32;
    int launches = 0;
    B5Plan P;
    if (tma_pass_b(Q, fp32) && state_base && b5_plan(hp, Q, fp32, P)) {
        static const bool tstore = [] {  // QCG_B5_STORE=stg: results leave from registers
            const char* e = std::getenv("QCG_B5_STORE");
            return !(e && std::string(e) == "stg");
        }();
        const B5Kernel kern = b5_lookup(P.nt, P.hm, fp32);
        for (int s0 = 0; s0 < n_slots; s0 += slots_per_launch(sms)) {
            const int n = std::min(n_slots - s0, slots_per_launch(sms));
            const uint32_t tiles = static_cast<uint32_t>(n) << (Q - 12);
            const uint32_t grid = pass_grid(tiles, n, sms, flags);
            P.dims[4] = (1ull << P.geo.hi_bits) * static_cast<cuuint64_t>(n);
            CUtensorMap tm;
            const cuuint32_t es[5] = {1, 1, 1, 1, 1};
            const CUresult r = tensor_encoder()(
                &tm, fp32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 5,
                const_cast<char*>(static_cast<const char*>(state_base)) + (static_cast<size_t>(s0) << Q) * (fp32 ? 8 : 16),
                P.dims, P.strides, P.box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                fp32 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B,
                CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            if (r != CUDA_SUCCESS) internal_error("pass B tensor map: " + std::to_string(static_cast<int>(r)));
            // refill a stored stage before waiting for the next tile: measured faster at 26
            // qubits (8 slots 1541 -> 1502 us), slower at 24 (22 slots 975 -> 988 us);
            // QCG_B5_EARLY=0|1 forces it
            static const int early_env = [] {
                const char* e = std::getenv("QCG_B5_EARLY");
                return e ? (e[0] == '1' ? 1 : 0) : -1;
            }();
            const uint32_t early = (early_env == 1 || (early_env < 0 && Q >= 25)) ? static_cast<uint32_t>(F_B5EARLY) : 0u;
            launch_ex(kern, dim3(grid), dim3(v4::kThreads), v4::kSmem + 1024, stream, pdl || s0 > 0,
                      d_slots + s0, d_lp, layer, Q, hp, flags | (tstore ? F_TSTORE : 0u) | early, tiles, P.geo, tm);
            ++launches;
        }
        return launches;
    }
    for (int s0 = 0; s0 < n_slots; s0 += slots_per_launch(sms)) {
        const int n = std::min(n_slots - s0, slots_per_launch(sms));
        const uint32_t tiles = static_cast<uint32_t>(n) << (Q - 12);
        const uint32_t grid = pass_grid(tiles, n, sms, flags);
        static const uint32_t nolev = [] {
            const char* e = std::getenv("QCG_LEVREG");
            return (e && e[0] == '0') ? static_cast<uint32_t>(F_NOLEVREG) : 0u;
        }();
        if (fp32)
            launch_ex(v4::k_pass_b<float2>, dim3(grid), dim3(v4::kThreads), v4::kSmem, stream,
                      pdl || s0 > 0, d_slots + s0, d_lp, layer, Q, hp, flags | nolev, tiles);
        else
            launch_ex(v4::k_pass_b<double2>, dim3(grid), dim3(v4::kThreads), v4::kSmem, stream,
                      pdl || s0 > 0, d_slots + s0, d_lp, layer, Q, hp, flags | nolev, tiles);
        ++launches;
    }
    return launches;
}

#ifdef QCG_TRACE
extern "C" int qc_trace_read(long long* out, int n) {
    const int cap = v4::kTraceCtas * 2 * v4::kTraceTiles * v4::kTraceEv;
    if (n > cap) n = cap;
    if (cudaMemcpyFromSymbol(out, v4::g_trace, n * sizeof(long long)) != cudaSuccess) return 4;
    static long long zero[v4::kTraceCtas * 2 * v4::kTraceTiles * v4::kTraceEv] = {};
    cudaMemcpyToSymbol(v4::g_trace, zero, sizeof(zero));
    return 0;
}
extern "C" int qc_trace_read_ctas(unsigned long long* out, int n) {
    if (n > v4::kTraceMaxCtas * 4) n = v4::kTraceMaxCtas * 4;
    if (cudaMemcpyFromSymbol(out, v4::g_cta, n * sizeof(unsigned long long)) != cudaSuccess) return 4;
    static unsigned long long zero[v4::kTraceMaxCtas * 4] = {};
    cudaMemcpyToSymbol(v4::g_cta, zero, sizeof(zero));
    return 0;
}
#endif
}  // namespace qcg
#ifdef QCG_TRACE
QCG_SPAN_READER(qc_span_read_pass)
#endif
