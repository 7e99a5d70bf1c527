// Internal declarations shared by the host C++ (g++) and the CUDA translation units.
#pragma once

#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <atomic>
#include <cstdint>
#include <mutex>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace qcg {

// NVTX ranges around the hot-path stages (SURVEY 5 tracing row): visible under nsys / ncu
// --nvtx; the header-only NVTX v3 API is a no-op branch when no tool is attached.
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};

// Status-coded exception; the C-ABI layer maps it to QC_ERR_* (qcgpu.h).
struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
[[noreturn]] inline void config_error(const std::string& m) { throw Error(1, m); }
[[noreturn]] inline void resource_error(const std::string& m) { throw Error(2, m); }
[[noreturn]] inline void internal_error(const std::string& m) { throw Error(4, m); }

void cuda_fail(cudaError_t e, const char* what, const char* file, int line);
#define QC_CUDA(x)                                                        \
    do {                                                                  \
        cudaError_t err_ = (x);                                           \
        if (err_ != cudaSuccess) ::qcg::cuda_fail(err_, #x, __FILE__, __LINE__); \
    } while (0)

// One-time setup per CUDA device, thread-safe. CUDA function attributes (the dynamic
// shared-memory opt-ins) live in each device's context, so an engine on another device of
// the same process needs its own; engines may also be driven from several host threads.
struct PerDeviceOnce {
    std::atomic<uint64_t> done{0};
    std::mutex mu;
    template <typename F>
    void run(F&& f) {
        int d = 0;
        QC_CUDA(cudaGetDevice(&d));
        const uint64_t bit = uint64_t{1} << (d & 63);
        if (done.load(std::memory_order_acquire) & bit) return;
        std::lock_guard<std::mutex> lk(mu);
        if (done.load(std::memory_order_relaxed) & bit) return;
        f();
        done.fetch_or(bit, std::memory_order_release);
    }
};
// SM count of the current device (cached per device).
inline int device_sm_count() {
    static std::atomic<int> cache[64];
    int d = 0;
    QC_CUDA(cudaGetDevice(&d));
    int v = cache[d & 63].load(std::memory_order_relaxed);
    if (!v) {
        QC_CUDA(cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, d));
        cache[d & 63].store(v, std::memory_order_relaxed);
    }
    return v;
}

// Largest simulated subgraph (stored half-state 2^25 amplitudes = 512 MiB fp64).
constexpr int kMaxQubits = 30;
constexpr int kLowBits = 12;   // pass A tile: 2^12 contiguous stored amplitudes
constexpr int kBlock = 4096;   // statevector.hpp:53 blocked_sum block

// ---------------------------------------------------------------------------
// Device-side descriptors. One "slot" = one state buffer evaluating one point.
// ---------------------------------------------------------------------------
struct SlotDesc {
    double2* state;        // 2^Q stored amplitudes
    double* fbuf;          // 2^Q per-amplitude expectation terms (scratch)
    const uint16_t* lev;   // integral cut levels, 2^Q entries (or null): the expectation's cost
    const double* val;     // fractional cut values, 2^Q entries (or null)
    const uint16_t* plev;  // phase LUT index per z: the integral levels, or for a fractional
                           // table the index of val[z] among its distinct values (qc_frac.cu);
                           // null: device sincos phases
    double amp0;           // 1/sqrt(2^q)
    int32_t layer_base;    // first LayerParam of this slot
    int32_t pad;
};

struct LayerParam {
    const double2* lut;    // integral: host-built std::polar(1,-gamma*c) table (device copy)
    double gamma;          // fractional path: per-amplitude phase angle factor
    double c, s;           // cos(beta), sin(beta) (host libm, statevector.hpp:192)
    int32_t phase;         // gamma != 0 (statevector.hpp:149)
    int32_t mix;           // !(s == 0 && c == 1) (statevector.hpp:193)
    int32_t lut_len;       // entries of lut
    int32_t pad;
};

// Mode flags for a launch chain.
enum : uint32_t {
    F_INIT = 1u,        // first layer starts from |+> (no state read)
    F_EXPECT = 2u,      // compute the blocked expectation after the last layer
    F_STATE_OUT = 4u,   // final state must be written back
    F_SYM = 8u,         // half-state storage (complement symmetry), else full state
    F_FP32 = 64u,       // optional fp32 mode: float2 amplitudes, float f(z), fp32 LUTs (1e-4)
    F_TSTORE = 128u,    // pass B (TMA): results leave by tensor stores (default)
    F_B5EARLY = 512u,   // pass B (TMA): refill a stored stage before the next tile's wait
    F_NOLEVREG = 256u,  // pass B (v4) f pass: levels read after the refill (experiment)
    F_A7EARLY = 2048u,  // split-buffer pass A: release the output buffer right after its store
    F_WHT = 1024u,      // fp32 mode only: Walsh–Hadamard form of the RX mixer (qc_amp.cuh)
    F_BALGRID = 4096u,  // chunks share the GPU: balanced pass grids (qc_pass.cu pass_grid)
};

// One high (gather) pass: 3 column bits (0,1,2) + kHighBits tile bits.
constexpr int kHighBits = 9;
struct HighPass {
    uint32_t mask[kHighBits];  // tile bit masks (single bit, or ALL for the mirror pseudo-bit)
    int32_t kind[kHighBits];   // 0 batch (no op), 1 RX target, 2 mirror (RX on qubit q-1)
    uint32_t freemask;         // stored-index bits enumerated by the tile index
    int32_t mpos;              // tile-bit index of the mirror pseudo-bit, -1 if none
};

struct ChainPlan {
    int Q;                         // stored index bits
    bool sym;
    bool onchip;                   // Q <= 12: whole state per CTA
    std::vector<HighPass> high;    // passes after pass A (bits >= 12)
};
ChainPlan plan_chain(int q, bool sym);

// ---------------------------------------------------------------------------
// Live kernel profiling: CUDA events recorded on the launching stream around each
// kernel, with the kernel's algorithmic bytes (bench.py roofline).
// ---------------------------------------------------------------------------
enum KernelKind : int {
    K_LEVELS = 0, K_ONCHIP, K_PASS_LOW, K_PASS_HIGH, K_BLOCKSUM, K_FINALSUM, K_TOPK,
    K_MERGE_TABLES, K_MERGE_SEARCH, K_MERGE_OTHER, K_COUNT
};
struct Prof {
    bool on = false;
    int stride = 1;  // record one launch in `stride` per kernel kind (sampling keeps the
                     // event overhead out of the timed region; averages stay per launch)
    uint64_t seen[K_COUNT] = {};
    bool open_ = false;
    struct Rec {
        int kind;
        cudaEvent_t a, b;
        double bytes, ops;
    };
    std::vector<Rec> recs;
    std::vector<cudaEvent_t> pool;
    double ms[K_COUNT] = {};
    double bytes[K_COUNT] = {};
    double ops[K_COUNT] = {};  // algorithmic FP64 operations (DMUL/DADD, no FMA)
    uint64_t count[K_COUNT] = {};
    cudaEvent_t ev() {
        if (!pool.empty()) {
            cudaEvent_t e = pool.back();
            pool.pop_back();
            return e;
        }
        cudaEvent_t e;
        cudaEventCreate(&e);
        return e;
    }
    void begin(int kind, double b, cudaStream_t s, double fp64_ops = 0.0) {
        open_ = false;
        if (!on) return;
        if ((seen[kind]++ % static_cast<uint64_t>(stride)) != 0) return;
        Rec r{kind, ev(), ev(), b, fp64_ops};
        cudaEventRecord(r.a, s);
        recs.push_back(r);
        open_ = true;
    }
    void end(cudaStream_t s) {
        if (!on || !open_ || recs.empty()) return;
        open_ = false;
        cudaEventRecord(recs.back().b, s);
        if (recs.size() >= 4096) resolve();
    }
    void resolve() {  // accumulate completed records
        for (auto& r : recs) {
            cudaEventSynchronize(r.b);
            float t = 0.f;
            cudaEventElapsedTime(&t, r.a, r.b);
            ms[r.kind] += t;
            bytes[r.kind] += r.bytes;
            ops[r.kind] += r.ops;
            count[r.kind] += 1;
            pool.push_back(r.a);
            pool.push_back(r.b);
        }
        recs.clear();
    }
    void reset() {
        resolve();
        for (int k = 0; k < K_COUNT; ++k) ms[k] = bytes[k] = ops[k] = 0, count[k] = 0, seen[k] = 0;
    }
    ~Prof() {
        for (auto& r : recs) {
            cudaEventDestroy(r.a);
            cudaEventDestroy(r.b);
        }
        for (auto e : pool) cudaEventDestroy(e);
    }
};

// Per-layer slot counts of one chain launch (for the algorithmic byte counts).
struct ChainStats {
    std::vector<int> phase, mix;  // per layer: slots with the phase / mixer active
};

// Launchers (qc_kernels.cu). All asynchronous on `stream`; return #kernels launched.
int launch_levels(const uint32_t* d_eu, const uint32_t* d_ev, const double* d_ew, int m,
                  int Q, bool integral, uint16_t* d_lev, double* d_val, cudaStream_t stream);
// qc_frac.cu: distinct values of a non-integral cost table (exact phases via a host LUT)
size_t distinct_scratch_bytes(uint32_t N);
const unsigned long long* launch_distinct(const double* d_val, uint32_t N, void* scratch, int* d_count,
                                          cudaStream_t st);
void launch_index_of(const double* d_val, uint32_t N, const unsigned long long* d_uniq, int D, uint16_t* d_lev,
                     cudaStream_t st);
constexpr int kMaxDistinct = 65535;  // uint16 level indices
// d_tickets: n_slots zero-initialised counters (left zeroed on return).
// d_fbuf: the f buffer of slot 0 of this launch (slots contiguous, 2^Q doubles each).
int launch_chain(const ChainPlan& plan, const SlotDesc* d_slots, const LayerParam* d_lp,
                 int n_slots, int p, uint32_t flags, double* d_fbuf, double* d_partials,
                 unsigned* d_tickets, double* d_out, cudaStream_t stream,
                 const ChainStats* stats = nullptr, Prof* prof = nullptr,
                 const void* state_base = nullptr, cudaEvent_t passes_done = nullptr);
size_t partials_per_slot(const ChainPlan& plan);
// v4 streaming passes (qc_pass.cu): persistent, one CTA per SM. pdl: launched with
// programmatic stream serialization (the kernel's prologue overlaps the previous kernel's
// tail; it waits with griddepcontrol.wait before touching state memory). Only for a
// kernel whose stream predecessor is a kernel of the same chain.
// state_base: the stored state of d_slots[0] (slots contiguous), for the TMA variant
int launch_pass_a4(const SlotDesc* d_slots, const LayerParam* d_lp, int layer, int Q, uint32_t flags,
                   int n_slots, cudaStream_t stream, bool pdl = false,
                   const void* state_base = nullptr);
int launch_pass_b4(const SlotDesc* d_slots, const LayerParam* d_lp, int layer, int Q,
                   const HighPass& hp, uint32_t flags, int n_slots, cudaStream_t stream,
                   bool pdl = false, const void* state_base = nullptr);

// cudaLaunchKernelEx with the programmatic-stream-serialization attribute
template <typename... KArgs, typename... Args>
void launch_ex(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
               bool pdl, Args&&... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    QC_CUDA(cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...));
}

// Top-K over the classes of one state (qc_topk.cu). Writes k (bits, prob) pairs,
// ordered by (prob desc, lex asc) (qaoa.hpp:179-182). d_scratch sized by topk_scratch_bytes.
size_t topk_scratch_bytes(int q, bool fold, int k);
// fp32: d_state holds float2 amplitudes (F_FP32 chains)
int launch_topk(const double2* d_state, int q, bool sym, bool fold, int k, void* d_scratch,
                uint32_t* d_bits, double* d_probs, cudaStream_t stream, Prof* prof = nullptr,
                bool fp32 = false);

}  // namespace qcg
