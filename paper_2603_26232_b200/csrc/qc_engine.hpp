// Engine internals shared by qc_engine.cpp and qc_pipeline.cpp.
#pragma once

#include <cuda_runtime.h>

#include <cstdlib>

#include <cstdint>
#include <string>
#include <vector>

#include "../../include/qcgpu.h"
#include "qc_internal.hpp"
#include "qc_merge.hpp"
#include <memory>

namespace qcg {

// Validated host copy of a qcut::Graph (graph.hpp:37-50 add_edge rules) plus the
// CostTable integrality rule (statevector.hpp:83-89).
struct HostGraph {
    int n = 0;
    std::vector<uint32_t> u, v;
    std::vector<double> w;
    bool integral = true;
    double total = 0.0;
    bool all_int = true;  // every weight a nonnegative integer, total <= 4e18 (merge scoring)
};
HostGraph load_graph(const qc_graph* g);

struct DevBuf {
    void* p = nullptr;
    size_t cap = 0;
    void* get(size_t bytes);
    void release();
    ~DevBuf() { release(); }
};
struct HostBuf {
    void* p = nullptr;
    size_t cap = 0;
    void* get(size_t bytes);
    ~HostBuf();
};

// Device cut table of one graph: 2^Q entries (levels or values).
struct DevGraph {
    int q = 0, Q = 0;
    bool sym = false;
    bool integral = true;
    bool unit_cost = false;  // norm_sq: cost 1 everywhere
    int lut_len = 0;
    uint16_t* lev = nullptr;   // integral: cut levels; else (when set) indices into fvals
    double* val = nullptr;     // non-integral: C(z) in edge order (the expectation's cost)
    std::vector<double> fvals; // non-integral: distinct values of val (host), the phase LUT's arguments
};

struct EvalPoint {
    int g;            // graph index
    const double* x;  // packed [gammas..., betas...]
};

// Staging + completion event of one in-flight launch chain ("chunk" of slots).
// Identity of a captured chain: everything the recorded nodes depend on (shape, flags and
// every buffer address baked into kernel arguments or copy nodes).
struct ChainKey {
    int Q = -1, n = 0, p = 0;
    bool sym = false;
    uint32_t flags = 0;
    const void* ptr[8] = {};  // states, f, partials, tickets, out, device/host staging, host out
    size_t copy_bytes = 0;
    bool operator==(const ChainKey& o) const {
        if (Q != o.Q || n != o.n || p != o.p || sym != o.sym || flags != o.flags || copy_bytes != o.copy_bytes)
            return false;
        for (int i = 0; i < 8; ++i)
            if (ptr[i] != o.ptr[i]) return false;
        return true;
    }
};

struct ChunkCtx {
    DevBuf dstage;
    HostBuf hstage, hout;
    cudaEvent_t done = nullptr;
    int n = 0;
    uint32_t flags = 0;
    double* d_out = nullptr;
    cudaStream_t st = nullptr;  // stream the chunk runs on (null: the engine stream)
    bool shared = false;        // other chunks run concurrently on other streams
    // lockstep ping-pong: `passes` is recorded after this chunk's last pass kernel (before
    // its block sum); the chunk's next step first waits on `wait_on` (the previous chunk's
    // `passes`), so chunks' pass chains alternate instead of interleaving launch by launch
    cudaEvent_t passes = nullptr;
    cudaEvent_t wait_on = nullptr;
    // CUDA graph of this chunk's step (staging upload -> launch chain -> result read),
    // captured once per ChainKey and replayed each lockstep step
    cudaGraphExec_t gexec = nullptr;
    ChainKey gkey;
    int glaunches = 0;
    ChunkCtx() = default;
    ChunkCtx(const ChunkCtx&) = delete;
    ChunkCtx& operator=(const ChunkCtx&) = delete;
    ~ChunkCtx() {
        if (gexec) cudaGraphExecDestroy(gexec);
        if (done) cudaEventDestroy(done);
        if (passes) cudaEventDestroy(passes);
    }
};

}  // namespace qcg

struct qc_engine {
    int device = 0;
    cudaStream_t stream = nullptr;
    cudaStream_t aux[3] = {nullptr, nullptr, nullptr};  // extra streams: chunks overlap on the device
    uint64_t launches = 0;
    uint64_t mem_budget = 0;
    mutable size_t auto_budget = 0;  // 60% of the free HBM seen at first use
    qcg::DevBuf tables, states, fbuf, partials, outd, stage, edges, topk_scratch, topk_out, tickets;
    qcg::DevBuf distinct;  // scratch of the non-integral tables' distinct-value search
    qcg::HostBuf hstage, hout;
    qcg::HostBuf topk_host;  // final top-K results of a batch, written by the kernels (zero-copy)
    qcg::Prof prof;        // live per-kernel CUDA-event timing (qc_engine_profile)
    qcg::DeviceArena merge_arena;                           // merge scratch, reused
    std::vector<std::unique_ptr<qcg::ChunkCtx>> chunk_pool;  // per-chunk staging, reused
    uint64_t h2d = 0, d2h = 0;  // bytes copied host<->device by this engine
    uint64_t graph_captures = 0;  // chunk chains captured as CUDA graphs
    // chunk chains run as captured CUDA graphs (QCG_GRAPH=0: direct launches)
    static bool use_graphs() {
        static const bool on = [] {
            const char* e = std::getenv("QCG_GRAPH");
            return !(e && e[0] == '0');
        }();
        return on;
    }
    double host_wait_s = 0.0, host_prep_s = 0.0;  // lockstep loop: waiting vs preparing
    // split of host_prep_s (QCG_HOST_PROFILE): results read + NM tell, staging build
    // (cos/sin, phase LUTs), launch (H2D record / graph launch)
    double host_tell_s = 0.0, host_stage_s = 0.0, host_launch_s = 0.0;
    uint64_t host_steps = 0;
    double t_optimize_s = 0.0, t_final_s = 0.0, t_merge_s = 0.0, t_execute_s = 0.0;

    // Build the device cut tables of graphs (sym: half state) into `target` (default:
    // the engine's shared `tables` buffer, valid until the next prepare()).
    std::vector<qcg::DevGraph> prepare(const std::vector<qcg::HostGraph>& hg, bool allow_sym,
                                       bool unit_cost = false, qcg::DevBuf* target = nullptr);
    void h2d_copy(void* dst, const void* src, size_t bytes, cudaStream_t st = nullptr);
    void d2h_copy(void* dst, const void* src, size_t bytes, cudaStream_t st = nullptr);
    // Evaluate points sharing (q, p) in chunks; out[k] = <C> of point k.
    // flags: qcg::F_* (F_STATE_OUT keeps each chunk's states for `on_chunk`).
    size_t max_slots(int Q, bool onchip) const;
    // Slots per pipelined chunk: sized so a chunk's working set stays L2-resident.
    size_t chunk_slots(int Q, bool onchip, size_t n) const;
    // Grow the shared slot buffers to `slots` slots of 2^Q (no work may be in flight).
    void reserve(int Q, bool need_fbuf, size_t slots);
    // Asynchronous chain on slots [slot0, slot0+n); wait_chunk collects <C> (F_EXPECT).
    void enqueue_chunk(const std::vector<qcg::DevGraph>& dg, const qcg::EvalPoint* pts, int n,
                       int p, uint32_t flags, size_t slot0, qcg::ChunkCtx& c);
    void wait_chunk(qcg::ChunkCtx& c, double* out);
    void eval_chunk(const std::vector<qcg::DevGraph>& dg, const qcg::EvalPoint* pts, int n, int p,
                    uint32_t flags, double* out);
    qcg::ChunkCtx sync_ctx;
    void eval(const std::vector<qcg::DevGraph>& dg, const std::vector<qcg::EvalPoint>& pts, int p,
              double* out);
    double2* slot_state(int q, bool sym, int k, bool fp32 = false);
    // 64: the exact fp64 path (default, bit-identical to the reference); 32: optional fp32
    // mode for the batched solve/eval paths (statevector-level calls stay fp64)
    int precision = 64;
    int mixer = 0;  // QC_MIXER_RX / QC_MIXER_WHT (fp32 mode only)
    uint32_t fp_flag() const {
        return precision == 32 ? (qcg::F_FP32 | (mixer == 1 ? qcg::F_WHT : 0u)) : 0u;
    }
    void sync();
};

namespace qcg {
// Lockstep batched optimisation (qaoa.hpp:85-117 for many graphs).
struct OptimizeOut {
    std::vector<double> params;
    double expectation = 0.0;
    int evals = 0;
};
std::vector<OptimizeOut> optimize_batch(qc_engine* e, const std::vector<DevGraph>& dg,
                                        const std::vector<int>& layers,
                                        const std::vector<int>& budget,
                                        const std::vector<uint64_t>& seeds,
                                        const std::vector<double>& tol,
                                        std::vector<std::vector<double>>* trace_x,
                                        std::vector<std::vector<double>>* trace_f);

struct SolveOut {
    int width = 0;
    bool folded = true;
    std::vector<uint32_t> bits;
    std::vector<double> probs;
    std::vector<double> params;
    double expectation = 0.0;
    int evals = 0;
};
void validate_solve(const std::vector<HostGraph>& hg, const std::vector<qc_solve_options>& opts);
std::vector<SolveOut> solve_batch(qc_engine* e, const std::vector<HostGraph>& hg,
                                  const std::vector<qc_solve_options>& opts);
// solve on graphs whose device cut tables are already resident (qc_pipeline_*)
std::vector<SolveOut> solve_prepared(qc_engine* e, const std::vector<HostGraph>& hg,
                                     const std::vector<DevGraph>& dg,
                                     const std::vector<qc_solve_options>& opts);

void set_error(const std::string& msg);

}  // namespace qcg
