/*
 * qcgpu.h — C-ABI of the B200-native ParaQAOA hot path (libqcgpu.so).
 *
 * Drop-in boundary for the reference's C++ API in /root/reference/proj/include/qcut/:
 * every entry point below replaces one reference function (cited per declaration),
 * takes caller-owned POD buffers (host memory), and reports errors as status codes
 * instead of exceptions. include/qcut_gpu.hpp rethrows them as the reference's
 * exception types (errors.hpp:8-24), so callers such as pipeline.hpp:263 keep their
 * error handling unchanged.
 *
 * Status codes: QC_OK 0, QC_ERR_CONFIG 1 (config_error), QC_ERR_RESOURCE 2
 * (resource_error, including device out-of-memory), QC_ERR_IO 3 (io_error),
 * QC_ERR_INTERNAL 4 (CUDA failure / internal). qc_last_error() returns the message
 * of the calling thread's last failure.
 *
 * Amplitude buffers are interleaved complex128 (re, im) of length 2^q, basis index z
 * with bit v = vertex v (statevector.hpp:22-23), i.e. the memory layout of
 * std::vector<std::complex<double>>.
 *
 * Numerics: fp64, bit-identical to the reference's canonical (no-FMA) build on the
 * integral-weight path (the phase LUT is built on the host with std::polar exactly
 * as statevector.hpp:154-157; the device uses explicitly rounded mul/add, ascending
 * RX targets and the 4096-blocked sequential expectation of statevector.hpp:48-65).
 * Non-integral weights (statevector.hpp:162-164) use a device sincos: agreement
 * within 1e-12 relative, not bit-exact.
 */
#ifndef QCGPU_H
#define QCGPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define QC_OK 0
#define QC_ERR_CONFIG 1
#define QC_ERR_RESOURCE 2
#define QC_ERR_IO 3
#define QC_ERR_INTERNAL 4

#define QC_ABI_VERSION 2

typedef struct qc_engine qc_engine;

/* graph.hpp:24-28 Edge: u < v not required on input (Graph::add_edge swaps). */
typedef struct {
    uint32_t u;
    uint32_t v;
    double w;
} qc_edge;

/* graph.hpp:32-81 Graph: vertex count + edge list (edge-list order is significant for
 * non-integral weights, statevector.hpp:103-107). */
typedef struct {
    int32_t n;
    int32_t m;
    const qc_edge* edges;
} qc_graph;

/* qaoa.hpp:136-145 SolveOptions. */
typedef struct {
    int32_t top_k;      /* default 2 */
    int32_t layers;     /* default 3 */
    int32_t budget;     /* default 200 */
    int32_t fold;       /* default 1 */
    uint64_t seed;      /* default 0 */
    uint64_t qubit_cap; /* default 20; the engine's hard cap (qc_qubit_cap) still binds */
    double tolerance;   /* default 1e-5 */
    int32_t threads;    /* accepted for API parity; ignored (device execution) */
    int32_t reserved;
} qc_solve_options;

/* qaoa.hpp:147-152 SolveResult + qaoa.hpp:130-134 CandidateSet. The caller owns bits
 * and probs (capacity >= top_k) and params (capacity 2*layers, [gammas..., betas...]). */
typedef struct {
    int32_t width;
    int32_t folded;
    int32_t count; /* entries written */
    int32_t evals;
    double expectation;
    uint32_t* bits;
    double* probs;
    double* params;
} qc_solve_result;

/* merge.hpp:19-25 CandidatePool, flattened: level i has counts[i] entries of width
 * widths[i], concatenated in bits. */
typedef struct {
    int32_t levels;
    const int32_t* widths;
    const int32_t* counts;
    const uint32_t* bits;
} qc_pool;

/* partition.hpp:22-34 PartitionResult reduced to what the merge reads: piece i covers
 * global ids [first[i], last[i]] and overlaps piece i+1 in exactly one vertex. */
typedef struct {
    int32_t pieces;
    const int32_t* first;
    const int32_t* last;
} qc_chain;

/* merge.hpp:85-91 MergeOptions (eval: 0 kFullGraph, 1 kIncremental). */
typedef struct {
    int32_t start_level;
    int32_t workers;
    int32_t incremental;
    int32_t halve_symmetry;
    double path_budget;
} qc_merge_options;

/* merge.hpp:333-338 ChainedMergeOptions. */
typedef struct {
    int64_t window;
    int64_t window_leaves;
    int32_t workers;
    int32_t halve_symmetry;
} qc_chained_merge_options;

/* merge.hpp:93-97 MergeResult; assignment: caller-owned, n bytes (0/1). */
typedef struct {
    double best_value;
    uint64_t candidates_evaluated;
    uint8_t* assignment;
} qc_merge_result;

/* pipeline.hpp:36-68 RunConfig (hot-path subset; graph given explicitly). */
typedef struct {
    int32_t qubit_cap;        /* 20 */
    int32_t subgraphs;        /* 0 = derive_subgraph_count */
    int32_t top_k;            /* 2; 0 = every class */
    int32_t start_level;      /* 1 */
    int32_t layers;           /* 3 */
    int32_t budget;           /* 200 */
    uint64_t seed;            /* 0 */
    int32_t fold;             /* 1 */
    int32_t halve_symmetry;   /* 0 */
    int32_t partition_mode;   /* 0 balanced, 1 tail-remainder */
    int32_t merge_incremental;/* 1 */
    int32_t merge_mode;       /* 0 auto, 1 level, 2 windowed */
    int32_t shard_index;      /* this process's shard of the subgraphs (multi-GPU) */
    int32_t shard_count;      /* 1 = single GPU */
    int32_t reserved;
    double path_budget;       /* 1e9 */
    double nm_tolerance;      /* 1e-5 */
} qc_run_config;

/* pipeline.hpp ExperimentReport: the fields the hot path produces. */
typedef struct {
    double cut;
    uint64_t candidates_evaluated;
    double partition_s, qaoa_s, merge_s, total_s;
    int32_t subgraphs;
    int32_t windowed;
    uint64_t evals; /* objective evaluations across all subgraphs */
} qc_run_report;

/* ---- engine ------------------------------------------------------------------- */
int qc_engine_create(int device, qc_engine** out);
void qc_engine_destroy(qc_engine* e);
const char* qc_last_error(void);
int qc_abi_version(void);
/* statevector.hpp:20 kQubitCap analogue: the largest subgraph the engine simulates. */
int qc_qubit_cap(void);
/* Kernel launches issued by this engine since creation (bench evidence). */
uint64_t qc_engine_launches(const qc_engine* e);
/* Device bytes of stored-state / scratch the engine may use; 0 = automatic. */
int qc_engine_set_memory_budget(qc_engine* e, uint64_t bytes);
/* Live profiling: with on=1 every engine kernel is bracketed by CUDA events on the
 * stream it runs on (on=N>1: one launch in N per kernel kind is sampled); qc_engine_profile_read returns, per kernel kind (0 levels, 1 onchip,
 * 2 pass_low, 3 pass_high, 4 blocksum, 5 finalsum, 6 topk, 7 merge_tables,
 * 8 merge_search, 9 merge_other), the launch count, summed device ms and summed
 * algorithmic bytes since the last qc_engine_profile call. */
/* Arithmetic of the batched solve / eval paths (qc_solve_batch, qc_eval_batch, the
 * pipeline): 64 = exact fp64, bit-identical to the reference (default); 32 = optional fp32
 * mode (float amplitudes, FMA; expectations within 1e-4 relative). The statevector-level
 * calls (qc_run_ansatz, qc_apply_*) always use fp64. Config error for other values. */
int qc_engine_set_precision(qc_engine* e, int bits);
/* Mixer form of the fp32 mode (replaces apply_mixer_layer,
 * statevector.hpp:187-221, behind the fp32 flag): QC_MIXER_RX (0, default) applies
 * mixer_pair rotations per target; QC_MIXER_WHT (1) applies RX(β)^{(x)T} =
 * H^{(x)T} diag(2^-n e^{-iβ(n-2|k|)}) H^{(x)T} with add/sub-only butterflies (per register
 * round in the streaming passes, over the whole state in the on-chip kernel). Config error
 * for other values, or for WHT while the precision is 64 (not bit-exact); setting
 * precision 64 resets the mixer to RX. */
#define QC_MIXER_RX 0
#define QC_MIXER_WHT 1
int qc_engine_set_mixer(qc_engine* e, int mixer);
int qc_engine_profile(qc_engine* e, int on);
int qc_engine_profile_read(qc_engine* e, int kind, uint64_t* launches, double* ms,
                           double* bytes);
/* Algorithmic FP64 operations (explicitly rounded DMUL/DADD; the path uses no FMA) of the
 * profiled launches of a kernel kind, same window as qc_engine_profile_read. */
int qc_engine_profile_read_fp64(qc_engine* e, int kind, double* fp64_ops);
/* Host time of the lockstep optimiser: waiting for chunk results vs preparing the next
 * step (NM tell/ask, phase LUTs, staging, launches), and chunk-steps serviced. */
int qc_engine_host_stats(qc_engine* e, double* wait_s, double* prep_s, uint64_t* steps,
                         int reset);
/* Host wall seconds accumulated since the last host_stats reset: [0] lockstep optimise,
 * [1] final circuits + top-K, [2] merge, [3] whole qc_pipeline_execute. */
int qc_engine_phase_times(const qc_engine* e, double* out4);
/* Split of qc_engine_host_stats' prep time (same reset): [0] result reads + NM tell,
 * [1] staging build (cos/sin beta, phase LUTs), [2] launch (staging copy + chain or
 * CUDA-graph launch, completion event). */
int qc_engine_host_split(const qc_engine* e, double* out3);
/* Host<->device bytes copied by this engine since creation. */
int qc_engine_transfers(const qc_engine* e, uint64_t* h2d, uint64_t* d2h);
/* The engine's cudaStream_t (all engine work is ordered on it). */
void* qc_engine_stream(const qc_engine* e);

/* ---- graph generators (host; instance prep, not timed by the reference) -------- */
/* graph.hpp:146-160 generate_er_graph: pairs (u<v) in lex order, one mt19937_64 draw
 * each, x = (draw >> 11) * 2^-53, edge iff x < p, weight 1. Two-call protocol: with
 * edges == NULL only *m is written. */
int qc_generate_er(int n, double p, uint64_t seed, qc_edge* edges, int64_t cap, int64_t* m);
/* Weighted random d-regular graph (BASELINE config 3; the reference has no generator):
 * configuration model over n*d stubs shuffled by Fisher-Yates with mt19937_64(seed)
 * (j = draw % (i+1)), consecutive stubs paired; a shuffle giving a self-loop or a
 * multi-edge is discarded and the next one drawn from the same stream. Integer weights
 * U{wlo..whi} (draw % span) in the same stream, edges sorted by (u, v). */
int qc_generate_regular(int n, int d, uint64_t seed, int wlo, int whi, qc_edge* edges,
                        int64_t cap, int64_t* m);

/* ---- statevector.hpp ---------------------------------------------------------- */
/* statevector.hpp:75-111 CostTable: out[z] = C(z) for z < 2^n. */
int qc_cost_table(qc_engine* e, const qc_graph* g, int cap, double* out, int* integral,
                  double* max_value);
/* statevector.hpp:134-143 plus_state. */
int qc_plus_state(qc_engine* e, int q, int cap, double* amps);
/* statevector.hpp:146-171 apply_cost_layer (in place on a host state). */
int qc_apply_cost_layer(qc_engine* e, int q, double* amps, const qc_graph* g, double gamma);
/* statevector.hpp:189-221 apply_mixer_layer (in place). */
int qc_apply_mixer_layer(qc_engine* e, int q, double* amps, double beta);
/* statevector.hpp:224-235 expectation. */
int qc_expectation(qc_engine* e, int q, const double* amps, const qc_graph* g, double* out);
/* statevector.hpp:237-241 norm_sq. */
int qc_norm_sq(qc_engine* e, int q, const double* amps, double* out);

/* ---- qaoa.hpp ----------------------------------------------------------------- */
/* qaoa.hpp:27-38 linear_ramp. */
int qc_linear_ramp(int p, double* gammas, double* betas);
/* qaoa.hpp:59-73 run_ansatz (+ statevector.hpp:224 expectation); amps/expectation
 * optional (NULL). */
int qc_run_ansatz(qc_engine* e, const qc_graph* g, int p, const double* gammas,
                  const double* betas, double* amps, double* expectation);
/* qaoa.hpp:89-91 objective, batched: for each point k, expectation of run_ansatz on
 * graphs[index[k]] at params[k*2p .. k*2p+2p) (packed [gammas..., betas...]). */
int qc_eval_batch(qc_engine* e, const qc_graph* graphs, int n_graphs, int p, int n_points,
                  const int32_t* index, const double* params, double* expectation);
/* qaoa.hpp:85-117 optimize_parameters for n graphs at once (lockstep ask/tell
 * Nelder-Mead; graph i uses seeds[i]). params: n x 2p. Optional trace (NULL): the
 * (x, f) of every objective call, trace_x n x budget x 2p, trace_f n x budget. */
int qc_optimize_batch(qc_engine* e, const qc_graph* graphs, int n, int p, int budget,
                      const uint64_t* seeds, double tolerance, double* params,
                      double* expectation, int32_t* evals, double* trace_x, double* trace_f);
/* qaoa.hpp:158-193 top_candidates on a host state. */
int qc_top_candidates(qc_engine* e, int q, const double* amps, int top_k, int fold,
                      uint32_t* bits, double* probs);
/* qaoa.hpp:198-216 solve_subgraph. */
int qc_solve_subgraph(qc_engine* e, const qc_graph* g, const qc_solve_options* opt,
                      qc_solve_result* res);
/* pipeline.hpp:239-263: solve_subgraph for n independent subgraphs (opts[i] each) in
 * one batched device pass. */
int qc_solve_batch(qc_engine* e, const qc_graph* graphs, int n, const qc_solve_options* opts,
                   qc_solve_result* results);

/* ---- ask/tell optimisers (host only, no device) --------------------------------
 * The engine's lockstep optimiser exposed for callers with their own objective.
 * qc_simplex: nelder_mead.hpp:29-120 nelder_mead_minimize (initial step 0.2,
 * coefficients 1/2/0.5/0.5); qc_optimizer: qaoa.hpp:85-117 optimize_parameters
 * (objective = -<C>; ramp start, seeded restarts). ask() yields the next point to
 * evaluate (done=1 once the run is over); tell() consumes its objective value. */
typedef struct qc_simplex qc_simplex;
int qc_simplex_create(const double* x0, int n, int max_evals, double tolerance,
                      qc_simplex** out);
int qc_simplex_ask(qc_simplex* s, double* x, int* done);
int qc_simplex_tell(qc_simplex* s, double f);
int qc_simplex_result(const qc_simplex* s, double* x, double* value, int* evals, int* converged);
void qc_simplex_destroy(qc_simplex* s);

typedef struct qc_optimizer qc_optimizer;
int qc_optimizer_create(int p, int budget, uint64_t seed, double tolerance, qc_optimizer** out);
int qc_optimizer_ask(qc_optimizer* o, double* x, int* done);
int qc_optimizer_tell(qc_optimizer* o, double f);
int qc_optimizer_result(const qc_optimizer* o, double* params, double* expectation, int* evals);
void qc_optimizer_destroy(qc_optimizer* o);

/* ---- merge.hpp ---------------------------------------------------------------- */
/* merge.hpp:280-331 level_aware_merge. */
int qc_level_merge(qc_engine* e, const qc_pool* pool, const qc_graph* g, const qc_chain* chain,
                   const qc_merge_options* opt, qc_merge_result* res);
/* merge.hpp:345-412 chained_merge. */
int qc_chained_merge(qc_engine* e, const qc_pool* pool, const qc_graph* g,
                     const qc_chain* chain, const qc_chained_merge_options* opt,
                     qc_merge_result* res);

/* ---- pipeline.hpp (hot-path stages) ------------------------------------------- */
/* pipeline.hpp:111-124 schedule rounds are replaced by one batched solve; this runs
 * partition (partition.hpp:111) -> QAOA stage (pipeline.hpp:219-296) -> merge
 * (pipeline.hpp:298-334) for graph g on one GPU and fills report + assignment (n bytes
 * '0'/'1' plus NUL). cfg->shard_count must be 1: multi-GPU callers use
 * qc_run_pipeline_multi (one process, n GPUs) or, one process per GPU,
 * qc_shard_solve -> qc_gather_topk -> qc_merge_records. */
int qc_run_pipeline(qc_engine* e, const qc_graph* g, const qc_run_config* cfg,
                    qc_run_report* report, char* assignment);

/* Resident-input session: partition + device cut tables built once
 * (qc_pipeline_prepare), then QAOA stage + top-K + merge on resident inputs
 * (qc_pipeline_execute, repeatable; same results as qc_run_pipeline). */
typedef struct qc_pipeline qc_pipeline;
int qc_pipeline_prepare(qc_engine* e, const qc_graph* g, const qc_run_config* cfg,
                        qc_pipeline** out);
int qc_pipeline_execute(qc_pipeline* pl, qc_run_report* report, char* assignment);
void qc_pipeline_destroy(qc_pipeline* pl);

/* SolveResults of the last qc_pipeline_execute as solve records (layout below), in
 * subgraph order; with records == NULL only *record_bytes / *subgraphs are written. */
int qc_pipeline_records(const qc_pipeline* pl, void* records, int64_t capacity,
                        int64_t* record_bytes, int32_t* subgraphs);

/* Sharded resident session (one process per GPU; replaces the rounds loop of
 * pipeline.hpp:271-280 for this rank's share): qc_pipeline_prepare with cfg->shard_count > 1
 * partitions once and builds device cut tables only for this rank's contiguous block
 * (qc_shard_range(M, shard_index, shard_count)); qc_pipeline_execute_shard runs that
 * block's QAOA stage and writes its (end - begin) solve records (record size from
 * qc_pipeline_records(pl, NULL, ...)); after the gather (qc_gather_topk), the rank holding
 * all M records merges them with qc_pipeline_merge_records (pipeline.hpp:298-334) without
 * partitioning again. */
int qc_pipeline_execute_shard(qc_pipeline* pl, void* records, int64_t capacity, int32_t* begin,
                              int32_t* end, double* qaoa_s);
int qc_pipeline_merge_records(qc_pipeline* pl, const void* records, int64_t capacity,
                              qc_run_report* report, char* assignment);

/* ---- multi-GPU: shards of subgraphs, one gather of solve records ----
 * Solve record (fixed size per run, qc_run_record_bytes): int32 {width, count, evals,
 * folded}, double expectation, uint32 bits[kcap] (padded to 8 bytes), double probs[kcap],
 * double params[2*layers] — one SolveResult (qaoa.hpp:147-152) of pipeline.hpp:263.
 * kcap = min(top_k, classes of the widest piece), or every class for top_k = 0. */
int64_t qc_record_bytes(int top_k_cap, int layers);
/* Record size and subgraph count of the run (g, cfg): the geometry every rank and the
 * merge must agree on (derived from the same chain partition as qc_shard_solve). */
int qc_run_record_bytes(const qc_graph* g, const qc_run_config* cfg, int64_t* record_bytes,
                        int32_t* subgraphs);
/* Contiguous balanced block [begin, end) of the M subgraphs for shard shard_index. */
int qc_shard_range(int M, int shard_index, int shard_count, int32_t* begin, int32_t* end);
/* pipeline.hpp:239-263 for subgraphs [begin, end) of g's partition on this engine:
 * writes end-begin records (capacity: bytes of `records`; config error if short). With
 * records == NULL only *subgraphs (= M) is written. */
int qc_shard_solve(qc_engine* e, const qc_graph* g, const qc_run_config* cfg, int32_t begin,
                   int32_t end, void* records, int64_t capacity, int32_t* subgraphs);
/* pipeline.hpp:298-334 on the M gathered records (all shards, subgraph order). */
int qc_merge_records(qc_engine* e, const qc_graph* g, const qc_run_config* cfg,
                     const void* records, int64_t capacity, int32_t M, qc_run_report* report,
                     char* assignment);

/* NCCL record gather (replaces the hand-over of SolveResults from the per-subgraph
 * threads of pipeline.hpp:271-280 to the merge at pipeline.hpp:300-305). One rank per
 * GPU: rank 0 calls qc_comm_id, the caller ships the 128 bytes to every rank (MPI, a
 * file, torch.distributed, ...), each rank calls qc_comm_create on its engine. One
 * process driving several GPUs: qc_comm_create_all (ncclCommInitAll; one engine per
 * distinct device) fills out[n]. NCCL is loaded at first use (libnccl.so.2). */
#define QC_COMM_ID_BYTES 128
typedef struct qc_comm qc_comm;
int qc_comm_id(void* id /* QC_COMM_ID_BYTES */);
int qc_comm_create(qc_engine* e, int nranks, int rank, const void* id, qc_comm** out);
int qc_comm_create_all(qc_engine* const* engines, int n, qc_comm** out);
int qc_comm_rank(const qc_comm* c, int32_t* rank, int32_t* nranks);
void qc_comm_destroy(qc_comm* c);
/* All-gather of solve records over NCCL on the engine's stream: this rank holds the
 * `count` records of its qc_shard_range block; `all` receives the M records of every
 * rank in subgraph order (M * record_bytes bytes). Collective: every rank calls it. */
int qc_gather_topk(qc_comm* c, const void* local, int32_t count, int32_t M, int64_t record_bytes,
                   void* all);
/* One process, n engines: shard -> per-engine solve (one host thread each) -> record
 * all-gather over comms (NCCL; comms[i] = rank i on engines[i], from
 * qc_comm_create_all) -> merge on engines[0]. comms == NULL (engines that share a
 * device, where NCCL cannot form a communicator): the records are concatenated in host
 * memory instead. An engine listed for several shards runs them back to back on one host
 * thread (an engine is never driven by two threads at once). Same results as
 * qc_run_pipeline. */
int qc_run_pipeline_multi(qc_engine* const* engines, qc_comm* const* comms, int n,
                          const qc_graph* g, const qc_run_config* cfg, qc_run_report* report,
                          char* assignment);

#ifdef __cplusplus
}
#endif
#endif /* QCGPU_H */
