/* TEST INFRASTRUCTURE ONLY — C restatement of the reference hot path, used as the
 * parity checker by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg.
 * Never linked into the product. Same signatures as oracle/ref_driver.cpp (prefix
 * orc_ instead of ref_) so both are interchangeable behind oracle/refpy.py.
 *
 * Status codes mirror qcut's exception taxonomy (errors.hpp:8-24):
 *   0 ok, 1 config_error, 2 resource_error, 3 io_error, 4 internal.
 */
#ifndef QCUT_ORACLE_H
#define QCUT_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
    uint32_t u, v;
    double w;
} orc_edge; /* graph.hpp:24-28 Edge layout */

typedef struct {
    int top_k, layers, budget;
    uint64_t seed;
    int fold, threads;
    uint64_t qubit_cap;
    double tolerance;
} orc_solve_options; /* qaoa.hpp:136-145 SolveOptions */

typedef struct {
    int qubit_cap, solvers, subgraphs, top_k, start_level, layers, budget;
    uint64_t seed;
    int fold, halve_symmetry, partition_mode, merge_incremental, merge_mode, workers;
    double path_budget, nm_tolerance;
    int baseline;
} orc_run_config; /* pipeline.hpp:36-68 RunConfig (hot-path subset) */

typedef struct {
    double cut;
    uint64_t leaves;
    double partition_s, qaoa_s, merge_s, total_s, baseline_value;
    int subgraphs, windowed;
} orc_run_result;

const char* orc_last_error(void);
int orc_qubit_cap(void);
void orc_set_qubit_cap(int cap); /* kQubitCap, statevector.hpp:20 (24; 26 for config 5) */

int orc_generate_er(int n, double p, uint64_t seed, orc_edge* out, long long cap, long long* m);
int orc_generate_regular(int n, int d, uint64_t seed, int wlo, int whi, orc_edge* out,
                         long long cap, long long* m);
int orc_partition(int n, int m, const orc_edge* e, int M, int mode, int cap, int* first, int* last,
                  int* local_m, long long* inter_m);
int orc_derive_subgraph_count(long long n, long long cap, int* out);

int orc_cost_table(int n, int m, const orc_edge* e, int cap, double* out, int* integral,
                   double* max_value);
int orc_plus_state(int q, int cap, double* amps);
int orc_apply_cost_layer(int q, double* amps, int n, int m, const orc_edge* e, double gamma,
                         int threads);
int orc_apply_mixer_layer(int q, double* amps, double beta, int threads);
int orc_expectation(int q, const double* amps, int n, int m, const orc_edge* e, int threads,
                    double* out);
int orc_norm_sq(int q, const double* amps, int threads, double* out);
int orc_run_ansatz(int n, int m, const orc_edge* e, int p, const double* gammas,
                   const double* betas, int threads, double* amps, double* expect);
int orc_linear_ramp(int p, double* gammas, double* betas);
int orc_optimize(int n, int m, const orc_edge* e, int p, int budget, uint64_t seed, int threads,
                 double tol, double* params, double* expect, int* evals, double* trace_x,
                 double* trace_f, int* trace_len);
int orc_top_candidates(int q, const double* amps, int top_k, int fold, uint32_t* bits,
                       double* probs);
int orc_solve_subgraph(int n, int m, const orc_edge* e, const orc_solve_options* o,
                       uint32_t* bits, double* probs, int* count, double* params, double* expect,
                       int* evals);
int orc_level_merge(int n, int m, const orc_edge* e, int M, int mode, const int* widths,
                    const int* counts, const uint32_t* bits, int start_level, int workers,
                    int incremental, double path_budget, int halve, double* value,
                    uint8_t* assignment, uint64_t* leaves);
int orc_chained_merge(int n, int m, const orc_edge* e, int M, int mode, const int* widths,
                      const int* counts, const uint32_t* bits, long long window,
                      long long window_leaves, int workers, int halve, double* value,
                      uint8_t* assignment, uint64_t* leaves);
int orc_run_pipeline(int n, int m, const orc_edge* e, const orc_run_config* c,
                     orc_run_result* out, char* assignment, double* sub_expect, int* sub_evals,
                     int M_cap);

#ifdef __cplusplus
}
#endif
#endif
