// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// extern "C" shim over the UNMODIFIED reference headers
// (/root/reference/proj/include/qcut/*.hpp), compiled by oracle/Makefile into
// oracle/_ref/libqcut_ref.so (and libqcut_ref26.so with kQubitCap raised to 26
// for BASELINE config 5). Only tests/, oracle/gen_golden.py and bench.py's
// reference / cpu_baseline legs load it. Every entry point forwards to the
// reference function named in its comment; nothing here re-implements the
// algorithm except ref_optimize_trace, which replays optimize_parameters'
// outer loop (qaoa.hpp:85-117) around the reference's own nelder_mead_minimize
// to record the (x, f) trajectory, and checks itself against
// optimize_parameters.
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <thread>
#include <vector>

#include "qcut/qcut.hpp"

namespace {

thread_local std::string g_err;

struct RefEdge {
    std::uint32_t u, v;
    double w;
};

int fail(int code, const char* what) {
    g_err = what;
    return code;
}

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const qcut::config_error& e) {
        return fail(1, e.what());
    } catch (const qcut::resource_error& e) {
        return fail(2, e.what());
    } catch (const qcut::io_error& e) {
        return fail(3, e.what());
    } catch (const qcut::pipeline_error& e) {
        int c = 4;
        switch (e.cause()) {
            case qcut::pipeline_error::Cause::kConfig: c = 1; break;
            case qcut::pipeline_error::Cause::kResource: c = 2; break;
            case qcut::pipeline_error::Cause::kIo: c = 3; break;
            default: c = 4;
        }
        return fail(c, e.what());
    } catch (const std::exception& e) {
        return fail(4, e.what());
    }
}

qcut::Graph make_graph(int n, int m, const RefEdge* e) {
    qcut::Graph g(static_cast<std::size_t>(n));
    for (int i = 0; i < m; ++i) g.add_edge(e[i].u, e[i].v, e[i].w);
    return g;
}

qcut::StateVector make_state(int q, const double* amps) {
    qcut::StateVector s;
    const std::size_t n = std::size_t{1} << q;
    s.amps.resize(n);
    std::memcpy(s.amps.data(), amps, n * 16);
    return s;
}

qcut::QaoaParams make_params(int p, const double* gammas, const double* betas) {
    qcut::QaoaParams qp;
    qp.gammas.assign(gammas, gammas + p);
    qp.betas.assign(betas, betas + p);
    return qp;
}

qcut::PartitionResult make_partition(const qcut::Graph& g, int M, int mode, int cap) {
    return qcut::partition(g, M, mode == 0 ? qcut::PartitionMode::kBalanced
                                           : qcut::PartitionMode::kTailRemainder,
                           static_cast<std::size_t>(cap));
}

qcut::CandidatePool make_pool(int M, const int* widths, const int* counts,
                              const std::uint32_t* bits) {
    qcut::CandidatePool pool;
    std::size_t off = 0;
    for (int i = 0; i < M; ++i) {
        qcut::CandidatePool::Level lv;
        lv.width = widths[i];
        lv.bits.assign(bits + off, bits + off + counts[i]);
        off += static_cast<std::size_t>(counts[i]);
        pool.levels.push_back(std::move(lv));
    }
    return pool;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_qubit_cap() { return static_cast<int>(qcut::kQubitCap); }

// graph.hpp:146 generate_er_graph. Two-call protocol: out may be null to query m.
int ref_generate_er(int n, double p, std::uint64_t seed, RefEdge* out, long long cap,
                    long long* m) {
    return guarded([&] {
        const qcut::Graph g = qcut::generate_er_graph(static_cast<std::size_t>(n), p, seed);
        *m = static_cast<long long>(g.edge_count());
        if (out) {
            if (cap < *m) throw qcut::config_error("edge buffer too small");
            for (std::size_t i = 0; i < g.edge_count(); ++i) {
                const auto& e = g.edges()[i];
                out[i] = {e.u, e.v, e.w};
            }
        }
    });
}

// statevector.hpp:75 CostTable; out[z] = value(z).
int ref_cost_table(int n, int m, const RefEdge* e, int cap, double* out, int* integral,
                   double* max_value) {
    return guarded([&] {
        const qcut::CostTable t(make_graph(n, m, e), static_cast<std::size_t>(cap));
        for (std::size_t z = 0; z < t.size(); ++z) out[z] = t.value(z);
        *integral = t.integral() ? 1 : 0;
        *max_value = t.max_value();
    });
}

// statevector.hpp:134 plus_state.
int ref_plus_state(int q, int cap, double* amps) {
    return guarded([&] {
        const auto s = qcut::plus_state(static_cast<std::size_t>(q), static_cast<std::size_t>(cap));
        std::memcpy(amps, s.amps.data(), s.size() * 16);
    });
}

// statevector.hpp:146 apply_cost_layer (CostTable overload) on a caller state.
int ref_apply_cost_layer(int q, double* amps, int n, int m, const RefEdge* e, double gamma,
                         int threads) {
    return guarded([&] {
        auto s = make_state(q, amps);
        const qcut::CostTable t(make_graph(n, m, e));
        qcut::apply_cost_layer(s, t, gamma, threads);
        std::memcpy(amps, s.amps.data(), s.size() * 16);
    });
}

// statevector.hpp:189 apply_mixer_layer.
int ref_apply_mixer_layer(int q, double* amps, double beta, int threads) {
    return guarded([&] {
        auto s = make_state(q, amps);
        qcut::apply_mixer_layer(s, beta, threads);
        std::memcpy(amps, s.amps.data(), s.size() * 16);
    });
}

// statevector.hpp:224 expectation / :237 norm_sq.
int ref_expectation(int q, const double* amps, int n, int m, const RefEdge* e, int threads,
                    double* out) {
    return guarded([&] {
        const auto s = make_state(q, amps);
        const qcut::CostTable t(make_graph(n, m, e));
        *out = qcut::expectation(s, t, threads);
    });
}

int ref_norm_sq(int q, const double* amps, int threads, double* out) {
    return guarded([&] { *out = qcut::norm_sq(make_state(q, amps), threads); });
}

// qaoa.hpp:59 run_ansatz + statevector.hpp:224 expectation. amps may be null.
int ref_run_ansatz(int n, int m, const RefEdge* e, int p, const double* gammas,
                   const double* betas, int threads, double* amps, double* expect) {
    return guarded([&] {
        const qcut::CostTable t(make_graph(n, m, e));
        const auto s = qcut::run_ansatz(t, make_params(p, gammas, betas), threads);
        if (amps) std::memcpy(amps, s.amps.data(), s.size() * 16);
        if (expect) *expect = qcut::expectation(s, t, threads);
    });
}

// qaoa.hpp:27 linear_ramp.
int ref_linear_ramp(int p, double* gammas, double* betas) {
    return guarded([&] {
        const auto r = qcut::linear_ramp(p);
        for (int i = 0; i < p; ++i) {
            gammas[i] = r.gammas[i];
            betas[i] = r.betas[i];
        }
    });
}

// qaoa.hpp:85 optimize_parameters. The trace (optional, capacity `budget`)
// records every objective call in order; it is produced by replaying the outer
// loop around qcut::nelder_mead_minimize and must agree with the direct call.
int ref_optimize(int n, int m, const RefEdge* e, int p, int budget, std::uint64_t seed,
                 int threads, double tol, double* params, double* expect, int* evals,
                 double* trace_x, double* trace_f, int* trace_len) {
    return guarded([&] {
        const qcut::CostTable table(make_graph(n, m, e));
        const auto direct = qcut::optimize_parameters(table, p, budget, seed, threads, tol);
        for (int i = 0; i < p; ++i) {
            params[i] = direct.params.gammas[i];
            params[p + i] = direct.params.betas[i];
        }
        *expect = direct.expectation;
        *evals = direct.evals;
        if (!trace_x) return;

        int len = 0;
        auto objective = [&](const std::vector<double>& x) {
            qcut::QaoaParams qp;
            qp.gammas.assign(x.begin(), x.begin() + p);
            qp.betas.assign(x.begin() + p, x.end());
            const double f = -qcut::expectation(qcut::run_ansatz(table, qp, threads), table, threads);
            if (len < budget) {
                std::memcpy(trace_x + static_cast<std::size_t>(len) * 2 * p, x.data(),
                            sizeof(double) * 2 * p);
                trace_f[len] = f;
            }
            ++len;
            return f;
        };
        const auto ramp = qcut::linear_ramp(p);
        std::vector<double> start(ramp.gammas);
        start.insert(start.end(), ramp.betas.begin(), ramp.betas.end());
        double best_neg = objective(start);
        std::vector<double> best_x = start;
        int used = 1;
        std::mt19937_64 rng(seed);
        std::uniform_real_distribution<double> angle(0.0, std::numbers::pi);
        while (used < budget) {
            qcut::NelderMeadOptions opt;
            opt.max_evals = budget - used;
            opt.tolerance = tol;
            const auto r = qcut::nelder_mead_minimize(objective, start, opt);
            used += r.evals;
            if (r.value < best_neg) {
                best_neg = r.value;
                best_x = r.x;
            }
            if (!r.converged) break;
            start.assign(2 * static_cast<std::size_t>(p), 0.0);
            for (double& v : start) v = angle(rng);
        }
        *trace_len = len;
        bool same = used == direct.evals && -best_neg == direct.expectation;
        for (int i = 0; i < 2 * p && same; ++i) same = best_x[i] == params[i];
        if (!same) throw std::runtime_error("trace replay diverged from optimize_parameters");
    });
}

// qaoa.hpp:158 top_candidates.
int ref_top_candidates(int q, const double* amps, int top_k, int fold, std::uint32_t* bits,
                       double* probs) {
    return guarded([&] {
        const auto set = qcut::top_candidates(make_state(q, amps), top_k, fold != 0);
        for (std::size_t i = 0; i < set.entries.size(); ++i) {
            bits[i] = set.entries[i].bits;
            probs[i] = set.entries[i].probability;
        }
    });
}

struct RefSolveOptions {
    int top_k, layers, budget;
    std::uint64_t seed;
    int fold, threads;
    std::uint64_t qubit_cap;
    double tolerance;
};

// qaoa.hpp:198 solve_subgraph. bits/probs capacity top_k, params 2*layers.
int ref_solve_subgraph(int n, int m, const RefEdge* e, const RefSolveOptions* o,
                       std::uint32_t* bits, double* probs, int* count, double* params,
                       double* expect, int* evals) {
    return guarded([&] {
        qcut::SolveOptions so;
        so.top_k = o->top_k;
        so.layers = o->layers;
        so.budget = o->budget;
        so.seed = o->seed;
        so.fold = o->fold != 0;
        so.threads = o->threads;
        so.qubit_cap = o->qubit_cap;
        so.tolerance = o->tolerance;
        const auto r = qcut::solve_subgraph(make_graph(n, m, e), so);
        *count = static_cast<int>(r.candidates.entries.size());
        for (std::size_t i = 0; i < r.candidates.entries.size(); ++i) {
            bits[i] = r.candidates.entries[i].bits;
            probs[i] = r.candidates.entries[i].probability;
        }
        for (int i = 0; i < o->layers; ++i) {
            params[i] = r.params.gammas[i];
            params[o->layers + i] = r.params.betas[i];
        }
        *expect = r.expectation;
        *evals = r.evals;
    });
}

// partition.hpp:111 partition. first/last: global id range per piece (M each);
// local_m: intra-edge count per piece; inter_m: number of inter edges.
int ref_partition(int n, int m, const RefEdge* e, int M, int mode, int cap, int* first,
                  int* last, int* local_m, long long* inter_m) {
    return guarded([&] {
        const auto part = make_partition(make_graph(n, m, e), M, mode, cap);
        for (std::size_t i = 0; i < part.subgraphs.size(); ++i) {
            first[i] = static_cast<int>(part.subgraphs[i].global_ids.front());
            last[i] = static_cast<int>(part.subgraphs[i].global_ids.back());
            local_m[i] = static_cast<int>(part.subgraphs[i].local_graph.edge_count());
        }
        *inter_m = static_cast<long long>(part.inter_edges.size());
    });
}

int ref_derive_subgraph_count(long long n, long long cap, int* out) {
    return guarded([&] {
        *out = qcut::derive_subgraph_count(static_cast<std::size_t>(n), static_cast<std::size_t>(cap));
    });
}

// merge.hpp:280 level_aware_merge over the partition (M, mode) of the graph.
int ref_level_merge(int n, int m, const RefEdge* e, int M, int mode, const int* widths,
                    const int* counts, const std::uint32_t* bits, int start_level, int workers,
                    int incremental, double path_budget, int halve, double* value,
                    std::uint8_t* assignment, std::uint64_t* leaves) {
    return guarded([&] {
        const auto g = make_graph(n, m, e);
        const auto part = make_partition(g, M, mode, 0);
        const auto pool = make_pool(M, widths, counts, bits);
        qcut::MergeOptions mo;
        mo.start_level = start_level;
        mo.workers = workers;
        mo.eval = incremental ? qcut::MergeEval::kIncremental : qcut::MergeEval::kFullGraph;
        mo.path_budget = path_budget;
        mo.halve_symmetry = halve != 0;
        const auto r = qcut::level_aware_merge(pool, g, part, mo);
        *value = r.best_value;
        std::memcpy(assignment, r.best_assignment.bits.data(), static_cast<std::size_t>(n));
        *leaves = r.candidates_evaluated;
    });
}

// merge.hpp:345 chained_merge.
int ref_chained_merge(int n, int m, const RefEdge* e, int M, int mode, const int* widths,
                      const int* counts, const std::uint32_t* bits, long long window,
                      long long window_leaves, int workers, int halve, double* value,
                      std::uint8_t* assignment, std::uint64_t* leaves) {
    return guarded([&] {
        const auto g = make_graph(n, m, e);
        const auto part = make_partition(g, M, mode, 0);
        const auto pool = make_pool(M, widths, counts, bits);
        qcut::ChainedMergeOptions co;
        co.window = static_cast<std::size_t>(window);
        co.window_leaves = static_cast<std::size_t>(window_leaves);
        co.workers = workers;
        co.halve_symmetry = halve != 0;
        const auto r = qcut::chained_merge(pool, g, part, co);
        *value = r.best_value;
        std::memcpy(assignment, r.best_assignment.bits.data(), static_cast<std::size_t>(n));
        *leaves = r.candidates_evaluated;
    });
}

struct RefRunConfig {
    int qubit_cap, solvers, subgraphs, top_k, start_level, layers, budget;
    std::uint64_t seed;
    int fold, halve_symmetry, partition_mode, merge_incremental, merge_mode, workers;
    double path_budget, nm_tolerance;
    int baseline;  // 0 auto, 1 brute, 2 local, 3 fixed value (no baseline work)
};

struct RefRunResult {
    double cut;
    std::uint64_t leaves;
    double partition_s, qaoa_s, merge_s, total_s, baseline_value;
    int subgraphs, windowed;
};

// pipeline.hpp:391 run_pipeline(Graph, RunConfig). Per-subgraph outputs
// (capacity `M_cap`): expectation, evals. Assignment: n bytes of '0'/'1'.
int ref_run_pipeline(int n, int m, const RefEdge* e, const RefRunConfig* c, RefRunResult* out,
                     char* assignment, double* sub_expect, int* sub_evals, int M_cap) {
    return guarded([&] {
        const auto g = make_graph(n, m, e);
        qcut::RunConfig cfg;
        cfg.qubit_cap = static_cast<std::size_t>(c->qubit_cap);
        cfg.solvers = c->solvers;
        cfg.subgraphs = c->subgraphs;
        cfg.top_k = c->top_k;
        cfg.start_level = c->start_level;
        cfg.layers = c->layers;
        cfg.budget = c->budget;
        cfg.seed = c->seed;
        cfg.fold = c->fold != 0;
        cfg.halve_symmetry = c->halve_symmetry != 0;
        cfg.partition_mode = c->partition_mode == 0 ? qcut::PartitionMode::kBalanced
                                                    : qcut::PartitionMode::kTailRemainder;
        cfg.merge_eval = c->merge_incremental ? qcut::MergeEval::kIncremental
                                              : qcut::MergeEval::kFullGraph;
        cfg.merge_mode = c->merge_mode == 1   ? qcut::MergeMode::kLevel
                         : c->merge_mode == 2 ? qcut::MergeMode::kWindowed
                                              : qcut::MergeMode::kAuto;
        cfg.workers = c->workers;
        cfg.path_budget = c->path_budget;
        cfg.nm_tolerance = c->nm_tolerance;
        switch (c->baseline) {
            case 1: cfg.baseline = qcut::BaselineKind::kBruteForce; break;
            case 2: cfg.baseline = qcut::BaselineKind::kLocalSearch; break;
            case 3:
                cfg.baseline = qcut::BaselineKind::kFixedValue;
                cfg.baseline_value = 1.0;
                cfg.baseline_seconds = 0.0;
                break;
            default: cfg.baseline = qcut::BaselineKind::kAuto;
        }
        const auto r = qcut::run_pipeline(g, cfg);
        out->cut = r.merge.best_value;
        out->leaves = r.merge.candidates_evaluated;
        out->partition_s = r.times.partition_s;
        out->qaoa_s = r.times.qaoa_s;
        out->merge_s = r.times.merge_s;
        out->total_s = r.times.total_s;
        out->baseline_value = r.baseline.value;
        out->subgraphs = r.config.subgraphs;
        out->windowed = r.config.merge_mode == "windowed" ? 1 : 0;
        std::memcpy(assignment, r.merge.assignment.data(), r.merge.assignment.size());
        for (std::size_t i = 0; i < r.subgraphs.size() && static_cast<int>(i) < M_cap; ++i) {
            sub_expect[i] = r.subgraphs[i].expectation;
            sub_evals[i] = r.subgraphs[i].evals;
        }
    });
}

// The QAOA stage of pipeline.hpp:219-296 for a chosen list of subgraph indices: the
// reference's own partition (partition.hpp:111), the stage's per-index SolveOptions
// (seed = base + idx, top_k clamp, pipeline.hpp:245-261) and its concurrency (`slots`
// std::threads per round, `threads` OpenMP threads each, pipeline.hpp:223-227). Every
// SolveResult is written out: widths/counts[count], bits/probs[count][kcap],
// params[count][2*layers] (gammas then betas), expect/evals[count]. seconds = wall time
// of the solves. Used by the GPU parity tests (full-budget solves of sampled subgraphs
// at configs 3-5) and by bench.py's parity block.
int ref_solve_stage(int n, int m, const RefEdge* e, int M, int mode, int qubit_cap,
                    const int* idx, int count, int top_k, int layers, int budget,
                    std::uint64_t seed, int fold, int slots, int threads, double tol, int kcap,
                    int* widths, int* counts, std::uint32_t* bits, double* probs, double* params,
                    double* expect, int* evals, double* seconds) {
    return guarded([&] {
        const auto g = make_graph(n, m, e);
        const auto part = make_partition(g, M, mode, qubit_cap);
        std::vector<std::exception_ptr> errs(static_cast<std::size_t>(count));
        auto solve_one = [&](int k) {
            try {
                const int id = idx[k];
                if (id < 0 || id >= static_cast<int>(part.subgraphs.size()))
                    throw qcut::config_error("subgraph index out of range");
                const auto& sub = part.subgraphs[static_cast<std::size_t>(id)];
                const std::size_t classes = fold ? (std::size_t{1} << (sub.size() - 1))
                                                 : (std::size_t{1} << sub.size());
                qcut::SolveOptions so;
                so.top_k = top_k == 0 ? static_cast<int>(classes)
                                      : static_cast<int>(std::min<std::size_t>(
                                            classes, static_cast<std::size_t>(top_k)));
                so.layers = layers;
                so.budget = budget;
                so.seed = seed + static_cast<std::uint64_t>(id);
                so.fold = fold != 0;
                so.threads = threads;
                so.qubit_cap = static_cast<std::size_t>(qubit_cap);
                so.tolerance = tol;
                if (so.top_k > kcap) throw qcut::config_error("kcap below the retained count");
                const auto r = qcut::solve_subgraph(sub.local_graph, so);
                const auto kk = static_cast<std::size_t>(k);
                widths[kk] = static_cast<int>(r.candidates.width);
                counts[kk] = static_cast<int>(r.candidates.entries.size());
                for (std::size_t i = 0; i < r.candidates.entries.size(); ++i) {
                    bits[kk * static_cast<std::size_t>(kcap) + i] = r.candidates.entries[i].bits;
                    probs[kk * static_cast<std::size_t>(kcap) + i] = r.candidates.entries[i].probability;
                }
                for (int l = 0; l < layers; ++l) {
                    params[kk * 2 * static_cast<std::size_t>(layers) + static_cast<std::size_t>(l)] = r.params.gammas[static_cast<std::size_t>(l)];
                    params[kk * 2 * static_cast<std::size_t>(layers) + static_cast<std::size_t>(layers + l)] = r.params.betas[static_cast<std::size_t>(l)];
                }
                expect[kk] = r.expectation;
                evals[kk] = r.evals;
            } catch (...) {
                errs[static_cast<std::size_t>(k)] = std::current_exception();
            }
        };
        const auto t0 = std::chrono::steady_clock::now();
        for (int start = 0; start < count; start += slots) {
            std::vector<std::thread> ts;
            for (int k = start; k < std::min(count, start + slots); ++k) ts.emplace_back(solve_one, k);
            for (auto& t : ts) t.join();
        }
        *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        for (auto& x : errs)
            if (x) std::rethrow_exception(x);
    });
}

// Per-eval CPU baseline: the objective of optimize_parameters
// (qaoa.hpp:89-91: run_ansatz + expectation on a prebuilt CostTable) evaluated `reps`
// times at fixed angles with `threads` OpenMP threads. Writes seconds per evaluation and
// the last expectation (so the loop cannot be elided).
int ref_eval_timing(int n, int m, const RefEdge* e, int p, const double* gammas,
                    const double* betas, int threads, int reps, double* sec_per_eval,
                    double* expect) {
    return guarded([&] {
        const auto g = make_graph(n, m, e);
        const qcut::CostTable table(g, qcut::kQubitCap);
        const auto params = make_params(p, gammas, betas);
        double x = 0.0;
        const auto t0 = std::chrono::steady_clock::now();
        for (int r = 0; r < reps; ++r)
            x = qcut::expectation(qcut::run_ansatz(table, params, threads), table, threads);
        *sec_per_eval = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() /
                        static_cast<double>(reps > 0 ? reps : 1);
        *expect = x;
    });
}

}  // extern "C"
