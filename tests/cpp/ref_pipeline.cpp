// Drop-in check on the reference's own types: the reference's run_pipeline (pipeline.hpp,
// unmodified, CPU) against the same stages with ONLY the QAOA stage replaced by
// qcut_gpu::reference::solve_batch (B200 engine): partition, per-subgraph SolveOptions
// (pipeline.hpp:247-262), candidate pools and merge are the reference's own functions, the
// solve results come back as qcut::SolveResult. Test infrastructure (built by
// oracle/Makefile against /root/reference; run by tests/test_gpu_cpp.py and
// tests/test_cpu_shim.py).
//
//   ref_pipeline run <n> <p> <seed> <cap> <top_k> <layers> <budget>   -> "ok cut ..."
//   ref_pipeline errors                                               -> error mapping
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include <qcut/pipeline.hpp>
#define QCUT_GPU_REFERENCE_TYPES
#include "qcut_gpu.hpp"

static int fail(const char* what) {
    std::printf("MISMATCH %s\n", what);
    return 1;
}

int main(int argc, char** argv) {
    if (argc >= 2 && std::strcmp(argv[1], "errors") == 0) {
        // codes come back as the reference's exception types (errors.hpp:8-24)
        qcut::Graph g(3);
        g.add_edge(0, 1);
        g.add_edge(1, 2);
        qcut::SolveOptions so;
        so.top_k = 0;  // qaoa.hpp:162-165: config_error
        try {
            (void)qcut_gpu::reference::solve_subgraph(g, so);
            std::printf("no exception\n");
        } catch (const qcut::config_error& e) {
            std::printf("qcut::config_error: %s\n", e.what());
        } catch (const qcut::resource_error& e) {  // no CUDA device: the engine refuses
            std::printf("qcut::resource_error: %s\n", e.what());
        }
        return 0;
    }
    if (argc < 9 || std::strcmp(argv[1], "run") != 0) {
        std::fprintf(stderr, "usage: ref_pipeline run n p seed cap top_k layers budget | errors\n");
        return 2;
    }
    qcut::RunConfig cfg;
    cfg.er_n = std::strtoull(argv[2], nullptr, 10);
    cfg.er_p = std::atof(argv[3]);
    cfg.er_seed = std::strtoull(argv[4], nullptr, 10);
    cfg.qubit_cap = std::strtoull(argv[5], nullptr, 10);
    cfg.top_k = std::atoi(argv[6]);
    cfg.layers = std::atoi(argv[7]);
    cfg.budget = std::atoi(argv[8]);
    cfg.baseline = qcut::BaselineKind::kFixedValue;  // no brute force / local search
    cfg.baseline_value = 1.0;
    const qcut::Graph g = qcut::generate_er_graph(cfg.er_n, cfg.er_p, cfg.er_seed);
    const qcut::ExperimentReport stock = qcut::run_pipeline(g, cfg);

    // the same stages, QAOA on the GPU (pipeline.hpp:206-334 with :263 swapped)
    const int M0 = qcut::derive_subgraph_count(g.n(), cfg.qubit_cap);
    const qcut::PartitionResult part = qcut::partition(g, M0, cfg.partition_mode, cfg.qubit_cap);
    const int M = static_cast<int>(part.subgraphs.size());
    std::vector<const qcut::Graph*> graphs;
    std::vector<qcut::SolveOptions> opts;
    for (int idx = 0; idx < M; ++idx) {
        const auto& sub = part.subgraphs[static_cast<std::size_t>(idx)];
        const std::size_t width = sub.size();
        const std::size_t classes = cfg.fold ? (std::size_t{1} << (width - 1)) : (std::size_t{1} << width);
        qcut::SolveOptions so;
        so.top_k = cfg.top_k == 0 ? static_cast<int>(classes)
                                  : static_cast<int>(std::min<std::size_t>(classes, static_cast<std::size_t>(cfg.top_k)));
        so.layers = cfg.layers;
        so.budget = cfg.budget;
        so.seed = cfg.seed + static_cast<std::uint64_t>(idx);
        so.fold = cfg.fold;
        so.qubit_cap = cfg.qubit_cap;
        so.tolerance = cfg.nm_tolerance;
        graphs.push_back(&sub.local_graph);
        opts.push_back(so);
    }
    std::vector<qcut::SolveResult> solves =
        qcut_gpu::reference::solve_batch(qcut_gpu::reference::default_engine(), graphs, opts);
    if (static_cast<int>(stock.subgraphs.size()) != M) return fail("subgraph count");
    for (int i = 0; i < M; ++i) {
        const auto& s = stock.subgraphs[static_cast<std::size_t>(i)];
        const auto& r = solves[static_cast<std::size_t>(i)];
        if (s.expectation != r.expectation) return fail("expectation");
        if (s.evals != r.evals) return fail("evals");
        if (s.retained != static_cast<int>(r.candidates.entries.size())) return fail("retained");
    }
    std::vector<qcut::CandidateSet> sets;
    for (auto& s : solves) sets.push_back(std::move(s.candidates));
    const qcut::CandidatePool pool = qcut::build_candidate_pools(sets);
    qcut::MergeResult merged;
    if (qcut::estimate_paths(pool, cfg.halve_symmetry) <= cfg.path_budget) {
        qcut::MergeOptions mo;
        mo.start_level = std::min(cfg.start_level, M);
        mo.workers = 1;
        mo.eval = cfg.merge_eval;
        mo.path_budget = cfg.path_budget;
        mo.halve_symmetry = cfg.halve_symmetry;
        merged = qcut::level_aware_merge(pool, g, part, mo);
    } else {
        qcut::ChainedMergeOptions co;
        co.workers = 1;
        merged = qcut::chained_merge(pool, g, part, co);
    }
    if (merged.best_value != stock.merge.best_value) return fail("cut");
    if (merged.best_assignment.to_string() != stock.merge.assignment) return fail("assignment");
    if (merged.candidates_evaluated != stock.merge.candidates_evaluated) return fail("leaves");
    std::printf("ok cut %.1f leaves %llu subgraphs %d\n", merged.best_value,
                static_cast<unsigned long long>(merged.candidates_evaluated), M);
    return 0;
}
