// qcut_gpu.hpp — header-only C++ shim over the C-ABI (qcgpu.h) with the reference's
// qcut:: signatures, value types and exception taxonomy (errors.hpp:8-24), so code
// written against /root/reference/proj/include/qcut switches to the B200 engine by
// replacing `qcut::solve_subgraph(g, so)` with `qcut_gpu::solve_subgraph(engine, g, so)`
// (or the whole QAOA stage with one `solve_batch`). Link with -lqcgpu.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "qcgpu.h"

namespace qcut_gpu {

// errors.hpp:8-24
class config_error : public std::runtime_error {
public:
    explicit config_error(const std::string& m) : std::runtime_error(m) {}
};
class resource_error : public std::runtime_error {
public:
    explicit resource_error(const std::string& m) : std::runtime_error(m) {}
};
class io_error : public std::runtime_error {
public:
    explicit io_error(const std::string& m) : std::runtime_error(m) {}
};

inline void check(int rc) {
    if (rc == QC_OK) return;
    const std::string msg = qc_last_error();
    switch (rc) {
        case QC_ERR_CONFIG: throw config_error(msg);
        case QC_ERR_RESOURCE: throw resource_error(msg);
        case QC_ERR_IO: throw io_error(msg);
        default: throw std::runtime_error(msg);
    }
}

// graph.hpp:24-81 (edge list; validation happens in the engine exactly as add_edge)
struct Edge {
    std::uint32_t u, v;
    double w = 1.0;
};
struct Graph {
    std::size_t n = 0;
    std::vector<Edge> edges;
    Graph() = default;
    explicit Graph(std::size_t nv) : n(nv) {}
    void add_edge(std::uint32_t u, std::uint32_t v, double w = 1.0) { edges.push_back({u, v, w}); }
    qc_graph view() const {
        static_assert(sizeof(Edge) == sizeof(qc_edge), "Edge layout must match qc_edge");
        return qc_graph{static_cast<int32_t>(n), static_cast<int32_t>(edges.size()),
                        reinterpret_cast<const qc_edge*>(edges.data())};
    }
};

// qaoa.hpp:17-23, :121-152
struct QaoaParams {
    std::vector<double> gammas, betas;
    bool operator==(const QaoaParams& o) const = default;
};
struct Candidate {
    std::uint32_t bits = 0;
    double probability = 0.0;
};
struct CandidateSet {
    int width = 0;
    bool folded = true;
    std::vector<Candidate> entries;
};
struct SolveOptions {
    int top_k = 2;
    int layers = 3;
    int budget = 200;
    std::uint64_t seed = 0;
    bool fold = true;
    int threads = 1;
    std::size_t qubit_cap = 20;
    double tolerance = 1e-5;
};
struct SolveResult {
    CandidateSet candidates;
    QaoaParams params;
    double expectation = 0.0;
    int evals = 0;
};

// merge.hpp:19-25, :85-97, :333-338
struct CandidatePool {
    struct Level {
        int width = 0;
        std::vector<std::uint32_t> bits;
    };
    std::vector<Level> levels;
};
struct Chain {  // partition.hpp PartitionResult: piece i = global ids [first[i], last[i]]
    std::vector<int32_t> first, last;
};
struct MergeOptions {
    int start_level = 1;
    int workers = 1;
    bool incremental = false;  // MergeEval::kIncremental
    double path_budget = 1e9;
    bool halve_symmetry = false;
};
struct ChainedMergeOptions {
    std::size_t window = 0;
    std::size_t window_leaves = 1 << 16;
    int workers = 1;
    bool halve_symmetry = true;
};
struct MergeResult {
    double best_value = 0.0;
    std::vector<std::uint8_t> best_assignment;
    std::uint64_t candidates_evaluated = 0;
};

// One CUDA device (RAII over qc_engine).
class Engine {
public:
    explicit Engine(int device = 0) { check(qc_engine_create(device, &h_)); }
    // with another error mapping (qcut_gpu::reference::check: the reference's own types)
    Engine(int device, void (*chk)(int)) { chk(qc_engine_create(device, &h_)); }
    ~Engine() { qc_engine_destroy(h_); }
    Engine(const Engine&) = delete;
    Engine& operator=(const Engine&) = delete;
    qc_engine* handle() const { return h_; }

private:
    qc_engine* h_ = nullptr;
};

inline QaoaParams linear_ramp(int p) {  // qaoa.hpp:27
    QaoaParams q;
    q.gammas.resize(static_cast<std::size_t>(p > 0 ? p : 1));
    q.betas.resize(q.gammas.size());
    check(qc_linear_ramp(p, q.gammas.data(), q.betas.data()));
    return q;
}

// qaoa.hpp:59 run_ansatz (full 2^n state, interleaved complex) + its expectation
inline std::pair<std::vector<double>, double> run_ansatz(Engine& e, const Graph& g,
                                                         const QaoaParams& p) {
    if (p.gammas.size() != p.betas.size())
        throw config_error("gamma and beta schedules must have equal length");
    std::vector<double> amps(2 * (std::size_t{1} << g.n));
    double ex = 0.0;
    const qc_graph v = g.view();
    check(qc_run_ansatz(e.handle(), &v, static_cast<int>(p.gammas.size()), p.gammas.data(),
                        p.betas.data(), amps.data(), &ex));
    return {std::move(amps), ex};
}

inline qc_solve_options to_c(const SolveOptions& o) {
    qc_solve_options c{};
    c.top_k = o.top_k;
    c.layers = o.layers;
    c.budget = o.budget;
    c.fold = o.fold ? 1 : 0;
    c.seed = o.seed;
    c.qubit_cap = o.qubit_cap;
    c.tolerance = o.tolerance;
    c.threads = o.threads;
    return c;
}

// pipeline.hpp:239-263 QAOA stage as ONE batched device call (graph i solves with opts[i])
inline std::vector<SolveResult> solve_batch(Engine& e, const std::vector<Graph>& graphs,
                                            const std::vector<SolveOptions>& opts) {
    const std::size_t n = graphs.size();
    if (opts.size() != n) throw config_error("one SolveOptions per graph");
    std::vector<qc_graph> gv(n);
    std::vector<qc_solve_options> ov(n);
    std::vector<qc_solve_result> rv(n);
    std::vector<std::vector<std::uint32_t>> bits(n);
    std::vector<std::vector<double>> probs(n), params(n);
    for (std::size_t i = 0; i < n; ++i) {
        gv[i] = graphs[i].view();
        ov[i] = to_c(opts[i]);
        bits[i].resize(static_cast<std::size_t>(opts[i].top_k > 0 ? opts[i].top_k : 1));
        probs[i].resize(bits[i].size());
        params[i].resize(2 * static_cast<std::size_t>(opts[i].layers > 0 ? opts[i].layers : 1));
        rv[i] = qc_solve_result{0, 0, 0, 0, 0.0, bits[i].data(), probs[i].data(), params[i].data()};
    }
    check(qc_solve_batch(e.handle(), gv.data(), static_cast<int>(n), ov.data(), rv.data()));
    std::vector<SolveResult> out(n);
    for (std::size_t i = 0; i < n; ++i) {
        SolveResult& r = out[i];
        r.candidates.width = rv[i].width;
        r.candidates.folded = rv[i].folded != 0;
        for (int k = 0; k < rv[i].count; ++k)
            r.candidates.entries.push_back({bits[i][static_cast<std::size_t>(k)], probs[i][static_cast<std::size_t>(k)]});
        const std::size_t p = static_cast<std::size_t>(opts[i].layers);
        r.params.gammas.assign(params[i].begin(), params[i].begin() + static_cast<long>(p));
        r.params.betas.assign(params[i].begin() + static_cast<long>(p), params[i].begin() + static_cast<long>(2 * p));
        r.expectation = rv[i].expectation;
        r.evals = rv[i].evals;
    }
    return out;
}

// qaoa.hpp:198 solve_subgraph
inline SolveResult solve_subgraph(Engine& e, const Graph& g, const SolveOptions& o = {}) {
    return solve_batch(e, {g}, {o})[0];
}

// merge.hpp:31-51 build_candidate_pools (host; complement-closed, first occurrence kept)
inline CandidatePool build_candidate_pools(const std::vector<CandidateSet>& sets) {
    if (sets.empty()) throw config_error("no candidate sets to merge");
    CandidatePool pool;
    for (const CandidateSet& cs : sets) {
        if (cs.width < 1 || cs.width > 32) throw config_error("candidate width out of range");
        if (cs.entries.empty()) throw config_error("candidate set has no entries");
        const std::uint32_t full = cs.width == 32 ? ~0u : ((1u << cs.width) - 1u);
        CandidatePool::Level lv;
        lv.width = cs.width;
        for (const Candidate& c : cs.entries) {
            if (c.bits > full) throw config_error("candidate bits exceed declared width");
            for (std::uint32_t b : {c.bits, c.bits ^ full}) {
                bool seen = false;
                for (std::uint32_t x : lv.bits) seen = seen || x == b;
                if (!seen) lv.bits.push_back(b);
            }
        }
        pool.levels.push_back(std::move(lv));
    }
    return pool;
}

namespace detail {
struct PoolView {
    std::vector<int32_t> widths, counts;
    std::vector<std::uint32_t> bits;
    qc_pool view() const {
        return qc_pool{static_cast<int32_t>(widths.size()), widths.data(), counts.data(), bits.data()};
    }
};
inline PoolView flatten(const CandidatePool& p) {
    PoolView v;
    for (const auto& lv : p.levels) {
        v.widths.push_back(lv.width);
        v.counts.push_back(static_cast<int32_t>(lv.bits.size()));
        v.bits.insert(v.bits.end(), lv.bits.begin(), lv.bits.end());
    }
    return v;
}
}  // namespace detail

// merge.hpp:280 level_aware_merge
inline MergeResult level_aware_merge(Engine& e, const CandidatePool& pool, const Graph& g,
                                     const Chain& chain, const MergeOptions& o = {}) {
    const auto pv = detail::flatten(pool);
    const qc_pool P = pv.view();
    const qc_graph G = g.view();
    const qc_chain C{static_cast<int32_t>(chain.first.size()), chain.first.data(), chain.last.data()};
    const qc_merge_options mo{o.start_level, o.workers, o.incremental ? 1 : 0,
                              o.halve_symmetry ? 1 : 0, o.path_budget};
    MergeResult r;
    r.best_assignment.resize(g.n);
    qc_merge_result cr{0.0, 0, r.best_assignment.data()};
    check(qc_level_merge(e.handle(), &P, &G, &C, &mo, &cr));
    r.best_value = cr.best_value;
    r.candidates_evaluated = cr.candidates_evaluated;
    return r;
}

// merge.hpp:345 chained_merge
inline MergeResult chained_merge(Engine& e, const CandidatePool& pool, const Graph& g,
                                 const Chain& chain, const ChainedMergeOptions& o = {}) {
    const auto pv = detail::flatten(pool);
    const qc_pool P = pv.view();
    const qc_graph G = g.view();
    const qc_chain C{static_cast<int32_t>(chain.first.size()), chain.first.data(), chain.last.data()};
    const qc_chained_merge_options co{static_cast<int64_t>(o.window),
                                      static_cast<int64_t>(o.window_leaves), o.workers,
                                      o.halve_symmetry ? 1 : 0};
    MergeResult r;
    r.best_assignment.resize(g.n);
    qc_merge_result cr{0.0, 0, r.best_assignment.data()};
    check(qc_chained_merge(e.handle(), &P, &G, &C, &co, &cr));
    r.best_value = cr.best_value;
    r.candidates_evaluated = cr.candidates_evaluated;
    return r;
}

}  // namespace qcut_gpu

// ---------------------------------------------------------------------------
// The reference's own types. Define QCUT_GPU_REFERENCE_TYPES after including the
// reference's <qcut/qaoa.hpp> (or <qcut/pipeline.hpp>): these overloads take qcut::Graph
// and qcut::SolveOptions, return qcut::SolveResult, and rethrow the engine's codes as
// qcut::config_error / resource_error / io_error, so the call site at pipeline.hpp:263 and
// the stage guard at pipeline.hpp:137-159 stay as they are (tests/cpp/ref_pipeline.cpp runs
// the reference's run_pipeline with only its QAOA stage replaced by reference::solve_batch).
// ---------------------------------------------------------------------------
#ifdef QCUT_GPU_REFERENCE_TYPES
namespace qcut_gpu::reference {

inline void check(int rc) {
    if (rc == QC_OK) return;
    const std::string msg = qc_last_error();
    switch (rc) {
        case QC_ERR_CONFIG: throw qcut::config_error(msg);
        case QC_ERR_RESOURCE: throw qcut::resource_error(msg);
        case QC_ERR_IO: throw qcut::io_error(msg);
        default: throw std::runtime_error(msg);
    }
}

inline Engine& default_engine(int device = 0) {  // one per process, created on first use
    static Engine e(device, &check);
    return e;
}

inline qc_graph view(const qcut::Graph& g) {  // graph.hpp:21-25 Edge {u, v, w} == qc_edge
    static_assert(sizeof(qcut::Edge) == sizeof(qc_edge), "qcut::Edge layout must match qc_edge");
    return qc_graph{static_cast<int32_t>(g.n()), static_cast<int32_t>(g.edge_count()),
                    reinterpret_cast<const qc_edge*>(g.edges().data())};
}

// pipeline.hpp:239-263: the whole QAOA stage as one batched device call
inline std::vector<qcut::SolveResult> solve_batch(Engine& e, const std::vector<const qcut::Graph*>& graphs,
                                                  const std::vector<qcut::SolveOptions>& opts) {
    const std::size_t n = graphs.size();
    if (opts.size() != n) throw qcut::config_error("one SolveOptions per graph");
    std::vector<qc_graph> gv(n);
    std::vector<qc_solve_options> ov(n);
    std::vector<qc_solve_result> rv(n);
    std::vector<std::vector<std::uint32_t>> bits(n);
    std::vector<std::vector<double>> probs(n), params(n);
    for (std::size_t i = 0; i < n; ++i) {
        gv[i] = view(*graphs[i]);
        const qcut::SolveOptions& o = opts[i];
        qc_solve_options& c = ov[i];
        c = qc_solve_options{};
        c.top_k = o.top_k;
        c.layers = o.layers;
        c.budget = o.budget;
        c.fold = o.fold ? 1 : 0;
        c.seed = o.seed;
        c.qubit_cap = o.qubit_cap;
        c.tolerance = o.tolerance;
        c.threads = o.threads;
        bits[i].resize(static_cast<std::size_t>(o.top_k > 0 ? o.top_k : 1));
        probs[i].resize(bits[i].size());
        params[i].resize(2 * static_cast<std::size_t>(o.layers > 0 ? o.layers : 1));
        rv[i] = qc_solve_result{0, 0, 0, 0, 0.0, bits[i].data(), probs[i].data(), params[i].data()};
    }
    check(qc_solve_batch(e.handle(), gv.data(), static_cast<int>(n), ov.data(), rv.data()));
    std::vector<qcut::SolveResult> out(n);
    for (std::size_t i = 0; i < n; ++i) {
        qcut::SolveResult& r = out[i];
        r.candidates.width = rv[i].width;
        r.candidates.folded = rv[i].folded != 0;
        for (int k = 0; k < rv[i].count; ++k)
            r.candidates.entries.push_back({bits[i][static_cast<std::size_t>(k)], probs[i][static_cast<std::size_t>(k)]});
        const auto p = static_cast<long>(opts[i].layers);
        r.params.gammas.assign(params[i].begin(), params[i].begin() + p);
        r.params.betas.assign(params[i].begin() + p, params[i].begin() + 2 * p);
        r.expectation = rv[i].expectation;
        r.evals = rv[i].evals;
    }
    return out;
}

// qaoa.hpp:198 solve_subgraph, on the process's default engine: the one-line replacement
// of the call at pipeline.hpp:263
inline qcut::SolveResult solve_subgraph(const qcut::Graph& g, const qcut::SolveOptions& so = {}) {
    return solve_batch(default_engine(), {&g}, {so})[0];
}

}  // namespace qcut_gpu::reference
#endif
