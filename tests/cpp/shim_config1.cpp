// C++ drop-in check: the reference's config-1 QAOA stage + merge written against the
// qcut_gpu shim exactly as pipeline.hpp:239-334 would call it (one batched solve
// instead of a std::thread per subgraph). Prints "cut <value> leaves <n>".
#include <cstdio>
#include <random>
#include <vector>

#include "qcut_gpu.hpp"

int main() {
    using namespace qcut_gpu;
    // generate_er_graph(100, 0.1, 0) (graph.hpp:146-160)
    Graph g(100);
    std::mt19937_64 rng(0);
    for (std::uint32_t u = 0; u + 1 < 100; ++u)
        for (std::uint32_t v = u + 1; v < 100; ++v)
            if (static_cast<double>(rng() >> 11) * 0x1.0p-53 < 0.1) g.add_edge(u, v);
    // partition(g, 11) (partition.hpp:111): 11 pieces of 10 vertices
    Chain chain;
    std::vector<Graph> subs;
    std::vector<SolveOptions> opts;
    for (int i = 0; i < 11; ++i) {
        const std::uint32_t a = 9u * static_cast<std::uint32_t>(i), b = a + 9u;
        chain.first.push_back(static_cast<int32_t>(a));
        chain.last.push_back(static_cast<int32_t>(b));
        Graph s(10);
        for (const Edge& e : g.edges)
            if (e.u >= a && e.v <= b && !(i + 1 < 11 && e.u == b)) s.add_edge(e.u - a, e.v - a, e.w);
        subs.push_back(s);
        SolveOptions so;
        so.top_k = 4;
        so.layers = 1;
        so.budget = 200;
        so.seed = static_cast<std::uint64_t>(i);  // pipeline.hpp:258
        so.qubit_cap = 10;
        opts.push_back(so);
    }
    Engine eng(0);
    const auto solves = solve_batch(eng, subs, opts);
    std::vector<CandidateSet> sets;
    for (const auto& s : solves) sets.push_back(s.candidates);
    const CandidatePool pool = build_candidate_pools(sets);
    MergeOptions mo;
    mo.incremental = true;
    const MergeResult m = level_aware_merge(eng, pool, g, chain, mo);
    std::printf("cut %.1f leaves %llu\n", m.best_value,
                static_cast<unsigned long long>(m.candidates_evaluated));
    try {
        SolveOptions bad;
        bad.top_k = 0;
        (void)solve_subgraph(eng, subs[0], bad);
    } catch (const config_error&) {
        std::printf("config_error ok\n");
    }
    return 0;
}
