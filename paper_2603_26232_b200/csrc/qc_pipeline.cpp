// Pipeline stages around the hot path (pipeline.hpp:135-336): chain partition
// (partition.hpp:58-160, host prep), the batched QAOA stage on the device, candidate
// pools (merge.hpp:31-51) and the device merge (qc_merge.cu). Also the merge.hpp entry
// points and the fixed-size solve records used by the multi-GPU gather.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <memory>
#include <cmath>
#include <cstring>
#include <random>
#include <string>
#include <unordered_set>
#include <vector>

#include "qc_engine.hpp"
#include "qc_merge.hpp"

using namespace qcg;

namespace {

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return QC_OK;
    } catch (const qcg::Error& e) {
        qcg::set_error(e.what());
        return e.code;
    } catch (const std::bad_alloc&) {
        qcg::set_error("host out of memory");
        return QC_ERR_RESOURCE;
    } catch (const std::exception& e) {
        qcg::set_error(e.what());
        return QC_ERR_INTERNAL;
    }
}

struct Partition {
    std::vector<int32_t> first, last;
    std::vector<HostGraph> local;  // local ids, global edge-list order
    long long inter = 0;
};

// partition.hpp:58-103 chain_intervals
void chain_intervals(int n, int M, int mode, std::vector<int32_t>& a, std::vector<int32_t>& b) {
    if (M < 1) config_error("subgraph count must be positive");
    if (n == 0) config_error("cannot partition an empty graph");
    a.assign(static_cast<size_t>(M), 0);
    b.assign(static_cast<size_t>(M), 0);
    if (M == 1) {
        b[0] = n - 1;
        return;
    }
    if (n < M + 1)
        config_error("need at least " + std::to_string(M + 1) + " vertices for " + std::to_string(M) +
                     " chained subgraphs, got " + std::to_string(n));
    std::vector<long long> spans(static_cast<size_t>(M));
    const long long total = n - 1;
    if (mode == 1) {
        const long long s = n / M - 1;
        if (s < 1)
            config_error("tail-remainder split needs n >= 2*M, got n=" + std::to_string(n) +
                         " M=" + std::to_string(M));
        for (int i = 0; i + 1 < M; ++i) spans[static_cast<size_t>(i)] = s;
        spans[static_cast<size_t>(M - 1)] = total - static_cast<long long>(M - 1) * s;
    } else {
        const long long s = (total + M - 1) / M;
        if (static_cast<long long>(M - 1) * s <= total - 1) {
            for (int i = 0; i + 1 < M; ++i) spans[static_cast<size_t>(i)] = s;
            spans[static_cast<size_t>(M - 1)] = total - static_cast<long long>(M - 1) * s;
        } else {
            const long long q = total / M, r = total % M;
            for (int i = 0; i < M; ++i) spans[static_cast<size_t>(i)] = q + (i < r ? 1 : 0);
        }
    }
    long long x = 0;
    for (int i = 0; i < M; ++i) {
        a[static_cast<size_t>(i)] = static_cast<int32_t>(x);
        x += spans[static_cast<size_t>(i)];
        b[static_cast<size_t>(i)] = static_cast<int32_t>(x);
    }
}

// partition.hpp:111-160 partition
Partition partition(const HostGraph& g, int M, int mode, int cap) {
    NvtxRange nv("qcgpu.partition");
    Partition P;
    chain_intervals(g.n, M, mode, P.first, P.last);
    if (cap > 0) {
        int largest = 0;
        for (int i = 0; i < M; ++i) largest = std::max(largest, P.last[static_cast<size_t>(i)] - P.first[static_cast<size_t>(i)] + 1);
        if (largest > cap) {
            const long long need = (static_cast<long long>(g.n) - 1 + cap - 2) / (cap - 1);
            resource_error("largest subgraph has " + std::to_string(largest) + " vertices, over the " +
                           std::to_string(cap) + "-qubit cap; use at least " + std::to_string(need) +
                           " subgraphs");
        }
    }
    std::vector<int32_t> last_piece(static_cast<size_t>(g.n));
    for (int i = 0; i < M; ++i)
        for (int v = P.first[static_cast<size_t>(i)]; v <= P.last[static_cast<size_t>(i)]; ++v)
            last_piece[static_cast<size_t>(v)] = i;
    P.local.resize(static_cast<size_t>(M));
    for (int i = 0; i < M; ++i) P.local[static_cast<size_t>(i)].n = P.last[static_cast<size_t>(i)] - P.first[static_cast<size_t>(i)] + 1;
    for (size_t k = 0; k < g.u.size(); ++k) {
        const uint32_t u = g.u[k], v = g.v[k];  // u < v
        const int i = last_piece[u];
        if (static_cast<int>(v) <= P.last[static_cast<size_t>(i)]) {
            HostGraph& L = P.local[static_cast<size_t>(i)];
            L.u.push_back(u - static_cast<uint32_t>(P.first[static_cast<size_t>(i)]));
            L.v.push_back(v - static_cast<uint32_t>(P.first[static_cast<size_t>(i)]));
            L.w.push_back(g.w[k]);
            L.total += g.w[k];
            if (g.w[k] != std::floor(g.w[k]) || g.w[k] < 0.0) L.integral = false;
        } else {
            ++P.inter;
        }
    }
    for (auto& L : P.local)
        if (L.total > 65535.0) L.integral = false;
    return P;
}

int derive_subgraph_count(long long n, long long cap) {  // partition.hpp:163-167
    if (cap < 2) config_error("qubit cap must be at least 2");
    if (n <= cap) return 1;
    return static_cast<int>((n - 1 + cap - 2) / (cap - 1));
}

struct Pool {
    std::vector<int32_t> widths, counts;
    std::vector<uint32_t> bits;
};

// merge.hpp:31-51 build_candidate_pools
Pool build_pools(const std::vector<SolveOut>& sets) {
    if (sets.empty()) config_error("no candidate sets to merge");
    Pool P;
    for (const auto& cs : sets) {
        if (cs.width < 1 || cs.width > 32) config_error("candidate width out of range");
        if (cs.bits.empty()) config_error("candidate set has no entries");
        const uint32_t full = cs.width == 32 ? ~0u : ((1u << cs.width) - 1u);
        std::unordered_set<uint32_t> seen;
        int cnt = 0;
        for (uint32_t b0 : cs.bits) {
            if (b0 > full) config_error("candidate bits exceed declared width");
            for (uint32_t b : {b0, b0 ^ full})
                if (seen.insert(b).second) {
                    P.bits.push_back(b);
                    ++cnt;
                }
        }
        P.widths.push_back(cs.width);
        P.counts.push_back(cnt);
    }
    return P;
}

MergeInput make_input(const HostGraph& g, std::vector<qc_edge_t>& store, const Pool& pool,
                      const std::vector<int32_t>& first, const std::vector<int32_t>& last) {
    (void)store;  // the merge reads the HostGraph's SoA edge arrays directly
    MergeInput in;
    in.n = g.n;
    in.m = static_cast<long long>(g.u.size());
    in.eu = g.u.data();
    in.ev = g.v.data();
    in.ew = g.w.data();
    in.all_int = g.all_int ? 1 : 0;
    in.levels = static_cast<int>(pool.widths.size());
    in.widths = pool.widths.data();
    in.counts = pool.counts.data();
    in.bits = pool.bits.data();
    in.pieces = static_cast<int>(first.size());
    in.first = first.data();
    in.last = last.data();
    return in;
}

// merge.hpp:280-331 level_aware_merge
MergeOutput level_merge(qc_engine* e, const MergeInput& in, int start_level, int workers,
                        bool incremental, double path_budget, bool halve) {
    check_pool(in);
    const int M = in.levels;
    if (start_level < 1 || start_level > M)
        config_error("start level must lie in [1, " + std::to_string(M) + "]");
    if (workers < 1) config_error("worker count must be positive");
    if (!(path_budget > 0)) config_error("path budget must be positive");
    const double est = estimate_paths(in.counts, M, halve);
    if (est > path_budget)
        resource_error("merge would enumerate about " + std::to_string(est) +
                       " complete chains, over the " + std::to_string(path_budget) +
                       " budget; lower the retained candidate count or the subgraph count, or "
                       "switch to the windowed merge");
    double prefix_est = static_cast<double>(in.counts[0]);
    if (halve) prefix_est /= 2.0;
    for (int i = 1; i < start_level; ++i) prefix_est *= static_cast<double>(in.counts[i]) / 2.0;
    if (prefix_est > static_cast<double>(size_t{1} << 22))
        resource_error("start level " + std::to_string(start_level) + " expands to about " +
                       std::to_string(prefix_est) + " prefixes; lower it");
    return run_merge(in, {Window{0, M, halve ? 3 : 2}}, !incremental, e->stream, &e->launches,
                     &e->prof, &e->h2d, &e->d2h, &e->merge_arena);
}

// merge.hpp:345-412 chained_merge
MergeOutput chained_merge(qc_engine* e, const MergeInput& in, long long window,
                          long long window_leaves, int workers, bool halve) {
    check_pool(in);
    const int M = in.levels;
    if (workers < 1) config_error("worker count must be positive");
    if (window_leaves < 2) config_error("window leaf target must be at least 2");
    std::vector<Window> wins;
    int s = 0;
    while (s < M) {
        int e_ = s + 1;
        double leaves = static_cast<double>(in.counts[s]);
        if (s == 0 && halve) leaves /= 2.0;
        if (s > 0) leaves /= 2.0;
        if (window > 0) {
            const int cap = static_cast<int>(std::min<long long>(M, s + window));
            for (; e_ < cap; ++e_) leaves *= static_cast<double>(in.counts[e_]) / 2.0;
        } else {
            while (e_ < M) {
                const double grown = leaves * static_cast<double>(in.counts[e_]) / 2.0;
                if (grown > static_cast<double>(window_leaves)) break;
                leaves = grown;
                ++e_;
            }
        }
        if (leaves > 1e9)
            resource_error("merge window spans about " + std::to_string(leaves) +
                           " combos; shrink the window");
        wins.push_back({s, e_, s == 0 ? (halve ? 3 : 2) : -1});
        s = e_;
    }
    return run_merge(in, wins, false, e->stream, &e->launches, &e->prof, &e->h2d, &e->d2h,
                     &e->merge_arena);
}

Pool pool_from_c(const qc_pool* p) {
    if (!p) config_error("null pool");
    Pool P;
    if (p->levels < 1) config_error("no candidate sets to merge");
    P.widths.assign(p->widths, p->widths + p->levels);
    P.counts.assign(p->counts, p->counts + p->levels);
    size_t tot = 0;
    for (int i = 0; i < p->levels; ++i) {
        if (p->counts[i] < 0) config_error("negative pool level size");
        tot += static_cast<size_t>(p->counts[i]);
    }
    P.bits.assign(p->bits, p->bits + tot);
    return P;
}

// ---- solve records (multi-GPU gather) -----------------------------------------
// [int32 width, count, evals, pad][double expectation][uint32 bits[K] pad8][double probs[K]]
// [double params[2p]]
int64_t record_bytes(int kcap, int layers) {
    return 24 + 8 * ((static_cast<int64_t>(kcap) * 4 + 7) / 8) + 8 * static_cast<int64_t>(kcap) +
           16 * static_cast<int64_t>(layers);
}

void pack_record(const SolveOut& s, int kcap, int layers, char* r) {
    std::memset(r, 0, static_cast<size_t>(record_bytes(kcap, layers)));
    const int32_t hdr[4] = {s.width, static_cast<int32_t>(s.bits.size()), s.evals, s.folded ? 1 : 0};
    std::memcpy(r, hdr, 16);
    std::memcpy(r + 16, &s.expectation, 8);
    char* p = r + 24;
    std::memcpy(p, s.bits.data(), s.bits.size() * 4);
    p += 8 * ((static_cast<int64_t>(kcap) * 4 + 7) / 8);
    std::memcpy(p, s.probs.data(), s.probs.size() * 8);
    p += 8 * static_cast<int64_t>(kcap);
    std::memcpy(p, s.params.data(), s.params.size() * 8);
}

SolveOut unpack_record(const char* r, int kcap, int layers) {
    SolveOut s;
    int32_t hdr[4];
    std::memcpy(hdr, r, 16);
    s.width = hdr[0];
    s.evals = hdr[2];
    s.folded = hdr[3] != 0;
    std::memcpy(&s.expectation, r + 16, 8);
    const int cnt = hdr[1];
    if (cnt < 0 || cnt > kcap) config_error("corrupt solve record");
    s.bits.resize(static_cast<size_t>(cnt));
    s.probs.resize(static_cast<size_t>(cnt));
    const char* p = r + 24;
    std::memcpy(s.bits.data(), p, static_cast<size_t>(cnt) * 4);
    p += 8 * ((static_cast<int64_t>(kcap) * 4 + 7) / 8);
    std::memcpy(s.probs.data(), p, static_cast<size_t>(cnt) * 8);
    p += 8 * static_cast<int64_t>(kcap);
    s.params.resize(2 * static_cast<size_t>(layers));
    std::memcpy(s.params.data(), p, s.params.size() * 8);
    return s;
}

void check_config(const qc_run_config* c) {  // pipeline.hpp:172-187
    if (!c) config_error("null run config");
    if (c->layers < 1) config_error("layer count must be positive");
    if (c->budget < 1) config_error("optimizer budget must be positive");
    if (c->top_k < 0) config_error("top_k cannot be negative");
    if (c->start_level < 1) config_error("start level must be positive");
    if (c->qubit_cap < 2 || c->qubit_cap > kMaxQubits)
        config_error("qubit cap must lie in [2, " + std::to_string(kMaxQubits) + "]");
    if (!(c->path_budget > 0)) config_error("path budget must be positive");
    if (c->subgraphs < 0) config_error("subgraph count cannot be negative");
    if (c->shard_count < 1 || c->shard_index < 0 || c->shard_index >= c->shard_count)
        config_error("invalid shard index/count");
}

int kcap_of(const qc_run_config* c, int max_width) {
    const uint64_t classes = c->fold ? (uint64_t{1} << (max_width - 1)) : (uint64_t{1} << max_width);
    if (c->top_k == 0) return static_cast<int>(std::min<uint64_t>(classes, 1u << 30));
    return static_cast<int>(std::min<uint64_t>(classes, static_cast<uint64_t>(c->top_k)));
}

// widest piece of the chain partition (partition.hpp:58-103), without building it
int max_width(int n, int M, const qc_run_config* c) {
    std::vector<int32_t> a, b;
    chain_intervals(n, M, c->partition_mode, a, b);
    int w = 1;
    for (size_t i = 0; i < a.size(); ++i) w = std::max(w, b[i] - a[i] + 1);
    return w;
}

// pipeline.hpp:239-263 per-subgraph options for subgraphs [begin, end)
std::vector<SolveOut> solve_range(qc_engine* e, const Partition& P, const qc_run_config* c,
                                  int begin, int end) {
    std::vector<HostGraph> hg;
    std::vector<qc_solve_options> opts;
    for (int idx = begin; idx < end; ++idx) {
        const HostGraph& L = P.local[static_cast<size_t>(idx)];
        const uint64_t classes = c->fold ? (uint64_t{1} << (L.n - 1)) : (uint64_t{1} << L.n);
        qc_solve_options so{};
        so.top_k = c->top_k == 0 ? static_cast<int>(classes)
                                 : static_cast<int>(std::min<uint64_t>(classes, static_cast<uint64_t>(c->top_k)));
        so.layers = c->layers;
        so.budget = c->budget;
        so.seed = c->seed + static_cast<uint64_t>(idx);
        so.fold = c->fold;
        so.qubit_cap = static_cast<uint64_t>(c->qubit_cap);
        so.tolerance = c->nm_tolerance;
        hg.push_back(L);
        opts.push_back(so);
    }
    return solve_batch(e, hg, opts);
}

MergeOutput merge_stage(qc_engine* e, const HostGraph& g, const Partition& P,
                        const std::vector<SolveOut>& solves, const qc_run_config* c, bool* windowed) {
    NvtxRange nv("qcgpu.merge");
    const auto tm0 = std::chrono::steady_clock::now();
    const Pool pool = build_pools(solves);
    std::vector<qc_edge_t> store;
    const MergeInput in = make_input(g, store, pool, P.first, P.last);
    if (std::getenv("QCG_TRACE_MERGE"))
        std::fprintf(stderr, "merge pools+input %8.2f ms\n",
                     std::chrono::duration<double>(std::chrono::steady_clock::now() - tm0).count() * 1e3);
    const int M = static_cast<int>(P.first.size());
    int mode = c->merge_mode;  // pipeline.hpp:307-311
    if (mode == 0)
        mode = estimate_paths(pool.counts.data(), M, c->halve_symmetry != 0) <= c->path_budget ? 1 : 2;
    *windowed = mode == 2;
    if (mode == 1)
        return level_merge(e, in, std::min(c->start_level, M), 1, c->merge_incremental != 0,
                           c->path_budget, c->halve_symmetry != 0);
    return chained_merge(e, in, 0, 1 << 16, 1, true);
}

double seconds_since(std::chrono::steady_clock::time_point t0) {
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

void write_assignment(const std::vector<uint8_t>& a, char* out) {
    if (!out) return;
    for (size_t v = 0; v < a.size(); ++v) out[v] = a[v] ? '1' : '0';
    out[a.size()] = 0;
}


// graph.hpp:146-160 and the config-3 regular generator (host instance prep)
std::vector<qc_edge_t> gen_er(int n, double p, uint64_t seed) {
    if (p < 0.0 || p > 1.0 || std::isnan(p)) config_error("edge probability must lie in [0,1]");
    if (n < 0) config_error("negative vertex count");
    std::vector<qc_edge_t> out;
    std::mt19937_64 rng(seed);
    for (uint32_t u = 0; u + 1 < static_cast<uint32_t>(n); ++u)
        for (uint32_t v = u + 1; v < static_cast<uint32_t>(n); ++v) {
            const double x = static_cast<double>(rng() >> 11) * 0x1.0p-53;
            if (x < p) out.push_back({u, v, 1.0});
        }
    return out;
}

std::vector<qc_edge_t> gen_regular(int n, int d, uint64_t seed, int wlo, int whi) {
    if (n < 1 || d < 1 || d >= n) config_error("regular graph needs 1 <= d < n");
    if ((static_cast<long long>(n) * d) % 2) config_error("n*d must be even");
    if (wlo < 0 || whi < wlo) config_error("weight range must satisfy 0 <= wlo <= whi");
    std::mt19937_64 rng(seed);
    const size_t S = static_cast<size_t>(n) * static_cast<size_t>(d);
    std::vector<uint32_t> stubs(S);
    std::vector<qc_edge_t> out;
    for (int attempt = 0; attempt < 100000; ++attempt) {
        for (size_t i = 0; i < S; ++i) stubs[i] = static_cast<uint32_t>(i / static_cast<size_t>(d));
        for (size_t i = S - 1; i > 0; --i) {
            const size_t j = static_cast<size_t>(rng() % (i + 1));
            std::swap(stubs[i], stubs[j]);
        }
        out.clear();
        std::unordered_set<uint64_t> seen;
        bool ok = true;
        for (size_t i = 0; i < S && ok; i += 2) {
            uint32_t u = stubs[i], v = stubs[i + 1];
            if (u == v) ok = false;
            if (u > v) std::swap(u, v);
            if (ok && !seen.insert(static_cast<uint64_t>(u) * static_cast<uint64_t>(n) + v).second) ok = false;
            if (ok) out.push_back({u, v, 0.0});
        }
        if (!ok) continue;
        std::sort(out.begin(), out.end(), [](const qc_edge_t& a, const qc_edge_t& b) {
            return a.u != b.u ? a.u < b.u : a.v < b.v;
        });
        const uint64_t span = static_cast<uint64_t>(whi - wlo + 1);
        for (auto& e : out) e.w = static_cast<double>(wlo + static_cast<int>(rng() % span));
        return out;
    }
    resource_error("no simple regular graph found");
}

int copy_edges(const std::vector<qc_edge_t>& g, qc_edge* edges, int64_t cap, int64_t* m) {
    *m = static_cast<int64_t>(g.size());
    if (!edges) return 0;
    if (cap < *m) config_error("edge buffer too small");
    std::memcpy(edges, g.data(), g.size() * sizeof(qc_edge_t));
    return 0;
}

}  // namespace

extern "C" {

int qc_generate_er(int n, double p, uint64_t seed, qc_edge* edges, int64_t cap, int64_t* m) {
    return guarded([&] { copy_edges(gen_er(n, p, seed), edges, cap, m); });
}

int qc_generate_regular(int n, int d, uint64_t seed, int wlo, int whi, qc_edge* edges,
                        int64_t cap, int64_t* m) {
    return guarded([&] { copy_edges(gen_regular(n, d, seed, wlo, whi), edges, cap, m); });
}

int qc_level_merge(qc_engine* e, const qc_pool* pool, const qc_graph* g, const qc_chain* chain,
                   const qc_merge_options* opt, qc_merge_result* res) {
    return guarded([&] {
        if (!e) config_error("null engine");
        QC_CUDA(cudaSetDevice(e->device));
        if (!opt || !res || !chain) config_error("null argument");
        const HostGraph hg = load_graph(g);
        const Pool P = pool_from_c(pool);
        std::vector<int32_t> first(chain->first, chain->first + chain->pieces);
        std::vector<int32_t> last(chain->last, chain->last + chain->pieces);
        std::vector<qc_edge_t> store;
        const MergeInput in = make_input(hg, store, P, first, last);
        const MergeOutput out = level_merge(e, in, opt->start_level, opt->workers,
                                            opt->incremental != 0, opt->path_budget,
                                            opt->halve_symmetry != 0);
        res->best_value = out.value;
        res->candidates_evaluated = out.leaves;
        if (res->assignment) std::memcpy(res->assignment, out.assignment.data(), out.assignment.size());
    });
}

int qc_chained_merge(qc_engine* e, const qc_pool* pool, const qc_graph* g, const qc_chain* chain,
                     const qc_chained_merge_options* opt, qc_merge_result* res) {
    return guarded([&] {
        if (!e) config_error("null engine");
        QC_CUDA(cudaSetDevice(e->device));
        if (!opt || !res || !chain) config_error("null argument");
        const HostGraph hg = load_graph(g);
        const Pool P = pool_from_c(pool);
        std::vector<int32_t> first(chain->first, chain->first + chain->pieces);
        std::vector<int32_t> last(chain->last, chain->last + chain->pieces);
        std::vector<qc_edge_t> store;
        const MergeInput in = make_input(hg, store, P, first, last);
        const MergeOutput out = chained_merge(e, in, opt->window, opt->window_leaves, opt->workers,
                                              opt->halve_symmetry != 0);
        res->best_value = out.value;
        res->candidates_evaluated = out.leaves;
        if (res->assignment) std::memcpy(res->assignment, out.assignment.data(), out.assignment.size());
    });
}

int qc_run_pipeline(qc_engine* e, const qc_graph* g, const qc_run_config* cfg,
                    qc_run_report* report, char* assignment) {
    return guarded([&] {
        if (!e) config_error("null engine");
        QC_CUDA(cudaSetDevice(e->device));
        check_config(cfg);
        if (cfg->shard_count != 1) config_error("qc_run_pipeline is single-shard; use qc_shard_solve");
        const HostGraph hg = load_graph(g);
        qc_run_report r{};
        auto t0 = std::chrono::steady_clock::now();
        const int M = cfg->subgraphs != 0 ? cfg->subgraphs : derive_subgraph_count(hg.n, cfg->qubit_cap);
        const Partition P = partition(hg, M, cfg->partition_mode, cfg->qubit_cap);
        r.partition_s = seconds_since(t0);
        r.subgraphs = M;

        t0 = std::chrono::steady_clock::now();
        const auto solves = solve_range(e, P, cfg, 0, M);
        r.qaoa_s = seconds_since(t0);
        for (const auto& s : solves) r.evals += static_cast<uint64_t>(s.evals);

        t0 = std::chrono::steady_clock::now();
        bool windowed = false;
        const MergeOutput out = merge_stage(e, hg, P, solves, cfg, &windowed);
        r.merge_s = seconds_since(t0);
        r.total_s = r.partition_s + r.qaoa_s + r.merge_s;
        r.cut = out.value;
        r.candidates_evaluated = out.leaves;
        r.windowed = windowed ? 1 : 0;
        if (report) *report = r;
        write_assignment(out.assignment, assignment);
    });
}

}  // extern "C"

struct qc_pipeline {
    qc_engine* e = nullptr;
    qc_run_config cfg{};
    HostGraph g;
    Partition P;
    std::vector<qc_solve_options> opts;
    qcg::DevBuf tables;  // resident device cut tables of every subgraph (of this shard)
    std::vector<DevGraph> dg;
    double partition_s = 0.0;
    std::vector<SolveOut> last;  // SolveResults of the last execute (qc_pipeline_records)
    // sharded session (cfg.shard_count > 1): this rank's contiguous block [begin, end)
    int begin = 0, end = 0;
    std::vector<HostGraph> shard_local;
    std::vector<qc_solve_options> shard_opts;
    int kcap = 1;
    int64_t rb = 0;  // record bytes of the run (widest piece of the whole partition)
};

extern "C" {

int qc_pipeline_prepare(qc_engine* e, const qc_graph* g, const qc_run_config* cfg,
                        qc_pipeline** out) {
    return guarded([&] {
        if (!e || !out) config_error("null argument");
        QC_CUDA(cudaSetDevice(e->device));
        check_config(cfg);
        auto pl = std::make_unique<qc_pipeline>();
        pl->e = e;
        pl->cfg = *cfg;
        pl->g = load_graph(g);
        auto t0 = std::chrono::steady_clock::now();
        const int M = cfg->subgraphs != 0 ? cfg->subgraphs : derive_subgraph_count(pl->g.n, cfg->qubit_cap);
        pl->P = partition(pl->g, M, cfg->partition_mode, cfg->qubit_cap);
        pl->partition_s = seconds_since(t0);
        for (int idx = 0; idx < M; ++idx) {
            const HostGraph& L = pl->P.local[static_cast<size_t>(idx)];
            const uint64_t classes = cfg->fold ? (uint64_t{1} << (L.n - 1)) : (uint64_t{1} << L.n);
            qc_solve_options so{};
            so.top_k = cfg->top_k == 0 ? static_cast<int>(classes)
                                       : static_cast<int>(std::min<uint64_t>(classes, static_cast<uint64_t>(cfg->top_k)));
            so.layers = cfg->layers;
            so.budget = cfg->budget;
            so.seed = cfg->seed + static_cast<uint64_t>(idx);
            so.fold = cfg->fold;
            so.qubit_cap = static_cast<uint64_t>(cfg->qubit_cap);
            so.tolerance = cfg->nm_tolerance;
            pl->opts.push_back(so);
        }
        validate_solve(pl->P.local, pl->opts);
        int maxw = 1;
        for (const auto& L : pl->P.local) maxw = std::max(maxw, L.n);
        pl->kcap = kcap_of(cfg, maxw);
        pl->rb = record_bytes(pl->kcap, cfg->layers);
        if (cfg->shard_count > 1) {  // only this rank's block gets device tables
            int32_t b = 0, en = 0;
            if (qc_shard_range(M, cfg->shard_index, cfg->shard_count, &b, &en) != 0)
                config_error("invalid shard request");
            pl->begin = b;
            pl->end = en;
            pl->shard_local.assign(pl->P.local.begin() + b, pl->P.local.begin() + en);
            pl->shard_opts.assign(pl->opts.begin() + b, pl->opts.begin() + en);
            pl->dg = e->prepare(pl->shard_local, true, false, &pl->tables);
        } else {
            pl->begin = 0;
            pl->end = M;
            pl->dg = e->prepare(pl->P.local, true, false, &pl->tables);
        }
        *out = pl.release();
    });
}

int qc_pipeline_execute_shard(qc_pipeline* pl, void* records, int64_t capacity, int32_t* begin,
                              int32_t* end, double* qaoa_s) {
    return guarded([&] {
        if (!pl) config_error("null pipeline");
        if (pl->cfg.shard_count <= 1) config_error("qc_pipeline_execute_shard needs a sharded session");
        qc_engine* e = pl->e;
        QC_CUDA(cudaSetDevice(e->device));
        const int n = pl->end - pl->begin;
        if (begin) *begin = pl->begin;
        if (end) *end = pl->end;
        if (!records) return;
        if (capacity < pl->rb * n)
            config_error("record buffer holds " + std::to_string(capacity) + " bytes, the shard needs " +
                         std::to_string(pl->rb * n) + " (qc_pipeline_records)");
        const auto t0 = std::chrono::steady_clock::now();
        pl->last = n ? solve_prepared(e, pl->shard_local, pl->dg, pl->shard_opts) : std::vector<SolveOut>{};
        for (int k = 0; k < n; ++k)
            pack_record(pl->last[static_cast<size_t>(k)], pl->kcap, pl->cfg.layers,
                        static_cast<char*>(records) + static_cast<int64_t>(k) * pl->rb);
        if (qaoa_s) *qaoa_s = seconds_since(t0);
    });
}

int qc_pipeline_merge_records(qc_pipeline* pl, const void* records, int64_t capacity, qc_run_report* report,
                              char* assignment) {
    return guarded([&] {
        if (!pl) config_error("null pipeline");
        qc_engine* e = pl->e;
        QC_CUDA(cudaSetDevice(e->device));
        const int M = static_cast<int>(pl->P.first.size());
        if (capacity < pl->rb * M)
            config_error("record buffer holds " + std::to_string(capacity) + " bytes, " + std::to_string(M) +
                         " records need " + std::to_string(pl->rb * M));
        std::vector<SolveOut> solves;
        solves.reserve(static_cast<size_t>(M));
        for (int i = 0; i < M; ++i)
            solves.push_back(unpack_record(static_cast<const char*>(records) + static_cast<int64_t>(i) * pl->rb,
                                           pl->kcap, pl->cfg.layers));
        const auto t0 = std::chrono::steady_clock::now();
        bool windowed = false;
        const MergeOutput out = merge_stage(e, pl->g, pl->P, solves, &pl->cfg, &windowed);
        qc_run_report r{};
        r.merge_s = seconds_since(t0);
        r.partition_s = pl->partition_s;
        r.subgraphs = M;
        r.cut = out.value;
        r.candidates_evaluated = out.leaves;
        r.windowed = windowed ? 1 : 0;
        for (const auto& sv : solves) r.evals += static_cast<uint64_t>(sv.evals);
        if (report) *report = r;
        write_assignment(out.assignment, assignment);
    });
}

int qc_pipeline_execute(qc_pipeline* pl, qc_run_report* report, char* assignment) {
    return guarded([&] {
        if (!pl) config_error("null pipeline");
        if (pl->cfg.shard_count > 1)
            config_error("sharded session: qc_pipeline_execute_shard + qc_pipeline_merge_records");
        qc_engine* e = pl->e;
        QC_CUDA(cudaSetDevice(e->device));
        qc_run_report r{};
        r.partition_s = pl->partition_s;
        r.subgraphs = static_cast<int32_t>(pl->P.first.size());
        auto t0 = std::chrono::steady_clock::now();
        pl->last = solve_prepared(e, pl->P.local, pl->dg, pl->opts);
        const auto& solves = pl->last;
        r.qaoa_s = seconds_since(t0);
        for (const auto& s : solves) r.evals += static_cast<uint64_t>(s.evals);
        t0 = std::chrono::steady_clock::now();
        bool windowed = false;
        const MergeOutput out = merge_stage(e, pl->g, pl->P, solves, &pl->cfg, &windowed);
        r.merge_s = seconds_since(t0);
        e->t_merge_s += r.merge_s;
        e->t_execute_s += r.qaoa_s + r.merge_s;
        r.total_s = r.partition_s + r.qaoa_s + r.merge_s;
        r.cut = out.value;
        r.candidates_evaluated = out.leaves;
        r.windowed = windowed ? 1 : 0;
        if (report) *report = r;
        write_assignment(out.assignment, assignment);
    });
}

void qc_pipeline_destroy(qc_pipeline* pl) {
    if (!pl) return;
    cudaSetDevice(pl->e->device);
    cudaStreamSynchronize(pl->e->stream);
    delete pl;
}

int64_t qc_record_bytes(int top_k_cap, int layers) { return record_bytes(top_k_cap, layers); }

int qc_run_record_bytes(const qc_graph* g, const qc_run_config* cfg, int64_t* bytes,
                        int32_t* subgraphs) {
    return guarded([&] {
        check_config(cfg);
        if (!bytes) config_error("null argument");
        const HostGraph hg = load_graph(g);
        const int M = cfg->subgraphs != 0 ? cfg->subgraphs : derive_subgraph_count(hg.n, cfg->qubit_cap);
        *bytes = record_bytes(kcap_of(cfg, max_width(hg.n, M, cfg)), cfg->layers);
        if (subgraphs) *subgraphs = M;
    });
}

int qc_pipeline_records(const qc_pipeline* pl, void* records, int64_t capacity, int64_t* bytes,
                        int32_t* subgraphs) {
    return guarded([&] {
        if (!pl) config_error("null pipeline");
        const int M = static_cast<int>(pl->P.first.size());
        int maxw = 1;
        for (const auto& L : pl->P.local) maxw = std::max(maxw, L.n);
        const int kcap = kcap_of(&pl->cfg, maxw);
        const int64_t rb = record_bytes(kcap, pl->cfg.layers);
        if (bytes) *bytes = rb;
        if (subgraphs) *subgraphs = M;
        if (!records) return;
        if (pl->cfg.shard_count > 1) config_error("sharded session: records come from qc_pipeline_execute_shard");
        if (pl->last.size() != static_cast<size_t>(M)) config_error("pipeline has not been executed");
        if (capacity < rb * M) config_error("record buffer too small");
        for (int i = 0; i < M; ++i)
            pack_record(pl->last[static_cast<size_t>(i)], kcap, pl->cfg.layers,
                        static_cast<char*>(records) + static_cast<int64_t>(i) * rb);
    });
}

int qc_shard_range(int M, int shard_index, int shard_count, int32_t* begin, int32_t* end) {
    return guarded([&] {
        if (M < 0 || shard_count < 1 || shard_index < 0 || shard_index >= shard_count)
            config_error("invalid shard request");
        // contiguous balanced blocks: the first M % count shards get one extra
        const int base = M / shard_count, rem = M % shard_count;
        *begin = shard_index * base + std::min(shard_index, rem);
        *end = *begin + base + (shard_index < rem ? 1 : 0);
    });
}

int qc_shard_solve(qc_engine* e, const qc_graph* g, const qc_run_config* cfg, int32_t begin,
                   int32_t end, void* records, int64_t capacity, int32_t* subgraphs) {
    return guarded([&] {
        if (!e) config_error("null engine");
        QC_CUDA(cudaSetDevice(e->device));
        check_config(cfg);
        const HostGraph hg = load_graph(g);
        const int M = cfg->subgraphs != 0 ? cfg->subgraphs : derive_subgraph_count(hg.n, cfg->qubit_cap);
        if (subgraphs) *subgraphs = M;
        if (!records) return;  // query M only
        if (begin < 0 || end > M || begin > end) config_error("shard range out of bounds");
        const Partition P = partition(hg, M, cfg->partition_mode, cfg->qubit_cap);
        int maxw = 1;
        for (const auto& L : P.local) maxw = std::max(maxw, L.n);
        const int kcap = kcap_of(cfg, maxw);
        const int64_t rb = record_bytes(kcap, cfg->layers);
        if (capacity < rb * (end - begin))
            config_error("record buffer holds " + std::to_string(capacity) + " bytes, the shard needs " +
                         std::to_string(rb * (end - begin)) + " (qc_run_record_bytes)");
        if (begin == end) return;
        const auto solves = solve_range(e, P, cfg, begin, end);
        for (size_t k = 0; k < solves.size(); ++k)
            pack_record(solves[k], kcap, cfg->layers, static_cast<char*>(records) + static_cast<int64_t>(k) * rb);
    });
}

int qc_merge_records(qc_engine* e, const qc_graph* g, const qc_run_config* cfg,
                     const void* records, int64_t capacity, int32_t M, qc_run_report* report,
                     char* assignment) {
    return guarded([&] {
        if (!e) config_error("null engine");
        QC_CUDA(cudaSetDevice(e->device));
        check_config(cfg);
        const HostGraph hg = load_graph(g);
        const Partition P = partition(hg, M, cfg->partition_mode, cfg->qubit_cap);
        int maxw = 1;
        for (const auto& L : P.local) maxw = std::max(maxw, L.n);
        const int kcap = kcap_of(cfg, maxw);
        const int64_t rb = record_bytes(kcap, cfg->layers);
        if (capacity < rb * M)
            config_error("record buffer holds " + std::to_string(capacity) + " bytes, " +
                         std::to_string(M) + " records need " + std::to_string(rb * M));
        std::vector<SolveOut> solves;
        for (int i = 0; i < M; ++i)
            solves.push_back(unpack_record(static_cast<const char*>(records) + static_cast<int64_t>(i) * rb,
                                           kcap, cfg->layers));
        auto t0 = std::chrono::steady_clock::now();
        bool windowed = false;
        const MergeOutput out = merge_stage(e, hg, P, solves, cfg, &windowed);
        qc_run_report r{};
        r.merge_s = seconds_since(t0);
        r.subgraphs = M;
        r.cut = out.value;
        r.candidates_evaluated = out.leaves;
        r.windowed = windowed ? 1 : 0;
        for (const auto& s : solves) r.evals += static_cast<uint64_t>(s.evals);
        if (report) *report = r;
        write_assignment(out.assignment, assignment);
    });
}

}  // extern "C"
