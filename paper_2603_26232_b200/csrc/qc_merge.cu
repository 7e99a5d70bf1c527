// GPU merge scoring (merge.hpp:280-331 level_aware_merge, merge.hpp:345-412
// chained_merge), sm_100a.
//
// Both merges are sequences of exhaustive "window" searches over compatible candidate
// chains (level mode = one window over all levels). A leaf is a tuple of pool entries,
// one per level, where entry i+1's bit 0 equals entry i's last bit (merge.hpp:55-58).
// The best leaf maximises the score; ties go to the lexicographically smallest
// assignment (merge.hpp:166-173). Because pieces are ascending contiguous vertex
// ranges, that order is the lexicographic order of per-level lex_less_mask ranks, so
// the engine enumerates every window's leaves in lex-DFS order (per-level candidate
// lists sorted by bit-reversed value) and breaks ties by the smaller leaf index.
//
// Scoring:
//   * integral weights (the ER/unit-weight configs): every summation order is exact, so
//     the score is a sum of per-level unary tables and per-level-pair tables
//     (edges bucketed by the levels of their endpoints; merge.hpp:103-113 groups the same
//     edges by max level) — O(levels) lookups per leaf instead of O(edges);
//   * fractional weights: the reference's floating-point association is reproduced
//     exactly (incremental: acc + bucket sums in edge-list order, merge.hpp:115-120,
//     182-184; full: cut_value in edge-list order at every leaf).
//
// Every window runs on the device back to back (no host round trip): unary tables
// from the fixed prefix, search, block reduction, commit of the winner into the
// device-resident assignment; the next window's seam bit is read on the device.
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>

#include <algorithm>
#include <cstdint>
#include <array>
#include <cstring>
#include <numeric>
#include <string>
#include <vector>

#include "qc_internal.hpp"
#include "qc_merge.hpp"

namespace qcg {

namespace {

constexpr int kSearchThreads = 128;
constexpr int kMaxL = 64;  // per-thread stacks (local memory)

struct WinLevel {
    int32_t count;        // pool entries
    int32_t bits_off;     // into entry bits (pool order)
    int32_t list_off[3];  // lex-sorted entry indices: parity 0, parity 1, all
    int32_t list_len[3];
    int32_t first;        // global id of local vertex 0
    int32_t width;
    int32_t u_off;        // unary table offset (count entries)
    int32_t pair_base;    // index into pair_off for (this level, j = s .. this-1)
    int32_t bucket_off;   // exact path: edges of this level's bucket
    int32_t bucket_len;
    int32_t fixed_off;    // fixed-prefix edges (integral path) for this level
    int32_t fixed_len;
    uint64_t nsub[2];     // leaves of levels [this, end) given incoming parity
};

struct XEdge {  // exact path edge with precomputed endpoint levels
    uint32_t u, v;
    double w;
    int32_t lu, lv;
};

struct FixedEdge {  // v_hi local index k in its level, v_lo global id, integral weight
    int32_t k;
    int32_t u;
    int64_t w;
};

struct SearchArgs {
    const WinLevel* lv;       // L levels
    const uint32_t* bits;     // entry bits
    const int32_t* lists;     // lex lists
    const int64_t* utab;      // unary tables (integral)
    const int64_t* ptab;      // pair tables (integral)
    const int32_t* pair_off;  // offsets of pair tables
    const XEdge* xedges;      // exact path buckets
    const XEdge* all_edges;   // full-graph scoring (edge-list order)
    int32_t m_all;
    const uint8_t* fixed;     // device assignment (fixed prefix)
    const int32_t* first_of_level;  // all levels (global)
    int32_t s;                // first level of the window (global index)
    int32_t L;
    int32_t need_mode;        // 2 free, 3 halve (bit0 == 0), -1 read from fixed[first[s]]
    int32_t integral;
    int32_t full_graph;       // exact path: score with cut_value at leaves
    int32_t leaves_per_thread;
    const double* base_acc;   // device acc of fixed prefix (exact path)
    const int64_t* base_iacc; // device acc (integral path)
    // windows longer than kMaxL levels (level mode with forced chains, e.g. top-K 1: few
    // leaves, hundreds of levels): per-thread odometer state in global scratch, L entries
    // per array per thread, instead of local arrays
    int32_t* sc_i;            // r, c, sel: 3 * L ints per thread
    int64_t* sc_ips;          // L per thread
    double* sc_dps;           // L per thread
    uint64_t* blk_idx;        // per-block best leaf index
    double* blk_val;          // per-block best value (exact path / integral as double)
    int64_t* blk_ival;
};

__device__ __forceinline__ int entry_bit(const SearchArgs& A, const WinLevel& L, int e, int k) {
    return (A.bits[L.bits_off + e] >> k) & 1u;
}

__device__ __forceinline__ int need_parity(const SearchArgs& A) {
    if (A.need_mode >= 0) return A.need_mode;
    return A.fixed[A.first_of_level[A.s]];
}

// list index for a level given incoming parity / need code
__device__ __forceinline__ int list_sel(int need) { return need == 2 ? 2 : (need == 3 ? 0 : need); }

template <bool INTEGRAL>
__device__ __forceinline__ void better(bool& has, int64_t& bi, double& bv, uint64_t& bidx,
                                       int64_t iv, double v, uint64_t idx) {
    if (INTEGRAL) {
        if (!has || iv > bi || (iv == bi && idx < bidx)) {
            has = true;
            bi = iv;
            bidx = idx;
        }
    } else {
        if (!has || v > bv || (v == bv && idx < bidx)) {
            has = true;
            bv = v;
            bidx = idx;
        }
    }
}

// bit of global vertex x for the current tuple (exact path)
__device__ __forceinline__ int vertex_bit(const SearchArgs& A, const int* c, int lvl, uint32_t x) {
    if (lvl < A.s) return A.fixed[x];
    const WinLevel& L = A.lv[lvl - A.s];
    return entry_bit(A, L, c[lvl - A.s], static_cast<int>(x) - L.first);
}

template <bool INTEGRAL, bool LONG>
__global__ void __launch_bounds__(kSearchThreads) k_search(SearchArgs A, uint64_t total_bound) {
    const int L = A.L;
    const int need0 = need_parity(A);
    // total leaves for this need
    uint64_t T = 0;
    {
        const WinLevel& l0 = A.lv[0];
        const int sel = list_sel(need0);
        for (int r = 0; r < l0.list_len[sel]; ++r) {
            const int e = A.lists[l0.list_off[sel] + r];
            const int out = entry_bit(A, l0, e, l0.width - 1);
            T += (L > 1) ? A.lv[1].nsub[out] : 1;
        }
    }
    const uint64_t t = static_cast<uint64_t>(blockIdx.x) * kSearchThreads + threadIdx.x;
    const uint64_t idx0 = t * static_cast<uint64_t>(A.leaves_per_thread);
    bool has = false;
    int64_t bi = 0;
    double bv = 0.0;
    uint64_t bidx = 0;

    if (idx0 < T) {
        int r_l[LONG ? 1 : kMaxL], c_l[LONG ? 1 : kMaxL], sel_l[LONG ? 1 : kMaxL];
        int64_t ips_l[LONG ? 1 : kMaxL] = {};  // score_level fills them in level order
        double dps_l[LONG ? 1 : kMaxL] = {};
        int *r = r_l, *c = c_l, *sel = sel_l;
        int64_t* ips = ips_l;
        double* dps = dps_l;
        if constexpr (LONG) {
            r = A.sc_i + t * 3 * static_cast<uint64_t>(L);
            c = r + L;
            sel = c + L;
            ips = A.sc_ips + t * static_cast<uint64_t>(L);
            dps = A.sc_dps + t * static_cast<uint64_t>(L);
        }
        // decode idx0
        uint64_t rem = idx0;
        int need = need0;
        for (int i = 0; i < L; ++i) {
            const WinLevel& lv = A.lv[i];
            sel[i] = list_sel(need);
            const int32_t* lst = A.lists + lv.list_off[sel[i]];
            int rr = 0;
            for (;; ++rr) {
                const int e = lst[rr];
                const int out = entry_bit(A, lv, e, lv.width - 1);
                const uint64_t cnt = (i + 1 < L) ? A.lv[i + 1].nsub[out] : 1;
                if (rem < cnt) break;
                rem -= cnt;
            }
            r[i] = rr;
            c[i] = lst[rr];
            need = entry_bit(A, lv, c[i], lv.width - 1);
        }
        auto score_level = [&](int i) {
            const WinLevel& lv = A.lv[i];
            if (INTEGRAL) {
                int64_t v = (i ? ips[i - 1] : 0) + A.utab[lv.u_off + c[i]];
                for (int j = 0; j < i; ++j) {
                    const int po = A.pair_off[lv.pair_base + j];
                    if (po >= 0) v += A.ptab[po + c[i] * A.lv[j].count + c[j]];
                }
                ips[i] = v;
            } else if (!A.full_graph) {
                double g = 0.0;
                const XEdge* es = A.xedges + lv.bucket_off;
                for (int k = 0; k < lv.bucket_len; ++k) {
                    const XEdge ed = es[k];
                    if (vertex_bit(A, c, ed.lu, ed.u) != vertex_bit(A, c, ed.lv, ed.v))
                        g = __dadd_rn(g, ed.w);
                }
                dps[i] = __dadd_rn(i ? dps[i - 1] : *A.base_acc, g);
            }
        };
        for (int i = 0; i < L; ++i) score_level(i);
        uint64_t idx = idx0;
        const uint64_t idx_end = min(T, idx0 + static_cast<uint64_t>(A.leaves_per_thread));
        for (;;) {
            if (INTEGRAL) {
                better<true>(has, bi, bv, bidx, ips[L - 1], 0.0, idx);
            } else if (A.full_graph) {
                double v = 0.0;
                for (int k = 0; k < A.m_all; ++k) {
                    const XEdge ed = A.all_edges[k];
                    if (vertex_bit(A, c, ed.lu, ed.u) != vertex_bit(A, c, ed.lv, ed.v))
                        v = __dadd_rn(v, ed.w);
                }
                better<false>(has, bi, bv, bidx, 0, v, idx);
            } else {
                better<false>(has, bi, bv, bidx, 0, dps[L - 1], idx);
            }
            if (++idx >= idx_end) break;
            // odometer
            int i = L - 1;
            for (;;) {
                const WinLevel& lv = A.lv[i];
                if (++r[i] < lv.list_len[sel[i]]) break;
                r[i] = 0;
                --i;  // never underflows: idx < T guarantees a successor exists
            }
            for (int k = i; k < L; ++k) {
                const WinLevel& lv = A.lv[k];
                if (k > i) {
                    const int inpar = entry_bit(A, A.lv[k - 1], c[k - 1], A.lv[k - 1].width - 1);
                    sel[k] = inpar;
                    r[k] = 0;
                }
                c[k] = A.lists[lv.list_off[sel[k]] + r[k]];
                score_level(k);
            }
        }
    }
    // block reduction: (value desc, idx asc)
    __shared__ int64_t s_i[kSearchThreads];
    __shared__ double s_v[kSearchThreads];
    __shared__ uint64_t s_x[kSearchThreads];
    __shared__ int s_h[kSearchThreads];
    s_i[threadIdx.x] = bi;
    s_v[threadIdx.x] = bv;
    s_x[threadIdx.x] = bidx;
    s_h[threadIdx.x] = has ? 1 : 0;
    __syncthreads();
    for (int off = kSearchThreads / 2; off > 0; off >>= 1) {
        if (threadIdx.x < off) {
            const int o = threadIdx.x + off;
            if (s_h[o]) {
                bool take;
                if (!s_h[threadIdx.x])
                    take = true;
                else if (INTEGRAL)
                    take = s_i[o] > s_i[threadIdx.x] ||
                           (s_i[o] == s_i[threadIdx.x] && s_x[o] < s_x[threadIdx.x]);
                else
                    take = s_v[o] > s_v[threadIdx.x] ||
                           (s_v[o] == s_v[threadIdx.x] && s_x[o] < s_x[threadIdx.x]);
                if (take) {
                    s_i[threadIdx.x] = s_i[o];
                    s_v[threadIdx.x] = s_v[o];
                    s_x[threadIdx.x] = s_x[o];
                    s_h[threadIdx.x] = 1;
                }
            }
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        A.blk_idx[blockIdx.x] = s_h[0] ? s_x[0] : ~uint64_t{0};
        A.blk_val[blockIdx.x] = s_v[0];
        A.blk_ival[blockIdx.x] = s_i[0];
    }
    (void)total_bound;
}

// Reduce block bests, decode the winning leaf, write its pieces into the device
// assignment, advance the accumulated value and the leaf counter.
constexpr int kCommitThreads = 256;
__global__ void __launch_bounds__(kCommitThreads) k_commit(SearchArgs A, int n_blocks, uint64_t* leaves_total,
                                                           int* dead_end, double* acc, int64_t* iacc) {
    // the window's winner over the search blocks' results: (value desc, leaf index asc),
    // reduced by the whole CTA (a single thread walking ~10^3 block results in order
    // waited on one global load at a time)
    __shared__ int s_best[kCommitThreads];
    const int t = threadIdx.x;
    auto better = [&](int b, int c) {  // is block b's result better than block c's?
        if (c < 0) return b >= 0;
        if (b < 0) return false;
        return A.integral ? (A.blk_ival[b] > A.blk_ival[c] ||
                             (A.blk_ival[b] == A.blk_ival[c] && A.blk_idx[b] < A.blk_idx[c]))
                          : (A.blk_val[b] > A.blk_val[c] ||
                             (A.blk_val[b] == A.blk_val[c] && A.blk_idx[b] < A.blk_idx[c]));
    };
    int mine = -1;
    for (int b = t; b < n_blocks; b += kCommitThreads)
        if (A.blk_idx[b] != ~uint64_t{0} && better(b, mine)) mine = b;
    s_best[t] = mine;
    __syncthreads();
    for (int off = kCommitThreads / 2; off > 0; off >>= 1) {
        if (t < off && better(s_best[t + off], s_best[t])) s_best[t] = s_best[t + off];
        __syncthreads();
    }
    if (t != 0 || blockIdx.x != 0) return;
    const int L = A.L;
    const int need0 = need_parity(A);
    uint64_t T = 0;
    {
        const WinLevel& l0 = A.lv[0];
        const int sel = list_sel(need0);
        for (int r = 0; r < l0.list_len[sel]; ++r) {
            const int e = A.lists[l0.list_off[sel] + r];
            const int out = entry_bit(A, l0, e, l0.width - 1);
            T += (L > 1) ? A.lv[1].nsub[out] : 1;
        }
    }
    if (T == 0) {
        *dead_end = 1;
        return;
    }
    *leaves_total += T;
    const int best = s_best[0];
    if (best < 0) {
        *dead_end = 1;
        return;
    }
    uint64_t rem = A.blk_idx[best];
    int need = need0;
    for (int i = 0; i < L; ++i) {
        const WinLevel& lv = A.lv[i];
        const int32_t* lst = A.lists + lv.list_off[list_sel(need)];
        int e = 0;
        for (int rr = 0;; ++rr) {
            e = lst[rr];
            const int out = entry_bit(A, lv, e, lv.width - 1);
            const uint64_t cnt = (i + 1 < L) ? A.lv[i + 1].nsub[out] : 1;
            if (rem < cnt) break;
            rem -= cnt;
        }
        const uint32_t b = A.bits[lv.bits_off + e];
        for (int k = 0; k < lv.width; ++k) const_cast<uint8_t*>(A.fixed)[lv.first + k] = (b >> k) & 1u;
        need = (b >> (lv.width - 1)) & 1u;
    }
    if (A.integral)
        *iacc = A.blk_ival[best];
    else
        *acc = A.blk_val[best];
}

// Unary tables of the window's levels: intra-level table + edges to the fixed prefix.
// One block per level; W0[k]/W1[k] = weight from local vertex k to fixed vertices on
// side 0/1 (exact integer sums), then U[a] = intra[a] + sum_k (bit_a(k) ? W0 : W1).
__global__ void k_unary(SearchArgs A, const int64_t* __restrict__ intra,
                        const FixedEdge* __restrict__ fixed_edges, int64_t* __restrict__ utab) {
    __shared__ unsigned long long W[2][32];
    const WinLevel& lv = A.lv[blockIdx.x];
    if (threadIdx.x < 64) W[threadIdx.x >> 5][threadIdx.x & 31] = 0;
    __syncthreads();
    for (int k = threadIdx.x; k < lv.fixed_len; k += blockDim.x) {
        const FixedEdge fe = fixed_edges[lv.fixed_off + k];
        atomicAdd(&W[A.fixed[fe.u]][fe.k], static_cast<unsigned long long>(fe.w));
    }
    __syncthreads();
    for (int a = threadIdx.x; a < lv.count; a += blockDim.x) {
        const uint32_t b = A.bits[lv.bits_off + a];
        int64_t u = intra[lv.u_off + a];
        for (int k = 0; k < lv.width; ++k)
            u += static_cast<int64_t>(((b >> k) & 1u) ? W[0][k] : W[1][k]);
        utab[lv.u_off + a] = u;
    }
}

// Pair / intra tables: one block per group, thread per table entry, loop over the
// group's edges (exact integer sums).
struct PairGroup {
    int32_t hi, lo;        // global levels (lo == hi: intra)
    int32_t out_off;       // table offset
    int32_t e_off, e_len;  // edges (v_hi local k, v_lo local k2, w)
};
struct PairEdge {
    int32_t khi, klo;
    int64_t w;
};

__global__ void k_pair_tables(const PairGroup* __restrict__ groups, const PairEdge* __restrict__ pe,
                              const uint32_t* __restrict__ bits, const int32_t* __restrict__ bits_off,
                              const int32_t* __restrict__ counts, int64_t* __restrict__ out) {
    const PairGroup g = groups[blockIdx.x];
    const int ch = counts[g.hi];
    const int cl = g.lo == g.hi ? 1 : counts[g.lo];
    for (int t = threadIdx.x; t < ch * cl; t += blockDim.x) {
        const int a = t / cl, b = t % cl;
        const uint32_t ba = bits[bits_off[g.hi] + a];
        const uint32_t bb = g.lo == g.hi ? ba : bits[bits_off[g.lo] + b];
        int64_t s = 0;
        for (int k = 0; k < g.e_len; ++k) {
            const PairEdge e = pe[g.e_off + k];
            if ((((ba >> e.khi) ^ (bb >> e.klo)) & 1u) != 0) s += e.w;
        }
        out[g.out_off + t] = s;
    }
}

// Integral re-score of the final assignment (cut_value, merge.hpp:327,:408).
__global__ void k_cut_int(const uint32_t* __restrict__ eu, const uint32_t* __restrict__ ev,
                          const double* __restrict__ ew, long long m, const uint8_t* __restrict__ a,
                          unsigned long long* __restrict__ out) {
    unsigned long long s = 0;
    for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < m;
         k += (long long)gridDim.x * blockDim.x)
        if (a[eu[k]] != a[ev[k]]) s += static_cast<unsigned long long>(ew[k]);
    for (int off = 16; off > 0; off >>= 1) s += __shfl_down_sync(0xffffffffu, s, off);
    if ((threadIdx.x & 31) == 0 && s) atomicAdd(out, s);
}

// ---------------------------------------------------------------------------
// Device-side edge classification for the integral windowed/level merge (replaces host
// bucketing of every edge: merge.hpp:103-113 level_edge_buckets, grouped for the unary /
// pair tables). Bins: fixed edges of level hi (lo in an earlier window) -> bin hi;
// in-window edges (hi, lo) -> bin M + hi*span + (lo - win_start[hi]). Sums over a bin are
// integers, so the scatter order is immaterial.
// ---------------------------------------------------------------------------
struct ClassArgs {
    const uint32_t* eu;
    const uint32_t* ev;
    const double* ew;
    long long m;
    const int32_t* fl;        // first level of each vertex
    const int32_t* ws;        // window start of each level
    const int32_t* first;     // first global vertex of each level
    int M;
    int span;                 // bin stride: the longest window (levels)
};

__device__ __forceinline__ void classify(const ClassArgs& A, long long k, int& bin, int32_t& khi,
                                         int32_t& kx, int64_t& w) {
    uint32_t a = A.eu[k], b = A.ev[k];
    int la = A.fl[a], lb = A.fl[b];
    if (la > lb) {
        const int t = la;
        la = lb;
        lb = t;
        const uint32_t tv = a;
        a = b;
        b = tv;
    }
    // b: vertex on the higher level lb, a: on the lower level la
    w = static_cast<int64_t>(A.ew[k]);
    khi = static_cast<int32_t>(b) - A.first[lb];
    if (la < A.ws[lb]) {
        bin = lb;
        kx = static_cast<int32_t>(a);  // global id of the fixed endpoint
    } else {
        bin = A.M + lb * A.span + (la - A.ws[lb]);
        kx = static_cast<int32_t>(a) - A.first[la];
    }
}

__global__ void k_edge_hist(ClassArgs A, unsigned* __restrict__ hist) {
    for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < A.m;
         k += (long long)gridDim.x * blockDim.x) {
        int bin;
        int32_t khi, kx;
        int64_t w;
        classify(A, k, bin, khi, kx, w);
        atomicAdd(hist + bin, 1u);
    }
}

__global__ void k_edge_scatter(ClassArgs A, unsigned* __restrict__ cursor,
                               FixedEdge* __restrict__ fixed, PairEdge* __restrict__ pairs) {
    for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < A.m;
         k += (long long)gridDim.x * blockDim.x) {
        int bin;
        int32_t khi, kx;
        int64_t w;
        classify(A, k, bin, khi, kx, w);
        const unsigned pos = atomicAdd(cursor + bin, 1u);
        if (bin < A.M)
            fixed[pos] = FixedEdge{khi, kx, w};
        else
            pairs[pos] = PairEdge{khi, kx, w};
    }
}

thread_local DeviceArena* g_arena = nullptr;

template <typename T>
T* dalloc(std::vector<void*>& keep, size_t n) {
    if (n == 0) n = 1;
    if (g_arena) {
        void* p = g_arena->get(n * sizeof(T));
        if (!p) resource_error("device out of memory (merge scratch)");
        return static_cast<T*>(p);
    }
    void* p = nullptr;
    QC_CUDA(cudaMalloc(&p, n * sizeof(T)));
    keep.push_back(p);
    return static_cast<T*>(p);
}

thread_local uint64_t* g_h2d_counter = nullptr;

template <typename T>
T* dupload(std::vector<void*>& keep, const std::vector<T>& h, cudaStream_t st) {
    T* d = dalloc<T>(keep, h.size());
    if (!h.empty()) {
        QC_CUDA(cudaMemcpyAsync(d, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice, st));
        if (g_h2d_counter) *g_h2d_counter += h.size() * sizeof(T);
    }
    return d;
}

uint32_t brev_w(uint32_t b) {
    uint32_t r = 0;
    for (int i = 0; i < 32; ++i) r |= ((b >> i) & 1u) << (31 - i);
    return r;
}

}  // namespace

// merge.hpp:122-141 check_pool_matches
void check_pool(const MergeInput& in) {
    const int M = in.levels;
    if (in.pieces < 1) config_error("merge needs at least one subgraph");
    if (M != in.pieces)
        config_error("pool has " + std::to_string(M) + " levels for " + std::to_string(in.pieces) +
                     " subgraphs");
    long long covered = 0;
    for (int i = 0; i < M; ++i) {
        const int piece = in.last[i] - in.first[i] + 1;
        if (in.widths[i] < 1 || in.widths[i] != piece)
            config_error("pool level " + std::to_string(i) + " width " + std::to_string(in.widths[i]) +
                         " does not match subgraph size " + std::to_string(piece));
        if (in.counts[i] == 0) config_error("pool level " + std::to_string(i) + " is empty");
        covered += piece;
    }
    if (covered != static_cast<long long>(in.n) + M - 1)
        config_error("subgraphs do not cover the graph as a chain");
}

double estimate_paths(const int32_t* counts, int M, bool halve) {
    if (M < 1) config_error("empty candidate pool");
    double est = static_cast<double>(counts[0]);
    if (halve) est /= 2.0;
    for (int i = 1; i < M; ++i) est *= static_cast<double>(counts[i]) / 2.0;
    return est;
}

namespace {
struct MTrace {
    bool on = std::getenv("QCG_TRACE_MERGE") != nullptr;
    std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
    void mark(const char* what) {
        if (!on) return;
        const auto now = std::chrono::steady_clock::now();
        std::fprintf(stderr, "merge %-12s %8.2f ms\n", what, std::chrono::duration<double>(now - t).count() * 1e3);
        t = now;
    }
};
}  // namespace

MergeOutput run_merge(const MergeInput& in, const std::vector<Window>& windows, bool full_graph,
                      cudaStream_t st, uint64_t* launches, Prof* prof, uint64_t* h2d, uint64_t* d2h,
                      DeviceArena* arena) {
    MTrace tr;
    Prof dummy;
    if (!prof) prof = &dummy;
    uint64_t h2d_local = 0, d2h_local = 0;
    if (!h2d) h2d = &h2d_local;
    if (!d2h) d2h = &d2h_local;
    const int M = in.levels;
    const int n = in.n;
    std::vector<void*> keep;
    struct Freer {
        std::vector<void*>* k;
        ~Freer() {
            for (void* p : *k) cudaFree(p);
            g_h2d_counter = nullptr;
            g_arena = nullptr;
        }
    } freer{&keep};
    g_h2d_counter = h2d;
    g_arena = arena;
    if (arena) arena->reset();
    auto S = [](int i) { return static_cast<size_t>(i); };

    // ---- first level of every vertex (merge.hpp:106-108), integrality
    // edges arrive either as the pipeline's SoA arrays or as qc_edge AoS (C-ABI merges)
    auto EU = [&](long long k) { return in.eu ? in.eu[k] : in.edges[k].u; };
    auto EV = [&](long long k) { return in.eu ? in.ev[k] : in.edges[k].v; };
    auto EW = [&](long long k) { return in.eu ? in.ew[k] : in.edges[k].w; };
    std::vector<int32_t> fl(S(n), 0);
    for (int i = M - 1; i >= 0; --i)
        for (int v = in.first[i]; v <= in.last[i]; ++v) fl[S(v)] = i;
    bool integral = in.all_int != 0;
    if (in.all_int < 0) {
        long double total = 0;
        for (long long k = 0; k < in.m; ++k) {
            const double w = EW(k);
            if (!(w >= 0) || w != static_cast<double>(static_cast<int64_t>(w))) integral = false;
            total += w;
        }
        if (total > 4.0e18L) integral = false;
    }
    for (int i = 0; i < M; ++i)
        if (in.widths[i] > 32) internal_error("piece wider than 32 vertices in merge");

    tr.mark("fl+integral");
    std::vector<int32_t> bits_off(S(M));
    for (int i = 0, off = 0; i < M; ++i) {
        bits_off[S(i)] = off;
        off += in.counts[i];
    }
    const size_t total_entries = static_cast<size_t>(bits_off[S(M - 1)] + in.counts[M - 1]);
    std::vector<uint32_t> hbits(in.bits, in.bits + total_entries);
    std::vector<int32_t> win_start(S(M));
    int span = 1;  // longest window (levels)
    for (const Window& W : windows) {
        for (int i = W.s; i < W.e; ++i) win_start[S(i)] = W.s;
        span = std::max(span, W.e - W.s);
    }

    // ---- lex-sorted candidate lists per level: parity 0, parity 1, all
    std::vector<int32_t> lists;
    std::vector<WinLevel> wl(S(M));
    for (int i = 0; i < M; ++i) {
        WinLevel& L = wl[S(i)];
        std::memset(&L, 0, sizeof L);
        L.count = in.counts[i];
        L.bits_off = bits_off[S(i)];
        L.first = in.first[i];
        L.width = in.widths[i];
        std::vector<int32_t> idx(S(L.count));
        std::iota(idx.begin(), idx.end(), 0);
        const uint32_t* b = in.bits + L.bits_off;
        std::sort(idx.begin(), idx.end(), [&](int a, int c) { return brev_w(b[a]) < brev_w(b[c]); });
        for (int sel = 0; sel < 3; ++sel) {
            L.list_off[sel] = static_cast<int32_t>(lists.size());
            int len = 0;
            for (int e : idx)
                if (sel == 2 || static_cast<int>(b[e] & 1u) == sel) {
                    lists.push_back(e);
                    ++len;
                }
            L.list_len[sel] = len;
        }
    }
    // subtree leaf counts per window (saturating)
    for (const Window& W : windows) {
        uint64_t next[2] = {1, 1};
        for (int i = W.e - 1; i >= W.s; --i) {
            WinLevel& L = wl[S(i)];
            uint64_t ns[2] = {0, 0};
            for (int par = 0; par < 2; ++par)
                for (int r = 0; r < L.list_len[par]; ++r) {
                    const uint32_t b = in.bits[L.bits_off + lists[S(L.list_off[par] + r)]];
                    const int out = static_cast<int>((b >> (L.width - 1)) & 1u);
                    const unsigned __int128 v = static_cast<unsigned __int128>(ns[par]) + next[out];
                    ns[par] = v > ~uint64_t{0} ? ~uint64_t{0} : static_cast<uint64_t>(v);
                }
            L.nsub[0] = ns[0];
            L.nsub[1] = ns[1];
            next[0] = ns[0];
            next[1] = ns[1];
        }
    }
    int64_t utab_size = 0;
    for (int i = 0; i < M; ++i) {
        wl[S(i)].u_off = static_cast<int32_t>(utab_size);
        utab_size += in.counts[i];
    }

    tr.mark("lists");
    // ---- scoring data
    std::vector<int32_t> pair_off;
    std::vector<XEdge> xedges, all_edges;
    int64_t* d_intra = nullptr;
    int64_t* d_ptab = nullptr;
    int64_t* d_utab = nullptr;
    FixedEdge* d_fixed_edges = nullptr;
    uint32_t* d_eu = nullptr;
    uint32_t* d_ev = nullptr;
    double* d_ew = nullptr;
    if (integral) {
        // Edges go to the device once (also used by the final re-score); the GPU bins them
        // by (higher level, lower level in the same window) or as "fixed" edges of their
        // higher level (lower endpoint in an earlier window: folded into the unary table
        // per window). The host only scans the bin histogram.
        const size_t m = static_cast<size_t>(in.m);
        d_eu = dalloc<uint32_t>(keep, m);
        d_ev = dalloc<uint32_t>(keep, m);
        d_ew = dalloc<double>(keep, m);
        if (m) {
            if (in.eu) {
                QC_CUDA(cudaMemcpyAsync(d_eu, in.eu, m * 4, cudaMemcpyHostToDevice, st));
                QC_CUDA(cudaMemcpyAsync(d_ev, in.ev, m * 4, cudaMemcpyHostToDevice, st));
                QC_CUDA(cudaMemcpyAsync(d_ew, in.ew, m * 8, cudaMemcpyHostToDevice, st));
            } else {
                std::vector<uint32_t> hu(m), hv(m);
                std::vector<double> hw(m);
                for (size_t k = 0; k < m; ++k) {
                    hu[k] = in.edges[k].u;
                    hv[k] = in.edges[k].v;
                    hw[k] = in.edges[k].w;
                }
                QC_CUDA(cudaMemcpyAsync(d_eu, hu.data(), m * 4, cudaMemcpyHostToDevice, st));
                QC_CUDA(cudaMemcpyAsync(d_ev, hv.data(), m * 4, cudaMemcpyHostToDevice, st));
                QC_CUDA(cudaMemcpyAsync(d_ew, hw.data(), m * 8, cudaMemcpyHostToDevice, st));
                QC_CUDA(cudaStreamSynchronize(st));  // host staging goes out of scope
            }
            *h2d += m * 16;
        }
        std::vector<int32_t> first_l(in.first, in.first + M);
        auto* d_fl = dupload(keep, fl, st);
        auto* d_ws = dupload(keep, win_start, st);
        auto* d_firstl = dupload(keep, first_l, st);
        const size_t nbins = S(M) + S(M) * S(span);
        auto* d_hist = dalloc<unsigned>(keep, nbins);
        QC_CUDA(cudaMemsetAsync(d_hist, 0, nbins * 4, st));
        ClassArgs CA{d_eu, d_ev, d_ew, in.m, d_fl, d_ws, d_firstl, M, span};
        const unsigned cblocks = static_cast<unsigned>(std::max<long long>(1, std::min<long long>((in.m + 255) / 256, 148 * 16)));
        if (m) {
            prof->begin(K_MERGE_OTHER, static_cast<double>(m) * 16.0, st);
            k_edge_hist<<<cblocks, 256, 0, st>>>(CA, d_hist);
            prof->end(st);
            ++*launches;
        }
        std::vector<unsigned> hist(nbins);
        QC_CUDA(cudaMemcpyAsync(hist.data(), d_hist, nbins * 4, cudaMemcpyDeviceToHost, st));
        QC_CUDA(cudaStreamSynchronize(st));
        *d2h += nbins * 4;
        // fixed edges: bins [0, M) in level order; pair edges: bins M + hi*span + (lo-ws)
        std::vector<unsigned> cursor(nbins);
        unsigned nfixed = 0, npair = 0;
        for (int i = 0; i < M; ++i) {
            WinLevel& L = wl[S(i)];
            L.fixed_off = static_cast<int32_t>(nfixed);
            L.fixed_len = static_cast<int32_t>(hist[S(i)]);
            cursor[S(i)] = nfixed;
            nfixed += hist[S(i)];
        }
        std::vector<PairGroup> gi, gp;
        int64_t ptab_size = 0;
        for (int i = 0; i < M; ++i) {
            const int s0 = win_start[S(i)];
            WinLevel& L = wl[S(i)];
            L.pair_base = static_cast<int32_t>(pair_off.size());
            for (int j = s0; j <= i; ++j) {
                const size_t bin = S(M) + S(i) * S(span) + S(j - s0);
                const unsigned len = hist[bin];
                cursor[bin] = npair;
                PairGroup G{i, j, 0, static_cast<int32_t>(npair), static_cast<int32_t>(len)};
                npair += len;
                if (j == i) {  // every level has an intra table
                    G.out_off = L.u_off;
                    gi.push_back(G);
                } else if (len) {
                    G.out_off = static_cast<int32_t>(ptab_size);
                    ptab_size += static_cast<int64_t>(in.counts[i]) * in.counts[j];
                    gp.push_back(G);
                    pair_off.push_back(G.out_off);
                } else {
                    pair_off.push_back(-1);
                }
            }
        }
        auto* d_cursor = dupload(keep, cursor, st);
        d_fixed_edges = dalloc<FixedEdge>(keep, nfixed);
        auto* d_pe = dalloc<PairEdge>(keep, npair);
        if (m) {
            prof->begin(K_MERGE_OTHER, static_cast<double>(m) * 32.0, st);
            k_edge_scatter<<<cblocks, 256, 0, st>>>(CA, d_cursor, d_fixed_edges, d_pe);
            prof->end(st);
            ++*launches;
        }
        std::vector<int32_t> counts_v(in.counts, in.counts + M);
        auto* d_bits0 = dupload(keep, hbits, st);
        auto* d_boff = dupload(keep, bits_off, st);
        auto* d_counts = dupload(keep, counts_v, st);
        d_intra = dalloc<int64_t>(keep, S(static_cast<int>(utab_size)));
        d_utab = dalloc<int64_t>(keep, S(static_cast<int>(utab_size)));
        d_ptab = dalloc<int64_t>(keep, static_cast<size_t>(ptab_size));
        if (!gi.empty()) {
            auto* d_gi = dupload(keep, gi, st);
            prof->begin(K_MERGE_TABLES, static_cast<double>(npair) * 16.0, st);
            k_pair_tables<<<static_cast<unsigned>(gi.size()), 128, 0, st>>>(d_gi, d_pe, d_bits0, d_boff,
                                                                           d_counts, d_intra);
            prof->end(st);
            ++*launches;
        }
        if (!gp.empty()) {
            auto* d_gp = dupload(keep, gp, st);
            prof->begin(K_MERGE_TABLES, static_cast<double>(ptab_size) * 8.0, st);
            k_pair_tables<<<static_cast<unsigned>(gp.size()), 128, 0, st>>>(d_gp, d_pe, d_bits0, d_boff,
                                                                           d_counts, d_ptab);
            prof->end(st);
            ++*launches;
        }
        QC_CUDA(cudaGetLastError());
    } else {
        std::vector<std::vector<XEdge>> buckets(S(M));
        for (long long k = 0; k < in.m; ++k) {
            const uint32_t eu = EU(k), ev = EV(k);
            XEdge x{eu, ev, EW(k), fl[S(eu)], fl[S(ev)]};
            all_edges.push_back(x);
            buckets[S(std::max(fl[S(eu)], fl[S(ev)]))].push_back(x);
        }
        for (int i = 0; i < M; ++i) {
            wl[S(i)].bucket_off = static_cast<int32_t>(xedges.size());
            wl[S(i)].bucket_len = static_cast<int32_t>(buckets[S(i)].size());
            xedges.insert(xedges.end(), buckets[S(i)].begin(), buckets[S(i)].end());
        }
    }

    tr.mark("tables");
    // ---- upload common data
    std::vector<int32_t> first_v(in.first, in.first + M);
    auto* d_wl = dupload(keep, wl, st);
    auto* d_lists = dupload(keep, lists, st);
    auto* d_bits = dupload(keep, hbits, st);
    auto* d_pair_off = dupload(keep, pair_off, st);
    auto* d_xedges = dupload(keep, xedges, st);
    auto* d_all = dupload(keep, all_edges, st);
    auto* d_first = dupload(keep, first_v, st);
    auto* d_asg = dalloc<uint8_t>(keep, S(n));
    auto* d_acc = dalloc<double>(keep, 1);
    auto* d_iacc = dalloc<int64_t>(keep, 1);
    auto* d_leaves = dalloc<uint64_t>(keep, 1);
    auto* d_dead = dalloc<int>(keep, 1);
    QC_CUDA(cudaMemsetAsync(d_asg, 0, S(n), st));
    QC_CUDA(cudaMemsetAsync(d_acc, 0, sizeof(double), st));
    QC_CUDA(cudaMemsetAsync(d_iacc, 0, sizeof(int64_t), st));
    QC_CUDA(cudaMemsetAsync(d_leaves, 0, sizeof(uint64_t), st));
    QC_CUDA(cudaMemsetAsync(d_dead, 0, sizeof(int), st));

    // per-window launch geometry (host upper bound on the leaf count)
    struct Geo {
        uint64_t bound;
        int per_thread;
        unsigned blocks;
    };
    std::vector<Geo> geo;
    unsigned max_blocks = 1;
    for (const Window& W : windows) {
        const WinLevel& L0 = wl[S(W.s)];
        auto total_for = [&](int sel) {
            uint64_t T = 0;
            for (int r = 0; r < L0.list_len[sel]; ++r) {
                const uint32_t b = in.bits[L0.bits_off + lists[S(L0.list_off[sel] + r)]];
                const int out = static_cast<int>((b >> (L0.width - 1)) & 1u);
                T += (W.e - W.s > 1) ? wl[S(W.s + 1)].nsub[out] : 1;
            }
            return T;
        };
        uint64_t bound = W.need == 2 ? total_for(2)
                         : W.need == 3 ? total_for(0)
                                       : std::max(total_for(0), total_for(1));
        // long windows keep their odometer state in global scratch: fewer threads
        const uint64_t target_threads = (W.e - W.s > kMaxL) ? 148ull * 64 : 148ull * 1024;
        uint64_t per = (bound + target_threads - 1) / target_threads;
        if (per < 1) per = 1;
        if (per > (1u << 20)) per = 1u << 20;
        const uint64_t threads = (bound + per - 1) / per;
        const uint64_t blocks64 = (threads + kSearchThreads - 1) / kSearchThreads;
        if (blocks64 > 0x7fffffffull) resource_error("merge enumeration too large");
        const unsigned blocks = static_cast<unsigned>(std::max<uint64_t>(blocks64, 1));
        geo.push_back({bound, static_cast<int>(per), blocks});
        max_blocks = std::max(max_blocks, blocks);
    }
    auto* d_bidx = dalloc<uint64_t>(keep, max_blocks);
    auto* d_bval = dalloc<double>(keep, max_blocks);
    auto* d_bival = dalloc<int64_t>(keep, max_blocks);

    for (size_t w = 0; w < windows.size(); ++w) {
        const Window& W = windows[w];
        SearchArgs A{};
        A.lv = d_wl + W.s;
        A.bits = d_bits;
        A.lists = d_lists;
        A.utab = d_utab;
        A.ptab = d_ptab;
        A.pair_off = d_pair_off;
        A.xedges = d_xedges;
        A.all_edges = d_all;
        A.m_all = static_cast<int32_t>(all_edges.size());
        A.fixed = d_asg;
        A.first_of_level = d_first;
        A.s = W.s;
        A.L = W.e - W.s;
        A.need_mode = W.need;
        A.integral = integral ? 1 : 0;
        A.full_graph = full_graph ? 1 : 0;
        A.leaves_per_thread = geo[w].per_thread;
        A.base_acc = d_acc;
        A.base_iacc = d_iacc;
        A.blk_idx = d_bidx;
        A.blk_val = d_bval;
        A.blk_ival = d_bival;
        const bool lng = A.L > kMaxL;
        if (lng) {  // per-thread odometer state for the long window (merge.hpp allows any M)
            const uint64_t thr = static_cast<uint64_t>(geo[w].blocks) * kSearchThreads;
            const uint64_t per = thr * static_cast<uint64_t>(A.L);
            A.sc_i = dalloc<int32_t>(keep, S(per * 3));
            A.sc_ips = dalloc<int64_t>(keep, S(per));
            A.sc_dps = dalloc<double>(keep, S(per));
        }
        auto search = [&](auto kern) {
            prof->begin(K_MERGE_SEARCH, static_cast<double>(geo[w].bound) * 8.0, st);
            kern<<<geo[w].blocks, kSearchThreads, 0, st>>>(A, geo[w].bound);
            prof->end(st);
        };
        if (integral) {
            prof->begin(K_MERGE_OTHER, 0.0, st);
            k_unary<<<static_cast<unsigned>(A.L), 128, 0, st>>>(A, d_intra, d_fixed_edges, d_utab);
            prof->end(st);
            if (lng)
                search(k_search<true, true>);
            else
                search(k_search<true, false>);
        } else {
            if (lng)
                search(k_search<false, true>);
            else
                search(k_search<false, false>);
        }
        prof->begin(K_MERGE_OTHER, 0.0, st);
        k_commit<<<1, kCommitThreads, 0, st>>>(A, static_cast<int>(geo[w].blocks), d_leaves, d_dead, d_acc, d_iacc);
        prof->end(st);
        *launches += integral ? 3 : 2;
        QC_CUDA(cudaGetLastError());
    }

    tr.mark("windows-enq");
    MergeOutput out;
    out.assignment.resize(S(n));
    int dead = 0;
    QC_CUDA(cudaMemcpyAsync(out.assignment.data(), d_asg, S(n), cudaMemcpyDeviceToHost, st));
    QC_CUDA(cudaMemcpyAsync(&out.leaves, d_leaves, sizeof(uint64_t), cudaMemcpyDeviceToHost, st));
    QC_CUDA(cudaMemcpyAsync(&dead, d_dead, sizeof(int), cudaMemcpyDeviceToHost, st));
    *d2h += S(n) + sizeof(uint64_t) + sizeof(int);
    if (integral && in.m > 0) {
        // cut_value re-score on the device (exact for integral weights), edges resident
        auto* d_cut = dalloc<unsigned long long>(keep, 1);
        QC_CUDA(cudaMemsetAsync(d_cut, 0, sizeof(unsigned long long), st));
        const long long blocks = std::min<long long>((in.m + 255) / 256, 148 * 8);
        prof->begin(K_MERGE_OTHER, static_cast<double>(in.m) * 16.0, st);
        k_cut_int<<<static_cast<unsigned>(blocks), 256, 0, st>>>(d_eu, d_ev, d_ew, in.m, d_asg, d_cut);
        prof->end(st);
        ++*launches;
        unsigned long long cut = 0;
        QC_CUDA(cudaMemcpyAsync(&cut, d_cut, sizeof cut, cudaMemcpyDeviceToHost, st));
        *d2h += sizeof cut;
        QC_CUDA(cudaStreamSynchronize(st));
        out.value = static_cast<double>(cut);
    } else {
        QC_CUDA(cudaStreamSynchronize(st));
        double v = 0.0;  // graph.hpp:126-134, edge-list order
        for (long long k = 0; k < in.m; ++k)
            if (out.assignment[EU(k)] != out.assignment[EV(k)]) v += EW(k);
        out.value = v;
    }
    tr.mark("rescore+sync");
    if (dead) config_error("no compatible candidate chain exists");
    return out;
}

}  // namespace qcg
