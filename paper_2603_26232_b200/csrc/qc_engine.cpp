// Engine: device memory, batched objective evaluation, lockstep optimisation, solve,
// and the statevector.hpp / qaoa.hpp entry points of the C-ABI (include/qcgpu.h).
// Host code is compiled with -ffp-contract=off: the phase LUT (std::polar), cos/sin(beta)
// and every Nelder-Mead expression round exactly like the reference's canonical build.
#include "qc_engine.hpp"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <complex>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <map>
#include <numbers>
#include <unordered_set>

#include "qc_nm.hpp"

namespace qcg {

namespace {
thread_local std::string g_last_error;
}

void set_error(const std::string& msg) { g_last_error = msg; }
const char* last_error() { return g_last_error.c_str(); }

void cuda_fail(cudaError_t e, const char* what, const char* file, int line) {
    if (e == cudaErrorMemoryAllocation) {
        (void)cudaGetLastError();
        resource_error(std::string("device out of memory (") + what + ")");
    }
    internal_error(std::string("CUDA error: ") + cudaGetErrorString(e) + " in " + what + " at " +
                   file + ":" + std::to_string(line));
}

void* DevBuf::get(size_t bytes) {
    if (bytes == 0) bytes = 16;
    if (bytes > cap) {
        release();
        QC_CUDA(cudaMalloc(&p, bytes));
        cap = bytes;
    }
    return p;
}
void DevBuf::release() {
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
}
void* HostBuf::get(size_t bytes) {
    if (bytes == 0) bytes = 16;
    if (bytes > cap) {
        if (p) cudaFreeHost(p);
        p = nullptr;
        cap = 0;
        QC_CUDA(cudaHostAlloc(&p, bytes, cudaHostAllocDefault));
        cap = bytes;
    }
    return p;
}
HostBuf::~HostBuf() {
    if (p) cudaFreeHost(p);
}

namespace {
// Parallel form of the validation loop below for large edge lists (C4: 9.3M edges, C5:
// 12.8M; the serial loop took ~65 ms of C4's end-to-end step): threads take contiguous edge
// ranges, the duplicate bitset is updated with atomic fetch-or. Any problem (range,
// self-loop, weight, duplicate) returns false and the serial loop re-runs to raise exactly
// the reference's first error; the weight total is summed in edge order as there.
bool load_graph_parallel(const qc_graph* g, HostGraph& h, uint64_t nn, int threads) {
    const int m = g->m;
    h.u.resize(static_cast<size_t>(m));
    h.v.resize(static_cast<size_t>(m));
    h.w.resize(static_cast<size_t>(m));
    std::vector<uint64_t> bits(static_cast<size_t>((nn * nn / 2 + nn) / 64 + 1), 0);
    int bad = 0, nonint = 0;
    const uint32_t n = static_cast<uint32_t>(g->n);
#pragma omp parallel for schedule(static) num_threads(threads) reduction(| : bad, nonint)
    for (int i = 0; i < m; ++i) {
        uint32_t u = g->edges[i].u, v = g->edges[i].v;
        const double w = g->edges[i].w;
        if (u >= n || v >= n || u == v || w < 0.0 || std::isnan(w)) {
            bad = 1;
            continue;
        }
        if (u > v) std::swap(u, v);
        const uint64_t k = static_cast<uint64_t>(u) * (2 * nn - u - 1) / 2 + (v - u - 1);
        const uint64_t bit = uint64_t{1} << (k & 63);
        if (__atomic_fetch_or(&bits[k >> 6], bit, __ATOMIC_RELAXED) & bit) {
            bad = 1;
            continue;
        }
        h.u[static_cast<size_t>(i)] = u;
        h.v[static_cast<size_t>(i)] = v;
        h.w[static_cast<size_t>(i)] = w;
        if (w != std::floor(w)) nonint = 1;
    }
    if (bad) return false;
    double total = 0.0;
    for (int i = 0; i < m; ++i) total += h.w[static_cast<size_t>(i)];
    h.total = total;
    h.integral = !nonint;
    return true;
}
}  // namespace

// graph.hpp:37-50 Graph::add_edge validation; statevector.hpp:83-89 integrality.
HostGraph load_graph(const qc_graph* g) {
    if (!g) config_error("null graph");
    if (g->n < 0) config_error("negative vertex count");
    if (g->m < 0) config_error("negative edge count");
    if (g->m > 0 && !g->edges) config_error("null edge list");
    HostGraph h;
    h.n = g->n;
    h.u.reserve(static_cast<size_t>(g->m));
    h.v.reserve(static_cast<size_t>(g->m));
    h.w.reserve(static_cast<size_t>(g->m));
    // duplicate detection (graph.hpp:37-50 add_edge rejects repeats): a bit per ordered
    // pair u < v when that fits in 64 MB (n <= ~32k: every BASELINE config), else a hash set
    const uint64_t nn = static_cast<uint64_t>(g->n);
    const bool use_bits = nn * nn / 2 <= (uint64_t{64} << 23);
    const int par = std::min(16, static_cast<int>(std::max(1u, std::thread::hardware_concurrency())));
    if (use_bits && g->m >= (1 << 18) && par > 1) {
        if (load_graph_parallel(g, h, nn, par)) {
            h.all_int = h.integral && h.total <= 4.0e18;
            if (h.total > 65535.0) h.integral = false;
            return h;
        }
        h = HostGraph{};  // a problem: the serial pass raises the reference's first error
        h.n = g->n;
    }
    std::vector<uint64_t> bits;
    std::unordered_set<uint64_t> keys;
    if (use_bits)
        bits.assign(static_cast<size_t>((nn * nn / 2 + nn) / 64 + 1), 0);
    else
        keys.reserve(static_cast<size_t>(g->m) * 2);
    for (int i = 0; i < g->m; ++i) {
        uint32_t u = g->edges[i].u, v = g->edges[i].v;
        const double w = g->edges[i].w;
        if (u >= static_cast<uint32_t>(g->n) || v >= static_cast<uint32_t>(g->n))
            config_error("edge endpoint out of range: (" + std::to_string(u) + "," +
                         std::to_string(v) + ") with n=" + std::to_string(g->n));
        if (u == v) config_error("self-loop rejected at vertex " + std::to_string(u));
        if (w < 0.0 || std::isnan(w)) config_error("negative or NaN edge weight rejected");
        if (u > v) std::swap(u, v);
        bool dup;
        if (use_bits) {  // row-major upper triangle: u*(2n-u-1)/2 + (v-u-1)
            const uint64_t k = static_cast<uint64_t>(u) * (2 * nn - u - 1) / 2 + (v - u - 1);
            dup = (bits[k >> 6] >> (k & 63)) & 1u;
            bits[k >> 6] |= uint64_t{1} << (k & 63);
        } else {
            dup = !keys.insert(static_cast<uint64_t>(u) * nn + v).second;
        }
        if (dup) config_error("duplicate edge (" + std::to_string(u) + "," + std::to_string(v) + ")");
        h.u.push_back(u);
        h.v.push_back(v);
        h.w.push_back(w);
        h.total += w;
        if (w != std::floor(w) || w < 0.0) h.integral = false;
    }
    h.all_int = h.integral && h.total <= 4.0e18;
    if (h.total > 65535.0) h.integral = false;
    return h;
}

}  // namespace qcg

using namespace qcg;

// ---------------------------------------------------------------------------
// engine
// ---------------------------------------------------------------------------
void qc_engine::h2d_copy(void* dst, const void* src, size_t bytes, cudaStream_t st) {
    QC_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st ? st : stream));
    h2d += bytes;
}
void qc_engine::d2h_copy(void* dst, const void* src, size_t bytes, cudaStream_t st) {
    QC_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, st ? st : stream));
    d2h += bytes;
}

std::vector<DevGraph> qc_engine::prepare(const std::vector<HostGraph>& hg, bool allow_sym,
                                         bool unit_cost, DevBuf* target) {
    std::vector<DevGraph> dg(hg.size());
    size_t bytes = 0, ebytes = 0;
    std::vector<size_t> off(hg.size()), eoff(hg.size());
    for (size_t i = 0; i < hg.size(); ++i) {
        DevGraph& d = dg[i];
        d.q = hg[i].n;
        d.sym = allow_sym && d.q >= 2;
        d.Q = d.sym ? d.q - 1 : d.q;
        d.integral = hg[i].integral;
        d.unit_cost = unit_cost;
        d.lut_len = d.integral ? static_cast<int>(hg[i].total) + 1 : 0;
        off[i] = bytes;
        if (!unit_cost) {
            const size_t entries = size_t{1} << d.Q;
            bytes += (d.integral ? 2 : 10) * entries;  // non-integral: values + index levels
            bytes = (bytes + 255) & ~size_t{255};
        }
        eoff[i] = ebytes;
        ebytes += hg[i].u.size() * 16 + 256;
    }
    char* base = static_cast<char*>((target ? target : &tables)->get(bytes));
    if (unit_cost) return dg;
    char* ebase = static_cast<char*>(edges.get(ebytes));
    char* hbase = static_cast<char*>(hstage.get(ebytes));
    for (size_t i = 0; i < hg.size(); ++i) {
        const size_t m = hg[i].u.size();
        char* h = hbase + eoff[i];
        std::memcpy(h, hg[i].u.data(), m * 4);
        std::memcpy(h + m * 4, hg[i].v.data(), m * 4);
        std::memcpy(h + m * 8, hg[i].w.data(), m * 8);
    }
    h2d_copy(ebase, hbase, ebytes);
    for (size_t i = 0; i < hg.size(); ++i) {
        DevGraph& d = dg[i];
        const size_t m = hg[i].u.size();
        char* de = ebase + eoff[i];
        if (d.integral)
            d.lev = reinterpret_cast<uint16_t*>(base + off[i]);
        else
            d.val = reinterpret_cast<double*>(base + off[i]);
        prof.begin(K_LEVELS, static_cast<double>(size_t{1} << d.Q) * (d.integral ? 2.0 : 8.0), stream);
        launches += launch_levels(reinterpret_cast<uint32_t*>(de), reinterpret_cast<uint32_t*>(de + m * 4),
                                  reinterpret_cast<double*>(de + m * 8), static_cast<int>(m), d.Q,
                                  d.integral, d.lev, d.val, stream);
        prof.end(stream);
    }
    // non-integral tables: exact phases through a LUT over the distinct values (qc_frac.cu)
    int* d_count = nullptr;
    for (size_t i = 0; i < hg.size(); ++i) {
        DevGraph& d = dg[i];
        if (d.integral) continue;
        const uint32_t N = uint32_t{1} << d.Q;
        void* scratch = distinct.get(distinct_scratch_bytes(N) + 64);
        d_count = reinterpret_cast<int*>(static_cast<char*>(scratch) + distinct_scratch_bytes(N));
        const unsigned long long* uniq = launch_distinct(d.val, N, scratch, d_count, stream);
        int D = 0;
        QC_CUDA(cudaMemcpyAsync(&D, d_count, sizeof(int), cudaMemcpyDeviceToHost, stream));
        QC_CUDA(cudaStreamSynchronize(stream));
        d2h += sizeof(int);
        if (D < 1 || D > kMaxDistinct) continue;  // device sincos (within 1e-10)
        std::vector<unsigned long long> bits(static_cast<size_t>(D));
        QC_CUDA(cudaMemcpyAsync(bits.data(), uniq, bits.size() * 8, cudaMemcpyDeviceToHost, stream));
        d2h += bits.size() * 8;
        d.lev = reinterpret_cast<uint16_t*>(base + off[i] + size_t{8} * N);
        launch_index_of(d.val, N, uniq, D, d.lev, stream);
        ++launches;
        QC_CUDA(cudaStreamSynchronize(stream));
        d.fvals.resize(bits.size());
        std::memcpy(d.fvals.data(), bits.data(), bits.size() * 8);
        d.lut_len = D;
    }
    // the host staging buffer is reused by the next upload: wait for this copy
    QC_CUDA(cudaStreamSynchronize(stream));
    return dg;
}

size_t qc_engine::max_slots(int Q, bool onchip) const {
    const size_t N = size_t{1} << Q;
    const size_t per = N * 16 + (onchip ? 0 : N * 8 + (N / 4096 + 2) * 16) + 64;
    size_t budget = mem_budget;
    if (budget == 0) {
        // queried once: cudaMemGetInfo can stall for tens of ms behind the driver's
        // deferred frees, and it sits on the per-step path
        if (auto_budget == 0) {
            size_t fr = 0, tot = 0;
            if (cudaMemGetInfo(&fr, &tot) != cudaSuccess) fr = size_t{8} << 30;
            auto_budget = static_cast<size_t>(static_cast<double>(fr + states.cap + fbuf.cap) * 0.6);
        }
        budget = auto_budget;
    }
    size_t s = budget / per;
    if (s < 1) s = 1;
    if (onchip) s = std::min<size_t>(s, 1u << 16);
    return s;
}

double2* qc_engine::slot_state(int q, bool sym, int k, bool fp32) {
    const int Q = sym ? q - 1 : q;
    return reinterpret_cast<double2*>(static_cast<char*>(states.p) +
                                      (static_cast<size_t>(k) << Q) * (fp32 ? 8 : 16));
}

void qc_engine::sync() { QC_CUDA(cudaStreamSynchronize(stream)); }

size_t qc_engine::chunk_slots(int Q, bool onchip, size_t n) const {
    if (const char* env = std::getenv("QCG_CHUNK_SLOTS")) {
        const long v = std::strtol(env, nullptr, 10);
        if (v > 0) return std::min<size_t>(n, static_cast<size_t>(v));
    }
    // Chunks on separate streams: while one chunk's NM step is prepared on the host the
    // other chunk's kernels run. With the persistent v4 pass kernels (one CTA per SM) two
    // chunks measured best on B200 for C2: 75.9 ms per solve vs 84.4 (1), 81.1 (3),
    // 82.5 (4), 82.5 (6) -- every extra chunk adds per-launch prologue/tail and a
    // latency-bound block-sum launch per lockstep step.
    size_t chunks = 2;
    if (const char* env = std::getenv("QCG_CHUNKS")) chunks = std::max(1L, std::strtol(env, nullptr, 10));
    chunks = std::min(chunks, n);
    return std::max<size_t>(1, (n + chunks - 1) / chunks);
}

void qc_engine::reserve(int Q, bool need_fbuf, size_t slots) {
    const size_t N = size_t{1} << Q;
    states.get(slots * N * 16);
    if (need_fbuf) fbuf.get(slots * N * 8);
    const size_t pps = Q > 12 ? (size_t{2} << (Q - 12)) : 0;
    partials.get(slots * pps * 8 + 8);
    outd.get(slots * 8);
    if (tickets.cap < slots * 4) {  // zeroed once; kernels leave them zeroed
        tickets.get(slots * 4);
        QC_CUDA(cudaMemsetAsync(tickets.p, 0, tickets.cap, stream));
    }
}

namespace {
// results written by the kernels into pinned host memory (default) or copied (QCG_ZC=0)
bool zero_copy_out() {
    static const bool on = [] {
        const char* e = std::getenv("QCG_ZC");
        return !(e && e[0] == '0');
    }();
    return on;
}
}  // namespace

void qc_engine::enqueue_chunk(const std::vector<DevGraph>& dg, const EvalPoint* pts, int n, int p,
                              uint32_t flags, size_t slot0, ChunkCtx& ctx) {
    const auto t_enq = std::chrono::steady_clock::now();
    if (ctx.shared) flags |= F_BALGRID;
    ctx.n = n;
    ctx.flags = flags;
    if (n <= 0) return;
    cudaStream_t cs = ctx.st ? ctx.st : stream;
    const DevGraph& g0 = dg[static_cast<size_t>(pts[0].g)];
    const ChainPlan plan = plan_chain(g0.q, g0.sym);
    const size_t N = size_t{1} << plan.Q;
    // fp32 mode: float2 amplitudes / float f(z) packed at half the fp64 stride
    const bool fp32 = flags & F_FP32;
    const size_t ab = fp32 ? 8 : 16, fbb = fp32 ? 4 : 8;
    char* st = static_cast<char*>(states.p) + slot0 * N * ab;
    char* fb = nullptr;
    if (!plan.onchip && (flags & F_EXPECT)) fb = static_cast<char*>(fbuf.p) + slot0 * N * fbb;
    const size_t pps = partials_per_slot(plan);
    auto* part = static_cast<double*>(partials.p) + slot0 * pps;
    auto* tick = static_cast<unsigned*>(tickets.p) + slot0;
    auto* od = static_cast<double*>(outd.p) + slot0;
    ctx.d_out = od;

    // staging: [SlotDesc n][LayerParam n*p][LUT entries]
    size_t lut_total = 0;
    for (int k = 0; k < n; ++k) {
        const DevGraph& d = dg[static_cast<size_t>(pts[k].g)];
        if (d.lev && !d.unit_cost)
            for (int l = 0; l < p; ++l)
                if (pts[k].x[l] != 0.0) lut_total += static_cast<size_t>(d.lut_len);
    }
    const size_t o_lp = (static_cast<size_t>(n) * sizeof(SlotDesc) + 255) & ~size_t{255};
    const size_t o_lut =
        (o_lp + static_cast<size_t>(n) * static_cast<size_t>(std::max(p, 1)) * sizeof(LayerParam) + 255) &
        ~size_t{255};
    const size_t lut_entry = fp32 ? 8 : 16;  // double2 (exact) or float2 LUT entries
    const size_t bytes = o_lut + lut_total * lut_entry;
    // a replayed graph copies a fixed-size staging block: sized for every slot phasing
    // every layer with the longest LUT of the solve, so it does not change step to step
    // the ping-pong wait binds to the other chunk's latest pass event at enqueue time, which
    // a replayed graph cannot express: those chunk steps launch directly
    const bool graph = use_graphs() && !prof.on && !ctx.passes;
    size_t copy_bytes = bytes;
    if (graph) {
        size_t maxl = 0;
        for (const DevGraph& x : dg) maxl = std::max(maxl, static_cast<size_t>(x.lut_len));
        copy_bytes = o_lut + static_cast<size_t>(n) * static_cast<size_t>(std::max(p, 1)) * maxl * lut_entry;
    }
    char* h = static_cast<char*>(ctx.hstage.get(copy_bytes));
    char* d = static_cast<char*>(ctx.dstage.get(copy_bytes));
    auto* hs = reinterpret_cast<SlotDesc*>(h);
    auto* hl = reinterpret_cast<LayerParam*>(h + o_lp);
    auto* hlut = reinterpret_cast<double*>(h + o_lut);
    size_t lut_pos = 0;
    ChainStats stats;
    stats.phase.assign(static_cast<size_t>(std::max(p, 0)), 0);
    stats.mix.assign(static_cast<size_t>(std::max(p, 0)), 0);
    const double amp0 = 1.0 / std::sqrt(static_cast<double>(size_t{1} << g0.q));  // :141
    struct LutJob {
        size_t pos;
        int len;
        double gamma;
        const double* fv;
    };
    std::vector<LutJob> jobs;
    jobs.reserve(static_cast<size_t>(n) * static_cast<size_t>(std::max(p, 1)));
    for (int k = 0; k < n; ++k) {
        const DevGraph& dgk = dg[static_cast<size_t>(pts[k].g)];
        SlotDesc& s = hs[k];
        s.state = reinterpret_cast<double2*>(st + static_cast<size_t>(k) * N * ab);
        s.fbuf = fb ? reinterpret_cast<double*>(fb + static_cast<size_t>(k) * N * fbb) : nullptr;
        // integral: lev = plev = cut levels; fractional: val = cut values, plev = the index
        // of each among the distinct values (null: device sincos), lev = null
        s.lev = (dgk.unit_cost || !dgk.integral) ? nullptr : dgk.lev;
        s.val = dgk.unit_cost ? nullptr : dgk.val;
        s.plev = dgk.unit_cost ? nullptr : dgk.lev;
        s.amp0 = amp0;
        s.layer_base = k * p;
        s.pad = 0;
        for (int l = 0; l < p; ++l) {
            LayerParam& L = hl[static_cast<size_t>(k) * static_cast<size_t>(p) + static_cast<size_t>(l)];
            const double gamma = pts[k].x[l];
            const double beta = pts[k].x[p + l];
            // statevector.hpp:192 (host libm, exactly like the reference)
            L.c = std::cos(beta);
            L.s = std::sin(beta);
            L.mix = (L.s == 0.0 && L.c == 1.0) ? 0 : 1;
            L.phase = gamma == 0.0 ? 0 : 1;  // :149
            L.gamma = gamma;
            stats.phase[static_cast<size_t>(l)] += L.phase;
            stats.mix[static_cast<size_t>(l)] += L.mix;
            L.lut = nullptr;
            L.lut_len = 0;
            L.pad = 0;
            if (L.phase && dgk.lev && !dgk.unit_cost) {
                jobs.push_back({lut_pos, dgk.lut_len, gamma, dgk.fvals.empty() ? nullptr : dgk.fvals.data()});
                L.lut = reinterpret_cast<const double2*>(d + o_lut + lut_pos * lut_entry);
                L.lut_len = dgk.lut_len;
                lut_pos += static_cast<size_t>(dgk.lut_len);
            }
        }
    }
    // statevector.hpp:154-157 lut[c] = std::polar(1.0, -gamma * c); non-integral tables
    // (:162-164) std::polar(1.0, -gamma * val) per distinct val. Host libm, exactly the
    // reference's operation. The LUTs sit on the chunk step's host critical path (results
    // in -> next step out), so from 256 entries they are split over 4 host threads (C2,
    // ~400-800 entries per step: staging 2.6 -> 1.5 ms per solve, C2 69.0-69.3 -> 68.5-68.6
    // ms). QCG_LUT_PAR_MIN / QCG_HOST_THREADS override.
    static const size_t lut_par_min = [] {
        const char* e = std::getenv("QCG_LUT_PAR_MIN");
        return e ? static_cast<size_t>(std::atol(e)) : static_cast<size_t>(256);
    }();
    static const int lut_threads_env = [] {
        const char* e = std::getenv("QCG_HOST_THREADS");
        if (e) return std::max(1, std::atoi(e));
        return static_cast<int>(std::max(1u, std::min(4u, std::thread::hardware_concurrency())));
    }();
    const int lut_threads = lut_pos >= lut_par_min ? lut_threads_env : 1;
#pragma omp parallel for schedule(static) num_threads(lut_threads) if (lut_threads > 1)
    for (size_t jb = 0; jb < jobs.size(); ++jb) {
        const LutJob& J = jobs[jb];
        auto arg = [&](int c) { return -J.gamma * (J.fv ? J.fv[c] : static_cast<double>(c)); };
        if (fp32) {
            float* dst = reinterpret_cast<float*>(h + o_lut) + 2 * J.pos;
            for (int c = 0; c < J.len; ++c) {
                const std::complex<double> z = std::polar(1.0, arg(c));
                dst[2 * c] = static_cast<float>(z.real());
                dst[2 * c + 1] = static_cast<float>(z.imag());
            }
        } else {
            double* dst = hlut + 2 * J.pos;
            for (int c = 0; c < J.len; ++c) {
                const std::complex<double> z = std::polar(1.0, arg(c));
                dst[2 * c] = z.real();
                dst[2 * c + 1] = z.imag();
            }
        }
    }
    const auto t_staged = std::chrono::steady_clock::now();
    double* ho = (flags & F_EXPECT) ? static_cast<double*>(ctx.hout.get(static_cast<size_t>(n) * 8)) : nullptr;
    if (ctx.wait_on) QC_CUDA(cudaStreamWaitEvent(cs, ctx.wait_on, 0));
    auto record = [&](size_t nbytes) {
        h2d_copy(d, h, nbytes, cs);
        // the expectations go straight to the pinned host block (zero-copy: pinned memory is
        // device-addressable under UVA), so no D2H copy node trails the block sum on the
        // chunk step's critical path
        const int k = launch_chain(plan, reinterpret_cast<const SlotDesc*>(d),
                                   reinterpret_cast<const LayerParam*>(d + o_lp), n, p, flags,
                                   reinterpret_cast<double*>(fb), part, tick, (ho && zero_copy_out()) ? ho : od, cs, &stats,
                                   graph ? nullptr : &prof, st, ctx.passes);
        if (ho && !zero_copy_out()) d2h_copy(ho, od, static_cast<size_t>(n) * 8, cs);
        else if (ho) d2h += static_cast<uint64_t>(n) * 8;
        return k;
    };
    if (!graph) {
        launches += record(bytes);
    } else {
        ChainKey key;
        key.Q = plan.Q;
        key.n = n;
        key.p = p;
        key.sym = plan.sym;
        key.flags = flags;
        const void* ptrs[8] = {st, fb, part, tick, od, d, h, ho};
        for (int i = 0; i < 8; ++i) key.ptr[i] = ptrs[i];
        key.copy_bytes = copy_bytes;
        if (!ctx.gexec || !(ctx.gkey == key)) {
            if (ctx.gexec) {
                QC_CUDA(cudaGraphExecDestroy(ctx.gexec));
                ctx.gexec = nullptr;
            }
            const uint64_t h0 = h2d, d0 = d2h;
            cudaGraph_t g = nullptr;
            QC_CUDA(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
            try {
                ctx.glaunches = record(copy_bytes);
            } catch (...) {  // never leave the stream in capture mode
                cudaGraph_t bad = nullptr;
                cudaStreamEndCapture(cs, &bad);
                if (bad) cudaGraphDestroy(bad);
                cudaGetLastError();
                h2d = h0;
                d2h = d0;
                throw;
            }
            QC_CUDA(cudaStreamEndCapture(cs, &g));
            QC_CUDA(cudaGraphInstantiate(&ctx.gexec, g, 0));
            QC_CUDA(cudaGraphDestroy(g));
            h2d = h0;  // counted per replay below
            d2h = d0;
            ctx.gkey = key;
            ++graph_captures;
        }
        QC_CUDA(cudaGraphLaunch(ctx.gexec, cs));
        launches += ctx.glaunches;
        h2d += copy_bytes;
        if (ho) d2h += static_cast<uint64_t>(n) * 8;
    }
    if (!ctx.done) QC_CUDA(cudaEventCreateWithFlags(&ctx.done, cudaEventDisableTiming));
    QC_CUDA(cudaEventRecord(ctx.done, cs));
    const auto t_launched = std::chrono::steady_clock::now();
    host_stage_s += std::chrono::duration<double>(t_staged - t_enq).count();
    host_launch_s += std::chrono::duration<double>(t_launched - t_staged).count();
}

void qc_engine::wait_chunk(ChunkCtx& ctx, double* out) {
    if (ctx.n <= 0) return;
    QC_CUDA(cudaEventSynchronize(ctx.done));
    if ((ctx.flags & F_EXPECT) && out) std::memcpy(out, ctx.hout.p, static_cast<size_t>(ctx.n) * 8);
}

void qc_engine::eval_chunk(const std::vector<DevGraph>& dg, const EvalPoint* pts, int n, int p,
                           uint32_t flags, double* out) {
    if (n <= 0) return;
    const DevGraph& g0 = dg[static_cast<size_t>(pts[0].g)];
    const ChainPlan plan = plan_chain(g0.q, g0.sym);
    reserve(plan.Q, !plan.onchip && (flags & F_EXPECT), static_cast<size_t>(n));
    enqueue_chunk(dg, pts, n, p, flags, 0, sync_ctx);
    wait_chunk(sync_ctx, out);
}

void qc_engine::eval(const std::vector<DevGraph>& dg, const std::vector<EvalPoint>& pts, int p,
                     double* out) {
    // group by qubit count (one launch chain per group and chunk)
    std::map<int, std::vector<int>> by_q;
    for (size_t k = 0; k < pts.size(); ++k) by_q[dg[static_cast<size_t>(pts[k].g)].q].push_back(static_cast<int>(k));
    std::vector<EvalPoint> buf;
    std::vector<double> res;
    for (auto& [q, idx] : by_q) {
        const DevGraph& g0 = dg[static_cast<size_t>(pts[static_cast<size_t>(idx[0])].g)];
        const ChainPlan plan = plan_chain(q, g0.sym);
        const size_t cap = max_slots(plan.Q, plan.onchip);
        for (size_t b = 0; b < idx.size(); b += cap) {
            const size_t e = std::min(idx.size(), b + cap);
            buf.clear();
            for (size_t k = b; k < e; ++k) buf.push_back(pts[static_cast<size_t>(idx[k])]);
            res.assign(buf.size(), 0.0);
            eval_chunk(dg, buf.data(), static_cast<int>(buf.size()), p, F_INIT | F_EXPECT | fp_flag(),
                       res.data());
            for (size_t k = b; k < e; ++k) out[idx[k]] = res[k - b];
        }
    }
}

namespace qcg {

std::vector<OptimizeOut> optimize_batch(qc_engine* e, const std::vector<DevGraph>& dg,
                                        const std::vector<int>& layers,
                                        const std::vector<int>& budget,
                                        const std::vector<uint64_t>& seeds,
                                        const std::vector<double>& tol,
                                        std::vector<std::vector<double>>* trace_x,
                                        std::vector<std::vector<double>>* trace_f) {
    const size_t n = dg.size();
    std::vector<AngleOptimizer> opt(n);
    for (size_t i = 0; i < n; ++i) {
        if (budget[i] < 1) config_error("optimizer budget must be positive");  // qaoa.hpp:88
        if (layers[i] < 1) config_error("layer count must be positive");      // qaoa.hpp:28
        opt[i].start(layers[i], budget[i], seeds[i], tol[i]);
    }
    // Tasks sharing (q, p) run as one lockstep group. The group is cut into chunks whose
    // working set fits L2; chunk c's next step is prepared on the host while the device
    // runs the chunks queued behind it (results are placement independent: every
    // evaluation restarts from |+>).
    std::map<std::pair<int, int>, std::vector<size_t>> groups;
    for (size_t i = 0; i < n; ++i) groups[{dg[i].q, layers[i]}].push_back(i);
    for (auto& [key, tasks] : groups) {
        const int p = key.second;
        const ChainPlan plan = plan_chain(dg[tasks[0]].q, dg[tasks[0]].sym);
        const size_t cap = e->max_slots(plan.Q, plan.onchip);
        for (size_t sb = 0; sb < tasks.size(); sb += cap) {
            const size_t se = std::min(tasks.size(), sb + cap);
            const size_t ns = se - sb;
            const size_t per = e->chunk_slots(plan.Q, plan.onchip, ns);
            const size_t nchunks = (ns + per - 1) / per;
            e->reserve(plan.Q, !plan.onchip, ns);
            while (e->chunk_pool.size() < nchunks) e->chunk_pool.push_back(std::make_unique<ChunkCtx>());
            std::vector<ChunkCtx*> ctxp(nchunks);
            for (size_t c = 0; c < nchunks; ++c) ctxp[c] = e->chunk_pool[c].get();
            auto ctx = [&](size_t c) -> ChunkCtx& { return *ctxp[c]; };
            // the aux stream must see the cut tables / zeroed tickets written on the main one
            cudaEvent_t ready;
            QC_CUDA(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
            QC_CUDA(cudaEventRecord(ready, e->stream));
            size_t nstreams = std::min<size_t>(nchunks, 4);
            if (const char* env = std::getenv("QCG_STREAMS"))
                nstreams = static_cast<size_t>(std::min(4L, std::max(1L, std::strtol(env, nullptr, 10))));
            for (size_t k = 0; k + 1 < nstreams; ++k) QC_CUDA(cudaStreamWaitEvent(e->aux[k], ready, 0));
            QC_CUDA(cudaEventDestroy(ready));
            for (size_t c = 0; c < nchunks; ++c) {
                ctx(c).st = (c % nstreams) ? e->aux[c % nstreams - 1] : e->stream;
                ctx(c).shared = nstreams > 1;
            }
            // Ping-pong (QCG_PINGPONG=1): whole-GPU pass kernels of concurrently queued chunks
            // otherwise interleave launch by launch, so the chunks stay in phase, their block
            // sums finish together and the device idles through every chunk's host step.
            // Chained on pass events, chunk c's passes follow chunk c-1's, and one chunk's
            // block sum + host step overlap the next chunk's passes.
            static const bool pingpong = [] {
                const char* v = std::getenv("QCG_PINGPONG");
                return v && v[0] == '1';
            }();
            for (size_t c = 0; c < nchunks; ++c) {
                ChunkCtx& x = ctx(c);
                if (pingpong && nchunks > 1) {
                    if (!x.passes) QC_CUDA(cudaEventCreateWithFlags(&x.passes, cudaEventDisableTiming));
                } else if (x.passes) {
                    QC_CUDA(cudaEventDestroy(x.passes));
                    x.passes = nullptr;
                }
            }
            for (size_t c = 0; c < nchunks; ++c)
                ctx(c).wait_on = (pingpong && nchunks > 1) ? ctx((c + nchunks - 1) % nchunks).passes : nullptr;
            std::vector<std::vector<EvalPoint>> pts(nchunks);
            std::vector<std::vector<size_t>> who(nchunks);
            std::vector<char> inflight(nchunks, 0);
            std::vector<double> vals;
            auto launch = [&](size_t c) {
                pts[c].clear();
                who[c].clear();
                const size_t b = sb + c * per, end = std::min(se, b + per);
                for (size_t k = b; k < end; ++k) {
                    const size_t i = tasks[k];
                    if (opt[i].done()) continue;
                    pts[c].push_back({static_cast<int>(i), opt[i].point().data()});
                    who[c].push_back(i);
                }
                inflight[c] = !pts[c].empty();
                if (inflight[c])
                    e->enqueue_chunk(dg, pts[c].data(), static_cast<int>(pts[c].size()), p,
                                     F_INIT | F_EXPECT | e->fp_flag(), c * per, ctx(c));
            };
            // Staggered start (QCG_STAGGER=1): chunk c+1's first step is enqueued only when
            // chunk c's first step completes. Measured: the interleaving of whole-GPU pass
            // kernels pulls the chunks back into phase within a few steps (C2 71.3 vs
            // 71.2 ms), so it is off; the ping-pong below keeps them apart.
            static const bool stagger = [] {
                const char* v = std::getenv("QCG_STAGGER");
                return v && v[0] == '1';
            }();
            size_t started = stagger ? 1 : nchunks;
            for (size_t c = 0; c < started; ++c) launch(c);
            // completion-order service: whichever chunk's step finished is told/asked and
            // re-enqueued first, so the device never idles behind a fixed host order
            size_t live = 0;
            for (size_t c = 0; c < nchunks; ++c) live += inflight[c] ? 1 : 0;
            live += nchunks - started;  // not yet started (staggered)
            using clk = std::chrono::steady_clock;
            while (live) {
                size_t c = nchunks;
                const auto tw = clk::now();
                for (;;) {
                    for (size_t k = 0; k < nchunks && c == nchunks; ++k) {
                        if (!inflight[k]) continue;
                        const cudaError_t q = cudaEventQuery(ctx(k).done);
                        if (q == cudaSuccess) c = k;
                        else if (q != cudaErrorNotReady) QC_CUDA(q);
                    }
                    if (c != nchunks) break;
                }
                if (started < nchunks) {  // staggered start: queue the next chunk first
                    launch(started);
                    if (!inflight[started]) --live;
                    ++started;
                }
                const auto tp = clk::now();
                e->host_wait_s += std::chrono::duration<double>(tp - tw).count();
                vals.assign(pts[c].size(), 0.0);
                e->wait_chunk(ctx(c), vals.data());
                for (size_t k = 0; k < who[c].size(); ++k) {
                    const size_t i = who[c][k];
                    const double f = -vals[k];  // qaoa.hpp:90
                    if (trace_x) {
                        const auto& x = opt[i].point();
                        (*trace_x)[i].insert((*trace_x)[i].end(), x.begin(), x.end());
                        (*trace_f)[i].push_back(f);
                    }
                    opt[i].tell(f);
                }
                e->host_tell_s += std::chrono::duration<double>(clk::now() - tp).count();
                launch(c);
                e->host_prep_s += std::chrono::duration<double>(clk::now() - tp).count();
                ++e->host_steps;
                if (!inflight[c]) --live;
            }
        }
    }
    std::vector<OptimizeOut> out(n);
    for (size_t i = 0; i < n; ++i) {
        out[i].params = opt[i].params;
        out[i].expectation = opt[i].expectation();
        out[i].evals = opt[i].evals;
    }
    return out;
}

void validate_solve(const std::vector<HostGraph>& hg, const std::vector<qc_solve_options>& opts) {
    const size_t n = hg.size();
    for (size_t i = 0; i < n; ++i) {  // qaoa.hpp:199-203, then :88, :28, :162-165
        const int q = hg[i].n;
        if (q < 1) config_error("cannot solve an empty subgraph");
        const uint64_t cap = std::min<uint64_t>(opts[i].qubit_cap, static_cast<uint64_t>(kMaxQubits));
        if (static_cast<uint64_t>(q) > cap)
            resource_error("subgraph has " + std::to_string(q) + " vertices, over the " +
                           std::to_string(cap) + "-qubit cap");
        if (opts[i].budget < 1) config_error("optimizer budget must be positive");
        if (opts[i].layers < 1) config_error("layer count must be positive");
        const uint64_t classes = opts[i].fold ? (uint64_t{1} << (q - 1)) : (uint64_t{1} << q);
        if (opts[i].top_k < 1 || static_cast<uint64_t>(opts[i].top_k) > classes)
            config_error("top_k must lie in [1, " + std::to_string(classes) + "] for " +
                         std::to_string(q) + " qubits" + (opts[i].fold ? " (folded)" : ""));
    }
}

std::vector<SolveOut> solve_batch(qc_engine* e, const std::vector<HostGraph>& hg,
                                  const std::vector<qc_solve_options>& opts) {
    validate_solve(hg, opts);
    NvtxRange r("qcgpu.solve_batch");
    const std::vector<DevGraph> dg = e->prepare(hg, true);
    return solve_prepared(e, hg, dg, opts);
}

std::vector<SolveOut> solve_prepared(qc_engine* e, const std::vector<HostGraph>& hg,
                                     const std::vector<DevGraph>& dg,
                                     const std::vector<qc_solve_options>& opts) {
    const size_t n = hg.size();
    std::vector<int> layers(n), budget(n);
    std::vector<uint64_t> seeds(n);
    std::vector<double> tol(n);
    for (size_t i = 0; i < n; ++i) {
        layers[i] = opts[i].layers;
        budget[i] = opts[i].budget;
        seeds[i] = opts[i].seed;
        tol[i] = opts[i].tolerance;
    }
    const auto t0 = std::chrono::steady_clock::now();
    const auto best = [&] {
        NvtxRange nv("qcgpu.optimize (lockstep Nelder-Mead)");
        return optimize_batch(e, dg, layers, budget, seeds, tol, nullptr, nullptr);
    }();
    const auto t1 = std::chrono::steady_clock::now();
    e->t_optimize_s += std::chrono::duration<double>(t1 - t0).count();
    struct FinalTimer {
        qc_engine* e;
        std::chrono::steady_clock::time_point t;
        ~FinalTimer() { e->t_final_s += std::chrono::duration<double>(std::chrono::steady_clock::now() - t).count(); }
    } final_timer{e, t1};
    NvtxRange nv_final("qcgpu.final_circuits_topk");

    // final circuit at the best angles (qaoa.hpp:208) + top-K (qaoa.hpp:211)
    std::vector<SolveOut> out(n);
    std::map<std::pair<int, int>, std::vector<size_t>> groups;  // (q, p)
    for (size_t i = 0; i < n; ++i) groups[{hg[i].n, layers[i]}].push_back(i);
    for (auto& [key, ids] : groups) {
        const int q = key.first, p = key.second;
        const ChainPlan plan = plan_chain(q, dg[ids[0]].sym);
        const size_t cap = e->max_slots(plan.Q, plan.onchip);
        for (size_t b = 0; b < ids.size(); b += cap) {
            const size_t end = std::min(ids.size(), b + cap);
            std::vector<EvalPoint> pts;
            for (size_t k = b; k < end; ++k) pts.push_back({static_cast<int>(ids[k]), best[ids[k]].params.data()});
            e->eval_chunk(dg, pts.data(), static_cast<int>(pts.size()), p,
                          F_INIT | F_STATE_OUT | e->fp_flag(),
                          nullptr);
            // every state's top-K is queued at once (scratch per state; the small results land
            // in pinned host memory, written by the kernels), spread over the engine's streams,
            // then one wait: no per-subgraph copy + sync round trip
            std::vector<size_t> soff(end - b + 1, 0), ooff(end - b + 1, 0);
            for (size_t k = b; k < end; ++k) {
                const size_t i = ids[k];
                const int K = opts[i].top_k;
                soff[k - b + 1] = soff[k - b] + ((topk_scratch_bytes(q, opts[i].fold != 0, K) + 255) & ~size_t{255});
                ooff[k - b + 1] = ooff[k - b] + ((static_cast<size_t>(K) * 12 + 64 + 255) & ~size_t{255});
            }
            char* scratch0 = static_cast<char*>(e->topk_scratch.get(soff[end - b]));
            char* host0 = static_cast<char*>(e->topk_host.get(ooff[end - b]));
            const int nst = 4;
            cudaEvent_t fork = nullptr;
            QC_CUDA(cudaEventCreateWithFlags(&fork, cudaEventDisableTiming));
            QC_CUDA(cudaEventRecord(fork, e->stream));  // the states are written on the main stream
            for (int sidx = 1; sidx < nst; ++sidx) QC_CUDA(cudaStreamWaitEvent(e->aux[sidx - 1], fork, 0));
            for (size_t k = b; k < end; ++k) {
                const size_t i = ids[k];
                const int K = opts[i].top_k;
                const bool fold = opts[i].fold != 0;
                char* ob = host0 + ooff[k - b];
                auto* d_bits = reinterpret_cast<uint32_t*>(ob);
                auto* d_probs = reinterpret_cast<double*>(ob + ((static_cast<size_t>(K) * 4 + 15) & ~size_t{15}));
                const int sidx = static_cast<int>((k - b) % nst);
                cudaStream_t sst = sidx == 0 ? e->stream : e->aux[sidx - 1];
                e->launches += launch_topk(e->slot_state(q, dg[i].sym, static_cast<int>(k - b),
                                                         e->precision == 32),
                                           q, dg[i].sym, fold, K, scratch0 + soff[k - b], d_bits, d_probs, sst,
                                           sidx == 0 ? &e->prof : nullptr, e->precision == 32);
                e->d2h += static_cast<uint64_t>(K) * 12;
            }
            for (int sidx = 1; sidx < nst; ++sidx) {  // join the side streams
                QC_CUDA(cudaEventRecord(fork, e->aux[sidx - 1]));
                QC_CUDA(cudaStreamWaitEvent(e->stream, fork, 0));
            }
            QC_CUDA(cudaEventDestroy(fork));
            e->sync();
            for (size_t k = b; k < end; ++k) {
                const size_t i = ids[k];
                const int K = opts[i].top_k;
                const char* ob = host0 + ooff[k - b];
                SolveOut& r = out[i];
                r.width = q;
                r.folded = opts[i].fold != 0;
                r.bits.assign(reinterpret_cast<const uint32_t*>(ob), reinterpret_cast<const uint32_t*>(ob) + K);
                const auto* pr = reinterpret_cast<const double*>(ob + ((static_cast<size_t>(K) * 4 + 15) & ~size_t{15}));
                r.probs.assign(pr, pr + K);
                r.params = best[i].params;
                r.expectation = best[i].expectation;
                r.evals = best[i].evals;
            }
        }
    }
    return out;
}

}  // namespace qcg

// ---------------------------------------------------------------------------
// C-ABI: engine + statevector.hpp + qaoa.hpp
// ---------------------------------------------------------------------------
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

void check_engine(qc_engine* e) {
    if (!e) config_error("null engine");
    QC_CUDA(cudaSetDevice(e->device));
}

// Run a FULL-mode single-state chain on a host state (statevector.hpp layer calls).
void full_state_op(qc_engine* e, int q, double* amps, const DevGraph& dg, int p,
                   const double* x, uint32_t flags, double* out_expect) {
    const ChainPlan plan = plan_chain(q, false);
    const size_t N = size_t{1} << q;
    auto* st = static_cast<double2*>(e->states.get(N * 16));
    if (!(flags & F_INIT)) {
        auto* h = static_cast<double*>(e->hstage.get(N * 16));
        std::memcpy(h, amps, N * 16);
        e->h2d_copy(st, h, N * 16);
        QC_CUDA(cudaStreamSynchronize(e->stream));
    }
    std::vector<DevGraph> v{dg};
    EvalPoint pt{0, x};
    double ex = 0.0;
    if (p == 0 && !plan.onchip) internal_error("layerless chain on a multi-pass state");
    e->eval_chunk(v, &pt, 1, p, flags, &ex);
    if (out_expect) *out_expect = ex;
    if (flags & F_STATE_OUT) {
        auto* h = static_cast<double*>(e->hout.get(N * 16));
        e->d2h_copy(h, e->states.p, N * 16);
        QC_CUDA(cudaStreamSynchronize(e->stream));
        std::memcpy(amps, h, N * 16);
    }
}

int check_q(int q, int cap_max) {
    if (q < 1) config_error("state needs at least one qubit");
    if (q > cap_max) resource_error("state rejected: " + std::to_string(q) + " qubits exceeds cap " + std::to_string(cap_max));
    return q;
}

}  // namespace

extern "C" {

const char* qc_last_error(void) { return qcg::last_error(); }
int qc_abi_version(void) { return QC_ABI_VERSION; }
int qc_qubit_cap(void) { return kMaxQubits; }
uint64_t qc_engine_launches(const qc_engine* e) { return e ? e->launches : 0; }

int qc_engine_create(int device, qc_engine** out) {
    return guarded([&] {
        if (!out) config_error("null output pointer");
        int count = 0;
        // no driver / no device is a resource failure (errors.hpp:14), not an internal one
        const cudaError_t dc = cudaGetDeviceCount(&count);
        if (dc != cudaSuccess) {
            cudaGetLastError();
            resource_error(std::string("no CUDA device: ") + cudaGetErrorString(dc));
        }
        if (device < 0 || device >= count)
            resource_error("CUDA device " + std::to_string(device) + " not available");
        QC_CUDA(cudaSetDevice(device));
        auto* e = new qc_engine();
        e->device = device;
        QC_CUDA(cudaStreamCreateWithFlags(&e->stream, cudaStreamNonBlocking));
        // chunk streams with descending priority (main stream = chunk 0 = highest): when
        // several chunks' kernels are runnable the device drains them in chunk order
        int lo = 0, hi = 0;
        QC_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
        QC_CUDA(cudaStreamDestroy(e->stream));
        QC_CUDA(cudaStreamCreateWithPriority(&e->stream, cudaStreamNonBlocking, hi));
        for (int k = 0; k < 3; ++k)
            QC_CUDA(cudaStreamCreateWithPriority(&e->aux[k], cudaStreamNonBlocking,
                                                 std::min(lo, hi + k + 1)));
        *out = e;
    });
}

void qc_engine_destroy(qc_engine* e) {
    if (!e) return;
    cudaSetDevice(e->device);
    cudaStreamSynchronize(e->stream);
    for (auto a : e->aux) {
        cudaStreamSynchronize(a);
        cudaStreamDestroy(a);
    }
    cudaStreamDestroy(e->stream);
    delete e;
}

int qc_engine_set_precision(qc_engine* e, int bits) {
    return guarded([&] {
        check_engine(e);
        if (bits != 64 && bits != 32) config_error("precision must be 64 (exact) or 32 (fp32 mode)");
        e->precision = bits;
        if (bits == 64) e->mixer = 0;  // the exact path replays mixer_pair only
    });
}

int qc_engine_set_mixer(qc_engine* e, int mixer) {
    return guarded([&] {
        check_engine(e);
        if (mixer != 0 && mixer != 1) config_error("mixer must be 0 (RX butterflies) or 1 (Walsh-Hadamard)");
        if (mixer == 1 && e->precision != 32)
            config_error("the Walsh-Hadamard mixer is an fp32-mode variant (not bit-exact): set precision 32 first");
        e->mixer = mixer;
    });
}

int qc_engine_profile(qc_engine* e, int on) {
    return guarded([&] {
        check_engine(e);
        e->prof.reset();
        e->prof.on = on != 0;
        e->prof.stride = on > 1 ? on : 1;  // on = N > 1: sample one launch in N per kind
    });
}

int qc_engine_profile_read(qc_engine* e, int kind, uint64_t* launches, double* ms,
                           double* bytes) {
    return guarded([&] {
        check_engine(e);
        if (kind < 0 || kind >= K_COUNT) config_error("unknown kernel kind");
        e->prof.resolve();
        if (launches) *launches = e->prof.count[kind];
        if (ms) *ms = e->prof.ms[kind];
        if (bytes) *bytes = e->prof.bytes[kind];
    });
}

int qc_engine_profile_read_fp64(qc_engine* e, int kind, double* fp64_ops) {
    return guarded([&] {
        check_engine(e);
        if (kind < 0 || kind >= K_COUNT) config_error("unknown kernel kind");
        e->prof.resolve();
        if (fp64_ops) *fp64_ops = e->prof.ops[kind];
    });
}

int qc_engine_host_stats(qc_engine* e, double* wait_s, double* prep_s, uint64_t* steps,
                         int reset) {
    return guarded([&] {
        if (!e) config_error("null engine");
        if (wait_s) *wait_s = e->host_wait_s;
        if (prep_s) *prep_s = e->host_prep_s;
        if (steps) *steps = e->host_steps;
        if (reset) {
            e->host_wait_s = e->host_prep_s = 0.0;
            e->host_tell_s = e->host_stage_s = e->host_launch_s = 0.0;
            e->host_steps = 0;
            e->t_optimize_s = e->t_final_s = e->t_merge_s = e->t_execute_s = 0.0;
        }
    });
}

int qc_engine_host_split(const qc_engine* e, double* out3) {
    return guarded([&] {
        if (!e || !out3) config_error("null argument");
        out3[0] = e->host_tell_s;
        out3[1] = e->host_stage_s;
        out3[2] = e->host_launch_s;
    });
}

int qc_engine_phase_times(const qc_engine* e, double* out4) {
    return guarded([&] {
        if (!e) config_error("null engine");
        out4[0] = e->t_optimize_s;
        out4[1] = e->t_final_s;
        out4[2] = e->t_merge_s;
        out4[3] = e->t_execute_s;
    });
}

int qc_engine_transfers(const qc_engine* e, uint64_t* h2d, uint64_t* d2h) {
    return guarded([&] {
        if (!e) config_error("null engine");
        if (h2d) *h2d = e->h2d;
        if (d2h) *d2h = e->d2h;
    });
}

void* qc_engine_stream(const qc_engine* e) { return e ? static_cast<void*>(e->stream) : nullptr; }

int qc_engine_set_memory_budget(qc_engine* e, uint64_t bytes) {
    return guarded([&] {
        check_engine(e);
        e->mem_budget = bytes;
    });
}

int qc_cost_table(qc_engine* e, const qc_graph* g, int cap, double* out, int* integral,
                  double* max_value) {
    return guarded([&] {
        check_engine(e);
        const HostGraph hg = load_graph(g);
        if (hg.n < 1) config_error("cost table needs at least one vertex");
        if (hg.n > cap || hg.n > kMaxQubits)
            resource_error("cost table rejected: " + std::to_string(hg.n) + " qubits exceeds cap " +
                           std::to_string(std::min(cap, kMaxQubits)));
        const auto dg = e->prepare({hg}, false);
        const size_t N = size_t{1} << hg.n;
        double mx = 0.0;
        if (dg[0].integral) {
            std::vector<uint16_t> lev(N);
            e->d2h_copy(lev.data(), dg[0].lev, N * 2);
            e->sync();
            for (size_t z = 0; z < N; ++z) {
                out[z] = static_cast<double>(lev[z]);
                mx = std::max(mx, out[z]);
            }
        } else {
            e->d2h_copy(out, dg[0].val, N * 8);
            e->sync();
            for (size_t z = 0; z < N; ++z) mx = std::max(mx, out[z]);
        }
        if (integral) *integral = dg[0].integral ? 1 : 0;
        if (max_value) *max_value = mx;
    });
}

int qc_plus_state(qc_engine* e, int q, int cap, double* amps) {
    return guarded([&] {
        check_engine(e);
        check_q(q, std::min(cap, kMaxQubits));
        if (q > 12) {
            // |+> of a multi-pass state: the first pass of a zero-angle layer writes it
            HostGraph hg;
            hg.n = q;
            const auto dg = e->prepare({hg}, false, true);
            const double x[2] = {0.0, 0.0};
            full_state_op(e, q, amps, dg[0], 1, x, F_INIT | F_STATE_OUT, nullptr);
            return;
        }
        HostGraph hg;
        hg.n = q;
        const auto dg = e->prepare({hg}, false, true);
        full_state_op(e, q, amps, dg[0], 0, nullptr, F_INIT | F_STATE_OUT, nullptr);
    });
}

int qc_apply_cost_layer(qc_engine* e, int q, double* amps, const qc_graph* g, double gamma) {
    return guarded([&] {
        check_engine(e);
        const HostGraph hg = load_graph(g);
        if (hg.n < 1) config_error("cost table needs at least one vertex");
        if (hg.n > kMaxQubits) resource_error("cost table rejected: qubits exceeds cap");
        if (hg.n != q) config_error("state and cost table disagree on qubit count");
        if (gamma == 0.0) return;  // statevector.hpp:149
        const auto dg = e->prepare({hg}, false);
        const double x[2] = {gamma, 0.0};  // beta 0 => mixer skipped exactly
        full_state_op(e, q, amps, dg[0], 1, x, F_STATE_OUT, nullptr);
    });
}

int qc_apply_mixer_layer(qc_engine* e, int q, double* amps, double beta) {
    return guarded([&] {
        check_engine(e);
        if (q < 1) config_error("mixer on empty state");
        if (q > kMaxQubits) resource_error("state exceeds the engine cap");
        HostGraph hg;
        hg.n = q;
        const auto dg = e->prepare({hg}, false, true);
        const double x[2] = {0.0, beta};
        full_state_op(e, q, amps, dg[0], 1, x, F_STATE_OUT, nullptr);
    });
}

int qc_expectation(qc_engine* e, int q, const double* amps, const qc_graph* g, double* out) {
    return guarded([&] {
        check_engine(e);
        const HostGraph hg = load_graph(g);
        if (hg.n < 1) config_error("cost table needs at least one vertex");
        if (hg.n > kMaxQubits) resource_error("cost table rejected: qubits exceeds cap");
        if (hg.n != q) config_error("state and cost table disagree on qubit count");
        const auto dg = e->prepare({hg}, false);
        const double x[2] = {0.0, 0.0};
        std::vector<double> tmp(amps, amps + 2 * (size_t{1} << q));
        // a zero-angle layer is an exact identity; its last pass emits the terms
        full_state_op(e, q, tmp.data(), dg[0], q > 12 ? 1 : 0, x, F_EXPECT, out);
    });
}

int qc_norm_sq(qc_engine* e, int q, const double* amps, double* out) {
    return guarded([&] {
        check_engine(e);
        check_q(q, kMaxQubits);
        HostGraph hg;
        hg.n = q;
        const auto dg = e->prepare({hg}, false, true);
        const double x[2] = {0.0, 0.0};
        std::vector<double> tmp(amps, amps + 2 * (size_t{1} << q));
        full_state_op(e, q, tmp.data(), dg[0], q > 12 ? 1 : 0, x, F_EXPECT, out);
    });
}

int qc_linear_ramp(int p, double* gammas, double* betas) {
    return guarded([&] {
        if (p < 1) config_error("layer count must be positive");
        const auto x = linear_ramp_packed(p);
        for (int l = 0; l < p; ++l) {
            gammas[l] = x[static_cast<size_t>(l)];
            betas[l] = x[static_cast<size_t>(p + l)];
        }
    });
}

int qc_run_ansatz(qc_engine* e, const qc_graph* g, int p, const double* gammas,
                  const double* betas, double* amps, double* expectation) {
    return guarded([&] {
        check_engine(e);
        const HostGraph hg = load_graph(g);
        if (hg.n < 1) config_error("cost table needs at least one vertex");
        if (hg.n > kMaxQubits) resource_error("cost table rejected: qubits exceeds cap");
        if (p < 0) config_error("gamma and beta schedules must have equal length");
        const auto dg = e->prepare({hg}, true);
        std::vector<double> x(static_cast<size_t>(2 * std::max(p, 1)), 0.0);
        for (int l = 0; l < p; ++l) {
            x[static_cast<size_t>(l)] = gammas[l];
            x[static_cast<size_t>(p + l)] = betas[l];
        }
        const ChainPlan plan = plan_chain(hg.n, dg[0].sym);
        if (p == 0 && !plan.onchip) {
            // |+> with no layers: the expectation of the uniform state
            std::vector<double> tmp(2 * (size_t{1} << hg.n));
            full_state_op(e, hg.n, tmp.data(), e->prepare({hg}, false, true)[0], 1,
                          std::vector<double>{0.0, 0.0}.data(), F_INIT | F_STATE_OUT, nullptr);
            if (amps) std::memcpy(amps, tmp.data(), tmp.size() * 8);
            if (expectation) {
                const auto dgf = e->prepare({hg}, false);
                full_state_op(e, hg.n, tmp.data(), dgf[0], 1, std::vector<double>{0.0, 0.0}.data(),
                              F_EXPECT, expectation);
            }
            return;
        }
        EvalPoint pt{0, x.data()};
        double ex = 0.0;
        e->eval_chunk(dg, &pt, 1, p, F_INIT | F_EXPECT | (amps ? F_STATE_OUT : 0u), &ex);
        if (expectation) *expectation = ex;
        if (amps) {
            const int q = hg.n;
            const size_t N = size_t{1} << plan.Q;
            std::vector<double> half(2 * N);
            e->d2h_copy(half.data(), e->states.p, N * 16);
            e->sync();
            const size_t full = (size_t{1} << q) - 1;
            for (size_t z = 0; z <= full; ++z) {  // a_{~z} == a_z (complement symmetry)
                const size_t i = (!dg[0].sym || z < N) ? z : (full ^ z);
                amps[2 * z] = half[2 * i];
                amps[2 * z + 1] = half[2 * i + 1];
            }
        }
    });
}

int qc_eval_batch(qc_engine* e, const qc_graph* graphs, int n_graphs, int p, int n_points,
                  const int32_t* index, const double* params, double* expectation) {
    return guarded([&] {
        check_engine(e);
        if (p < 1) config_error("layer count must be positive");
        std::vector<HostGraph> hg;
        for (int i = 0; i < n_graphs; ++i) {
            hg.push_back(load_graph(&graphs[i]));
            if (hg.back().n < 1) config_error("cost table needs at least one vertex");
            if (hg.back().n > kMaxQubits) resource_error("graph exceeds the engine qubit cap");
        }
        const auto dg = e->prepare(hg, true);
        std::vector<EvalPoint> pts(static_cast<size_t>(n_points));
        for (int k = 0; k < n_points; ++k) {
            if (index[k] < 0 || index[k] >= n_graphs) config_error("point graph index out of range");
            pts[static_cast<size_t>(k)] = {index[k], params + static_cast<size_t>(k) * 2 * static_cast<size_t>(p)};
        }
        e->eval(dg, pts, p, expectation);
    });
}

int qc_optimize_batch(qc_engine* e, const qc_graph* graphs, int n, int p, int budget,
                      const uint64_t* seeds, double tolerance, double* params, double* expectation,
                      int32_t* evals, double* trace_x, double* trace_f) {
    return guarded([&] {
        check_engine(e);
        std::vector<HostGraph> hg;
        for (int i = 0; i < n; ++i) {
            hg.push_back(load_graph(&graphs[i]));
            if (hg.back().n < 1) config_error("cost table needs at least one vertex");
            if (hg.back().n > kMaxQubits) resource_error("graph exceeds the engine qubit cap");
        }
        if (budget < 1) config_error("optimizer budget must be positive");
        if (p < 1) config_error("layer count must be positive");
        const auto dg = e->prepare(hg, true);
        std::vector<int> L(static_cast<size_t>(n), p), B(static_cast<size_t>(n), budget);
        std::vector<uint64_t> S(seeds, seeds + n);
        std::vector<double> T(static_cast<size_t>(n), tolerance);
        std::vector<std::vector<double>> tx(static_cast<size_t>(n)), tf(static_cast<size_t>(n));
        const auto out = optimize_batch(e, dg, L, B, S, T, trace_x ? &tx : nullptr,
                                        trace_x ? &tf : nullptr);
        for (int i = 0; i < n; ++i) {
            const auto& o = out[static_cast<size_t>(i)];
            std::memcpy(params + static_cast<size_t>(i) * 2 * p, o.params.data(), 16 * static_cast<size_t>(p));
            expectation[i] = o.expectation;
            evals[i] = o.evals;
            if (trace_x) {
                const size_t stride_x = static_cast<size_t>(budget) * 2 * p;
                std::fill(trace_x + i * stride_x, trace_x + (i + 1) * stride_x, 0.0);
                std::fill(trace_f + static_cast<size_t>(i) * budget, trace_f + static_cast<size_t>(i + 1) * budget, 0.0);
                std::memcpy(trace_x + i * stride_x, tx[static_cast<size_t>(i)].data(),
                            std::min(tx[static_cast<size_t>(i)].size(), stride_x) * 8);
                std::memcpy(trace_f + static_cast<size_t>(i) * budget, tf[static_cast<size_t>(i)].data(),
                            std::min<size_t>(tf[static_cast<size_t>(i)].size(), static_cast<size_t>(budget)) * 8);
            }
        }
    });
}

int qc_top_candidates(qc_engine* e, int q, const double* amps, int top_k, int fold,
                      uint32_t* bits, double* probs) {
    return guarded([&] {
        check_engine(e);
        if (q < 1) config_error("cannot rank candidates of an empty state");
        if (q > 32) resource_error("candidate bits limited to 32 qubits");
        if (q > kMaxQubits) resource_error("state exceeds the engine qubit cap");
        const uint64_t classes = fold ? (uint64_t{1} << (q - 1)) : (uint64_t{1} << q);
        if (top_k < 1 || static_cast<uint64_t>(top_k) > classes)
            config_error("top_k must lie in [1, " + std::to_string(classes) + "] for " +
                         std::to_string(q) + " qubits" + (fold ? " (folded)" : ""));
        const size_t N = size_t{1} << q;
        auto* st = static_cast<double2*>(e->states.get(N * 16));
        auto* h = static_cast<double*>(e->hstage.get(N * 16));
        std::memcpy(h, amps, N * 16);
        e->h2d_copy(st, h, N * 16);
        void* scratch = e->topk_scratch.get(topk_scratch_bytes(q, fold != 0, top_k));
        char* ob = static_cast<char*>(e->topk_out.get(static_cast<size_t>(top_k) * 12 + 64));
        auto* d_bits = reinterpret_cast<uint32_t*>(ob);
        auto* d_probs = reinterpret_cast<double*>(ob + ((static_cast<size_t>(top_k) * 4 + 15) & ~size_t{15}));
        e->launches += launch_topk(st, q, false, fold != 0, top_k, scratch, d_bits, d_probs, e->stream,
                                   &e->prof);
        e->d2h_copy(bits, d_bits, static_cast<size_t>(top_k) * 4);
        e->d2h_copy(probs, d_probs, static_cast<size_t>(top_k) * 8);
        e->sync();
    });
}

static void fill_result(const SolveOut& s, qc_solve_result* r) {
    r->width = s.width;
    r->folded = s.folded ? 1 : 0;
    r->count = static_cast<int32_t>(s.bits.size());
    r->evals = s.evals;
    r->expectation = s.expectation;
    if (r->bits) std::memcpy(r->bits, s.bits.data(), s.bits.size() * 4);
    if (r->probs) std::memcpy(r->probs, s.probs.data(), s.probs.size() * 8);
    if (r->params) std::memcpy(r->params, s.params.data(), s.params.size() * 8);
}

int qc_solve_subgraph(qc_engine* e, const qc_graph* g, const qc_solve_options* opt,
                      qc_solve_result* res) {
    return guarded([&] {
        check_engine(e);
        if (!opt || !res) config_error("null options/result");
        const auto out = solve_batch(e, {load_graph(g)}, {*opt});
        fill_result(out[0], res);
    });
}

int qc_solve_batch(qc_engine* e, const qc_graph* graphs, int n, const qc_solve_options* opts,
                   qc_solve_result* results) {
    return guarded([&] {
        check_engine(e);
        std::vector<HostGraph> hg;
        std::vector<qc_solve_options> o(opts, opts + n);
        for (int i = 0; i < n; ++i) hg.push_back(load_graph(&graphs[i]));
        const auto out = solve_batch(e, hg, o);
        for (int i = 0; i < n; ++i) fill_result(out[static_cast<size_t>(i)], &results[i]);
    });
}

}  // extern "C"
