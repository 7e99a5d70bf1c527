/* TEST INFRASTRUCTURE ONLY — plain-C restatement of the reference's hot path
 * (/root/reference/proj/include/qcut/*.hpp), written independently from the
 * published algorithm and pinned bit-for-bit against oracle/_ref (the reference
 * itself, compiled here) and the committed fixtures in tests/golden/.
 *
 * It is the parity CHECKER: tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg call it. The product (paper_2603_26232_b200/) never links,
 * loads or falls back to it.
 *
 * Floating point is restated operation by operation (compile with
 * -ffp-contract=off: the reference's canonical Release build has no FMA).
 */
#define _GNU_SOURCE
#include "qcut_oracle.h"

#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

#define PI_D 3.141592653589793238462643383279502884 /* std::numbers::pi */

static __thread char g_err[512];
static int g_qubit_cap = 24; /* statevector.hpp:20 kQubitCap */

static int set_err(int code, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof g_err, fmt, ap);
    va_end(ap);
    return code;
}
#define CHECK(x)                 \
    do {                         \
        int rc_ = (x);           \
        if (rc_) return rc_;     \
    } while (0)

const char* orc_last_error(void) { return g_err; }
int orc_qubit_cap(void) { return g_qubit_cap; }
void orc_set_qubit_cap(int cap) { g_qubit_cap = cap; }

static double now_s(void) {
    struct timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

/* ------------------------------------------------------------------------ */
/* mt19937_64 (the standard engine used by graph.hpp:150 and qaoa.hpp:98)    */
/* ------------------------------------------------------------------------ */
typedef struct {
    uint64_t s[312];
    int i;
} mt64;

static void mt64_seed(mt64* r, uint64_t seed) {
    r->s[0] = seed;
    for (int k = 1; k < 312; ++k)
        r->s[k] = 6364136223846793005ULL * (r->s[k - 1] ^ (r->s[k - 1] >> 62)) + (uint64_t)k;
    r->i = 312;
}

static uint64_t mt64_next(mt64* r) {
    if (r->i >= 312) {
        for (int k = 0; k < 312; ++k) {
            uint64_t y = (r->s[k] & 0xFFFFFFFF80000000ULL) | (r->s[(k + 1) % 312] & 0x7FFFFFFFULL);
            uint64_t v = r->s[(k + 156) % 312] ^ (y >> 1);
            if (y & 1) v ^= 0xB5026F5AA96619E9ULL;
            r->s[k] = v;
        }
        r->i = 0;
    }
    uint64_t x = r->s[r->i++];
    x ^= (x >> 29) & 0x5555555555555555ULL;
    x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
    x ^= (x << 37) & 0xFFF7EEE000000000ULL;
    x ^= x >> 43;
    return x;
}

/* libstdc++ uniform_real_distribution<double>(a, b) over a 64-bit engine:
 * generate_canonical<double,53> = (double)draw / 2^64 (clamped below 1), then
 * canonical * (b - a) + a. Used for NM restarts, qaoa.hpp:98-99,113. */
static double uniform_real(mt64* r, double a, double b) {
    double c = (double)mt64_next(r) / 18446744073709551616.0;
    if (c >= 1.0) c = nextafter(1.0, 0.0);
    return c * (b - a) + a;
}

/* ------------------------------------------------------------------------ */
/* graph.hpp                                                                 */
/* ------------------------------------------------------------------------ */
static int cmp_u64(const void* a, const void* b) {
    uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
    return x < y ? -1 : x > y;
}

/* Graph::add_edge validation (graph.hpp:37-50): range, self-loop, weight, duplicates. */
static int validate_graph(int n, int m, const orc_edge* e) {
    if (n < 0) return set_err(1, "negative vertex count");
    uint64_t* keys = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)(m > 0 ? m : 1));
    for (int i = 0; i < m; ++i) {
        uint32_t u = e[i].u, v = e[i].v;
        if (u >= (uint32_t)n || v >= (uint32_t)n) {
            free(keys);
            return set_err(1, "edge endpoint out of range: (%u,%u) with n=%d", u, v, n);
        }
        if (u == v) {
            free(keys);
            return set_err(1, "self-loop rejected at vertex %u", u);
        }
        if (e[i].w < 0.0 || isnan(e[i].w)) {
            free(keys);
            return set_err(1, "negative or NaN edge weight rejected");
        }
        if (u > v) {
            uint32_t t = u;
            u = v;
            v = t;
        }
        keys[i] = (uint64_t)u * (uint64_t)n + v;
    }
    qsort(keys, (size_t)m, sizeof(uint64_t), cmp_u64);
    for (int i = 1; i < m; ++i)
        if (keys[i] == keys[i - 1]) {
            free(keys);
            return set_err(1, "duplicate edge");
        }
    free(keys);
    return 0;
}

/* graph.hpp:126-134 cut_value: edge-list order sum of crossing weights. */
static double cut_value(int m, const orc_edge* e, const uint8_t* a) {
    double v = 0.0;
    for (int i = 0; i < m; ++i)
        if (a[e[i].u] != a[e[i].v]) v += e[i].w;
    return v;
}

/* graph.hpp:167-171 lex_less_mask: bit 0 is the most significant character. */
static int lex_less_mask(uint64_t a, uint64_t b) {
    uint64_t d = a ^ b;
    if (d == 0) return 0;
    return (a & (d & (~d + 1))) == 0;
}

/* graph.hpp:146-160 generate_er_graph: one 53-bit draw per pair (u<v) in lex order. */
int orc_generate_er(int n, double p, uint64_t seed, orc_edge* out, long long cap, long long* m) {
    if (p < 0.0 || p > 1.0 || isnan(p)) return set_err(1, "edge probability must lie in [0,1]");
    mt64 r;
    mt64_seed(&r, seed);
    long long cnt = 0;
    for (uint32_t u = 0; u + 1 < (uint32_t)n; ++u)
        for (uint32_t v = u + 1; v < (uint32_t)n; ++v) {
            double x = (double)(mt64_next(&r) >> 11) * 0x1.0p-53;
            if (x < p) {
                if (out) {
                    if (cnt >= cap) return set_err(1, "edge buffer too small");
                    out[cnt].u = u;
                    out[cnt].v = v;
                    out[cnt].w = 1.0;
                }
                ++cnt;
            }
        }
    *m = cnt;
    return 0;
}

/* Weighted random d-regular graph for BASELINE config 3 (the reference has no generator):
 * configuration model, Fisher-Yates shuffle of n*d stubs with mt19937_64(seed)
 * (j = draw % (i+1)), consecutive pairs; shuffles with a loop or multi-edge are
 * discarded; then integer weights wlo + draw % span in (u, v)-sorted edge order. */
static int cmp_edge_uv(const void* a, const void* b) {
    const orc_edge* x = (const orc_edge*)a;
    const orc_edge* y = (const orc_edge*)b;
    if (x->u != y->u) return x->u < y->u ? -1 : 1;
    return x->v < y->v ? -1 : (x->v > y->v);
}

int orc_generate_regular(int n, int d, uint64_t seed, int wlo, int whi, orc_edge* out,
                         long long cap, long long* m) {
    if (n < 1 || d < 1 || d >= n) return set_err(1, "regular graph needs 1 <= d < n");
    if (((long long)n * d) % 2) return set_err(1, "n*d must be even");
    if (wlo < 0 || whi < wlo) return set_err(1, "weight range must satisfy 0 <= wlo <= whi");
    mt64 r;
    mt64_seed(&r, seed);
    size_t S = (size_t)n * (size_t)d, E = S / 2;
    uint32_t* stubs = (uint32_t*)malloc(sizeof(uint32_t) * S);
    orc_edge* es = (orc_edge*)malloc(sizeof(orc_edge) * (E ? E : 1));
    uint64_t* keys = (uint64_t*)malloc(sizeof(uint64_t) * (E ? E : 1));
    for (int attempt = 0; attempt < 100000; ++attempt) {
        for (size_t i = 0; i < S; ++i) stubs[i] = (uint32_t)(i / (size_t)d);
        for (size_t i = S - 1; i > 0; --i) {
            size_t j = (size_t)(mt64_next(&r) % (uint64_t)(i + 1));
            uint32_t t = stubs[i];
            stubs[i] = stubs[j];
            stubs[j] = t;
        }
        int ok = 1;
        for (size_t k = 0; k < E && ok; ++k) {
            uint32_t u = stubs[2 * k], v = stubs[2 * k + 1];
            if (u == v) ok = 0;
            if (u > v) {
                uint32_t t = u;
                u = v;
                v = t;
            }
            es[k].u = u;
            es[k].v = v;
            es[k].w = 0.0;
            keys[k] = (uint64_t)u * (uint64_t)n + v;
        }
        if (ok) { /* multi-edge check (the product checks in pairing order; same verdict) */
            qsort(keys, E, sizeof(uint64_t), cmp_u64);
            for (size_t k = 1; k < E; ++k)
                if (keys[k] == keys[k - 1]) ok = 0;
        }
        if (!ok) continue;
        qsort(es, E, sizeof(orc_edge), cmp_edge_uv);
        uint64_t span = (uint64_t)(whi - wlo + 1);
        for (size_t k = 0; k < E; ++k) es[k].w = (double)(wlo + (int)(mt64_next(&r) % span));
        *m = (long long)E;
        int rc = 0;
        if (out) {
            if (cap < (long long)E) rc = set_err(1, "edge buffer too small");
            else memcpy(out, es, sizeof(orc_edge) * E);
        }
        free(stubs);
        free(es);
        free(keys);
        return rc;
    }
    free(stubs);
    free(es);
    free(keys);
    return set_err(2, "no simple regular graph found");
}

/* ------------------------------------------------------------------------ */
/* partition.hpp                                                             */
/* ------------------------------------------------------------------------ */
/* partition.hpp:58-103 chain_intervals: inclusive [a_i, b_i], b_i = a_{i+1}. */
static int chain_intervals(int n, int M, int mode, int* a, int* b) {
    if (M < 1) return set_err(1, "subgraph count must be positive");
    if (n == 0) return set_err(1, "cannot partition an empty graph");
    if (M == 1) {
        a[0] = 0;
        b[0] = n - 1;
        return 0;
    }
    if (n < M + 1) return set_err(1, "need at least %d vertices for %d chained subgraphs, got %d",
                                  M + 1, M, n);
    long long total = n - 1;
    long long* spans = (long long*)malloc(sizeof(long long) * (size_t)M);
    if (mode == 1) { /* kTailRemainder */
        long long s = (long long)(n / M) - 1;
        if (s < 1) {
            free(spans);
            return set_err(1, "tail-remainder split needs n >= 2*M, got n=%d M=%d", n, M);
        }
        for (int i = 0; i + 1 < M; ++i) spans[i] = s;
        spans[M - 1] = total - (long long)(M - 1) * s;
    } else {
        long long s = (total + M - 1) / M;
        if ((long long)(M - 1) * s <= total - 1) {
            for (int i = 0; i + 1 < M; ++i) spans[i] = s;
            spans[M - 1] = total - (long long)(M - 1) * s;
        } else {
            long long q = total / M, r = total % M;
            for (int i = 0; i < M; ++i) spans[i] = q + (i < r ? 1 : 0);
        }
    }
    long long x = 0;
    for (int i = 0; i < M; ++i) {
        a[i] = (int)x;
        x += spans[i];
        b[i] = (int)x;
    }
    free(spans);
    return 0;
}

typedef struct {
    int M;
    int *a, *b;       /* global id range per piece */
    int* local_m;     /* intra edges per piece */
    orc_edge** local; /* local edge lists (local ids), global edge-list order */
    long long inter_m;
} partition_t;

static void partition_free(partition_t* p) {
    if (p->local)
        for (int i = 0; i < p->M; ++i) free(p->local[i]);
    free(p->local);
    free(p->a);
    free(p->b);
    free(p->local_m);
    memset(p, 0, sizeof *p);
}

/* partition.hpp:111-160 partition: intra iff the edge fits u's right-most piece. */
static int do_partition(int n, int m, const orc_edge* e, int M, int mode, int cap,
                        partition_t* out) {
    memset(out, 0, sizeof *out);
    int* a = (int*)malloc(sizeof(int) * (size_t)(M > 0 ? M : 1));
    int* b = (int*)malloc(sizeof(int) * (size_t)(M > 0 ? M : 1));
    int rc = chain_intervals(n, M, mode, a, b);
    if (rc) {
        free(a);
        free(b);
        return rc;
    }
    if (cap > 0) {
        int largest = 0;
        for (int i = 0; i < M; ++i)
            if (b[i] - a[i] + 1 > largest) largest = b[i] - a[i] + 1;
        if (largest > cap) {
            long long need = ((long long)n - 1 + cap - 2) / (cap - 1);
            free(a);
            free(b);
            return set_err(2, "largest subgraph has %d vertices, over the %d-qubit cap; use at "
                              "least %lld subgraphs", largest, cap, need);
        }
    }
    int* last_piece = (int*)malloc(sizeof(int) * (size_t)(n > 0 ? n : 1));
    for (int i = 0; i < M; ++i)
        for (int v = a[i]; v <= b[i]; ++v) last_piece[v] = i;
    out->M = M;
    out->a = a;
    out->b = b;
    out->local_m = (int*)calloc((size_t)M, sizeof(int));
    out->local = (orc_edge**)calloc((size_t)M, sizeof(orc_edge*));
    int* capv = (int*)calloc((size_t)M, sizeof(int));
    for (int k = 0; k < m; ++k) {
        uint32_t u = e[k].u < e[k].v ? e[k].u : e[k].v;
        uint32_t v = e[k].u < e[k].v ? e[k].v : e[k].u;
        int i = last_piece[u];
        if ((int)v <= b[i]) {
            if (out->local_m[i] == capv[i]) {
                capv[i] = capv[i] ? 2 * capv[i] : 16;
                out->local[i] = (orc_edge*)realloc(out->local[i], sizeof(orc_edge) * (size_t)capv[i]);
            }
            orc_edge le = {u - (uint32_t)a[i], v - (uint32_t)a[i], e[k].w};
            out->local[i][out->local_m[i]++] = le;
        } else {
            out->inter_m++;
        }
    }
    free(capv);
    free(last_piece);
    return 0;
}

int orc_partition(int n, int m, const orc_edge* e, int M, int mode, int cap, int* first, int* last,
                  int* local_m, long long* inter_m) {
    CHECK(validate_graph(n, m, e));
    partition_t p;
    CHECK(do_partition(n, m, e, M, mode, cap, &p));
    for (int i = 0; i < M; ++i) {
        first[i] = p.a[i];
        last[i] = p.b[i];
        local_m[i] = p.local_m[i];
    }
    *inter_m = p.inter_m;
    partition_free(&p);
    return 0;
}

/* partition.hpp:163-167 derive_subgraph_count. */
int orc_derive_subgraph_count(long long n, long long cap, int* out) {
    if (cap < 2) return set_err(1, "qubit cap must be at least 2");
    *out = n <= cap ? 1 : (int)((n - 1 + cap - 2) / (cap - 1));
    return 0;
}

/* ------------------------------------------------------------------------ */
/* statevector.hpp                                                           */
/* ------------------------------------------------------------------------ */
typedef struct {
    int q;
    int integral;
    double max_value;
    uint16_t* lev; /* integral path */
    double* val;   /* fractional path */
} cost_t;

static void cost_free(cost_t* c) {
    free(c->lev);
    free(c->val);
    memset(c, 0, sizeof *c);
}

/* statevector.hpp:75-111 CostTable: uint16 levels when every weight is a
 * nonnegative integer and the total <= 65535, else doubles summed in edge order. */
static int cost_build(int n, int m, const orc_edge* e, int cap, cost_t* c) {
    memset(c, 0, sizeof *c);
    if (n < 1) return set_err(1, "cost table needs at least one vertex");
    if (n > cap) return set_err(2, "cost table rejected: %d qubits exceeds cap %d", n, cap);
    size_t size = (size_t)1 << n;
    double total = 0.0;
    int integral = 1;
    for (int i = 0; i < m; ++i) {
        total += e[i].w;
        if (e[i].w != floor(e[i].w) || e[i].w < 0.0) integral = 0;
    }
    if (total > 65535.0) integral = 0;
    c->q = n;
    c->integral = integral;
    if (integral) {
        c->lev = (uint16_t*)calloc(size, sizeof(uint16_t));
        for (int i = 0; i < m; ++i) {
            size_t bu = (size_t)1 << e[i].u, bv = (size_t)1 << e[i].v;
            uint16_t w = (uint16_t)e[i].w;
            for (size_t z = 0; z < size; ++z)
                if (((z & bu) != 0) != ((z & bv) != 0)) c->lev[z] = (uint16_t)(c->lev[z] + w);
        }
        double mx = 0.0;
        for (size_t z = 0; z < size; ++z)
            if ((double)c->lev[z] > mx) mx = (double)c->lev[z];
        c->max_value = mx;
    } else {
        c->val = (double*)calloc(size, sizeof(double));
        for (int i = 0; i < m; ++i) {
            size_t bu = (size_t)1 << e[i].u, bv = (size_t)1 << e[i].v;
            for (size_t z = 0; z < size; ++z)
                if (((z & bu) != 0) != ((z & bv) != 0)) c->val[z] += e[i].w;
        }
        double mx = 0.0;
        for (size_t z = 0; z < size; ++z)
            if (c->val[z] > mx) mx = c->val[z];
        c->max_value = mx;
    }
    return 0;
}

static inline double cost_value(const cost_t* c, size_t z) {
    return c->integral ? (double)c->lev[z] : c->val[z];
}

int orc_cost_table(int n, int m, const orc_edge* e, int cap, double* out, int* integral,
                   double* max_value) {
    CHECK(validate_graph(n, m, e));
    cost_t c;
    CHECK(cost_build(n, m, e, cap, &c));
    for (size_t z = 0; z < ((size_t)1 << n); ++z) out[z] = cost_value(&c, z);
    *integral = c.integral;
    *max_value = c.max_value;
    cost_free(&c);
    return 0;
}

/* statevector.hpp:134-143 plus_state: every amplitude (1/sqrt(2^q), 0). */
static int plus_fill(int q, int cap, double* amps) {
    if (q < 1) return set_err(1, "state needs at least one qubit");
    if (q > cap) return set_err(2, "state rejected: %d qubits exceeds cap %d", q, cap);
    size_t size = (size_t)1 << q;
    double a = 1.0 / sqrt((double)size);
    for (size_t z = 0; z < size; ++z) {
        amps[2 * z] = a;
        amps[2 * z + 1] = 0.0;
    }
    return 0;
}

int orc_plus_state(int q, int cap, double* amps) { return plus_fill(q, cap, amps); }

/* std::complex<double> *= : (a+bi)(c+di) = (ac - bd) + (ad + bc)i, no FMA. */
static inline void cmul_inplace(double* z, double c, double d) {
    double a = z[0], b = z[1];
    double re = a * c - b * d;
    double im = a * d + b * c;
    z[0] = re;
    z[1] = im;
}

/* statevector.hpp:146-166 apply_cost_layer. */
static int cost_layer(double* amps, const cost_t* c, double gamma, int threads) {
    if (gamma == 0.0) return 0; /* exact identity */
    long long n = (long long)1 << c->q;
    if (c->integral) {
        size_t nlut = (size_t)c->max_value + 1;
        double* lut = (double*)malloc(sizeof(double) * 2 * nlut);
        for (size_t k = 0; k < nlut; ++k) { /* std::polar(1, -gamma*k) */
            double th = -gamma * (double)k;
            lut[2 * k] = cos(th);
            lut[2 * k + 1] = sin(th);
        }
#pragma omp parallel for schedule(static) num_threads(threads) if (threads > 1)
        for (long long z = 0; z < n; ++z) {
            const double* l = lut + 2 * c->lev[z];
            cmul_inplace(amps + 2 * z, l[0], l[1]);
        }
        free(lut);
    } else {
#pragma omp parallel for schedule(static) num_threads(threads) if (threads > 1)
        for (long long z = 0; z < n; ++z) {
            double th = -gamma * c->val[z];
            cmul_inplace(amps + 2 * z, cos(th), sin(th));
        }
    }
    return 0;
}

int orc_apply_cost_layer(int q, double* amps, int n, int m, const orc_edge* e, double gamma,
                         int threads) {
    CHECK(validate_graph(n, m, e));
    cost_t c;
    CHECK(cost_build(n, m, e, g_qubit_cap, &c));
    if (q != n) {
        cost_free(&c);
        return set_err(1, "state and cost table disagree on qubit count");
    }
    cost_layer(amps, &c, gamma, threads);
    cost_free(&c);
    return 0;
}

/* statevector.hpp:176-180 mixer_pair: e^{-i beta X} on (a0, a1). */
static inline void rx_pair(double* a0, double* a1, double c, double s) {
    double r0 = a0[0], i0 = a0[1], r1 = a1[0], i1 = a1[1];
    a0[0] = c * r0 + s * i1;
    a0[1] = c * i0 - s * r1;
    a1[0] = s * i0 + c * r1;
    a1[1] = c * i1 - s * r0;
}

/* statevector.hpp:189-221 apply_mixer_layer. Every amplitude sees targets in
 * ascending order; the reference's 2^11 chunking only reorders independent
 * pairs, so a plain target-major loop yields identical bits. */
static int mixer_layer(int q, double* amps, double beta, int threads) {
    if (q == 0) return set_err(1, "mixer on empty state");
    double c = cos(beta), s = sin(beta);
    if (s == 0.0 && c == 1.0) return 0;
    long long pairs = ((long long)1 << q) >> 1;
    for (int t = 0; t < q; ++t) {
        long long half = (long long)1 << t, lo = half - 1;
#pragma omp parallel for schedule(static) num_threads(threads) if (threads > 1)
        for (long long k = 0; k < pairs; ++k) {
            long long i = ((k & ~lo) << 1) | (k & lo);
            rx_pair(amps + 2 * i, amps + 2 * (i + half), c, s);
        }
    }
    return 0;
}

int orc_apply_mixer_layer(int q, double* amps, double beta, int threads) {
    return mixer_layer(q, amps, beta, threads);
}

/* statevector.hpp:48-65 blocked_sum with f(z) = norm(a_z) * C(z)
 * (statevector.hpp:224-235): 4096-blocks summed in z order, partials in block order. */
static double blocked_expectation(int q, const double* amps, const cost_t* c, int threads) {
    const long long kBlock = 4096;
    long long count = (long long)1 << q;
    long long blocks = (count + kBlock - 1) / kBlock;
    double* partial = (double*)calloc((size_t)blocks, sizeof(double));
#pragma omp parallel for schedule(static) num_threads(threads) if (threads > 1)
    for (long long b = 0; b < blocks; ++b) {
        long long lo = b * kBlock, hi = lo + kBlock < count ? lo + kBlock : count;
        double acc = 0.0;
        for (long long z = lo; z < hi; ++z) {
            double x = amps[2 * z], y = amps[2 * z + 1];
            double nrm = x * x + y * y;
            acc += c ? nrm * cost_value(c, (size_t)z) : nrm;
        }
        partial[b] = acc;
    }
    double total = 0.0;
    for (long long b = 0; b < blocks; ++b) total += partial[b];
    free(partial);
    return total;
}

int orc_expectation(int q, const double* amps, int n, int m, const orc_edge* e, int threads,
                    double* out) {
    CHECK(validate_graph(n, m, e));
    cost_t c;
    CHECK(cost_build(n, m, e, g_qubit_cap, &c));
    if (q != n) {
        cost_free(&c);
        return set_err(1, "state and cost table disagree on qubit count");
    }
    *out = blocked_expectation(q, amps, &c, threads);
    cost_free(&c);
    return 0;
}

int orc_norm_sq(int q, const double* amps, int threads, double* out) {
    *out = blocked_expectation(q, amps, NULL, threads);
    return 0;
}

/* qaoa.hpp:59-68 run_ansatz: |+> then (cost gamma_l, mixer beta_l) per layer. */
static int ansatz(const cost_t* c, int p, const double* gammas, const double* betas, int threads,
                  double* amps) {
    CHECK(plus_fill(c->q, g_qubit_cap, amps));
    for (int l = 0; l < p; ++l) {
        cost_layer(amps, c, gammas[l], threads);
        CHECK(mixer_layer(c->q, amps, betas[l], threads));
    }
    return 0;
}

int orc_run_ansatz(int n, int m, const orc_edge* e, int p, const double* gammas,
                   const double* betas, int threads, double* amps, double* expect) {
    CHECK(validate_graph(n, m, e));
    cost_t c;
    CHECK(cost_build(n, m, e, g_qubit_cap, &c));
    double* s = amps ? amps : (double*)malloc(sizeof(double) * 2 * ((size_t)1 << n));
    int rc = ansatz(&c, p, gammas, betas, threads, s);
    if (!rc && expect) *expect = blocked_expectation(n, s, &c, threads);
    if (!amps) free(s);
    cost_free(&c);
    return rc;
}

/* qaoa.hpp:27-38 linear_ramp. */
int orc_linear_ramp(int p, double* gammas, double* betas) {
    if (p < 1) return set_err(1, "layer count must be positive");
    for (int l = 1; l <= p; ++l) {
        double frac = (double)l / (double)p;
        gammas[l - 1] = frac * PI_D / 2.0;
        betas[l - 1] = (1.0 - frac) * PI_D / 2.0;
    }
    return 0;
}

/* ------------------------------------------------------------------------ */
/* nelder_mead.hpp + qaoa.hpp:85-117                                         */
/* ------------------------------------------------------------------------ */
typedef struct {
    const cost_t* c;
    int p, threads;
    double* state;
    double* trace_x;
    double* trace_f;
    int trace_cap, trace_len;
} objective_t;

/* qaoa.hpp:89-91: -expectation(run_ansatz(unpack(x))). */
static double objective(objective_t* o, const double* x) {
    ansatz(o->c, o->p, x, x + o->p, o->threads, o->state);
    double f = -blocked_expectation(o->c->q, o->state, o->c, o->threads);
    if (o->trace_x && o->trace_len < o->trace_cap) {
        memcpy(o->trace_x + (size_t)o->trace_len * 2 * o->p, x, sizeof(double) * 2 * o->p);
        o->trace_f[o->trace_len] = f;
    }
    o->trace_len++;
    return f;
}

typedef struct {
    double* x;
    double value;
    int evals, converged, has_x, n, max_evals;
    objective_t* obj;
} nm_res;

/* std::vector<double> operator< : lexicographic. */
static int vec_less(const double* a, const double* b, int n) {
    for (int i = 0; i < n; ++i) {
        if (a[i] < b[i]) return 1;
        if (b[i] < a[i]) return 0;
    }
    return 0;
}

/* nelder_mead.hpp:36-46 eval: budget check, call, best-point tracking. */
static int nm_eval(nm_res* r, const double* x, double* out) {
    if (r->evals >= r->max_evals) return 0;
    *out = objective(r->obj, x);
    ++r->evals;
    if (!r->has_x || *out < r->value || (*out == r->value && vec_less(x, r->x, r->n))) {
        r->value = *out;
        memcpy(r->x, x, sizeof(double) * (size_t)r->n);
        r->has_x = 1;
    }
    return 1;
}

/* nelder_mead.hpp:29-120 nelder_mead_minimize (coefficients 1, 2, 0.5, 0.5). */
static void nelder_mead(objective_t* obj, const double* x0, int n, int max_evals, double tol,
                        nm_res* r) {
    const double step = 0.2;
    r->n = n;
    r->max_evals = max_evals;
    r->obj = obj;
    r->evals = 0;
    r->converged = 0;
    r->has_x = 0;
    r->value = 0.0;
    double* pts = (double*)malloc(sizeof(double) * (size_t)(n + 1) * n);
    double* fv = (double*)malloc(sizeof(double) * (size_t)(n + 1));
    int* order = (int*)malloc(sizeof(int) * (size_t)(n + 1));
    double* cen = (double*)malloc(sizeof(double) * n);
    double* xr = (double*)malloc(sizeof(double) * n);
    double* xe = (double*)malloc(sizeof(double) * n);
    double* xc = (double*)malloc(sizeof(double) * n);
#define PT(i) (pts + (size_t)(i) * n)
    for (int i = 0; i <= n; ++i) memcpy(PT(i), x0, sizeof(double) * n);
    int ok = nm_eval(r, PT(0), &fv[0]);
    for (int i = 1; i <= n && ok; ++i) {
        PT(i)[i - 1] += step;
        ok = nm_eval(r, PT(i), &fv[i]);
    }
    while (ok) {
        /* stable sort of indices by fv (insertion sort is stable) */
        for (int i = 0; i <= n; ++i) order[i] = i;
        for (int i = 1; i <= n; ++i) {
            int k = order[i], j = i - 1;
            while (j >= 0 && fv[k] < fv[order[j]]) {
                order[j + 1] = order[j];
                --j;
            }
            order[j + 1] = k;
        }
        int best = order[0], worst = order[n], second = order[n - 1];
        if (fv[worst] - fv[best] <= tol) {
            r->converged = 1;
            break;
        }
        for (int d = 0; d < n; ++d) cen[d] = 0.0;
        for (int i = 0; i <= n; ++i)
            if (i != worst)
                for (int d = 0; d < n; ++d) cen[d] += PT(i)[d];
        for (int d = 0; d < n; ++d) cen[d] /= (double)n;
#define BLEND(dst, t) \
    for (int d = 0; d < n; ++d) (dst)[d] = cen[d] + (t) * (cen[d] - PT(worst)[d]);
        BLEND(xr, 1.0);
        double fr, fe, fc;
        if (!nm_eval(r, xr, &fr)) break;
        if (fr < fv[best]) {
            BLEND(xe, 2.0);
            if (!nm_eval(r, xe, &fe)) break;
            if (fe < fr) {
                memcpy(PT(worst), xe, sizeof(double) * n);
                fv[worst] = fe;
            } else {
                memcpy(PT(worst), xr, sizeof(double) * n);
                fv[worst] = fr;
            }
        } else if (fr < fv[second]) {
            memcpy(PT(worst), xr, sizeof(double) * n);
            fv[worst] = fr;
        } else {
            int outside = fr < fv[worst];
            BLEND(xc, outside ? 0.5 : -0.5);
            if (!nm_eval(r, xc, &fc)) break;
            if (fc < (outside ? fr : fv[worst])) {
                memcpy(PT(worst), xc, sizeof(double) * n);
                fv[worst] = fc;
            } else {
                int stop = 0;
                for (int i = 0; i <= n && !stop; ++i) {
                    if (i == best) continue;
                    for (int d = 0; d < n; ++d) PT(i)[d] = PT(best)[d] + 0.5 * (PT(i)[d] - PT(best)[d]);
                    if (!nm_eval(r, PT(i), &fv[i])) stop = 1;
                }
                if (stop) break;
            }
        }
#undef BLEND
    }
#undef PT
    free(pts);
    free(fv);
    free(order);
    free(cen);
    free(xr);
    free(xe);
    free(xc);
}

/* qaoa.hpp:85-117 optimize_parameters. params out: [gammas..., betas...]. */
static int optimize(const cost_t* c, int p, int budget, uint64_t seed, int threads, double tol,
                    double* params, double* expect, int* evals, double* trace_x, double* trace_f,
                    int* trace_len) {
    if (budget < 1) return set_err(1, "optimizer budget must be positive");
    if (p < 1) return set_err(1, "layer count must be positive");
    int n = 2 * p;
    objective_t obj = {c, p, threads, NULL, trace_x, trace_f, budget, 0};
    obj.state = (double*)malloc(sizeof(double) * 2 * ((size_t)1 << c->q));
    double* start = (double*)malloc(sizeof(double) * n);
    orc_linear_ramp(p, start, start + p);
    memcpy(params, start, sizeof(double) * n);
    double best_neg = objective(&obj, start);
    int used = 1;
    mt64 rng;
    mt64_seed(&rng, seed);
    nm_res r;
    r.x = (double*)malloc(sizeof(double) * n);
    while (used < budget) {
        nelder_mead(&obj, start, n, budget - used, tol, &r);
        used += r.evals;
        if (r.value < best_neg) {
            best_neg = r.value;
            memcpy(params, r.x, sizeof(double) * n);
        }
        if (!r.converged) break;
        for (int i = 0; i < n; ++i) start[i] = uniform_real(&rng, 0.0, PI_D);
    }
    *expect = -best_neg;
    *evals = used;
    if (trace_len) *trace_len = obj.trace_len;
    free(r.x);
    free(start);
    free(obj.state);
    return 0;
}

int orc_optimize(int n, int m, const orc_edge* e, int p, int budget, uint64_t seed, int threads,
                 double tol, double* params, double* expect, int* evals, double* trace_x,
                 double* trace_f, int* trace_len) {
    CHECK(validate_graph(n, m, e));
    cost_t c;
    CHECK(cost_build(n, m, e, g_qubit_cap, &c));
    int rc = optimize(&c, p, budget, seed, threads, tol, params, expect, evals, trace_x, trace_f,
                      trace_len);
    cost_free(&c);
    return rc;
}

/* ------------------------------------------------------------------------ */
/* qaoa.hpp:158-193 top_candidates                                           */
/* ------------------------------------------------------------------------ */
typedef struct {
    uint32_t bits;
    double prob;
} cand_t;

/* total order: probability descending, then lex_less_mask ascending (qaoa.hpp:179-182) */
static int cand_cmp(const void* pa, const void* pb) {
    const cand_t* a = (const cand_t*)pa;
    const cand_t* b = (const cand_t*)pb;
    if (a->prob != b->prob) return a->prob > b->prob ? -1 : 1;
    if (lex_less_mask(a->bits, b->bits)) return -1;
    if (lex_less_mask(b->bits, a->bits)) return 1;
    return 0;
}

static int top_candidates(int q, const double* amps, int top_k, int fold, uint32_t* bits,
                          double* probs) {
    if (q < 1) return set_err(1, "cannot rank candidates of an empty state");
    if (q > 32) return set_err(2, "candidate bits limited to 32 qubits");
    size_t classes = fold ? ((size_t)1 << (q - 1)) : ((size_t)1 << q);
    if (top_k < 1 || (size_t)top_k > classes)
        return set_err(1, "top_k must lie in [1, %zu] for %d qubits%s", classes, q,
                       fold ? " (folded)" : "");
    size_t size = (size_t)1 << q;
    cand_t* all = (cand_t*)malloc(sizeof(cand_t) * classes);
    if (fold) {
        uint32_t full = (uint32_t)(size - 1);
        size_t k = 0;
        for (size_t z = 0; z < size; z += 2) {
            const double* a = amps + 2 * z;
            const double* b = amps + 2 * (z ^ full);
            all[k].bits = (uint32_t)z;
            all[k].prob = (a[0] * a[0] + a[1] * a[1]) + (b[0] * b[0] + b[1] * b[1]);
            ++k;
        }
    } else {
        for (size_t z = 0; z < size; ++z) {
            const double* a = amps + 2 * z;
            all[z].bits = (uint32_t)z;
            all[z].prob = a[0] * a[0] + a[1] * a[1];
        }
    }
    qsort(all, classes, sizeof(cand_t), cand_cmp);
    for (int i = 0; i < top_k; ++i) {
        bits[i] = all[i].bits;
        probs[i] = all[i].prob;
    }
    free(all);
    return 0;
}

int orc_top_candidates(int q, const double* amps, int top_k, int fold, uint32_t* bits,
                       double* probs) {
    return top_candidates(q, amps, top_k, fold, bits, probs);
}

/* qaoa.hpp:198-216 solve_subgraph. */
int orc_solve_subgraph(int n, int m, const orc_edge* e, const orc_solve_options* o,
                       uint32_t* bits, double* probs, int* count, double* params, double* expect,
                       int* evals) {
    CHECK(validate_graph(n, m, e));
    if (n < 1) return set_err(1, "cannot solve an empty subgraph");
    if ((uint64_t)n > o->qubit_cap || n > g_qubit_cap)
        return set_err(2, "subgraph has %d vertices, over the qubit cap", n);
    cost_t c;
    CHECK(cost_build(n, m, e, g_qubit_cap, &c));
    int rc = optimize(&c, o->layers, o->budget, o->seed, o->threads, o->tolerance, params, expect,
                      evals, NULL, NULL, NULL);
    if (!rc) {
        double* s = (double*)malloc(sizeof(double) * 2 * ((size_t)1 << n));
        rc = ansatz(&c, o->layers, params, params + o->layers, o->threads, s);
        if (!rc) rc = top_candidates(n, s, o->top_k, o->fold, bits, probs);
        if (!rc) *count = o->top_k;
        free(s);
    }
    cost_free(&c);
    return rc;
}

/* ------------------------------------------------------------------------ */
/* merge.hpp                                                                 */
/* ------------------------------------------------------------------------ */
typedef struct {
    int M;
    const int* width;
    const int* count;
    const uint32_t** bits; /* per level */
} pool_t;

typedef struct {
    double value;
    uint8_t* asg;
    int has;
    uint64_t leaves;
} best_t;

typedef struct {
    int n, m;
    const orc_edge* e;
    const pool_t* pool;
    const partition_t* part;
    orc_edge** bucket; /* null => full-graph scoring */
    int* bucket_m;
    int stop, compare_end;
} walk_t;

/* merge.hpp:63-66 apply_candidate */
static inline void apply_cand(uint8_t* a, const partition_t* part, int level, uint32_t b) {
    for (int j = 0; j <= part->b[level] - part->a[level]; ++j)
        a[part->a[level] + j] = (uint8_t)((b >> j) & 1u);
}

/* merge.hpp:115-120 bucket_gain */
static inline double bucket_gain(const orc_edge* es, int m, const uint8_t* a) {
    double s = 0.0;
    for (int i = 0; i < m; ++i)
        if (a[es[i].u] != a[es[i].v]) s += es[i].w;
    return s;
}

/* merge.hpp:161-186 walk_levels */
static void walk(const walk_t* c, int level, double acc, uint8_t* a, best_t* out) {
    if (level == c->stop) {
        double value = c->bucket ? acc : cut_value(c->m, c->e, a);
        ++out->leaves;
        if (value > out->value ||
            (value == out->value && memcmp(a, out->asg, (size_t)c->compare_end) < 0)) {
            out->value = value;
            memcpy(out->asg, a, (size_t)c->n);
            out->has = 1;
        }
        return;
    }
    uint8_t need = a[c->part->a[level]];
    for (int k = 0; k < c->pool->count[level]; ++k) {
        uint32_t b = c->pool->bits[level][k];
        if ((b & 1u) != need) continue;
        apply_cand(a, c->part, level, b);
        double next = c->bucket ? acc + bucket_gain(c->bucket[level], c->bucket_m[level], a) : 0.0;
        walk(c, level + 1, next, a, out);
    }
}

/* merge.hpp:192-216 collect_prefixes */
static void collect(const pool_t* pool, int from, int depth, int need_first, uint32_t* cur,
                    int cur_len, uint32_t** out, size_t* out_len, size_t* out_cap) {
    if (cur_len == depth) {
        if (*out_len + (size_t)depth > *out_cap) {
            *out_cap = (*out_cap ? *out_cap * 2 : 64) + (size_t)depth;
            *out = (uint32_t*)realloc(*out, sizeof(uint32_t) * *out_cap);
        }
        memcpy(*out + *out_len, cur, sizeof(uint32_t) * (size_t)depth);
        *out_len += (size_t)depth;
        return;
    }
    int level = from + cur_len;
    int need = cur_len == 0 ? need_first
                            : (int)((cur[cur_len - 1] >> (pool->width[level - 1] - 1)) & 1u);
    for (int k = 0; k < pool->count[level]; ++k) {
        uint32_t b = pool->bits[level][k];
        uint32_t lead = b & 1u;
        if (need <= 1 && (int)lead != need) continue;
        if (need == 3 && lead != 0) continue;
        cur[cur_len] = b;
        collect(pool, from, depth, need_first, cur, cur_len + 1, out, out_len, out_cap);
    }
}

/* merge.hpp:223-270 sharded_search with one worker (the result is worker-invariant,
 * test_merge.cpp:187-213). */
static void search(const walk_t* c, const uint32_t* prefixes, size_t count, int depth, int from,
                   const uint8_t* base, double base_acc, best_t* best) {
    uint8_t* a = (uint8_t*)malloc((size_t)c->n + 1);
    memcpy(a, base, (size_t)c->n);
    for (size_t pi = 0; pi < count; ++pi) {
        double acc = base_acc;
        for (int d = 0; d < depth; ++d) {
            int level = from + d;
            apply_cand(a, c->part, level, prefixes[pi * (size_t)depth + (size_t)d]);
            if (c->bucket) acc += bucket_gain(c->bucket[level], c->bucket_m[level], a);
        }
        walk(c, from + depth, acc, a, best);
    }
    free(a);
}

/* merge.hpp:122-141 check_pool_matches */
static int check_pool(const pool_t* pool, int n, const partition_t* part) {
    if (part->M < 1) return set_err(1, "merge needs at least one subgraph");
    if (pool->M != part->M)
        return set_err(1, "pool has %d levels for %d subgraphs", pool->M, part->M);
    long long covered = 0;
    for (int i = 0; i < pool->M; ++i) {
        int piece = part->b[i] - part->a[i] + 1;
        if (pool->width[i] < 1 || pool->width[i] != piece)
            return set_err(1, "pool level %d width %d does not match subgraph size %d", i,
                           pool->width[i], piece);
        if (pool->count[i] == 0) return set_err(1, "pool level %d is empty", i);
        covered += piece;
    }
    if (covered != (long long)n + part->M - 1)
        return set_err(1, "subgraphs do not cover the graph as a chain");
    return 0;
}

/* merge.hpp:103-113 level_edge_buckets: edge -> max(first_level[u], first_level[v]). */
static void make_buckets(int n, int m, const orc_edge* e, const partition_t* part,
                         orc_edge*** bucket, int** bucket_m) {
    int M = part->M;
    int* fl = (int*)calloc((size_t)(n > 0 ? n : 1), sizeof(int));
    for (int i = M - 1; i >= 0; --i)
        for (int v = part->a[i]; v <= part->b[i]; ++v) fl[v] = i;
    int* cnt = (int*)calloc((size_t)M, sizeof(int));
    for (int k = 0; k < m; ++k) {
        int L = fl[e[k].u] > fl[e[k].v] ? fl[e[k].u] : fl[e[k].v];
        cnt[L]++;
    }
    orc_edge** bk = (orc_edge**)calloc((size_t)M, sizeof(orc_edge*));
    int* bm = (int*)calloc((size_t)M, sizeof(int));
    for (int i = 0; i < M; ++i) bk[i] = (orc_edge*)malloc(sizeof(orc_edge) * (size_t)(cnt[i] + 1));
    for (int k = 0; k < m; ++k) {
        int L = fl[e[k].u] > fl[e[k].v] ? fl[e[k].u] : fl[e[k].v];
        bk[L][bm[L]++] = e[k];
    }
    free(cnt);
    free(fl);
    *bucket = bk;
    *bucket_m = bm;
}

static void free_buckets(orc_edge** bk, int* bm, int M) {
    if (bk)
        for (int i = 0; i < M; ++i) free(bk[i]);
    free(bk);
    free(bm);
}

static void make_pool(pool_t* pool, int M, const int* widths, const int* counts,
                      const uint32_t* bits) {
    pool->M = M;
    pool->width = widths;
    pool->count = counts;
    pool->bits = (const uint32_t**)malloc(sizeof(uint32_t*) * (size_t)(M > 0 ? M : 1));
    size_t off = 0;
    for (int i = 0; i < M; ++i) {
        pool->bits[i] = bits + off;
        off += (size_t)counts[i];
    }
}

/* merge.hpp:71-78 estimate_paths */
static double estimate_paths(const pool_t* pool, int halve) {
    double est = (double)pool->count[0];
    if (halve) est /= 2.0;
    for (int i = 1; i < pool->M; ++i) est *= (double)pool->count[i] / 2.0;
    return est;
}

static int level_merge_impl(int n, int m, const orc_edge* e, const partition_t* part,
                            const pool_t* pool, int start_level, int workers, int incremental,
                            double path_budget, int halve, double* value, uint8_t* assignment,
                            uint64_t* leaves) {
    CHECK(check_pool(pool, n, part));
    int M = pool->M;
    if (start_level < 1 || start_level > M)
        return set_err(1, "start level must lie in [1, %d]", M);
    if (workers < 1) return set_err(1, "worker count must be positive");
    if (!(path_budget > 0)) return set_err(1, "path budget must be positive");
    double est = estimate_paths(pool, halve);
    if (est > path_budget)
        return set_err(2, "merge would enumerate about %g complete chains, over the %g budget", est,
                       path_budget);
    int depth = start_level;
    double prefix_est = (double)pool->count[0];
    if (halve) prefix_est /= 2.0;
    for (int i = 1; i < depth; ++i) prefix_est *= (double)pool->count[i] / 2.0;
    if (prefix_est > (double)((size_t)1 << 22))
        return set_err(2, "start level %d expands to about %g prefixes; lower it", start_level,
                       prefix_est);
    walk_t c = {n, m, e, pool, part, NULL, NULL, M, n};
    if (incremental) make_buckets(n, m, e, part, &c.bucket, &c.bucket_m);
    uint32_t* cur = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)depth);
    uint32_t* prefixes = NULL;
    size_t plen = 0, pcap = 0;
    collect(pool, 0, depth, halve ? 3 : 2, cur, 0, &prefixes, &plen, &pcap);
    uint8_t* base = (uint8_t*)calloc((size_t)n + 1, 1);
    best_t best = {-INFINITY, (uint8_t*)calloc((size_t)n + 1, 1), 0, 0};
    search(&c, prefixes, plen / (size_t)depth, depth, 0, base, 0.0, &best);
    int rc = 0;
    if (best.leaves == 0) {
        rc = set_err(1, "no compatible candidate chain exists");
    } else {
        *value = cut_value(m, e, best.asg);
        memcpy(assignment, best.asg, (size_t)n);
        *leaves = best.leaves;
    }
    free(best.asg);
    free(base);
    free(prefixes);
    free(cur);
    free_buckets(c.bucket, c.bucket_m, M);
    return rc;
}

int orc_level_merge(int n, int m, const orc_edge* e, int M, int mode, const int* widths,
                    const int* counts, const uint32_t* bits, int start_level, int workers,
                    int incremental, double path_budget, int halve, double* value,
                    uint8_t* assignment, uint64_t* leaves) {
    CHECK(validate_graph(n, m, e));
    partition_t part;
    CHECK(do_partition(n, m, e, M, mode, 0, &part));
    pool_t pool;
    make_pool(&pool, M, widths, counts, bits);
    int rc = level_merge_impl(n, m, e, &part, &pool, start_level, workers, incremental,
                              path_budget, halve, value, assignment, leaves);
    free(pool.bits);
    partition_free(&part);
    return rc;
}

/* merge.hpp:345-412 chained_merge */
static int chained_merge_impl(int n, int m, const orc_edge* e, const partition_t* part,
                              const pool_t* pool, long long window, long long window_leaves,
                              int workers, int halve, double* value, uint8_t* assignment,
                              uint64_t* leaves_out) {
    CHECK(check_pool(pool, n, part));
    int M = pool->M;
    if (workers < 1) return set_err(1, "worker count must be positive");
    if (window_leaves < 2) return set_err(1, "window leaf target must be at least 2");
    walk_t c = {n, m, e, pool, part, NULL, NULL, M, n};
    make_buckets(n, m, e, part, &c.bucket, &c.bucket_m);
    uint8_t* asg = (uint8_t*)calloc((size_t)n + 1, 1);
    double acc = 0.0;
    uint64_t total_leaves = 0;
    int rc = 0;
    int s = 0;
    while (s < M) {
        int e_ = s + 1;
        double lv = (double)pool->count[s];
        if (s == 0 && halve) lv /= 2.0;
        if (s > 0) lv /= 2.0;
        if (window > 0) {
            int cap = (int)(M < s + window ? M : s + window);
            for (; e_ < cap; ++e_) lv *= (double)pool->count[e_] / 2.0;
        } else {
            while (e_ < M) {
                double grown = lv * (double)pool->count[e_] / 2.0;
                if (grown > (double)window_leaves) break;
                lv = grown;
                ++e_;
            }
        }
        if (lv > 1e9) {
            rc = set_err(2, "merge window spans about %g combos; shrink the window", lv);
            break;
        }
        c.stop = e_;
        c.compare_end = part->b[e_ - 1] + 1;
        int need_first = s == 0 ? (halve ? 3 : 2) : asg[part->a[s]];
        uint32_t cur[1];
        uint32_t* prefixes = NULL;
        size_t plen = 0, pcap = 0;
        collect(pool, s, 1, need_first, cur, 0, &prefixes, &plen, &pcap);
        best_t best = {-INFINITY, (uint8_t*)calloc((size_t)n + 1, 1), 0, 0};
        search(&c, prefixes, plen, 1, s, asg, acc, &best);
        free(prefixes);
        if (best.leaves == 0) {
            free(best.asg);
            rc = set_err(1, "no compatible candidate chain exists");
            break;
        }
        memcpy(asg, best.asg, (size_t)n);
        free(best.asg);
        acc = best.value;
        total_leaves += best.leaves;
        s = e_;
    }
    if (!rc) {
        *value = cut_value(m, e, asg);
        memcpy(assignment, asg, (size_t)n);
        *leaves_out = total_leaves;
    }
    free(asg);
    free_buckets(c.bucket, c.bucket_m, M);
    return rc;
}

int orc_chained_merge(int n, int m, const orc_edge* e, int M, int mode, const int* widths,
                      const int* counts, const uint32_t* bits, long long window,
                      long long window_leaves, int workers, int halve, double* value,
                      uint8_t* assignment, uint64_t* leaves) {
    CHECK(validate_graph(n, m, e));
    partition_t part;
    CHECK(do_partition(n, m, e, M, mode, 0, &part));
    pool_t pool;
    make_pool(&pool, M, widths, counts, bits);
    int rc = chained_merge_impl(n, m, e, &part, &pool, window, window_leaves, workers, halve,
                                value, assignment, leaves);
    free(pool.bits);
    partition_free(&part);
    return rc;
}

/* ------------------------------------------------------------------------ */
/* pipeline.hpp:135-336 (partition -> QAOA stage -> merge; baseline omitted)  */
/* ------------------------------------------------------------------------ */
int orc_run_pipeline(int n, int m, const orc_edge* e, const orc_run_config* c,
                     orc_run_result* out, char* assignment, double* sub_expect, int* sub_evals,
                     int M_cap) {
    CHECK(validate_graph(n, m, e));
    if (c->layers < 1) return set_err(1, "layer count must be positive");
    if (c->budget < 1) return set_err(1, "optimizer budget must be positive");
    if (c->top_k < 0) return set_err(1, "top_k cannot be negative");
    if (c->start_level < 1) return set_err(1, "start level must be positive");
    if (c->qubit_cap < 2 || c->qubit_cap > g_qubit_cap)
        return set_err(1, "qubit cap must lie in [2, %d]", g_qubit_cap);
    if (!(c->path_budget > 0)) return set_err(1, "path budget must be positive");
    if (c->solvers < 0) return set_err(1, "solver slot count cannot be negative");
    if (c->subgraphs < 0) return set_err(1, "subgraph count cannot be negative");
    int workers = c->workers > 0 ? c->workers : 1;
    memset(out, 0, sizeof *out);

    double t0 = now_s();
    int M = c->subgraphs;
    if (M == 0) CHECK(orc_derive_subgraph_count(n, c->qubit_cap, &M));
    partition_t part;
    CHECK(do_partition(n, m, e, M, c->partition_mode, c->qubit_cap, &part));
    out->partition_s = now_s() - t0;
    out->subgraphs = M;

    /* QAOA stage: subgraph i solves with seed + i (pipeline.hpp:258), top_k clamp (:251-255) */
    t0 = now_s();
    int* widths = (int*)malloc(sizeof(int) * (size_t)M);
    int* kept = (int*)calloc((size_t)M, sizeof(int));
    uint32_t** cbits = (uint32_t**)calloc((size_t)M, sizeof(uint32_t*));
    int rc = 0;
#pragma omp parallel for schedule(dynamic, 1) num_threads(workers) if (workers > 1)
    for (int i = 0; i < M; ++i) {
        int w = part.b[i] - part.a[i] + 1;
        widths[i] = w;
        size_t classes = c->fold ? ((size_t)1 << (w - 1)) : ((size_t)1 << w);
        orc_solve_options so;
        so.top_k = c->top_k == 0 ? (int)classes
                                 : (int)((size_t)c->top_k < classes ? (size_t)c->top_k : classes);
        so.layers = c->layers;
        so.budget = c->budget;
        so.seed = c->seed + (uint64_t)i;
        so.fold = c->fold;
        so.threads = 1;
        so.qubit_cap = (uint64_t)c->qubit_cap;
        so.tolerance = c->nm_tolerance;
        uint32_t* bits = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)so.top_k);
        double* probs = (double*)malloc(sizeof(double) * (size_t)so.top_k);
        double* params = (double*)malloc(sizeof(double) * 2 * (size_t)c->layers);
        double ex = 0;
        int ev = 0, cnt = 0;
        int r = orc_solve_subgraph(w, part.local_m[i], part.local[i], &so, bits, probs, &cnt,
                                   params, &ex, &ev);
        if (r) {
#pragma omp critical
            rc = r;
        } else {
            if (i < M_cap) {
                sub_expect[i] = ex;
                sub_evals[i] = ev;
            }
            /* merge.hpp:31-51 build_candidate_pools: (b, ~b) per entry, first occurrence kept */
            uint32_t full = w == 32 ? ~0u : ((1u << w) - 1u);
            cbits[i] = (uint32_t*)malloc(sizeof(uint32_t) * 2 * (size_t)cnt);
            int k = 0;
            for (int j = 0; j < cnt; ++j) {
                uint32_t cand[2] = {bits[j], bits[j] ^ full};
                for (int t = 0; t < 2; ++t) {
                    int dup = 0;
                    for (int s2 = 0; s2 < k; ++s2)
                        if (cbits[i][s2] == cand[t]) dup = 1;
                    if (!dup) cbits[i][k++] = cand[t];
                }
            }
            kept[i] = k;
        }
        free(bits);
        free(probs);
        free(params);
    }
    out->qaoa_s = now_s() - t0;

    if (!rc) {
        t0 = now_s();
        size_t tot = 0;
        for (int i = 0; i < M; ++i) tot += (size_t)kept[i];
        uint32_t* flat = (uint32_t*)malloc(sizeof(uint32_t) * (tot ? tot : 1));
        size_t off = 0;
        for (int i = 0; i < M; ++i) {
            memcpy(flat + off, cbits[i], sizeof(uint32_t) * (size_t)kept[i]);
            off += (size_t)kept[i];
        }
        pool_t pool;
        make_pool(&pool, M, widths, kept, flat);
        int mode = c->merge_mode;
        if (mode == 0) mode = estimate_paths(&pool, c->halve_symmetry) <= c->path_budget ? 1 : 2;
        uint8_t* asg = (uint8_t*)calloc((size_t)n + 1, 1);
        double val = 0;
        uint64_t leaves = 0;
        if (mode == 1)
            rc = level_merge_impl(n, m, e, &part, &pool, c->start_level < M ? c->start_level : M,
                                  workers, c->merge_incremental, c->path_budget,
                                  c->halve_symmetry, &val, asg, &leaves);
        else
            rc = chained_merge_impl(n, m, e, &part, &pool, 0, 1 << 16, workers, 1, &val, asg,
                                    &leaves);
        out->windowed = mode == 2;
        out->cut = val;
        out->leaves = leaves;
        for (int v = 0; v < n; ++v) assignment[v] = asg[v] ? '1' : '0';
        assignment[n] = 0;
        free(asg);
        free(pool.bits);
        free(flat);
        out->merge_s = now_s() - t0;
    }
    out->total_s = out->partition_s + out->qaoa_s + out->merge_s;
    for (int i = 0; i < M; ++i) free(cbits[i]);
    free(cbits);
    free(kept);
    free(widths);
    partition_free(&part);
    return rc;
}
