// Host-only ask/tell optimisers of the C-ABI (qc_simplex_*, qc_optimizer_*): the same
// state machines the engine steps in lockstep (qc_nm.hpp), for external objectives.
#include <cstring>
#include <string>

#include "../../include/qcgpu.h"
#include "qc_engine.hpp"
#include "qc_nm.hpp"

struct qc_simplex {
    qcg::NelderMead nm;
    int n = 0;
};
struct qc_optimizer {
    qcg::AngleOptimizer opt;
    int p = 0;
};

namespace {
template <typename F>
int guarded(F&& f) {
    try {
        f();
        return QC_OK;
    } catch (const qcg::Error& e) {
        qcg::set_error(e.what());
        return e.code;
    } catch (const std::exception& e) {
        qcg::set_error(e.what());
        return QC_ERR_INTERNAL;
    }
}
}  // namespace

extern "C" {

int qc_simplex_create(const double* x0, int n, int max_evals, double tolerance,
                      qc_simplex** out) {
    return guarded([&] {
        if (n <= 0) qcg::config_error("optimizer needs at least one dimension");  // :33
        if (max_evals < 1) qcg::config_error("optimizer budget must be positive"); // :34
        auto* s = new qc_simplex();
        s->n = n;
        s->nm.start(std::vector<double>(x0, x0 + n), max_evals, tolerance);
        *out = s;
    });
}

int qc_simplex_ask(qc_simplex* s, double* x, int* done) {
    return guarded([&] {
        if (!s) qcg::config_error("null simplex");
        *done = s->nm.done() ? 1 : 0;
        if (!*done) std::memcpy(x, s->nm.point().data(), sizeof(double) * static_cast<size_t>(s->n));
    });
}

int qc_simplex_tell(qc_simplex* s, double f) {
    return guarded([&] {
        if (!s || s->nm.done()) qcg::config_error("simplex is not waiting for a value");
        s->nm.tell(f);
    });
}

int qc_simplex_result(const qc_simplex* s, double* x, double* value, int* evals, int* converged) {
    return guarded([&] {
        if (!s) qcg::config_error("null simplex");
        if (x && !s->nm.best_x.empty())
            std::memcpy(x, s->nm.best_x.data(), sizeof(double) * static_cast<size_t>(s->n));
        if (value) *value = s->nm.best_f;
        if (evals) *evals = s->nm.evals;
        if (converged) *converged = s->nm.converged ? 1 : 0;
    });
}

void qc_simplex_destroy(qc_simplex* s) { delete s; }

int qc_optimizer_create(int p, int budget, uint64_t seed, double tolerance, qc_optimizer** out) {
    return guarded([&] {
        if (budget < 1) qcg::config_error("optimizer budget must be positive");  // qaoa.hpp:88
        if (p < 1) qcg::config_error("layer count must be positive");           // qaoa.hpp:28
        auto* o = new qc_optimizer();
        o->p = p;
        o->opt.start(p, budget, seed, tolerance);
        *out = o;
    });
}

int qc_optimizer_ask(qc_optimizer* o, double* x, int* done) {
    return guarded([&] {
        if (!o) qcg::config_error("null optimizer");
        *done = o->opt.done() ? 1 : 0;
        if (!*done) std::memcpy(x, o->opt.point().data(), sizeof(double) * 2 * static_cast<size_t>(o->p));
    });
}

int qc_optimizer_tell(qc_optimizer* o, double f) {
    return guarded([&] {
        if (!o || o->opt.done()) qcg::config_error("optimizer is not waiting for a value");
        o->opt.tell(f);
    });
}

int qc_optimizer_result(const qc_optimizer* o, double* params, double* expectation, int* evals) {
    return guarded([&] {
        if (!o) qcg::config_error("null optimizer");
        if (params) std::memcpy(params, o->opt.params.data(), sizeof(double) * 2 * static_cast<size_t>(o->p));
        if (expectation) *expectation = o->opt.expectation();
        if (evals) *evals = o->opt.evals;
    });
}

void qc_optimizer_destroy(qc_optimizer* o) { delete o; }

}  // extern "C"
