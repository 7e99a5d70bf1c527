// Nelder-Mead (nelder_mead.hpp:29-120) and the QAOA angle optimiser
// (qaoa.hpp:85-117) restated as ask/tell state machines, so that one host thread can
// step every subgraph of a batch in lockstep and hand the device one batched launch
// per step. Each machine issues exactly the sequence of objective calls the
// reference's recursive code issues (same points, same order, same budget
// accounting, same best-point tie rule), so the optimisation trajectory is
// reproduced bit for bit. Compiled with -ffp-contract=off.
#pragma once

#include <algorithm>
#include <cstddef>
#include <numbers>
#include <numeric>
#include <random>
#include <vector>

namespace qcg {

class NelderMead {
public:
    // nelder_mead.hpp:30 nelder_mead_minimize(f, x0, {max_evals, tolerance, 0.2})
    void start(const std::vector<double>& x0, int max_evals, double tol) {
        n_ = x0.size();
        max_evals_ = max_evals;
        tol_ = tol;
        evals = 0;
        converged = false;
        has_best = false;
        best_x.clear();
        best_f = 0.0;
        pts_.assign(n_ + 1, x0);
        fv_.assign(n_ + 1, 0.0);
        i_ = 0;
        state_ = kInit;
        request(pts_[0]);
    }

    bool done() const { return state_ == kDone; }
    const std::vector<double>& point() const { return pending_; }

    void tell(double f) {
        // nelder_mead.hpp:36-46 eval(): count, then best-point tracking
        ++evals;
        if (!has_best || f < best_f || (f == best_f && pending_ < best_x)) {
            best_f = f;
            best_x = pending_;
            has_best = true;
        }
        switch (state_) {
            case kInit:  // :48-54
                fv_[i_] = f;
                ++i_;
                if (i_ <= n_) {
                    pts_[i_][i_ - 1] += kStep;
                    request(pts_[i_]);
                } else {
                    order_and_reflect();
                }
                break;
            case kReflect:  // :83-100
                fr_ = f;
                if (fr_ < fv_[best_]) {
                    blend(2.0, xe_);
                    state_ = kExpand;
                    request(xe_);
                } else if (fr_ < fv_[second_]) {
                    pts_[worst_] = xr_;
                    fv_[worst_] = fr_;
                    order_and_reflect();
                } else {
                    outside_ = fr_ < fv_[worst_];
                    blend(outside_ ? 0.5 : -0.5, xc_);
                    state_ = kContract;
                    request(xc_);
                }
                break;
            case kExpand:  // :88-97
                if (f < fr_) {
                    pts_[worst_] = xe_;
                    fv_[worst_] = f;
                } else {
                    pts_[worst_] = xr_;
                    fv_[worst_] = fr_;
                }
                order_and_reflect();
                break;
            case kContract:  // :101-108
                if (f < (outside_ ? fr_ : fv_[worst_])) {
                    pts_[worst_] = xc_;
                    fv_[worst_] = f;
                    order_and_reflect();
                } else {
                    i_ = 0;
                    shrink_next();
                }
                break;
            case kShrink:  // :110-116
                fv_[i_] = f;
                ++i_;
                shrink_next();
                break;
            case kDone:
                break;
        }
    }

    // NelderMeadResult
    std::vector<double> best_x;
    double best_f = 0.0;
    int evals = 0;
    bool converged = false;
    bool has_best = false;

private:
    static constexpr double kStep = 0.2;  // NelderMeadOptions::initial_step
    enum State { kInit, kReflect, kExpand, kContract, kShrink, kDone };

    bool request(const std::vector<double>& x) {
        if (evals >= max_evals_) {  // :37 budget exhausted
            state_ = kDone;
            return false;
        }
        pending_ = x;
        return true;
    }

    void blend(double t, std::vector<double>& out) const {  // :72-79
        out.resize(n_);
        for (std::size_t d = 0; d < n_; ++d)
            out[d] = centroid_[d] + t * (centroid_[d] - pts_[worst_][d]);
    }

    void order_and_reflect() {  // :57-85
        order_.resize(n_ + 1);
        std::iota(order_.begin(), order_.end(), std::size_t{0});
        std::stable_sort(order_.begin(), order_.end(),
                         [&](std::size_t a, std::size_t b) { return fv_[a] < fv_[b]; });
        best_ = order_[0];
        worst_ = order_[n_];
        second_ = order_[n_ - 1];
        if (fv_[worst_] - fv_[best_] <= tol_) {
            converged = true;
            state_ = kDone;
            return;
        }
        centroid_.assign(n_, 0.0);
        for (std::size_t i = 0; i <= n_; ++i)
            if (i != worst_)
                for (std::size_t d = 0; d < n_; ++d) centroid_[d] += pts_[i][d];
        for (double& c : centroid_) c /= static_cast<double>(n_);
        blend(1.0, xr_);
        state_ = kReflect;
        request(xr_);
    }

    void shrink_next() {  // :110-116
        while (i_ <= n_ && i_ == best_) ++i_;
        if (i_ > n_) {
            order_and_reflect();
            return;
        }
        for (std::size_t d = 0; d < n_; ++d)
            pts_[i_][d] = pts_[best_][d] + 0.5 * (pts_[i_][d] - pts_[best_][d]);
        state_ = kShrink;
        request(pts_[i_]);
    }

    std::size_t n_ = 0;
    int max_evals_ = 0;
    double tol_ = 0.0;
    State state_ = kDone;
    std::vector<std::vector<double>> pts_;
    std::vector<double> fv_;
    std::vector<std::size_t> order_;
    std::size_t i_ = 0, best_ = 0, worst_ = 0, second_ = 0;
    std::vector<double> centroid_, xr_, xe_, xc_, pending_;
    double fr_ = 0.0;
    bool outside_ = false;
};

// qaoa.hpp:27-38 linear_ramp, packed [gammas..., betas...]
inline std::vector<double> linear_ramp_packed(int p) {
    std::vector<double> x(2 * static_cast<std::size_t>(p));
    for (int l = 1; l <= p; ++l) {
        const double frac = static_cast<double>(l) / static_cast<double>(p);
        x[static_cast<std::size_t>(l - 1)] = frac * std::numbers::pi / 2.0;
        x[static_cast<std::size_t>(p + l - 1)] = (1.0 - frac) * std::numbers::pi / 2.0;
    }
    return x;
}

// qaoa.hpp:85-117 optimize_parameters as ask/tell.
class AngleOptimizer {
public:
    void start(int p, int budget, std::uint64_t seed, double tol) {
        p_ = p;
        budget_ = budget;
        tol_ = tol;
        rng_.seed(seed);
        params = linear_ramp_packed(p);
        start_ = params;
        evals = 0;
        state_ = kRamp;
    }
    bool done() const { return state_ == kDone; }
    const std::vector<double>& point() const { return state_ == kRamp ? start_ : nm_.point(); }

    void tell(double f) {
        if (state_ == kRamp) {  // :94-96
            best_neg_ = f;
            evals = 1;
            next_run();
            return;
        }
        nm_.tell(f);
        if (!nm_.done()) return;
        evals += nm_.evals;  // :106
        if (nm_.best_f < best_neg_) {  // :107-110
            best_neg_ = nm_.best_f;
            params = nm_.best_x;
        }
        if (!nm_.converged) {  // :111
            state_ = kDone;
            return;
        }
        std::uniform_real_distribution<double> angle(0.0, std::numbers::pi);
        start_.assign(2 * static_cast<std::size_t>(p_), 0.0);  // :112-113
        for (double& v : start_) v = angle(rng_);
        next_run();
    }

    double expectation() const { return -best_neg_; }

    std::vector<double> params;
    int evals = 0;

private:
    enum State { kRamp, kNm, kDone };
    void next_run() {  // :101-105 while (evals < budget) { nelder_mead_minimize(...) }
        if (evals < budget_) {
            nm_.start(start_, budget_ - evals, tol_);
            state_ = nm_.done() ? kDone : kNm;
        } else {
            state_ = kDone;
        }
    }

    int p_ = 1, budget_ = 0;
    double tol_ = 1e-5;
    std::mt19937_64 rng_;
    std::vector<double> start_;
    double best_neg_ = 0.0;
    NelderMead nm_;
    State state_ = kDone;
};

}  // namespace qcg
