// Scalar coordinate rules shared by the host C-ABI and the device CCD loop.
// Restates proj/src/optimizer.cpp:32-78 (newton_step, apply_trust_region,
// l1_coordinate_update); the constants are proj/include/stratcox/optimizer.hpp:47
// and likelihood.hpp:21. Compiled for host and device from one source so the
// on-device coordinate update is the same code the host API exposes.
#pragma once

#include <cmath>
#include <cstdint>

namespace scx {

constexpr double kLinearPredictorBound = 700.0;  // likelihood.hpp:21
constexpr double kFlatCurvature = 1e-12;         // optimizer.hpp:47
constexpr uint32_t kRefreshEvery = 256;          // likelihood.cpp:82
constexpr int kMaxHalvings = 10;                 // optimizer.cpp:115
constexpr double kMonotoneSlack = 1e-8;          // optimizer.cpp:131

// Rule failures map onto the reference exception taxonomy.
enum RuleCode : int {
    kRuleOk = 0,
    kRuleNonFiniteNewton = 1,  // numeric_error("non-finite gradient or Hessian in Newton step")
    kRuleNonFiniteTrust = 2,   // numeric_error("non-finite trust-region inputs")
    kRuleBothNegative = 3,     // internal_error("both directional derivatives negative at the origin")
};

// std::max / std::min argument conventions (first argument wins ties/NaN).
__host__ __device__ inline double dmax(double a, double b) { return a < b ? b : a; }
__host__ __device__ inline double dmin(double a, double b) { return b < a ? b : a; }

// optimizer.cpp:32-41
__host__ __device__ inline int newton_step(double g1, double g2, double* step, int* flat) {
    if (!isfinite(g1) || !isfinite(g2)) return kRuleNonFiniteNewton;
    *flat = 0;
    if (g2 < kFlatCurvature) {
        *flat = 1;
        *step = 0.0;
        return kRuleOk;
    }
    *step = -g1 / g2;
    return kRuleOk;
}

// optimizer.cpp:43-49
__host__ __device__ inline int apply_trust_region(double proposed, double trust, double* applied,
                                                  double* next_trust) {
    if (!isfinite(proposed) || !isfinite(trust)) return kRuleNonFiniteTrust;
    const double magnitude = dmin(fabs(proposed), trust);
    const double a = copysign(magnitude, proposed);
    *applied = a;
    *next_trust = dmax(2.0 * fabs(a), trust * 0.5);
    return kRuleOk;
}

// optimizer.cpp:51-78: penalised Newton proposal with the directional-
// derivative rule at the origin and zero-crossing truncation.
__host__ __device__ inline int l1_coordinate_update(double g1, double g2, double beta_j,
                                                    double gamma_j, double* step, int* skipped,
                                                    int* flat) {
    *step = 0.0;
    *skipped = 0;
    *flat = 0;
    if (gamma_j == 0.0) return newton_step(g1, g2, step, flat);
    if (beta_j != 0.0) {
        const double penalized = g1 + (beta_j > 0.0 ? gamma_j : -gamma_j);
        const int rc = newton_step(penalized, g2, step, flat);
        if (rc) return rc;
        if ((beta_j > 0.0 && beta_j + *step < 0.0) || (beta_j < 0.0 && beta_j + *step > 0.0))
            *step = -beta_j;
        return kRuleOk;
    }
    const double up = g1 + gamma_j;
    const double down = -g1 + gamma_j;
    if (up < 0.0 && down < 0.0) return kRuleBothNegative;
    if (up >= 0.0 && down >= 0.0) {
        *skipped = 1;
        return kRuleOk;
    }
    const double penalized = up < 0.0 ? g1 + gamma_j : g1 - gamma_j;
    return newton_step(penalized, g2, step, flat);
}

// Elastic-net rule (extension; not in the reference — BASELINE config 1's
// "L2 prior"): the ridge term l2_j beta_j^2 / 2 adds l2_j beta_j to g' and l2_j
// to g'', then the reference's L1 rule runs on the penalised pair. With
// l2_j = 0 this is l1_coordinate_update bit for bit (g1 + 0*beta == g1).
__host__ __device__ inline int coordinate_update(double g1, double g2, double beta_j,
                                                 double gamma_j, double l2_j, double* step,
                                                 int* skipped, int* flat) {
#ifdef __CUDA_ARCH__
    const double pg = __dadd_rn(g1, __dmul_rn(l2_j, beta_j));  // no FMA: the host's rounding
#else
    const double pg = g1 + l2_j * beta_j;
#endif
    return l1_coordinate_update(pg, g2 + l2_j, beta_j, gamma_j, step, skipped, flat);
}

}  // namespace scx
