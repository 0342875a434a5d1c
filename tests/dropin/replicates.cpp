// TEST INFRASTRUCTURE ONLY — a bootstrap-style caller of the reference C++ API.
//
// Like bootstrap_intervals (proj/src/resample.cpp:207-230), every replicate
// builds a STACK-LOCAL SortedDesign (`const SortedDesign design = ...` inside
// the loop, so the object sits at the same address each time) of the SAME
// shape (n, p, nnz: the covariate columns are shared, only the observed times
// are reshuffled) and fits it. Linked twice by oracle/Makefile: against the
// unmodified reference (replicates_ref) and against the CUDA drop-in
// (replicates_b200); tests/test_dropin.py compares the two outputs. A design
// cache keyed on object identity would fit the first replicate's data every
// time and fail the comparison.
//
// Output: one line per replicate: "r cycles converged beta_0 ... beta_{p-1}".
#include <algorithm>
#include <cstdio>
#include <random>

#include "stratcox/data.hpp"
#include "stratcox/optimizer.hpp"
#include "stratcox/simulate.hpp"

using namespace stratcox;

int main() {
    SimulateConfig cfg;
    cfg.n = 3000;
    cfg.p = 8;
    cfg.density = 0.2;
    cfg.strata = 5;
    cfg.seed = 42;
    const Simulated base = simulate(cfg);
    for (int r = 0; r < 6; ++r) {
        SurvivalDataset d = base.data;
        std::mt19937_64 rng(1000 + r);
        std::shuffle(d.time.begin(), d.time.end(), rng);
        const SortedDesign design = build_sorted_design(d);
        const FitResult fit = ccd_fit(design, PenaltySpec::shared(cfg.p, 0.0), OptimizerConfig{});
        std::printf("%d %d %d", r, fit.cycles_used, fit.converged ? 1 : 0);
        for (const double b : fit.beta) std::printf(" %.17g", b);
        std::printf("\n");
    }
    return 0;
}
