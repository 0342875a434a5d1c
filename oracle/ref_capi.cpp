// TEST INFRASTRUCTURE ONLY — never linked into the product path.
//
// A thin extern "C" face over the UNMODIFIED reference library ("stratcox",
// /root/reference/proj/src/*.cpp, compiled in place by oracle/Makefile into
// oracle/_ref/libstratcox_ref.so). It exists so that Python tests, the golden
// fixture generator (tests/golden/make_golden.py) and bench.py's CPU-baseline
// leg can drive the reference's own public C++ API:
//   simulate            proj/src/simulate.cpp:9-102
//   random_dataset      proj/tests/oracles.hpp:58-85
//   build_sorted_design proj/src/data.cpp:68-147
//   make_state / gradient_hessian / log_partial_likelihood / naive_*
//                       proj/src/likelihood.cpp:19-244
//   segmented_inclusive_scan  proj/src/scan.cpp:124-190
//   ccd_fit             proj/src/optimizer.cpp:82-160
//   gamma_max / default_gamma_grid  proj/src/resample.cpp:42-68
//   run_iteration timing semantics  proj/src/benchmark.cpp:27-41,71-105
// Handles are opaque heap objects; every call returns 0 on success and a
// non-zero code (1 validation, 2 numeric, 3 internal, 9 other) with the
// exception text retrievable from ref_last_error().

#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <random>
#include <string>
#include <vector>

#include "oracles.hpp"  // proj/tests/oracles.hpp (header-only test oracle)
#include "stratcox/likelihood.hpp"
#include "stratcox/optimizer.hpp"
#include "stratcox/resample.hpp"
#include "stratcox/transforms.hpp"
#include "stratcox/io.hpp"
#include <sstream>
#include "stratcox/scan.hpp"
#include "stratcox/simulate.hpp"

#ifdef _OPENMP
#include <omp.h>
#endif

using namespace stratcox;

namespace {

thread_local std::string g_last_error;

template <class F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const validation_error& e) {
        g_last_error = e.what();
        return 1;
    } catch (const numeric_error& e) {
        g_last_error = e.what();
        return 2;
    } catch (const internal_error& e) {
        g_last_error = e.what();
        return 3;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return 9;
    }
}

struct Dataset {
    SurvivalDataset data;
    std::vector<double> true_beta;
};

void copy_dataset(const SurvivalDataset& d, double* time, uint8_t* event, int32_t* stratum,
                  int64_t* col_ptr, int64_t* row_idx, double* values) {
    const std::size_t n = d.n_rows();
    if (time) std::memcpy(time, d.time.data(), n * sizeof(double));
    if (event) std::memcpy(event, d.event.data(), n);
    if (stratum) std::memcpy(stratum, d.stratum.data(), n * sizeof(int32_t));
    int64_t off = 0;
    if (col_ptr) col_ptr[0] = 0;
    for (std::size_t j = 0; j < d.n_covariates(); ++j) {
        const SparseColumn& c = d.columns[j];
        if (row_idx) std::memcpy(row_idx + off, c.rows.data(), c.nnz() * sizeof(int64_t));
        if (values) std::memcpy(values + off, c.values.data(), c.nnz() * sizeof(double));
        off += static_cast<int64_t>(c.nnz());
        if (col_ptr) col_ptr[j + 1] = off;
    }
}

SurvivalDataset make_dataset(int64_t n, const double* time, const uint8_t* event,
                             const int32_t* stratum, int64_t p, const int64_t* col_ptr,
                             const int64_t* row_idx, const double* values) {
    SurvivalDataset d;
    d.time.assign(time, time + n);
    d.event.assign(event, event + n);
    d.stratum.assign(stratum, stratum + n);
    d.subject.resize(static_cast<std::size_t>(n));
    for (int64_t i = 0; i < n; ++i) d.subject[static_cast<std::size_t>(i)] = i + 1;
    d.columns.resize(static_cast<std::size_t>(p));
    for (int64_t j = 0; j < p; ++j) {
        for (int64_t t = col_ptr[j]; t < col_ptr[j + 1]; ++t)
            d.columns[static_cast<std::size_t>(j)].push(row_idx[t], values ? values[t] : 1.0);
    }
    return d;
}

ExecutionConfig exec_of(int64_t chunk, int workers) {
    ExecutionConfig c;
    if (chunk > 0) c.chunk_size = static_cast<std::size_t>(chunk);
    if (workers > 0) c.worker_count = workers;
    return c;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_last_error.c_str(); }

int ref_max_threads() { return default_worker_count(); }

// ---------------------------------------------------------------- datasets
int ref_simulate(int64_t n, int64_t p, double density, double beta_sparsity, int32_t strata,
                 double censoring, uint64_t seed, void** out) {
    return guard([&] {
        SimulateConfig c;
        c.n = static_cast<std::size_t>(n);
        c.p = static_cast<std::size_t>(p);
        c.density = density;
        c.beta_sparsity = beta_sparsity;
        c.strata = strata;
        c.censoring = censoring;
        c.seed = seed;
        Simulated s = simulate(c);
        auto* h = new Dataset{std::move(s.data), std::move(s.true_beta)};
        *out = h;
    });
}

int ref_random_dataset(uint64_t seed, int64_t n, int32_t strata, int64_t p, double density,
                       double time_grid, void** out) {
    return guard([&] {
        std::mt19937_64 rng(seed);
        auto* h = new Dataset{oracles::random_dataset(rng, static_cast<std::size_t>(n), strata,
                                                      static_cast<std::size_t>(p), density,
                                                      time_grid),
                              {}};
        *out = h;
    });
}

int ref_dataset_from_arrays(int64_t n, const double* time, const uint8_t* event,
                            const int32_t* stratum, int64_t p, const int64_t* col_ptr,
                            const int64_t* row_idx, const double* values, void** out) {
    return guard([&] {
        auto* h = new Dataset{make_dataset(n, time, event, stratum, p, col_ptr, row_idx, values), {}};
        *out = h;
    });
}

void ref_dataset_sizes(void* h, int64_t* n, int64_t* p, int64_t* nnz) {
    const auto& d = static_cast<Dataset*>(h)->data;
    *n = static_cast<int64_t>(d.n_rows());
    *p = static_cast<int64_t>(d.n_covariates());
    int64_t z = 0;
    for (const auto& c : d.columns) z += static_cast<int64_t>(c.nnz());
    *nnz = z;
}

void ref_dataset_copy(void* h, double* time, uint8_t* event, int32_t* stratum, int64_t* col_ptr,
                      int64_t* row_idx, double* values, double* true_beta) {
    const auto* ds = static_cast<Dataset*>(h);
    copy_dataset(ds->data, time, event, stratum, col_ptr, row_idx, values);
    if (true_beta && !ds->true_beta.empty())
        std::memcpy(true_beta, ds->true_beta.data(), ds->true_beta.size() * sizeof(double));
}

void ref_dataset_free(void* h) { delete static_cast<Dataset*>(h); }

void ref_dataset_subject(void* h, int64_t* out) {
    const auto& d = static_cast<Dataset*>(h)->data;
    std::memcpy(out, d.subject.data(), d.subject.size() * sizeof(int64_t));
}

void ref_dataset_set_subject(void* h, const int64_t* subject) {
    auto& d = static_cast<Dataset*>(h)->data;
    d.subject.assign(subject, subject + d.n_rows());
}

// ---------------------------------------------------------------- lowering
// make_time_varying (time-fixed columns of the subject dataset h) + lower_pipeline.
int ref_lower_pipeline(void* h, const double* cuts, int64_t n_cuts, const int64_t* split_cov,
                       const int64_t* split_ptr, const double* split_times, int64_t n_splits,
                       void** out, int64_t* map_source, int32_t* map_window) {
    return guard([&] {
        const auto& d = static_cast<Dataset*>(h)->data;
        std::vector<std::string> names;
        TimeVaryingDataset tv = make_time_varying(d.time, d.event, d.subject, d.columns, names,
                                                  std::vector<double>(cuts, cuts + n_cuts));
        TimeVaryingSpec spec;
        spec.cut_points.assign(cuts, cuts + n_cuts);
        for (int64_t s = 0; s < n_splits; ++s) {
            TimeVaryingSpec::Split sp;
            sp.covariate = static_cast<std::size_t>(split_cov[s]);
            sp.times.assign(split_times + split_ptr[s], split_times + split_ptr[s + 1]);
            spec.splits.push_back(sp);
        }
        LoweredDataset low = lower_pipeline(tv, spec);
        for (std::size_t c = 0; c < low.column_map.size(); ++c) {
            map_source[c] = static_cast<int64_t>(low.column_map[c].source);
            map_window[c] = low.column_map[c].window;
        }
        *out = new Dataset{std::move(low.data), {}};
    });
}

// ---------------------------------------------------------------- resample
int ref_fold_assignment(void* h, int folds, uint64_t seed, int32_t* out) {
    return guard([&] {
        const auto f = fold_assignment(static_cast<Dataset*>(h)->data, folds, seed);
        for (std::size_t i = 0; i < f.size(); ++i) out[i] = f[i];
    });
}

int ref_kfold_select_gamma(void* h, const double* tmpl, int folds, const double* grid, int64_t ng,
                           uint64_t seed, int max_cycles, double tolerance, double initial_trust,
                           int workers, double* fold_scores, double* mean_scores,
                           double* gamma_star, int* n_warnings) {
    return guard([&] {
        const auto& d = static_cast<Dataset*>(h)->data;
        PenaltySpec pen{std::vector<double>(tmpl, tmpl + d.n_covariates())};
        CvConfig cv;
        cv.folds = folds;
        cv.gamma_grid.assign(grid, grid + ng);
        cv.seed = seed;
        OptimizerConfig cfg;
        cfg.max_cycles = max_cycles;
        cfg.tolerance = tolerance;
        cfg.initial_trust = initial_trust;
        cfg.exec = exec_of(0, workers);
        const CvResult r = kfold_select_gamma(d, pen, cv, cfg);
        for (int64_t g = 0; g < ng; ++g) {
            mean_scores[g] = r.mean_scores[static_cast<std::size_t>(g)];
            for (int f = 0; f < folds; ++f)
                fold_scores[g * folds + f] = r.fold_scores[static_cast<std::size_t>(g)][static_cast<std::size_t>(f)];
        }
        *gamma_star = r.gamma_star;
        *n_warnings = static_cast<int>(r.warnings.size());
    });
}

// ---------------------------------------------------------------- design
int ref_design_build(void* dataset, void** out) {
    return guard([&] {
        auto* d = new SortedDesign(build_sorted_design(static_cast<Dataset*>(dataset)->data));
        *out = d;
    });
}

void ref_design_sizes(void* h, int64_t* n, int64_t* p, int32_t* k, int64_t* nnz) {
    const auto& d = *static_cast<SortedDesign*>(h);
    *n = static_cast<int64_t>(d.n_rows());
    *p = static_cast<int64_t>(d.n_covariates());
    *k = d.n_strata();
    int64_t z = 0;
    for (const auto& c : d.data.columns) z += static_cast<int64_t>(c.nnz());
    *nnz = z;
}

void ref_design_copy(void* h, int64_t* perm, uint8_t* head, int64_t* tie_end, int64_t* offsets,
                     double* time, uint8_t* event, int32_t* stratum, int64_t* col_ptr,
                     int64_t* row_idx, double* values) {
    const auto& d = *static_cast<SortedDesign*>(h);
    const std::size_t n = d.n_rows();
    if (perm) std::memcpy(perm, d.perm.data(), n * sizeof(int64_t));
    if (head) std::memcpy(head, d.head_flags.data(), n);
    if (tie_end) std::memcpy(tie_end, d.tie_group_end.data(), n * sizeof(int64_t));
    if (offsets)
        std::memcpy(offsets, d.stratum_offsets.data(), d.stratum_offsets.size() * sizeof(int64_t));
    copy_dataset(d.data, time, event, stratum, col_ptr, row_idx, values);
}

void ref_design_free(void* h) { delete static_cast<SortedDesign*>(h); }

// ---------------------------------------------------------------- likelihood
int ref_make_state(void* design, const double* beta, double* xbeta, double* exp_xbeta) {
    return guard([&] {
        const auto& d = *static_cast<SortedDesign*>(design);
        const auto st = make_state(d, std::span<const double>(beta, d.n_covariates()));
        std::memcpy(xbeta, st.xbeta.data(), st.xbeta.size() * sizeof(double));
        std::memcpy(exp_xbeta, st.exp_xbeta.data(), st.exp_xbeta.size() * sizeof(double));
    });
}

static CoefficientState state_of(const SortedDesign& d, const double* beta, const double* xbeta,
                                 const double* exp_xbeta) {
    CoefficientState st;
    st.beta.assign(beta, beta + d.n_covariates());
    st.xbeta.assign(xbeta, xbeta + d.n_rows());
    st.exp_xbeta.assign(exp_xbeta, exp_xbeta + d.n_rows());
    return st;
}

int ref_gradient_hessian(void* design, const double* beta, const double* xbeta,
                         const double* exp_xbeta, int64_t j, int64_t chunk, int workers,
                         double* g, double* hs) {
    return guard([&] {
        const auto& d = *static_cast<SortedDesign*>(design);
        const auto st = state_of(d, beta, xbeta, exp_xbeta);
        ScanWorkspace ws;
        const auto gh = gradient_hessian(d, st, static_cast<std::size_t>(j), ws,
                                         exec_of(chunk, workers));
        *g = gh.gradient;
        *hs = gh.hessian;
    });
}

int ref_naive_gradient_hessian(void* design, const double* beta, const double* xbeta,
                               const double* exp_xbeta, int64_t j, double* g, double* hs) {
    return guard([&] {
        const auto& d = *static_cast<SortedDesign*>(design);
        const auto st = state_of(d, beta, xbeta, exp_xbeta);
        const auto gh = naive_gradient_hessian(d, st, static_cast<std::size_t>(j));
        *g = gh.gradient;
        *hs = gh.hessian;
    });
}

int ref_log_partial_likelihood(void* design, const double* beta, const double* xbeta,
                               const double* exp_xbeta, int64_t chunk, int workers, double* ll) {
    return guard([&] {
        const auto& d = *static_cast<SortedDesign*>(design);
        const auto st = state_of(d, beta, xbeta, exp_xbeta);
        *ll = log_partial_likelihood(d, st, exec_of(chunk, workers));
    });
}

int ref_naive_log_partial_likelihood(void* design, const double* beta, const double* xbeta,
                                     const double* exp_xbeta, double* ll) {
    return guard([&] {
        const auto& d = *static_cast<SortedDesign*>(design);
        const auto st = state_of(d, beta, xbeta, exp_xbeta);
        *ll = naive_log_partial_likelihood(d, st);
    });
}

// update_xbeta on a full state; the state arrays are updated in place
// (beta[p], xbeta[n], exp_xbeta[n], *updates).
int ref_update_xbeta(void* design, double* beta, double* xbeta, double* exp_xbeta,
                     uint32_t* updates, int64_t j, double delta) {
    return guard([&] {
        const auto& d = *static_cast<SortedDesign*>(design);
        auto st = state_of(d, beta, xbeta, exp_xbeta);
        st.updates_since_refresh = *updates;
        update_xbeta(d, st, static_cast<std::size_t>(j), delta);
        std::memcpy(beta, st.beta.data(), st.beta.size() * sizeof(double));
        std::memcpy(xbeta, st.xbeta.data(), st.xbeta.size() * sizeof(double));
        std::memcpy(exp_xbeta, st.exp_xbeta.data(), st.exp_xbeta.size() * sizeof(double));
        *updates = st.updates_since_refresh;
    });
}

int ref_segmented_scan(int64_t n, const double* values, const uint8_t* flags, int64_t chunk,
                       int workers, double* out) {
    return guard([&] {
        segmented_inclusive_scan(std::span<const double>(values, static_cast<std::size_t>(n)),
                                 std::span<const uint8_t>(flags, static_cast<std::size_t>(n)),
                                 std::span<double>(out, static_cast<std::size_t>(n)),
                                 exec_of(chunk, workers));
    });
}

// ---------------------------------------------------------------- optimizer
int ref_ccd_fit(void* design, const double* gamma, int max_cycles, double tolerance,
                double initial_trust, int64_t chunk, int workers, const double* initial_beta,
                double* beta_out, double* trace_out, int trace_cap, int* trace_len, int* cycles,
                int* converged, double* trust_out, int* n_warnings) {
    return guard([&] {
        const auto& d = *static_cast<SortedDesign*>(design);
        const std::size_t p = d.n_covariates();
        PenaltySpec pen{std::vector<double>(gamma, gamma + p)};
        OptimizerConfig cfg;
        cfg.max_cycles = max_cycles;
        cfg.tolerance = tolerance;
        cfg.initial_trust = initial_trust;
        cfg.exec = exec_of(chunk, workers);
        const FitResult r = initial_beta
                                ? ccd_fit(d, pen, cfg, std::span<const double>(initial_beta, p))
                                : ccd_fit(d, pen, cfg);
        std::memcpy(beta_out, r.beta.data(), p * sizeof(double));
        const int len = static_cast<int>(r.objective_trace.size());
        *trace_len = len;
        std::memcpy(trace_out, r.objective_trace.data(),
                    static_cast<std::size_t>(std::min(len, trace_cap)) * sizeof(double));
        *cycles = r.cycles_used;
        *converged = r.converged ? 1 : 0;
        if (trust_out) std::memcpy(trust_out, r.trust.data(), p * sizeof(double));
        *n_warnings = static_cast<int>(r.warnings.size());
    });
}

int ref_gamma_max(void* design, int64_t chunk, int workers, double* out) {
    return guard([&] {
        const auto& d = *static_cast<SortedDesign*>(design);
        *out = gamma_max(d, PenaltySpec::shared(d.n_covariates(), 1.0), exec_of(chunk, workers));
    });
}

int ref_default_gamma_grid(double gmax, int64_t size, double* out) {
    return guard([&] {
        const auto g = default_gamma_grid(gmax, static_cast<std::size_t>(size));
        std::memcpy(out, g.data(), g.size() * sizeof(double));
    });
}

// ---------------------------------------------------------------- timing
// CPU baseline with run_benchmark semantics (benchmark.cpp:27-41,71-105):
// state at beta = 0, one untimed warm-up coordinate iteration, then `reps`
// timed sweeps of `sweep` coordinate iterations (gradient_hessian, L1
// proposal, trust clip, update_xbeta). Writes the per-rep seconds/iteration.
int ref_time_iterations(void* design, double gamma, int reps, int sweep, int workers,
                        double* seconds_per_iteration) {
    return guard([&] {
        const auto& d = *static_cast<SortedDesign*>(design);
        const std::size_t p = d.n_covariates();
        ExecutionConfig exec = exec_of(0, workers);
#ifdef _OPENMP
        if (workers > 0) omp_set_num_threads(workers);
#endif
        const PenaltySpec penalty = PenaltySpec::shared(p, gamma);
        CoefficientState state = make_state(d, std::vector<double>(p, 0.0));
        ScanWorkspace ws;
        std::vector<double> trust(p, 1.0);
        std::size_t coordinate = 0;
        auto iteration = [&](std::size_t j) {
            GradHess gh{0.0, 0.0};
            if (d.data.columns[j].nnz() > 0) gh = gradient_hessian(d, state, j, ws, exec);
            const ProposedStep prop =
                l1_coordinate_update(gh.gradient, gh.hessian, state.beta[j], penalty.gamma[j]);
            const TrustOutcome out = apply_trust_region(prop.step, trust[j]);
            trust[j] = out.next_trust;
            if (out.applied != 0.0) update_xbeta(d, state, j, out.applied);
        };
        iteration(coordinate);
        coordinate = (coordinate + 1) % p;
        for (int rep = 0; rep < reps; ++rep) {
            const auto t0 = std::chrono::steady_clock::now();
            for (int it = 0; it < sweep; ++it) {
                iteration(coordinate);
                coordinate = (coordinate + 1) % p;
            }
            const std::chrono::duration<double> el = std::chrono::steady_clock::now() - t0;
            seconds_per_iteration[rep] = el.count() / sweep;
        }
    });
}

// Wall time of one full ccd_fit (design build excluded), seconds.
int ref_time_fit(void* design, double gamma, int max_cycles, double tolerance, int workers,
                 double* seconds, int* cycles) {
    return guard([&] {
        const auto& d = *static_cast<SortedDesign*>(design);
#ifdef _OPENMP
        if (workers > 0) omp_set_num_threads(workers);
#endif
        OptimizerConfig cfg;
        cfg.max_cycles = max_cycles;
        cfg.tolerance = tolerance;
        cfg.exec = exec_of(0, workers);
        const auto t0 = std::chrono::steady_clock::now();
        const auto r = ccd_fit(d, PenaltySpec::shared(d.n_covariates(), gamma), cfg);
        const std::chrono::duration<double> el = std::chrono::steady_clock::now() - t0;
        *seconds = el.count();
        *cycles = r.cycles_used;
    });
}


// ---------------------------------------------------------------- io (proj/src/io.cpp)
thread_local std::string g_str;

int ref_read_wide_csv(const char* path, void** out) {
    return guard([&] { *out = new Dataset{read_wide_csv(path), {}}; });
}
const char* ref_dataset_name(void* h, int64_t j) {
    g_str = static_cast<Dataset*>(h)->data.covariate_name(static_cast<std::size_t>(j));
    return g_str.c_str();
}
int32_t ref_dataset_n_labels(void* h) {
    return static_cast<int32_t>(static_cast<Dataset*>(h)->data.stratum_labels.size());
}
const char* ref_dataset_label(void* h, int32_t k) {
    g_str = static_cast<Dataset*>(h)->data.stratum_label(k);
    return g_str.c_str();
}
int ref_write_wide_csv(void* h, const char* path) {
    return guard([&] { write_wide_csv(path, static_cast<Dataset*>(h)->data); });
}
int ref_read_long_csv(const char* path, void** out) {
    return guard([&] { *out = new LongData(read_long_csv(path)); });
}
void ref_long_sizes(void* h, int64_t* ns, int64_t* nr, int64_t* p, double* max_stop) {
    const auto& d = *static_cast<LongData*>(h);
    int64_t r = 0;
    for (const auto& s : d.subjects) r += static_cast<int64_t>(s.size());
    *ns = static_cast<int64_t>(d.subjects.size());
    *nr = r;
    *p = static_cast<int64_t>(d.covariate_names.size());
    *max_stop = d.max_stop;
}
const char* ref_long_name(void* h, int64_t j) {
    g_str = static_cast<LongData*>(h)->covariate_names[static_cast<std::size_t>(j)];
    return g_str.c_str();
}
int ref_write_long_csv(void* h, const char* path) {
    return guard([&] { write_long_csv(path, *static_cast<LongData*>(h)); });
}
void ref_long_free(void* h) { delete static_cast<LongData*>(h); }
// to_time_varying + lower_pipeline; the lowered dataset keeps its covariate names
int ref_long_lower(void* h, const double* cuts, int64_t n_cuts, const int64_t* split_cov,
                   const int64_t* split_ptr, const double* split_times, int64_t n_splits,
                   void** out, int64_t* map_source, int32_t* map_window) {
    return guard([&] {
        const auto& d = *static_cast<LongData*>(h);
        const std::vector<double> cp(cuts, cuts + n_cuts);
        TimeVaryingDataset tv = to_time_varying(d, cp);
        TimeVaryingSpec spec;
        spec.cut_points = cp;
        for (int64_t s = 0; s < n_splits; ++s) {
            TimeVaryingSpec::Split sp;
            sp.covariate = static_cast<std::size_t>(split_cov[s]);
            sp.times.assign(split_times + split_ptr[s], split_times + split_ptr[s + 1]);
            spec.splits.push_back(sp);
        }
        LoweredDataset low = lower_pipeline(tv, spec);
        for (std::size_t c = 0; c < low.column_map.size(); ++c) {
            map_source[c] = static_cast<int64_t>(low.column_map[c].source);
            map_window[c] = low.column_map[c].window;
        }
        *out = new Dataset{std::move(low.data), {}};
    });
}
// ConfigMap driven by a script of "OP key [fallback]" lines (S string, D double,
// I int, DL double list, SL string list, H has, F finish); one output line per op
// (results joined by '|', errors as "ERR:<message>"); a from_string failure
// gives a single "ERR:" line.
int ref_config_script(const char* text, const char* origin, const char* script, char* out,
                      int cap) {
    std::ostringstream res;
    try {
        ConfigMap cfg = ConfigMap::from_string(text, origin);
        std::istringstream sc(script);
        std::string line;
        while (std::getline(sc, line)) {
            std::istringstream ls(line);
            std::string op, key, fb;
            ls >> op >> key;
            std::getline(ls, fb);
            if (!fb.empty() && fb[0] == ' ') fb.erase(0, 1);
            try {
                if (op == "S") {
                    res << cfg.get_string(key, fb);
                } else if (op == "D") {
                    res << format_double(cfg.get_double(key, std::stod(fb)));
                } else if (op == "I") {
                    res << cfg.get_int(key, std::stoll(fb));
                } else if (op == "DL") {
                    const auto v = cfg.get_double_list(key);
                    for (std::size_t i = 0; i < v.size(); ++i) res << (i ? "|" : "") << format_double(v[i]);
                } else if (op == "SL") {
                    const auto v = cfg.get_string_list(key);
                    for (std::size_t i = 0; i < v.size(); ++i) res << (i ? "|" : "") << v[i];
                } else if (op == "H") {
                    res << (cfg.has(key) ? 1 : 0);
                } else if (op == "F") {
                    cfg.finish();
                    res << "OK";
                }
            } catch (const std::exception& e) {
                res << "ERR:" << e.what();
            }
            res << "\n";
        }
    } catch (const std::exception& e) {
        res << "ERR:" << e.what() << "\n";
    }
    std::strncpy(out, res.str().c_str(), static_cast<std::size_t>(cap) - 1);
    out[cap - 1] = 0;
    return 0;
}
}  // extern "C"
