/*
 * stratcox_b200 — C-ABI of the B200-native (sm_100a) stratified Cox CCD hot path.
 *
 * This is the drop-in boundary. Each entry point replaces one function of the
 * reference C++ API (namespace stratcox, /root/reference/proj/include/stratcox/);
 * the reference interface it replaces is cited beside it. Arguments are plain
 * pointers and sizes — no C++ or torch types — so a C++ shim (see
 * INTEGRATION.md and paper_2310_16238_b200/csrc/dropin/) or a ctypes/cffi
 * binding can bind it directly.
 *
 * Object model
 *   scx_ctx     one device + one stream + one uploaded SortedDesign + one
 *               CoefficientState. Not thread-safe; create one per thread
 *               (the reference calls ccd_fit concurrently from OpenMP threads,
 *               proj/src/resample.cpp:121,207 — each gets its own context).
 *   errors      every call returns scx_status; scx_last_error(ctx) holds the
 *               message, identical to the reference exception text
 *               (proj/include/stratcox/errors.hpp:9-26 taxonomy:
 *               validation_error / numeric_error / internal_error).
 *
 * Row space: all row indices are SORTED rows (stratum ascending, time
 * descending, stable — proj/src/data.cpp:75-81), i.e. a SortedDesign.
 */
#ifndef STRATCOX_B200_H
#define STRATCOX_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct scx_ctx scx_ctx;

typedef enum {
    SCX_OK = 0,
    SCX_ERR_VALIDATION = 1, /* stratcox::validation_error */
    SCX_ERR_NUMERIC = 2,    /* stratcox::numeric_error   */
    SCX_ERR_INTERNAL = 3,   /* stratcox::internal_error  */
    SCX_ERR_CUDA = 4        /* device/runtime failure (no reference equivalent) */
} scx_status;

/* ---------------------------------------------------------------- context */
const char* scx_version(void);
/* Number of visible CUDA devices (0 when none / no driver). */
int scx_device_count(void);
scx_status scx_create(int device, scx_ctx** out);
void scx_destroy(scx_ctx* ctx);
const char* scx_last_error(const scx_ctx* ctx);

/* ---------------------------------------------------------------- design
 * Replaces the device-side view of SortedDesign (data.hpp:50-62) as produced
 * by build_sorted_design (data.cpp:68-147).
 *   stratum_offsets  int64[n_strata+1]   SortedDesign::stratum_offsets
 *   event            uint8[n_rows]       SortedDesign::data.event (0/1)
 *   tie_group_end    int64[n_rows]       SortedDesign::tie_group_end
 *   col_ptr          int64[p+1]          concatenation of data.columns[j]
 *   row_idx          int64[nnz]          SparseColumn::rows (sorted rows, strictly increasing)
 *   values           double[nnz] or NULL SparseColumn::values (NULL = every value 1.0)
 * Columns whose values are all 1.0 are stored as indicators (row index only).
 * Uploading resets the coefficient state to beta = 0. */
scx_status scx_upload_design(scx_ctx* ctx, int64_t n_rows, int32_t n_strata,
                             const int64_t* stratum_offsets, const uint8_t* event,
                             const int64_t* tie_group_end, int64_t n_covariates,
                             const int64_t* col_ptr, const int64_t* row_idx,
                             const double* values);

/* Same design, row indices already int32 (no host->device narrowing pass). */
scx_status scx_upload_design_i32(scx_ctx* ctx, int64_t n_rows, int32_t n_strata,
                                 const int64_t* stratum_offsets, const uint8_t* event,
                                 const int64_t* tie_group_end, int64_t n_covariates,
                                 const int64_t* col_ptr, const int32_t* row_idx,
                                 const double* values);

/* Design statistics: n_rows, n_strata, p, nnz, event-code width in bytes,
 * number of 4096-row tiles, indicator-column count. Any pointer may be NULL. */
scx_status scx_design_info(const scx_ctx* ctx, int64_t* n_rows, int32_t* n_strata, int64_t* p,
                           int64_t* nnz, int32_t* code_bytes, int64_t* n_tiles,
                           int64_t* n_indicator);

/* The uploaded SortedDesign back on the host (any pointer may be NULL):
 * stratum_offsets [n_strata+1], event [n], tie_group_end [n], col_ptr [p+1],
 * row_idx [nnz] (sorted rows), values [nnz] (1.0 for indicator columns).
 * With scx_build_design this is build_sorted_design (data.cpp:68-147) run on
 * the device; the C++ drop-in returns it as the reference's SortedDesign. */
scx_status scx_design_export(scx_ctx* ctx, int64_t* stratum_offsets, uint8_t* event,
                             int64_t* tie_group_end, int64_t* col_ptr, int64_t* row_idx,
                             double* values);

/* ---------------------------------------------------------------- state
 * CoefficientState (likelihood.hpp:23-29) lives on the device. */
/* make_state (likelihood.hpp:33, likelihood.cpp:19-29): beta[p] -> eta, D. */
scx_status scx_make_state(scx_ctx* ctx, const double* beta);
/* Load an arbitrary host CoefficientState (used at the parity boundary by the
 * C++ shim for gradient_hessian / log_partial_likelihood calls). */
scx_status scx_set_state(scx_ctx* ctx, const double* beta, const double* xbeta,
                         const double* exp_xbeta, uint32_t updates_since_refresh);
/* Read the state back; any pointer may be NULL. */
scx_status scx_get_state(scx_ctx* ctx, double* beta, double* xbeta, double* exp_xbeta,
                         uint32_t* updates_since_refresh);
/* refresh_xbeta (likelihood.hpp:37, likelihood.cpp:31-58). */
scx_status scx_refresh_xbeta(scx_ctx* ctx);
/* update_xbeta (likelihood.hpp:43-44, likelihood.cpp:60-83): "step overflow"
 * leaves the state untouched; refresh every 256 accepted updates. */
scx_status scx_update_xbeta(scx_ctx* ctx, int64_t j, double delta);

/* ---------------------------------------------------------------- likelihood */
/* gradient_hessian (likelihood.hpp:75-77, likelihood.cpp:129-189). */
scx_status scx_gradient_hessian(scx_ctx* ctx, int64_t j, double* gradient, double* hessian);
/* The same (g', g'') by the risk-suffix formulation the fit uses on the chunked
 * layout (no reference counterpart; replaces likelihood.cpp:129-189 inside
 * run_ccd, optimizer.cpp:104): one fused scan of the state gives per row the
 * within-stratum prefixes of w/S0 and w/S0^2, then column j costs O(nnz_j)
 * gathers. Agrees with scx_gradient_hessian within rounding. Needs the
 * chunked layout (many small strata); else SCX_ERR_VALIDATION. */
scx_status scx_gradient_hessian_rs(scx_ctx* ctx, int64_t j, double* gradient, double* hessian);
/* The risk-suffix fused scan alone over the current state (timing kind 3). */
scx_status scx_risk_prefix(scx_ctx* ctx);
/* reps back-to-back risk scans in ONE launch (timing kind 3): the scan's
 * throughput as it runs inside the persistent fit kernel, without the launch
 * and pipeline fill of a single scan. reps >= 1. */
scx_status scx_risk_prefix_n(scx_ctx* ctx, int reps);
/* CCD cycle implementation: 0 = automatic (risk-suffix cycle on the chunked
 * layout while max|eta| <= 300, the per-coordinate fused-scan cycle otherwise
 * and for coordinates whose g'' cancels), 1 = fused-scan cycle only.
 * *risk_suffix (may be NULL) receives whether the risk-suffix cycle can run. */
scx_status scx_set_fit_path(scx_ctx* ctx, int path, int* risk_suffix);
/* Path counters of the last scx_ccd_fit: out[0] risk-suffix cycle launches,
 * out[1] coordinates handed to the exact fused scan (rounding bound not
 * certified), out[2] hand-offs on the |eta| bound, out[3] fused-scan cycle launches. */
scx_status scx_fit_path_stats(const scx_ctx* ctx, int64_t out[4]);
/* log_partial_likelihood (likelihood.hpp:60-65, likelihood.cpp:93-121). */
scx_status scx_log_partial_likelihood(scx_ctx* ctx, double* loglik);
/* naive_gradient_hessian / naive_log_partial_likelihood (likelihood.hpp:80-82,
 * likelihood.cpp:191-244): literal O(sum n_k^2) risk-set loops, on device. */
scx_status scx_naive_gradient_hessian(scx_ctx* ctx, int64_t j, double* gradient,
                                      double* hessian);
scx_status scx_naive_log_partial_likelihood(scx_ctx* ctx, double* loglik);

/* segmented_inclusive_scan (scan.hpp:71-79, scan.cpp:124-190) on the device.
 * Host in/out buffers; n >= 1, flags[0] must be 1. Uses the context's stream
 * and scratch but not its design. */
scx_status scx_segmented_inclusive_scan(scx_ctx* ctx, int64_t n, const double* values,
                                        const uint8_t* flags, double* out);

/* ---------------------------------------------------------------- optimizer */
/* Scalar rules (optimizer.hpp:47-68, optimizer.cpp:32-78). The same code runs
 * on the device inside scx_ccd_fit. */
scx_status scx_newton_step(double g1, double g2, double* step, int* flat);
scx_status scx_apply_trust_region(double proposed, double trust, double* applied,
                                  double* next_trust);
scx_status scx_l1_coordinate_update(double g1, double g2, double beta_j, double gamma_j,
                                    double* step, int* skipped, int* flat);

/* Elastic-net rule (EXTENSION, no reference counterpart; BASELINE config 1's
 * "L2 prior"): the ridge term l2_j beta_j^2 / 2 adds l2_j beta_j to g' and l2_j
 * to g'', then l1_coordinate_update (optimizer.cpp:51-78) runs on the
 * penalised pair. l2_j = 0 is scx_l1_coordinate_update exactly. */
scx_status scx_coordinate_update(double g1, double g2, double beta_j, double gamma_j, double l2_j,
                                 double* step, int* skipped, int* flat);

/* Message of the last failing scalar-rule call on this thread. */
const char* scx_rule_error(void);

typedef struct {
    int32_t max_cycles;   /* OptimizerConfig::max_cycles   (default 1000) */
    double tolerance;     /* OptimizerConfig::tolerance    (default 1e-6) */
    double initial_trust; /* OptimizerConfig::initial_trust (default 1.0) */
} scx_fit_options;

typedef struct {
    double* beta;            /* [p]  FitResult::beta */
    double* trust;           /* [p]  FitResult::trust (may be NULL) */
    double* objective_trace; /* [max_cycles+1] FitResult::objective_trace */
    int32_t trace_len;       /* entries written */
    int32_t cycles_used;     /* FitResult::cycles_used */
    int32_t converged;       /* FitResult::converged */
    int32_t n_warnings;      /* coordinates skipped after 10 halvings (exact count; the first
                                min(warning_cap, 65536) are listed in warning_coords) */
    int64_t* warning_coords; /* [warning_cap] coordinate of each warning, in order (may be NULL) */
    int32_t warning_cap;
    uint32_t updates_since_refresh;
    int64_t n_evaluations;   /* gradient/Hessian evaluations performed (nnz_j > 0 coordinates) */
} scx_fit_result;

/* ccd_fit (optimizer.hpp:70-73, optimizer.cpp:82-160). gamma[p] = PenaltySpec::gamma;
 * initial_beta NULL = zeros. The whole cycle runs on the device; the host
 * synchronises once per cycle (objective, max step, error word). */
scx_status scx_ccd_fit(scx_ctx* ctx, const double* gamma, const scx_fit_options* options,
                       const double* initial_beta, scx_fit_result* result);

/* ccd_fit with an optional L2 (ridge / Gaussian) prior l2[p] >= 0 (NULL: none,
 * = scx_ccd_fit). EXTENSION, no reference counterpart: the objective becomes
 * -log L + sum gamma_j |beta_j| + sum l2_j beta_j^2 / 2 and every coordinate
 * uses scx_coordinate_update's rule. Parity unpinned against the reference
 * (it has no L2 prior); checked by KKT conditions and against the oracle's
 * restatement of the same rule. */
scx_status scx_ccd_fit_prior(scx_ctx* ctx, const double* gamma, const double* l2,
                             const scx_fit_options* options, const double* initial_beta,
                             scx_fit_result* result);

/* gamma_max (resample.hpp:38-39, resample.cpp:42-55) with a penalty template
 * gamma_template[p] (NULL = every coefficient penalized). */
scx_status scx_gamma_max(scx_ctx* ctx, const double* gamma_template, double* out);

/* ---------------------------------------------------------------- data sets, path and CV
 * SurvivalDataset (data.hpp:31-45) in INPUT row order, for the drivers below. */
typedef struct {
    int64_t n_rows;
    const double* time;       /* [n] observed time, >= 0 */
    const uint8_t* event;     /* [n] 1 event, 0 censored */
    const int32_t* stratum;   /* [n] dense labels 1..K */
    const int64_t* subject;   /* [n] originating subject, or NULL (row + 1) */
    int64_t n_covariates;
    const int64_t* col_ptr;   /* [p+1] */
    const int64_t* row_idx;   /* [nnz] input rows, strictly increasing per column */
    const double* values;     /* [nnz] or NULL (every value 1.0) */
} scx_dataset;

/* build_sorted_design (data.cpp:68-147) with validate_invariants
 * (data.cpp:27-66) ON THE DEVICE: stable LSD radix sorts by (stratum asc,
 * time desc), heads, tie-group ends and the CSC re-index (a segmented radix
 * sort per column), then the upload (as scx_upload_design). Same permutation,
 * same arrays and same validation messages as the reference. perm_out [n]
 * may be NULL: sorted row s is input row perm_out[s]. */
scx_status scx_build_design(scx_ctx* ctx, const scx_dataset* data, int64_t* perm_out);

/* Lowering + build on the device (BASELINE configs 2-3; PAPER.md:582-583
 * "mappings on the original data" instead of duplication): only the
 * SUBJECT-level data (scx_dataset over subjects, time-fixed covariates) is
 * uploaded; the subject x interval -> augmented-row mapping, the augmented
 * rows and columns (augment_to_strata + split_time_varying_coefficient,
 * transforms.cpp:98-223, same arrays as scx_lower_time_varying) and then
 * build_sorted_design run on the device. The duplicated design never exists
 * on the host. map_* [p_out] (may be NULL) receive the column map,
 * p_out = p + sum over splits of their number of times. */
scx_status scx_build_lowered_design(scx_ctx* ctx, const scx_dataset* subjects,
                                    const double* cut_points, int64_t n_cuts,
                                    const int64_t* split_covariate, const int64_t* split_ptr,
                                    const double* split_times, int64_t n_splits,
                                    int64_t* perm_out, int64_t* map_source, int32_t* map_window,
                                    double* map_start, double* map_end);

/* default_gamma_grid (resample.hpp:42, resample.cpp:57-68): `size` values
 * log-spaced over [gamma_max / 1e4, gamma_max]. */
scx_status scx_default_gamma_grid(double gamma_max, int64_t size, double* out);

/* fold_assignment (resample.hpp:45, resample.cpp:70-91): subjects shuffled by
 * mt19937_64(seed) and dealt round-robin; fold_of_row [n]. */
scx_status scx_fold_assignment(const scx_dataset* data, int folds, uint64_t seed,
                               int32_t* fold_of_row);

typedef struct {               /* CvConfig (resample.hpp:15-19) */
    int folds;
    const double* gamma_grid;  /* strictly increasing, positive */
    int64_t grid_size;
    uint64_t seed;
} scx_cv_config;

typedef struct {               /* CvResult (resample.hpp:21-27) */
    double gamma_star;
    double* fold_scores;       /* [grid_size][folds] caller-allocated (may be NULL) */
    double* mean_scores;       /* [grid_size] caller-allocated (may be NULL) */
    int32_t n_warnings;        /* fits / scores that failed (score -inf) */
} scx_cv_result;

/* kfold_select_gamma (resample.hpp:53-54, resample.cpp:93-172): per fold, the
 * warm-started gamma path from the sparse end on the training folds with
 * held-out partial-likelihood scoring; fits and scores run on the device.
 * Folds are dealt round-robin over devices[0..n_devices) (NULL/0: device 0),
 * one host thread per device. error_out (cap bytes, may be NULL) receives the
 * error message, or the fold warnings one per line on success. */
scx_status scx_kfold_select_gamma(const scx_dataset* data, const double* penalty_template,
                                  const scx_cv_config* cv, const scx_fit_options* options,
                                  const int* devices, int n_devices, scx_cv_result* result,
                                  char* error_out, int error_cap);

/* ---------------------------------------------------------------- lowering (transforms.hpp)
 * Subjects with time-fixed covariates (scx_dataset over SUBJECTS; stratum is
 * ignored) and cut points 0 = t0 < ... < tK: make_time_varying, then
 * split_time_varying_coefficient for the covariates listed in split_covariate
 * (split times of split s: split_times[split_ptr[s] .. split_ptr[s+1]), each a
 * cut point), then augment_to_strata (transforms.cpp:64-223): one row per
 * (subject, interval at risk), interval-major, stratum = interval. The result
 * is library-owned: sizes, a scx_dataset view (feed it to scx_build_design or
 * scx_kfold_select_gamma) and the column map (source covariate, effect window
 * -1 = unsplit, window bounds). */
typedef struct scx_lowered scx_lowered;
scx_status scx_lower_time_varying(const scx_dataset* subjects, const double* cut_points,
                                  int64_t n_cuts, const int64_t* split_covariate,
                                  const int64_t* split_ptr, const double* split_times,
                                  int64_t n_splits, scx_lowered** out, char* error_out,
                                  int error_cap);
scx_status scx_lowered_sizes(const scx_lowered* lowered, int64_t* n_rows, int64_t* n_covariates,
                             int64_t* nnz);
scx_status scx_lowered_dataset(const scx_lowered* lowered, scx_dataset* view);
scx_status scx_lowered_column_map(const scx_lowered* lowered, int64_t* source, int32_t* window,
                                  double* window_start, double* window_end);
void scx_lowered_free(scx_lowered* lowered);

/* ---------------------------------------------------------------- files and configuration
 * io.hpp (proj/src/io.cpp): the two CSV layouts and the key = value config,
 * same formats, canonical order and error messages as the reference; files
 * are parsed by a thread pool. Every *err / cap pair receives the message of
 * a failure (the reference's validation_error text). */
typedef struct scx_table scx_table;   /* SurvivalDataset + names and stratum labels */
typedef struct scx_long scx_long;     /* LongData (io.hpp:32-43) */
typedef struct scx_config scx_config; /* ConfigMap (io.hpp:57-76) */
/* read_wide_csv (io.cpp:123-193): rows in file order, strata relabelled 1..K
 * by label (numeric order when every label is a number), columns in name order. */
scx_status scx_read_wide_csv(const char* path, scx_table** out, char* err, int cap);
scx_status scx_table_dataset(const scx_table* table, scx_dataset* view);
const char* scx_table_covariate_name(const scx_table* table, int64_t j);
int32_t scx_table_n_strata(const scx_table* table);
const char* scx_table_stratum_label(const scx_table* table, int32_t k); /* k = 1..K */
void scx_table_free(scx_table* table);
/* write_wide_csv (io.cpp:195-223); names / labels may be NULL (x1.., 1..). */
scx_status scx_write_wide_csv(const char* path, const scx_dataset* data,
                              const char* const* covariate_names, const char* const* stratum_labels,
                              char* err, int cap);
/* read_long_csv (io.cpp:225-272) / write_long_csv (io.cpp:274-291). */
scx_status scx_read_long_csv(const char* path, scx_long** out, char* err, int cap);
scx_status scx_long_sizes(const scx_long* data, int64_t* n_subjects, int64_t* n_records,
                          int64_t* n_covariates, double* max_stop);
const char* scx_long_covariate_name(const scx_long* data, int64_t j);
scx_status scx_write_long_csv(const char* path, const scx_long* data, char* err, int cap);
/* to_time_varying (io.cpp:293-345) + lower_pipeline (transforms.cpp:98-231):
 * the long records' per-interval covariate values, effect-window splits as in
 * scx_lower_time_varying, augmented to strata (interval-major rows). */
scx_status scx_long_lower(const scx_long* data, const double* cut_points, int64_t n_cuts,
                          const int64_t* split_covariate, const int64_t* split_ptr,
                          const double* split_times, int64_t n_splits, scx_lowered** out,
                          char* err, int cap);
void scx_long_free(scx_long* data);
/* Augmented covariate names of a lowered dataset (window names
 * "NAME[a-b)" as transforms.cpp:18-21; NULL when the source had no names). */
const char* scx_lowered_covariate_name(const scx_lowered* lowered, int64_t j);
/* ConfigMap: from_string / from_file (io.cpp:347-375), typed getters that mark
 * a key consumed (io.cpp:377-429), finish() naming unconsumed keys (:431-438).
 * Returned strings live as long as the config. */
scx_status scx_config_from_string(const char* text, const char* origin, scx_config** out,
                                  char* err, int cap);
scx_status scx_config_from_file(const char* path, scx_config** out, char* err, int cap);
int scx_config_has(const scx_config* config, const char* key);
const char* scx_config_get_string(scx_config* config, const char* key, const char* fallback);
scx_status scx_config_get_double(scx_config* config, const char* key, double fallback,
                                 double* out, char* err, int cap);
scx_status scx_config_get_int(scx_config* config, const char* key, int64_t fallback,
                              int64_t* out, char* err, int cap);
scx_status scx_config_get_double_list(scx_config* config, const char* key, double* out,
                                      int64_t cap_out, int64_t* n, char* err, int cap);
/* newline-joined list items; *n = count */
const char* scx_config_get_string_list(scx_config* config, const char* key, int64_t* n);
scx_status scx_config_finish(const scx_config* config, char* err, int cap);
void scx_config_free(scx_config* config);

/* ---------------------------------------------------------------- measurement
 * Device time of the kernels launched by the last call, for bench/roofline:
 * per-kernel-class accumulated milliseconds and launch counts since the last
 * scx_timing_reset. Enabled by scx_timing_enable(ctx, 1) (adds events). */
scx_status scx_timing_enable(scx_ctx* ctx, int on);
scx_status scx_timing_reset(scx_ctx* ctx);
/* kind: 0 = fused scan+reduce (K1), 1 = update (K3), 2 = log-likelihood (K2),
 * 3 = risk-suffix cycle / risk prefix */
scx_status scx_timing_get(scx_ctx* ctx, int kind, double* total_ms, int64_t* launches);

/* Fused scan+reduce decomposition: 0 = automatic (stratum-aligned chunk per
 * CTA when the strata are small enough, else cross-CTA look-back), 1 = always
 * look-back, 2 = chunks when available. *chunked (may be NULL) receives
 * whether the chunked kernel will run. Results agree within rounding. */
scx_status scx_set_k1_mode(scx_ctx* ctx, int mode, int* chunked);

/* Profiling: per-event clock64 trace of the last fused scan+reduce launch made
 * with SCX_K1_DBG bit 8 set (CTAs 0 and 73, tiles < 511): out[2][512][8]. */
scx_status scx_debug_k1_trace(long long* out);

/* Debug: the risk scan's arrays after scx_risk_prefix — tile-local suffix sums
 * R[n], Q[n], tile carries CR / CQ [2048-row tiles] and each tile's last-head
 * offset; R of row r = R[r] + (r mod 2048 >= lasth[r / 2048] ? CR[r / 2048] : 0). */
scx_status scx_debug_risk_arrays(scx_ctx* ctx, double* R, double* Q, double* CR, double* CQ,
                                 int32_t* lasth);

/* Number of kernels this context has launched so far (bench bookkeeping). */
int64_t scx_launch_count(const scx_ctx* ctx);

/* Raw device pointers of the context's stream (cudaStream_t) for callers that
 * want to time on it; returns NULL without a context. */
void* scx_stream(scx_ctx* ctx);

/* ---------------------------------------------------------------- multi-GPU
 * Row-sharded fits: each rank uploads the rows of whole
 * strata it owns (shards cut at stratum boundaries: no scan carry crosses
 * ranks), so every rank's risk sets are local; per coordinate the ranks only
 * exchange a few partial sums. The exchange is device-side, inside the
 * persistent risk-suffix cycle kernel and a few one-thread kernels, through
 * 2 x 128-byte slots per rank in device memory that every rank can load:
 * peer-mapped (P2P over NVLink/NVSwitch) for ranks in one process,
 * IPC-opened across processes, plain device memory for ranks sharing one
 * GPU. Partials are summed in rank order, so every rank applies a
 * bit-identical step; no host round trip per coordinate.
 * Protocol: [scx_set_sm_budget] -> upload -> scx_xchg_slots / _ipc_handle
 * -> scx_xchg_connect / _connect_ipc (all ranks) -> combine the ranks'
 * scx_shard_local_columns (OR nonempty, SUM lin in rank order, MAX xmax,
 * AND rs_ok) -> scx_shard_set_columns -> scx_ccd_fit on every rank at once.
 * (Replaces the reference's shared-memory OpenMP parallelism over rows,
 * scan.cpp:124-190; the reference has no multi-device path.) */
/* Cycle-kernel CTAs / stratum-aligned chunks (before upload; 0 = every SM):
 * ranks sharing one GPU split its SMs so their persistent kernels co-reside. */
scx_status scx_set_sm_budget(scx_ctx* ctx, int sms);
/* This context's exchange slots (device pointer, zeroed). */
scx_status scx_xchg_slots(scx_ctx* ctx, void** slots);
/* The same as a 64-byte cudaIpcMemHandle for other processes. */
scx_status scx_xchg_ipc_handle(scx_ctx* ctx, char out[64]);
/* Attach this context as rank `rank` of `nranks` (<= 8): rank_slots[r] =
 * rank r's slots (rank_slots[rank] = this context's own). Enables P2P to
 * peer devices. */
scx_status scx_xchg_connect(scx_ctx* ctx, int nranks, int rank, void* const* rank_slots);
/* The same from the ranks' IPC handles (handles = nranks x 64 bytes). */
scx_status scx_xchg_connect_ipc(scx_ctx* ctx, int nranks, int rank, const char* handles);
/* Per-column facts of this rank's rows: nonempty[p], lin[p] = sum x*delta,
 * xmax[p] = max |x|; rs_ok: the risk-suffix cycle can run on this shard. */
scx_status scx_shard_local_columns(scx_ctx* ctx, uint8_t* nonempty, double* lin, double* xmax,
                                   int* rs_ok);
/* The combined (global) facts: the same column set, lin and xmax on every rank. */
scx_status scx_shard_set_columns(scx_ctx* ctx, const uint8_t* nonempty, const double* lin,
                                 const double* xmax, int rs_ok);

#ifdef __cplusplus
}
#endif
#endif /* STRATCOX_B200_H */
