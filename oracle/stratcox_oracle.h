/* TEST INFRASTRUCTURE ONLY — the CPU oracle for parity tests.
 *
 * A plain-C restatement of the reference ("stratcox", /root/reference/proj)
 * algorithm on the hot path: sorted-design construction, the chunked
 * flag-value segmented scan, the per-coordinate gradient/Hessian, the
 * stratified log partial likelihood, the X*beta cache and the L1 cyclic
 * coordinate descent loop. Serial, with the reference's chunk order, so its
 * output bits equal the reference's for the same chunk_size (the reference's
 * bits depend on chunk_size only: proj/include/stratcox/scan.hpp:8-12).
 *
 * Pinned against the compiled reference (oracle/_ref/libstratcox_ref.so) and
 * the fixtures in tests/golden/ by tests/test_oracle.py.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load this library. The product (paper_2310_16238_b200) never does.
 */
#ifndef STRATCOX_ORACLE_H
#define STRATCOX_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { ORC_OK = 0, ORC_VALIDATION = 1, ORC_NUMERIC = 2, ORC_INTERNAL = 3 };

/* Sorted layout (proj/include/stratcox/data.hpp:50-62). All arrays in sorted
 * row space; CSC columns re-indexed to sorted rows, strictly increasing. */
typedef struct {
    int64_t n;
    int64_t p;
    int32_t k;
    const double* time;
    const uint8_t* event;
    const uint8_t* head;
    const int64_t* tie_end;
    const int64_t* offsets; /* k+1 */
    const int64_t* col_ptr; /* p+1 */
    const int64_t* row_idx;
    const double* values;
} orc_design;

const char* orc_last_error(void);

/* data.cpp:68-147 */
int orc_build_sorted_design(int64_t n, const double* time, const uint8_t* event,
                            const int32_t* stratum, int64_t p, const int64_t* col_ptr,
                            const int64_t* row_idx, const double* values, int64_t* perm,
                            uint8_t* head, int64_t* tie_end, int64_t* offsets, int32_t* k_out,
                            double* s_time, uint8_t* s_event, int32_t* s_stratum,
                            int64_t* s_row_idx, double* s_values);

/* scan.cpp:124-190 */
int orc_segmented_scan(int64_t n, const double* values, const uint8_t* flags, int64_t chunk,
                       double* out);
/* scan.cpp:63-115 */
int orc_inclusive_scan(int64_t n, const double* values, int64_t chunk, double* out);

/* likelihood.cpp:19-83 */
int orc_make_state(const orc_design* d, const double* beta, double* xbeta, double* exp_xbeta);
int orc_update_xbeta(const orc_design* d, double* beta, double* xbeta, double* exp_xbeta,
                     uint32_t* updates, int64_t j, double delta);

/* likelihood.cpp:93-121 */
int orc_log_partial_likelihood(const orc_design* d, const double* xbeta, const double* exp_xbeta,
                               int64_t chunk, double* ll);
/* likelihood.cpp:129-189 */
int orc_gradient_hessian(const orc_design* d, const double* exp_xbeta, int64_t j, int64_t chunk,
                         double* g, double* h);
/* likelihood.cpp:191-244 */
int orc_naive_gradient_hessian(const orc_design* d, const double* exp_xbeta, int64_t j,
                               double* g, double* h);
int orc_naive_log_partial_likelihood(const orc_design* d, const double* xbeta,
                                     const double* exp_xbeta, double* ll);

/* optimizer.cpp:32-78 */
int orc_newton_step(double g1, double g2, double* step, int* flat);
int orc_apply_trust_region(double proposed, double trust, double* applied, double* next_trust);
int orc_l1_coordinate_update(double g1, double g2, double beta_j, double gamma_j, double* step,
                             int* skipped, int* flat);

/* optimizer.cpp:82-160. trace_out needs max_cycles+1 slots. */
int orc_ccd_fit(const orc_design* d, const double* gamma, int max_cycles, double tolerance,
                double initial_trust, int64_t chunk, const double* initial_beta,
                double* beta_out, double* trace_out, int* trace_len, int* cycles,
                int* converged, double* trust_out, int* n_warnings);

/* Extension (not in the reference; BASELINE config 1 "L2 prior"): ridge term
 * sum l2_j beta_j^2 / 2 added to the objective, g' += l2 beta, g'' += l2 before
 * the L1 rule. l2 == NULL is orc_ccd_fit. */
int orc_coordinate_update(double g1, double g2, double beta_j, double gamma_j, double l2_j,
                          double* step, int* skipped, int* flat);
int orc_ccd_fit_prior(const orc_design* d, const double* gamma, const double* l2, int max_cycles,
                      double tolerance, double initial_trust, int64_t chunk,
                      const double* initial_beta, double* beta_out, double* trace_out,
                      int* trace_len, int* cycles, int* converged, double* trust_out,
                      int* n_warnings);

/* resample.cpp:42-55 (every coefficient penalized, as PenaltySpec::shared) */
int orc_gamma_max(const orc_design* d, int64_t chunk, double* out);

#ifdef __cplusplus
}
#endif
#endif
