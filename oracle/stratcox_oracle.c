/* TEST INFRASTRUCTURE ONLY — CPU oracle (see stratcox_oracle.h).
 *
 * Plain-C restatement of the reference's hot path. Every function cites the
 * reference file:line it follows; paths are relative to /root/reference/proj.
 * Built with -ffp-contract=off so that no multiply-add is fused: the reference
 * build (g++ -O3, baseline x86-64, no FMA) evaluates every product and sum
 * separately, and the serial chunk order below reproduces its bits.
 */
#include "stratcox_oracle.h"

#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define LP_BOUND 700.0       /* kLinearPredictorBound, include/stratcox/likelihood.hpp:21 */
#define FLAT_CURVATURE 1e-12 /* kFlatCurvature, include/stratcox/optimizer.hpp:47 */
#define REFRESH_EVERY 256u   /* src/likelihood.cpp:82 */

static _Thread_local char g_err[512];

const char* orc_last_error(void) { return g_err; }

static int fail(int code, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof g_err, fmt, ap);
    va_end(ap);
    return code;
}

/* std::max / std::min semantics (return the first argument on ties/NaN). */
static double dmax(double a, double b) { return a < b ? b : a; }
static double dmin(double a, double b) { return b < a ? b : a; }

/* ------------------------------------------------------------------ design */

typedef struct {
    const int32_t* stratum;
    const double* time;
} sort_ctx;

/* Comparator of data.cpp:77-81: stratum ascending, then time descending. */
static int key_less(const sort_ctx* c, int64_t a, int64_t b) {
    if (c->stratum[a] != c->stratum[b]) return c->stratum[a] < c->stratum[b];
    return c->time[a] > c->time[b];
}

/* Stable merge sort (std::stable_sort semantics: equal keys keep input order). */
static void merge_sort(const sort_ctx* c, int64_t* a, int64_t* tmp, int64_t n) {
    if (n < 2) return;
    const int64_t mid = n / 2;
    merge_sort(c, a, tmp, mid);
    merge_sort(c, a + mid, tmp, n - mid);
    int64_t i = 0, j = mid, o = 0;
    while (i < mid && j < n) {
        if (key_less(c, a[j], a[i]))
            tmp[o++] = a[j++];
        else
            tmp[o++] = a[i++];
    }
    while (i < mid) tmp[o++] = a[i++];
    while (j < n) tmp[o++] = a[j++];
    memcpy(a, tmp, (size_t)n * sizeof(int64_t));
}

typedef struct {
    int64_t key;
    int64_t src;
} pair64;

static int pair_cmp(const void* x, const void* y) {
    const pair64* a = (const pair64*)x;
    const pair64* b = (const pair64*)y;
    return (a->key > b->key) - (a->key < b->key);
}

int orc_build_sorted_design(int64_t n, const double* time, const uint8_t* event,
                            const int32_t* stratum, int64_t p, const int64_t* col_ptr,
                            const int64_t* row_idx, const double* values, int64_t* perm,
                            uint8_t* head, int64_t* tie_end, int64_t* offsets, int32_t* k_out,
                            double* s_time, uint8_t* s_event, int32_t* s_stratum,
                            int64_t* s_row_idx, double* s_values) {
    /* validate_invariants, data.cpp:27-66 */
    int32_t k = 0;
    for (int64_t i = 0; i < n; ++i)
        if (stratum[i] > k) k = stratum[i];
    if (n > 0 && k < 1) return fail(ORC_VALIDATION, "dataset has no strata");
    int64_t* per = (int64_t*)calloc((size_t)k + 1, sizeof(int64_t));
    for (int64_t i = 0; i < n; ++i) {
        const double t = time[i];
        if (!isfinite(t) || t < 0.0) {
            free(per);
            return fail(ORC_VALIDATION, "negative or non-finite time at row %lld", (long long)i);
        }
        if (event[i] > 1) {
            free(per);
            return fail(ORC_VALIDATION, "event indicator must be 0 or 1 at row %lld", (long long)i);
        }
        if (stratum[i] < 1 || stratum[i] > k) {
            free(per);
            return fail(ORC_VALIDATION, "stratum label out of range at row %lld", (long long)i);
        }
        ++per[stratum[i]];
    }
    for (int32_t s = 1; s <= k; ++s) {
        if (per[s] == 0) {
            free(per);
            return fail(ORC_VALIDATION, "stratum %d has zero rows", s);
        }
    }
    free(per);
    for (int64_t j = 0; j < p; ++j) {
        int64_t prev = -1;
        for (int64_t t = col_ptr[j]; t < col_ptr[j + 1]; ++t) {
            const int64_t r = row_idx[t];
            if (r <= prev)
                return fail(ORC_VALIDATION, "column x%lld row indices must be strictly increasing",
                            (long long)(j + 1));
            if (r < 0 || r >= n)
                return fail(ORC_VALIDATION, "column x%lld row index out of range", (long long)(j + 1));
            if (values && !isfinite(values[t]))
                return fail(ORC_VALIDATION, "column x%lld has a non-finite value", (long long)(j + 1));
            prev = r;
        }
    }
    if (n == 0) return fail(ORC_VALIDATION, "dataset has no rows");

    /* stable sort of the row permutation, data.cpp:75-81 */
    for (int64_t i = 0; i < n; ++i) perm[i] = i;
    int64_t* tmp = (int64_t*)malloc((size_t)n * sizeof(int64_t));
    sort_ctx c = {stratum, time};
    merge_sort(&c, perm, tmp, n);
    int64_t* inverse = tmp; /* reuse: inverse[perm[s]] = s, data.cpp:83-84 */
    for (int64_t s = 0; s < n; ++s) inverse[perm[s]] = s;

    for (int64_t s = 0; s < n; ++s) { /* data.cpp:91-97 */
        const int64_t r = perm[s];
        s_time[s] = time[r];
        s_event[s] = event[r];
        s_stratum[s] = stratum[r];
    }

    /* per-column CSC re-index, data.cpp:102-119 (rows distinct -> keys distinct) */
    int64_t maxnnz = 0;
    for (int64_t j = 0; j < p; ++j)
        if (col_ptr[j + 1] - col_ptr[j] > maxnnz) maxnnz = col_ptr[j + 1] - col_ptr[j];
    pair64* pairs = (pair64*)malloc((size_t)(maxnnz > 0 ? maxnnz : 1) * sizeof(pair64));
    for (int64_t j = 0; j < p; ++j) {
        const int64_t b = col_ptr[j], m = col_ptr[j + 1] - b;
        for (int64_t t = 0; t < m; ++t) {
            pairs[t].key = inverse[row_idx[b + t]];
            pairs[t].src = b + t;
        }
        qsort(pairs, (size_t)m, sizeof(pair64), pair_cmp);
        for (int64_t t = 0; t < m; ++t) {
            s_row_idx[b + t] = pairs[t].key;
            s_values[b + t] = values ? values[pairs[t].src] : 1.0;
        }
    }
    free(pairs);
    free(tmp);

    /* heads and stratum offsets, data.cpp:121-131 */
    int64_t nk = 0;
    memset(head, 0, (size_t)n);
    head[0] = 1;
    offsets[nk++] = 0;
    for (int64_t s = 1; s < n; ++s) {
        if (s_stratum[s] != s_stratum[s - 1]) {
            head[s] = 1;
            offsets[nk++] = s;
        }
    }
    offsets[nk] = n;
    *k_out = (int32_t)nk;

    /* tie groups, data.cpp:133-145 */
    int64_t s = 0;
    while (s < n) {
        int64_t e = s;
        while (e + 1 < n && s_stratum[e + 1] == s_stratum[s] && s_time[e + 1] == s_time[s]) ++e;
        for (int64_t i = s; i <= e; ++i) tie_end[i] = e;
        s = e + 1;
    }
    return ORC_OK;
}

/* ------------------------------------------------------------------ scans */

/* segmented_inclusive_scan, scan.cpp:124-190, run serially chunk by chunk. */
int orc_segmented_scan(int64_t n, const double* values, const uint8_t* flags, int64_t chunk,
                       double* out) {
    if (n == 0) return fail(ORC_VALIDATION, "empty scan input");
    if (!flags[0]) return fail(ORC_VALIDATION, "first element must head a segment");
    if (chunk < 1) return fail(ORC_VALIDATION, "chunk_size must be >= 1");
    const int64_t count = (n + chunk - 1) / chunk;
    uint8_t* agg_f = (uint8_t*)malloc((size_t)count);
    double* agg_v = (double*)malloc((size_t)count * sizeof(double));
    int64_t* first_head = (int64_t*)malloc((size_t)count * sizeof(int64_t));
    int64_t bad = -1;
    for (int64_t c = 0; c < count; ++c) { /* pass 1, scan.cpp:140-163 */
        const int64_t begin = c * chunk;
        const int64_t end = begin + chunk < n ? begin + chunk : n;
        const int64_t length = end - begin;
        double run = 0.0;
        int64_t h = length;
        for (int64_t i = begin; i < end; ++i) {
            const double v = values[i];
            if (!isfinite(v)) {
                if (bad < 0 || i < bad) bad = i;
                break;
            }
            const int f = flags[i] != 0;
            if (h == length && f) h = i - begin;
            run = run * (double)(1 - f) + v;
            out[i] = run;
        }
        agg_f[c] = h < length ? 1 : 0;
        agg_v[c] = run;
        first_head[c] = h;
    }
    if (bad >= 0) {
        free(agg_f);
        free(agg_v);
        free(first_head);
        return fail(ORC_VALIDATION, "non-finite input at index %lld", (long long)bad);
    }
    /* pass 2: serial fold of chunk aggregates with combine(), scan.cpp:166-171 */
    uint8_t rf = 0;
    double rv = 0.0;
    for (int64_t c = 0; c < count; ++c) {
        const double carry = rv;
        rv = agg_f[c] ? agg_v[c] : rv + agg_v[c]; /* combine, scan.hpp:41-44 */
        rf = (uint8_t)(rf | agg_f[c]);
        agg_v[c] = carry; /* reuse as carry[c] */
    }
    (void)rf;
    /* pass 3: carry only left of each chunk's first head, scan.cpp:176-182 */
    for (int64_t c = 1; c < count; ++c) {
        const int64_t begin = c * chunk;
        const int64_t stop = begin + first_head[c];
        for (int64_t i = begin; i < stop; ++i) out[i] += agg_v[c];
    }
    free(agg_f);
    free(agg_v);
    free(first_head);
    return ORC_OK;
}

/* inclusive_scan, scan.cpp:63-115 */
int orc_inclusive_scan(int64_t n, const double* values, int64_t chunk, double* out) {
    if (n == 0) return fail(ORC_VALIDATION, "empty scan input");
    if (chunk < 1) return fail(ORC_VALIDATION, "chunk_size must be >= 1");
    const int64_t count = (n + chunk - 1) / chunk;
    double* agg = (double*)malloc((size_t)count * sizeof(double));
    for (int64_t c = 0; c < count; ++c) {
        const int64_t begin = c * chunk;
        const int64_t end = begin + chunk < n ? begin + chunk : n;
        double run = 0.0;
        for (int64_t i = begin; i < end; ++i) {
            if (!isfinite(values[i])) {
                free(agg);
                return fail(ORC_VALIDATION, "non-finite input at index %lld", (long long)i);
            }
            run += values[i];
            out[i] = run;
        }
        agg[c] = run;
    }
    double run = 0.0;
    for (int64_t c = 0; c < count; ++c) {
        const double carry = run;
        run += agg[c];
        agg[c] = carry;
    }
    for (int64_t c = 1; c < count; ++c) {
        const int64_t begin = c * chunk;
        const int64_t end = begin + chunk < n ? begin + chunk : n;
        for (int64_t i = begin; i < end; ++i) out[i] += agg[c];
    }
    free(agg);
    return ORC_OK;
}

/* ------------------------------------------------------------------ state */

/* refresh_xbeta, likelihood.cpp:31-58 (release build: no drift assert) */
static int refresh(const orc_design* d, const double* beta, double* xbeta, double* exp_xbeta) {
    memset(xbeta, 0, (size_t)d->n * sizeof(double));
    for (int64_t j = 0; j < d->p; ++j) {
        const double b = beta[j];
        if (b == 0.0) continue;
        for (int64_t t = d->col_ptr[j]; t < d->col_ptr[j + 1]; ++t)
            xbeta[d->row_idx[t]] += d->values[t] * b;
    }
    for (int64_t s = 0; s < d->n; ++s) {
        const double v = xbeta[s];
        if (!isfinite(v) || fabs(v) > LP_BOUND) /* check_linear_predictor, likelihood.cpp:12-15 */
            return fail(ORC_NUMERIC, "linear predictor overflow at row %lld", (long long)s);
        exp_xbeta[s] = exp(v);
    }
    return ORC_OK;
}

/* make_state, likelihood.cpp:19-29 */
int orc_make_state(const orc_design* d, const double* beta, double* xbeta, double* exp_xbeta) {
    return refresh(d, beta, xbeta, exp_xbeta);
}

/* update_xbeta, likelihood.cpp:60-83 */
int orc_update_xbeta(const orc_design* d, double* beta, double* xbeta, double* exp_xbeta,
                     uint32_t* updates, int64_t j, double delta) {
    if (j < 0 || j >= d->p) return fail(ORC_VALIDATION, "covariate index out of range");
    if (!isfinite(delta)) return fail(ORC_NUMERIC, "non-finite coordinate step");
    const int64_t b = d->col_ptr[j], e = d->col_ptr[j + 1];
    if (delta == 0.0 || e == b) {
        beta[j] += delta;
        return ORC_OK;
    }
    for (int64_t t = b; t < e; ++t) {
        const double next = xbeta[d->row_idx[t]] + d->values[t] * delta;
        if (!isfinite(next) || fabs(next) > LP_BOUND) return fail(ORC_NUMERIC, "step overflow");
    }
    for (int64_t t = b; t < e; ++t) {
        const int64_t s = d->row_idx[t];
        xbeta[s] += d->values[t] * delta;
        exp_xbeta[s] = exp(xbeta[s]);
    }
    beta[j] += delta;
    if (++*updates >= REFRESH_EVERY) {
        *updates = 0;
        return refresh(d, beta, xbeta, exp_xbeta);
    }
    return ORC_OK;
}

/* ------------------------------------------------------------------ likelihood */

/* log_partial_likelihood, likelihood.cpp:93-121; the event-row sum is
 * chunked_transform_sum (scan.hpp:115-154): serial per chunk, chunk partials
 * folded in order. */
int orc_log_partial_likelihood(const orc_design* d, const double* xbeta, const double* exp_xbeta,
                               int64_t chunk, double* ll) {
    const int64_t n = d->n;
    double* sd = (double*)malloc((size_t)n * sizeof(double));
    int rc = orc_segmented_scan(n, exp_xbeta, d->head, chunk, sd);
    if (rc) {
        free(sd);
        return rc;
    }
    double total = 0.0;
    for (int64_t begin = 0; begin < n; begin += chunk) {
        const int64_t end = begin + chunk < n ? begin + chunk : n;
        double sa = 0.0;
        for (int64_t i = begin; i < end; ++i) {
            double v = 0.0;
            if (d->event[i]) v = xbeta[i] - log(sd[d->tie_end[i]]);
            sa += v;
        }
        total += sa;
    }
    if (!isfinite(total)) {
        for (int64_t i = 0; i < n; ++i) {
            if (!d->event[i]) continue;
            const double den = sd[d->tie_end[i]];
            if (!(den > 0.0) || !isfinite(den)) {
                free(sd);
                return fail(ORC_INTERNAL, "risk-set sum not positive at sorted row %lld",
                            (long long)i);
            }
        }
        free(sd);
        return fail(ORC_NUMERIC, "non-finite log partial likelihood");
    }
    free(sd);
    *ll = total;
    return ORC_OK;
}

/* gradient_hessian, likelihood.cpp:129-189 */
int orc_gradient_hessian(const orc_design* d, const double* exp_xbeta, int64_t j, int64_t chunk,
                         double* g, double* h) {
    const int64_t n = d->n;
    if (j < 0 || j >= d->p) return fail(ORC_VALIDATION, "covariate index out of range");
    double* n1 = (double*)calloc((size_t)n, sizeof(double));
    double* n2 = (double*)calloc((size_t)n, sizeof(double));
    double* sd = (double*)malloc((size_t)n * sizeof(double));
    double* s1 = (double*)malloc((size_t)n * sizeof(double));
    double* s2 = (double*)malloc((size_t)n * sizeof(double));
    double linear = 0.0;
    for (int64_t t = d->col_ptr[j]; t < d->col_ptr[j + 1]; ++t) { /* :141-148 */
        const int64_t s = d->row_idx[t];
        const double x = d->values[t];
        const double e = exp_xbeta[s];
        n1[s] = x * e;
        n2[s] = x * x * e;
        linear += x * (double)d->event[s];
    }
    int rc = orc_segmented_scan(n, exp_xbeta, d->head, chunk, sd);
    if (!rc) rc = orc_segmented_scan(n, n1, d->head, chunk, s1);
    if (!rc) rc = orc_segmented_scan(n, n2, d->head, chunk, s2);
    if (rc) goto done;
    {
        double ta = 0.0, tb = 0.0; /* chunked_transform_sum2, scan.hpp:115-144 */
        for (int64_t begin = 0; begin < n; begin += chunk) {
            const int64_t end = begin + chunk < n ? begin + chunk : n;
            double sa = 0.0, sb = 0.0;
            for (int64_t i = begin; i < end; ++i) { /* :165-175 */
                const double w = (double)d->event[i];
                const int64_t gi = d->tie_end[i];
                const double den = sd[gi];
                const double r1 = s1[gi] / den;
                const double r2 = s2[gi] / den;
                sa += w * r1;
                sb += w * (r2 - r1 * r1);
            }
            ta += sa;
            tb += sb;
        }
        const double gg = -linear + ta, hh = tb;
        if (!isfinite(gg) || !isfinite(hh)) { /* :178-187 */
            for (int64_t i = 0; i < n; ++i) {
                if (!d->event[i]) continue;
                const double den = sd[d->tie_end[i]];
                if (!(den > 0.0) || !isfinite(den)) {
                    rc = fail(ORC_INTERNAL, "risk-set sum not positive at sorted row %lld",
                              (long long)i);
                    goto done;
                }
            }
            rc = fail(ORC_NUMERIC, "non-finite gradient/Hessian for covariate x%lld",
                      (long long)(j + 1));
            goto done;
        }
        *g = gg;
        *h = hh;
    }
done:
    free(n1);
    free(n2);
    free(sd);
    free(s1);
    free(s2);
    return rc;
}

/* naive_gradient_hessian, likelihood.cpp:191-224 */
int orc_naive_gradient_hessian(const orc_design* d, const double* exp_xbeta, int64_t j,
                               double* g, double* h) {
    if (j < 0 || j >= d->p) return fail(ORC_VALIDATION, "covariate index out of range");
    double* xj = (double*)calloc((size_t)d->n, sizeof(double));
    for (int64_t t = d->col_ptr[j]; t < d->col_ptr[j + 1]; ++t) xj[d->row_idx[t]] = d->values[t];
    double og = 0.0, oh = 0.0;
    for (int32_t k = 0; k < d->k; ++k) {
        const int64_t b = d->offsets[k], e = d->offsets[k + 1];
        for (int64_t i = b; i < e; ++i) {
            if (!d->event[i]) continue;
            double den = 0.0, num1 = 0.0, num2 = 0.0;
            for (int64_t r = b; r < e; ++r) {
                if (d->time[r] < d->time[i]) continue;
                const double ex = exp_xbeta[r];
                const double x = xj[r];
                den += ex;
                num1 += x * ex;
                num2 += x * x * ex;
            }
            og += num1 / den - xj[i];
            oh += num2 / den - (num1 / den) * (num1 / den);
        }
    }
    free(xj);
    *g = og;
    *h = oh;
    return ORC_OK;
}

/* naive_log_partial_likelihood, likelihood.cpp:226-244 */
int orc_naive_log_partial_likelihood(const orc_design* d, const double* xbeta,
                                     const double* exp_xbeta, double* ll) {
    double out = 0.0;
    for (int32_t k = 0; k < d->k; ++k) {
        const int64_t b = d->offsets[k], e = d->offsets[k + 1];
        for (int64_t i = b; i < e; ++i) {
            if (!d->event[i]) continue;
            double den = 0.0;
            for (int64_t r = b; r < e; ++r)
                if (d->time[r] >= d->time[i]) den += exp_xbeta[r];
            out += xbeta[i] - log(den);
        }
    }
    *ll = out;
    return ORC_OK;
}

/* ------------------------------------------------------------------ optimizer */

/* newton_step, optimizer.cpp:32-41 */
int orc_newton_step(double g1, double g2, double* step, int* flat) {
    if (!isfinite(g1) || !isfinite(g2))
        return fail(ORC_NUMERIC, "non-finite gradient or Hessian in Newton step");
    if (flat) *flat = 0;
    if (g2 < FLAT_CURVATURE) {
        if (flat) *flat = 1;
        *step = 0.0;
        return ORC_OK;
    }
    *step = -g1 / g2;
    return ORC_OK;
}

/* apply_trust_region, optimizer.cpp:43-49 */
int orc_apply_trust_region(double proposed, double trust, double* applied, double* next_trust) {
    if (!isfinite(proposed) || !isfinite(trust))
        return fail(ORC_NUMERIC, "non-finite trust-region inputs");
    const double magnitude = dmin(fabs(proposed), trust);
    const double a = copysign(magnitude, proposed);
    *applied = a;
    if (next_trust) *next_trust = dmax(2.0 * fabs(a), trust * 0.5);
    return ORC_OK;
}

/* l1_coordinate_update, optimizer.cpp:51-78 */
int orc_l1_coordinate_update(double g1, double g2, double beta_j, double gamma_j, double* step,
                             int* skipped, int* flat) {
    int fl = 0, rc;
    *skipped = 0;
    *step = 0.0;
    if (gamma_j == 0.0) {
        rc = orc_newton_step(g1, g2, step, &fl);
        if (flat) *flat = fl;
        return rc;
    }
    if (beta_j != 0.0) {
        const double penalized = g1 + (beta_j > 0.0 ? gamma_j : -gamma_j);
        rc = orc_newton_step(penalized, g2, step, &fl);
        if (rc) return rc;
        if ((beta_j > 0.0 && beta_j + *step < 0.0) || (beta_j < 0.0 && beta_j + *step > 0.0))
            *step = -beta_j;
        if (flat) *flat = fl;
        return ORC_OK;
    }
    const double up = g1 + gamma_j;
    const double down = -g1 + gamma_j;
    if (up < 0.0 && down < 0.0)
        return fail(ORC_INTERNAL, "both directional derivatives negative at the origin");
    if (up >= 0.0 && down >= 0.0) {
        *skipped = 1;
        if (flat) *flat = 0;
        return ORC_OK;
    }
    const double penalized = up < 0.0 ? g1 + gamma_j : g1 - gamma_j;
    rc = orc_newton_step(penalized, g2, step, &fl);
    if (flat) *flat = fl;
    return rc;
}

/* PenaltySpec::value, optimizer.cpp:18-22; with an L2 (ridge / Gaussian)
 * prior l2 (NOT in the reference: BASELINE config 1's "L2 prior", parity
 * unpinned) the value adds sum_j l2_j beta_j^2 / 2 after the L1 sum. */
static double penalty_value(const double* gamma, const double* l2, const double* beta, int64_t p) {
    double total = 0.0;
    for (int64_t j = 0; j < p; ++j) total += gamma[j] * fabs(beta[j]);
    if (l2)
        for (int64_t j = 0; j < p; ++j) total += 0.5 * l2[j] * beta[j] * beta[j];
    return total;
}

/* Elastic-net coordinate rule (extension, not in the reference): the ridge
 * term adds l2*beta to g' and l2 to g'', then the reference's L1 rule
 * (optimizer.cpp:51-78) runs on the penalised pair. l2 = 0 is the reference
 * rule bit for bit (g1 + 0*beta == g1, g2 + 0 == g2). */
int orc_coordinate_update(double g1, double g2, double beta_j, double gamma_j, double l2_j,
                          double* step, int* skipped, int* flat) {
    return orc_l1_coordinate_update(g1 + l2_j * beta_j, g2 + l2_j, beta_j, gamma_j, step, skipped,
                                    flat);
}

/* run_ccd + ccd_fit, optimizer.cpp:82-160 */
int orc_ccd_fit(const orc_design* d, const double* gamma, int max_cycles, double tolerance,
                double initial_trust, int64_t chunk, const double* initial_beta,
                double* beta_out, double* trace_out, int* trace_len, int* cycles,
                int* converged, double* trust_out, int* n_warnings) {
    return orc_ccd_fit_prior(d, gamma, NULL, max_cycles, tolerance, initial_trust, chunk,
                             initial_beta, beta_out, trace_out, trace_len, cycles, converged,
                             trust_out, n_warnings);
}

/* The same with an optional L2 prior l2[p] (NULL: none). */
int orc_ccd_fit_prior(const orc_design* d, const double* gamma, const double* l2, int max_cycles,
                      double tolerance, double initial_trust, int64_t chunk,
                      const double* initial_beta, double* beta_out, double* trace_out,
                      int* trace_len, int* cycles, int* converged, double* trust_out,
                      int* n_warnings) {
    const int64_t p = d->p, n = d->n;
    for (int64_t j = 0; j < p; ++j) /* PenaltySpec::validate, optimizer.cpp:24-30 */
        if (!isfinite(gamma[j]) || gamma[j] < 0.0)
            return fail(ORC_VALIDATION, "penalty weights must be finite and non-negative");
    for (int64_t j = 0; l2 && j < p; ++j)
        if (!isfinite(l2[j]) || l2[j] < 0.0)
            return fail(ORC_VALIDATION, "L2 prior weights must be finite and non-negative");
    if (max_cycles < 1) return fail(ORC_VALIDATION, "max_cycles must be >= 1");
    if (!(tolerance > 0.0)) return fail(ORC_VALIDATION, "tolerance must be positive");
    if (!(initial_trust > 0.0)) return fail(ORC_VALIDATION, "initial_trust must be positive");

    double* beta = beta_out;
    for (int64_t j = 0; j < p; ++j) beta[j] = initial_beta ? initial_beta[j] : 0.0;
    double* xb = (double*)malloc((size_t)n * sizeof(double));
    double* ex = (double*)malloc((size_t)n * sizeof(double));
    double* trust = trust_out;
    uint32_t updates = 0;
    int warnings = 0, rc;
    int len = 0;
    *cycles = 0;
    *converged = 0;
    rc = orc_make_state(d, beta, xb, ex);
    if (rc) goto out;
    for (int64_t j = 0; j < p; ++j) trust[j] = initial_trust;
    double ll;
    rc = orc_log_partial_likelihood(d, xb, ex, chunk, &ll);
    if (rc) goto out;
    double objective = -ll + penalty_value(gamma, l2, beta, p);
    trace_out[len++] = objective;

    for (int cycle = 1; cycle <= max_cycles; ++cycle) {
        double max_step = 0.0;
        for (int64_t j = 0; j < p; ++j) {
            double g = 0.0, h = 0.0;
            if (d->col_ptr[j + 1] > d->col_ptr[j]) {
                rc = orc_gradient_hessian(d, ex, j, chunk, &g, &h);
                if (rc) goto out;
            }
            double step;
            int skipped, flat;
            rc = orc_coordinate_update(g, h, beta[j], gamma[j], l2 ? l2[j] : 0.0, &step, &skipped, &flat);
            if (rc) goto out;
            double applied;
            rc = orc_apply_trust_region(step, trust[j], &applied, NULL);
            if (rc) goto out;
            int halvings = 0;
            while (applied != 0.0) { /* :110-123 */
                rc = orc_update_xbeta(d, beta, xb, ex, &updates, j, applied);
                if (rc == ORC_OK) break;
                if (rc != ORC_NUMERIC) goto out;
                rc = ORC_OK;
                if (++halvings > 10) {
                    ++warnings;
                    applied = 0.0;
                    break;
                }
                applied *= 0.5;
            }
            trust[j] = dmax(2.0 * fabs(applied), trust[j] * 0.5); /* :124 */
            max_step = dmax(max_step, fabs(applied));
        }
        rc = orc_log_partial_likelihood(d, xb, ex, chunk, &ll);
        if (rc) goto out;
        const double next = -ll + penalty_value(gamma, l2, beta, p);
        if (next > objective + 1e-8) {
            rc = fail(ORC_NUMERIC, "monotonicity violated: objective rose from %f to %f", objective,
                      next);
            goto out;
        }
        objective = next;
        trace_out[len++] = objective;
        *cycles = cycle;
        if (max_step < tolerance) {
            *converged = 1;
            break;
        }
    }
out:
    *trace_len = len;
    *n_warnings = warnings;
    free(xb);
    free(ex);
    return rc;
}

/* gamma_max, resample.cpp:42-55 */
int orc_gamma_max(const orc_design* d, int64_t chunk, double* out) {
    double* beta = (double*)calloc((size_t)d->p, sizeof(double));
    double* xb = (double*)malloc((size_t)d->n * sizeof(double));
    double* ex = (double*)malloc((size_t)d->n * sizeof(double));
    int rc = orc_make_state(d, beta, xb, ex);
    double best = 0.0;
    for (int64_t j = 0; !rc && j < d->p; ++j) {
        if (d->col_ptr[j + 1] == d->col_ptr[j]) continue;
        double g, h;
        rc = orc_gradient_hessian(d, ex, j, chunk, &g, &h);
        if (!rc) best = dmax(best, fabs(g));
    }
    free(beta);
    free(xb);
    free(ex);
    if (!rc) *out = best;
    return rc;
}
