// Drop-in replacement for the reference's proj/src/likelihood.cpp,
// proj/src/optimizer.cpp and proj/src/scan.cpp: the same `namespace stratcox` symbols
// (proj/include/stratcox/likelihood.hpp, optimizer.hpp) implemented over the
// C-ABI of libstratcox_b200.so (include/stratcox_b200.h).
//
// Build it against the reference headers and link it in place of the two
// reference translation units (oracle/Makefile target
// `dropin` builds the reference's own acceptance suite this way).
//
// Contexts: one scx_ctx per calling thread (thread_local), because the
// reference calls ccd_fit concurrently from OpenMP threads
// (proj/src/resample.cpp:121,207). The uploaded design is cached per thread
// and keyed by a 64-bit hash of its CONTENT (offsets, tie ends, events, times
// and every column's rows and values) plus its shape: the reference builds a
// stack-local SortedDesign per bootstrap replicate and per fold
// (resample.cpp:129-130,218-219), so an address can be reused by a different
// design of the same shape and identity alone would return a stale upload. A
// CoefficientState passed by the caller is uploaded per call (parity
// boundary), while ccd_fit keeps its whole loop on the device.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#ifdef _OPENMP
#include <omp.h>
#endif

#include "stratcox/likelihood.hpp"
#include "stratcox/optimizer.hpp"
#include "stratcox/scan.hpp"
#include "stratcox_b200.h"

namespace stratcox {

namespace {

struct ThreadCtx {
    scx_ctx* h = nullptr;
    bool valid = false;
    uint64_t hash = 0;
    std::size_t n = 0, p = 0, nnz = 0;
    ~ThreadCtx() {
        if (h) scx_destroy(h);
    }
};

thread_local ThreadCtx g_ctx;

// Replace the C-ABI's default covariate name "xN" with the design's own.
std::string with_names(std::string msg, const SortedDesign* d) {
    const std::string tag = "for covariate x";
    const auto pos = msg.find(tag);
    if (d && pos != std::string::npos) {
        const std::size_t j = std::stoul(msg.substr(pos + tag.size())) - 1;
        msg = msg.substr(0, pos) + "for covariate " + d->data.covariate_name(j);
    }
    return msg;
}

[[noreturn]] void raise(scx_status s, const std::string& msg) {
    switch (s) {
        case SCX_ERR_VALIDATION: throw validation_error(msg);
        case SCX_ERR_NUMERIC: throw numeric_error(msg);
        case SCX_ERR_INTERNAL: throw internal_error(msg);
        default: throw error("CUDA backend: " + msg);
    }
}

void check(scx_status s, const SortedDesign* d = nullptr) {
    if (s != SCX_OK) raise(s, with_names(scx_last_error(g_ctx.h), d));
}

void check_rule(scx_status s) {
    if (s != SCX_OK) raise(s, scx_rule_error());
}

// 64-bit content hash: four independent multiply-rotate lanes over 8-byte
// words (a tail is zero-padded), folded with the byte count.
struct Hasher {
    uint64_t a = 0x9e3779b97f4a7c15ull, b = 0xc2b2ae3d27d4eb4full, c = 0x165667b19e3779f9ull,
             e = 0x27d4eb2f165667c5ull;
    uint64_t bytes = 0;
    static uint64_t mix(uint64_t h, uint64_t w) {
        h ^= w * 0x87c37b91114253d5ull;
        h = (h << 31) | (h >> 33);
        return h * 0x4cf5ad432745937full + 0x52dce729ull;
    }
    void add(const void* p, std::size_t nbytes) {
        const unsigned char* s = static_cast<const unsigned char*>(p);
        std::size_t i = 0;
        for (; i + 32 <= nbytes; i += 32) {
            uint64_t w[4];
            std::memcpy(w, s + i, 32);
            a = mix(a, w[0]);
            b = mix(b, w[1]);
            c = mix(c, w[2]);
            e = mix(e, w[3]);
        }
        for (; i < nbytes; i += 8) {
            uint64_t w = 0;
            std::memcpy(&w, s + i, std::min<std::size_t>(8, nbytes - i));
            a = mix(a, w);
        }
        bytes += nbytes;
        b = mix(b, nbytes);
    }
    uint64_t value() const { return mix(mix(mix(mix(a, b), c), e), bytes); }
};

uint64_t content_hash(const SortedDesign& d) {
    Hasher h;
    h.add(d.stratum_offsets.data(), d.stratum_offsets.size() * sizeof(d.stratum_offsets[0]));
    h.add(d.tie_group_end.data(), d.tie_group_end.size() * sizeof(d.tie_group_end[0]));
    h.add(d.data.event.data(), d.data.event.size() * sizeof(d.data.event[0]));
    h.add(d.data.time.data(), d.data.time.size() * sizeof(d.data.time[0]));
    for (const auto& c : d.data.columns) {
        h.add(c.rows.data(), c.rows.size() * sizeof(c.rows[0]));
        h.add(c.values.data(), c.values.size() * sizeof(c.values[0]));
    }
    return h.value();
}

scx_ctx* ctx_for(const SortedDesign& d) {
    std::size_t nnz = 0;
    for (const auto& c : d.data.columns) nnz += c.nnz();
    const uint64_t hash = content_hash(d);
    ThreadCtx& t = g_ctx;
    if (t.h && t.valid && t.hash == hash && t.n == d.n_rows() && t.p == d.n_covariates() &&
        t.nnz == nnz)
        return t.h;
    if (!t.h) {
        if (scx_create(0, &t.h) != SCX_OK) {
            t.h = nullptr;
            throw error("CUDA backend: no usable sm_100 device");
        }
    }
    std::vector<int64_t> col_ptr(d.n_covariates() + 1, 0);
    std::vector<int64_t> rows;
    std::vector<double> values;
    rows.reserve(nnz);
    values.reserve(nnz);
    for (std::size_t j = 0; j < d.n_covariates(); ++j) {
        const SparseColumn& c = d.data.columns[j];
        rows.insert(rows.end(), c.rows.begin(), c.rows.end());
        values.insert(values.end(), c.values.begin(), c.values.end());
        col_ptr[j + 1] = static_cast<int64_t>(rows.size());
    }
    t.valid = false;
    check(scx_upload_design(t.h, static_cast<int64_t>(d.n_rows()), d.n_strata(),
                            d.stratum_offsets.data(), d.data.event.data(), d.tie_group_end.data(),
                            static_cast<int64_t>(d.n_covariates()), col_ptr.data(), rows.data(),
                            values.data()),
          &d);
    t.valid = true;
    t.hash = hash;
    t.n = d.n_rows();
    t.p = d.n_covariates();
    t.nnz = nnz;
    return t.h;
}

void put_state(scx_ctx* h, const SortedDesign& d, const CoefficientState& st) {
    check(scx_set_state(h, st.beta.data(), st.xbeta.data(), st.exp_xbeta.data(),
                        st.updates_since_refresh),
          &d);
}

void get_state(scx_ctx* h, const SortedDesign& d, CoefficientState& st) {
    st.beta.resize(d.n_covariates());
    st.xbeta.resize(d.n_rows());
    st.exp_xbeta.resize(d.n_rows());
    uint32_t u = 0;
    check(scx_get_state(h, st.beta.data(), st.xbeta.data(), st.exp_xbeta.data(), &u), &d);
    st.updates_since_refresh = u;
}

}  // namespace

// ------------------------------------------------------------------ scan.hpp
// Replaces proj/src/scan.cpp: the scans run on the device (same flag-value
// tile scan as the likelihood kernels); the chunk-runner and config helpers
// stay host utilities.

int default_worker_count() {
#ifdef _OPENMP
    return std::max(1, omp_get_max_threads());
#else
    return 1;
#endif
}

void validate(const ExecutionConfig& config) {
    if (config.chunk_size < 1) throw validation_error("chunk_size must be >= 1");
    if (config.worker_count < 1) throw validation_error("worker_count must be >= 1");
}

namespace detail {
void run_chunks(const ChunkPlan& plan, int worker_count, void* ctx,
                void (*body)(void*, std::int64_t)) {
    (void)worker_count;
    for (std::int64_t c = 0; c < plan.count; ++c) body(ctx, c);
}
}  // namespace detail

namespace {
scx_ctx* scan_ctx() {
    ThreadCtx& t = g_ctx;
    if (!t.h && scx_create(0, &t.h) != SCX_OK) {
        t.h = nullptr;
        throw error("CUDA backend: no usable sm_100 device");
    }
    return t.h;
}
}  // namespace

void segmented_inclusive_scan(std::span<const double> values, std::span<const std::uint8_t> flags,
                              std::span<double> out, const ExecutionConfig& config,
                              ScanCounters* counters) {
    if (values.empty()) throw validation_error("empty scan input");
    if (flags.size() != values.size())
        throw validation_error("values and flags must have equal length");
    if (out.size() != values.size()) throw validation_error("scan output size mismatch");
    if (!flags[0]) throw validation_error("first element must head a segment");
    validate(config);
    check(scx_segmented_inclusive_scan(scan_ctx(), static_cast<int64_t>(values.size()),
                                       values.data(), flags.data(), out.data()));
    if (counters) counters->elements.fetch_add(values.size(), std::memory_order_relaxed);
}

std::vector<double> segmented_inclusive_scan(std::span<const double> values,
                                             std::span<const std::uint8_t> flags,
                                             const ExecutionConfig& config,
                                             ScanCounters* counters) {
    std::vector<double> out(values.size());
    segmented_inclusive_scan(values, flags, out, config, counters);
    return out;
}

void inclusive_scan(std::span<const double> values, std::span<double> out,
                    const ExecutionConfig& config, ScanCounters* counters) {
    if (values.empty()) throw validation_error("empty scan input");
    if (out.size() != values.size()) throw validation_error("scan output size mismatch");
    std::vector<std::uint8_t> flags(values.size(), 0);
    flags[0] = 1;
    segmented_inclusive_scan(values, flags, out, config, counters);
}

std::vector<double> inclusive_scan(std::span<const double> values, const ExecutionConfig& config,
                                   ScanCounters* counters) {
    std::vector<double> out(values.size());
    inclusive_scan(values, out, config, counters);
    return out;
}

double chunked_sum(std::span<const double> values, const ExecutionConfig& config,
                   ScanCounters* counters) {
    return chunked_transform_sum(
        values.size(), [&](std::size_t i) { return values[i]; }, config, counters);
}

// ------------------------------------------------------------------ likelihood.hpp

CoefficientState make_state(const SortedDesign& design, std::span<const double> beta) {
    if (beta.size() != design.n_covariates())
        throw validation_error("beta length does not match covariate count");
    scx_ctx* h = ctx_for(design);
    check(scx_make_state(h, beta.data()), &design);
    CoefficientState st;
    get_state(h, design, st);
    st.updates_since_refresh = 0;
    return st;
}

void refresh_xbeta(const SortedDesign& design, CoefficientState& state) {
    scx_ctx* h = ctx_for(design);
    put_state(h, design, state);
    check(scx_refresh_xbeta(h), &design);
    get_state(h, design, state);
}

void update_xbeta(const SortedDesign& design, CoefficientState& state, std::size_t j,
                  double delta) {
    if (j >= design.n_covariates()) throw validation_error("covariate index out of range");
    if (!std::isfinite(delta)) throw numeric_error("non-finite coordinate step");
    scx_ctx* h = ctx_for(design);
    put_state(h, design, state);
    check(scx_update_xbeta(h, static_cast<int64_t>(j), delta), &design);  // throws: host state untouched
    get_state(h, design, state);
}

void ScanWorkspace::resize(std::size_t n) {
    n1.resize(n);
    n2.resize(n);
    scanned_d.resize(n);
    scanned_n1.resize(n);
    scanned_n2.resize(n);
}

double log_partial_likelihood(const SortedDesign& design, const CoefficientState& state,
                              const ExecutionConfig& config, ScanWorkspace& /*workspace*/,
                              ScanCounters* /*counters*/) {
    validate(config);
    if (state.xbeta.size() != design.n_rows()) throw validation_error("state does not match design");
    scx_ctx* h = ctx_for(design);
    put_state(h, design, state);
    double ll = 0.0;
    check(scx_log_partial_likelihood(h, &ll), &design);
    return ll;
}

double log_partial_likelihood(const SortedDesign& design, const CoefficientState& state,
                              const ExecutionConfig& config, ScanCounters* counters) {
    ScanWorkspace ws;
    return log_partial_likelihood(design, state, config, ws, counters);
}

GradHess gradient_hessian(const SortedDesign& design, const CoefficientState& state,
                          std::size_t j, ScanWorkspace& /*workspace*/,
                          const ExecutionConfig& config, ScanCounters* /*counters*/) {
    if (j >= design.n_covariates()) throw validation_error("covariate index out of range");
    if (state.xbeta.size() != design.n_rows()) throw validation_error("state does not match design");
    validate(config);
    scx_ctx* h = ctx_for(design);
    put_state(h, design, state);
    GradHess out;
    check(scx_gradient_hessian(h, static_cast<int64_t>(j), &out.gradient, &out.hessian), &design);
    return out;
}

GradHess naive_gradient_hessian(const SortedDesign& design, const CoefficientState& state,
                                std::size_t j) {
    if (j >= design.n_covariates()) throw validation_error("covariate index out of range");
    scx_ctx* h = ctx_for(design);
    put_state(h, design, state);
    GradHess out;
    check(scx_naive_gradient_hessian(h, static_cast<int64_t>(j), &out.gradient, &out.hessian),
          &design);
    return out;
}

double naive_log_partial_likelihood(const SortedDesign& design, const CoefficientState& state) {
    scx_ctx* h = ctx_for(design);
    put_state(h, design, state);
    double ll = 0.0;
    check(scx_naive_log_partial_likelihood(h, &ll), &design);
    return ll;
}

// ------------------------------------------------------------------ optimizer.hpp

PenaltySpec PenaltySpec::shared(std::size_t p, double gamma_value,
                                std::span<const std::size_t> unpenalized) {
    PenaltySpec spec{std::vector<double>(p, gamma_value)};
    for (const std::size_t j : unpenalized) {
        if (j >= p) throw validation_error("unpenalized index out of range");
        spec.gamma[j] = 0.0;
    }
    return spec;
}

double PenaltySpec::value(std::span<const double> beta) const {
    double total = 0.0;
    for (std::size_t j = 0; j < beta.size(); ++j) total += gamma[j] * std::abs(beta[j]);
    return total;
}

void PenaltySpec::validate(std::size_t p) const {
    if (gamma.size() != p) throw validation_error("penalty length does not match covariate count");
    for (const double g : gamma)
        if (!std::isfinite(g) || g < 0.0)
            throw validation_error("penalty weights must be finite and non-negative");
}

double newton_step(double g1, double g2, bool* flat) {
    double step = 0.0;
    int fl = 0;
    check_rule(scx_newton_step(g1, g2, &step, &fl));
    if (flat) *flat = fl != 0;
    return step;
}

TrustOutcome apply_trust_region(double delta_proposed, double trust) {
    TrustOutcome out{};
    check_rule(scx_apply_trust_region(delta_proposed, trust, &out.applied, &out.next_trust));
    return out;
}

ProposedStep l1_coordinate_update(double g1, double g2, double beta_j, double gamma_j) {
    ProposedStep out;
    int sk = 0, fl = 0;
    check_rule(scx_l1_coordinate_update(g1, g2, beta_j, gamma_j, &out.step, &sk, &fl));
    out.skipped = sk != 0;
    out.flat = fl != 0;
    return out;
}

namespace {

FitResult run_fit(const SortedDesign& design, const PenaltySpec& penalty,
                  const OptimizerConfig& config, const double* initial_beta) {
    const std::size_t p = design.n_covariates();
    penalty.validate(p);
    validate(config.exec);
    scx_ctx* h = ctx_for(design);
    FitResult r;
    r.beta.assign(p, 0.0);
    r.trust.assign(p, 0.0);
    std::vector<double> trace(static_cast<std::size_t>(std::max(1, config.max_cycles)) + 1);
    std::vector<int64_t> warn(1 << 16);  // kWarnCap
    scx_fit_options opt{config.max_cycles, config.tolerance, config.initial_trust};
    scx_fit_result out{};
    out.beta = r.beta.data();
    out.trust = r.trust.data();
    out.objective_trace = trace.data();
    out.warning_coords = warn.data();
    out.warning_cap = static_cast<int32_t>(warn.size());
    check(scx_ccd_fit(h, penalty.gamma.data(), &opt, initial_beta, &out), &design);
    r.objective_trace.assign(trace.begin(), trace.begin() + out.trace_len);
    r.cycles_used = out.cycles_used;
    r.converged = out.converged != 0;
    for (int w = 0; w < out.n_warnings; ++w) {
        const std::string name =
            w < out.warning_cap ? design.data.covariate_name(static_cast<std::size_t>(warn[w])) : "?";
        r.warnings.push_back("coordinate " + name +
                             " skipped: step overflow persisted after 10 halvings");
    }
    return r;
}

}  // namespace

FitResult ccd_fit(const SortedDesign& design, const PenaltySpec& penalty,
                  const OptimizerConfig& config) {
    return run_fit(design, penalty, config, nullptr);
}

FitResult ccd_fit(const SortedDesign& design, const PenaltySpec& penalty,
                  const OptimizerConfig& config, std::span<const double> initial_beta) {
    if (initial_beta.size() != design.n_covariates())
        throw validation_error("initial beta length does not match covariate count");
    return run_fit(design, penalty, config, initial_beta.data());
}

}  // namespace stratcox
