// Regularisation path and k-fold cross-validation over the device fits
// (SURVEY.md §8(f)1): the caller that turns one fit into BASELINE configs
// 4/5's gamma-grid x folds workload.
//
// Host side (input preparation, run once per fold) restates the reference's
// data handling with the same standard-library algorithms, so fold labels and
// sorted layouts are identical to the reference's:
//   build_sorted_design  proj/src/data.cpp:68-147   stable sort (stratum asc,
//                        time desc), CSC re-index, heads, offsets, tie ends
//   subset_rows          proj/src/data.cpp:219-275  dense stratum relabel
//   fold_assignment      proj/src/resample.cpp:70-91 mt19937_64 + std::shuffle
//   default_gamma_grid   proj/src/resample.cpp:57-68
//   kfold_select_gamma   proj/src/resample.cpp:93-172
// Every fit and every held-out score runs on the device through this
// library's own C-ABI (scx_ccd_fit, scx_make_state, scx_log_partial_likelihood);
// folds are dealt round-robin over the given devices, one host thread per
// device (the reference runs folds in an OpenMP loop, resample.cpp:121).
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>
#include <numeric>
#include <random>
#include <stdexcept>
#include <string>
#include <thread>
#include <unordered_map>
#include <utility>
#include <vector>

#include "../../include/stratcox_b200.h"

// capi.cu: record a message on a context (scx_last_error)
void scx_note_error(scx_ctx* ctx, const char* msg);

namespace {

struct ScxError : std::runtime_error {
    scx_status status;
    ScxError(scx_status s, const std::string& m) : std::runtime_error(m), status(s) {}
};

// Owned copy of a dataset in input row order (SurvivalDataset, data.hpp:31-45).
struct Data {
    std::vector<double> time;
    std::vector<uint8_t> event;
    std::vector<int32_t> stratum;
    std::vector<int64_t> subject;
    std::vector<int64_t> col_ptr;  // [p+1]
    std::vector<int64_t> rows;     // [nnz]
    std::vector<double> values;    // [nnz]
    int64_t n() const { return (int64_t)time.size(); }
    int64_t p() const { return (int64_t)col_ptr.size() - 1; }
    int32_t n_strata() const {
        int32_t k = 0;
        for (int32_t s : stratum) k = std::max(k, s);
        return k;
    }
};

Data copy_in(const scx_dataset* d) {
    Data o;
    const int64_t n = d->n_rows, p = d->n_covariates;
    o.time.assign(d->time, d->time + n);
    o.event.assign(d->event, d->event + n);
    o.stratum.assign(d->stratum, d->stratum + n);
    if (d->subject)
        o.subject.assign(d->subject, d->subject + n);
    else {
        o.subject.resize(n);
        for (int64_t i = 0; i < n; ++i) o.subject[i] = i + 1;
    }
    o.col_ptr.assign(d->col_ptr, d->col_ptr + p + 1);
    const int64_t nnz = o.col_ptr[p];
    o.rows.assign(d->row_idx, d->row_idx + nnz);
    if (d->values)
        o.values.assign(d->values, d->values + nnz);
    else
        o.values.assign(nnz, 1.0);
    return o;
}

// validate_invariants (data.cpp:27-66), same checks and messages.
void validate(const Data& d) {
    const int64_t n = d.n();
    const int32_t kc = d.n_strata();
    if (n > 0 && kc < 1) throw ScxError(SCX_ERR_VALIDATION, "dataset has no strata");
    std::vector<int64_t> per(kc, 0);
    for (int64_t i = 0; i < n; ++i) {
        const double t = d.time[i];
        if (!std::isfinite(t) || t < 0.0)
            throw ScxError(SCX_ERR_VALIDATION, "negative or non-finite time at row " + std::to_string(i));
        if (d.event[i] > 1)
            throw ScxError(SCX_ERR_VALIDATION, "event indicator must be 0 or 1 at row " + std::to_string(i));
        const int32_t s = d.stratum[i];
        if (s < 1 || s > kc)
            throw ScxError(SCX_ERR_VALIDATION, "stratum label out of range at row " + std::to_string(i));
        ++per[s - 1];
    }
    for (int32_t k = 1; k <= kc; ++k)
        if (per[k - 1] == 0)
            throw ScxError(SCX_ERR_VALIDATION, "stratum " + std::to_string(k) + " has zero rows");
    for (int64_t j = 0; j < d.p(); ++j) {
        const std::string name = "x" + std::to_string(j + 1);
        int64_t prev = -1;
        for (int64_t t = d.col_ptr[j]; t < d.col_ptr[j + 1]; ++t) {
            const int64_t r = d.rows[t];
            if (r <= prev)
                throw ScxError(SCX_ERR_VALIDATION, "column " + name + " row indices must be strictly increasing");
            if (r < 0 || r >= n)
                throw ScxError(SCX_ERR_VALIDATION, "column " + name + " row index out of range");
            if (!std::isfinite(d.values[t]))
                throw ScxError(SCX_ERR_VALIDATION, "column " + name + " has a non-finite value");
            prev = r;
        }
    }
}

// SortedDesign arrays (data.hpp:50-62) in the layout scx_upload_design takes.
struct Sorted {
    std::vector<int64_t> perm, offsets, tie_end, col_ptr, rows;
    std::vector<uint8_t> event;
    std::vector<double> values;
    int32_t k = 0;
};

// Worker threads for the host preparation (design build, CV folds' subsets).
int host_threads() {
    const unsigned h = std::thread::hardware_concurrency();
    return (int)std::max(1u, std::min(h, 32u));
}

template <class F>
void parallel_for(int64_t count, F&& body) {
    const int nt = (int)std::min<int64_t>(host_threads(), std::max<int64_t>(count, 1));
    if (nt <= 1) {
        for (int64_t i = 0; i < count; ++i) body(i);
        return;
    }
    std::atomic<int64_t> next{0};
    std::vector<std::thread> pool;
    for (int t = 0; t < nt; ++t)
        pool.emplace_back([&] {
            for (int64_t i; (i = next.fetch_add(1)) < count;) body(i);
        });
    for (auto& th : pool) th.join();
}

// The reference's std::stable_sort by (stratum asc, time desc) is done as a
// stable counting sort by stratum followed by a stable sort by time desc
// inside each stratum (in parallel over strata): the same permutation.
Sorted build_sorted(const Data& data) {
    validate(data);
    const int64_t n = data.n();
    if (n == 0) throw ScxError(SCX_ERR_VALIDATION, "dataset has no rows");
    Sorted s;
    const int32_t kc = data.n_strata();
    std::vector<int64_t> start(kc + 2, 0);
    for (int64_t i = 0; i < n; ++i) ++start[data.stratum[i] + 1];
    for (int32_t k = 1; k <= kc + 1; ++k) start[k] += start[k - 1];
    s.perm.resize(n);
    {
        std::vector<int64_t> fill(start.begin(), start.end());
        for (int64_t i = 0; i < n; ++i) s.perm[fill[data.stratum[i]]++] = i;
    }
    parallel_for(kc, [&](int64_t q) {
        const int32_t k = (int32_t)q + 1;
        std::stable_sort(s.perm.begin() + start[k], s.perm.begin() + start[k + 1],
                         [&](int64_t a, int64_t b) { return data.time[a] > data.time[b]; });
    });
    std::vector<int64_t> inverse(n);
    for (int64_t i = 0; i < n; ++i) inverse[s.perm[i]] = i;
    std::vector<int32_t> sstr(n);
    std::vector<double> stime(n);
    s.event.resize(n);
    for (int64_t i = 0; i < n; ++i) {
        sstr[i] = data.stratum[s.perm[i]];
        stime[i] = data.time[s.perm[i]];
        s.event[i] = data.event[s.perm[i]];
    }
    const int64_t p = data.p();
    s.col_ptr = data.col_ptr;
    s.rows.resize(data.rows.size());
    s.values.resize(data.values.size());
    parallel_for(p, [&](int64_t j) {
        std::vector<std::pair<int64_t, double>> buf;
        buf.reserve(data.col_ptr[j + 1] - data.col_ptr[j]);
        for (int64_t t = data.col_ptr[j]; t < data.col_ptr[j + 1]; ++t)
            buf.emplace_back(inverse[data.rows[t]], data.values[t]);
        std::sort(buf.begin(), buf.end(),
                  [](const auto& a, const auto& b) { return a.first < b.first; });
        for (size_t t = 0; t < buf.size(); ++t) {
            s.rows[data.col_ptr[j] + t] = buf[t].first;
            s.values[data.col_ptr[j] + t] = buf[t].second;
        }
    });
    s.offsets.push_back(0);
    for (int64_t i = 1; i < n; ++i)
        if (sstr[i] != sstr[i - 1]) s.offsets.push_back(i);
    s.offsets.push_back(n);
    s.k = (int32_t)s.offsets.size() - 1;
    s.tie_end.resize(n);
    int64_t a = 0;
    while (a < n) {
        int64_t e = a;
        while (e + 1 < n && sstr[e + 1] == sstr[a] && stime[e + 1] == stime[a]) ++e;
        for (int64_t i = a; i <= e; ++i) s.tie_end[i] = e;
        a = e + 1;
    }
    return s;
}

// subset_rows (data.cpp:219-275): rows in the given order, strata relabelled
// densely in ascending label order, columns gathered and row-sorted.
Data subset(const Data& data, const std::vector<int64_t>& rows) {
    Data o;
    const int32_t kc = data.n_strata();
    std::vector<int32_t> remap(kc + 1, 0);
    for (int64_t r : rows) {
        if (r < 0 || r >= data.n()) throw ScxError(SCX_ERR_VALIDATION, "subset row index out of range");
        remap[data.stratum[r]] = 1;
    }
    int32_t next = 0;
    for (int32_t k = 1; k <= kc; ++k)
        if (remap[k]) remap[k] = ++next;
    for (int64_t r : rows) {
        o.time.push_back(data.time[r]);
        o.event.push_back(data.event[r]);
        o.subject.push_back(data.subject[r]);
        o.stratum.push_back(remap[data.stratum[r]]);
    }
    std::vector<std::vector<int64_t>> hits(data.n());
    for (size_t s = 0; s < rows.size(); ++s) hits[rows[s]].push_back((int64_t)s);
    o.col_ptr.push_back(0);
    std::vector<std::pair<int64_t, double>> scratch;
    for (int64_t j = 0; j < data.p(); ++j) {
        scratch.clear();
        for (int64_t t = data.col_ptr[j]; t < data.col_ptr[j + 1]; ++t)
            for (int64_t nr : hits[data.rows[t]]) scratch.emplace_back(nr, data.values[t]);
        std::sort(scratch.begin(), scratch.end(),
                  [](const auto& a, const auto& b) { return a.first < b.first; });
        for (const auto& [r, v] : scratch) {
            o.rows.push_back(r);
            o.values.push_back(v);
        }
        o.col_ptr.push_back((int64_t)o.rows.size());
    }
    return o;
}

// fold_assignment (resample.cpp:70-91): subjects in order of first
// appearance, shuffled by mt19937_64(seed), dealt round-robin.
std::vector<int32_t> folds_of(const Data& data, int folds, uint64_t seed) {
    if (folds < 2) throw ScxError(SCX_ERR_VALIDATION, "folds must be >= 2");
    std::vector<int64_t> ids;
    std::vector<std::vector<int64_t>> rows;
    std::unordered_map<int64_t, size_t> pos;
    for (int64_t r = 0; r < data.n(); ++r) {
        const auto [it, inserted] = pos.try_emplace(data.subject[r], ids.size());
        if (inserted) {
            ids.push_back(data.subject[r]);
            rows.emplace_back();
        }
        rows[it->second].push_back(r);
    }
    const size_t ns = ids.size();
    if ((size_t)folds > ns) throw ScxError(SCX_ERR_VALIDATION, "degenerate fold; reduce folds or reseed");
    std::vector<size_t> order(ns);
    for (size_t i = 0; i < ns; ++i) order[i] = i;
    std::mt19937_64 rng(seed);
    std::shuffle(order.begin(), order.end(), rng);
    std::vector<int32_t> fold_of(ns);
    for (size_t i = 0; i < ns; ++i) fold_of[order[i]] = (int32_t)(i % (size_t)folds);
    std::vector<int32_t> by_row(data.n());
    for (size_t s = 0; s < ns; ++s)
        for (int64_t r : rows[s]) by_row[r] = fold_of[s];
    return by_row;
}

void check(scx_status st, scx_ctx* ctx) {
    if (st != SCX_OK) throw ScxError(st, ctx ? scx_last_error(ctx) : "device error");
}

struct Ctx {
    scx_ctx* c = nullptr;
    explicit Ctx(int device) {
        if (scx_create(device, &c) != SCX_OK) throw ScxError(SCX_ERR_CUDA, "cannot create a device context");
    }
    ~Ctx() { scx_destroy(c); }
};

void upload_sorted(scx_ctx* ctx, const Sorted& s, int64_t p) {
    check(scx_upload_design(ctx, (int64_t)s.event.size(), s.k, s.offsets.data(), s.event.data(),
                            s.tie_end.data(), p, s.col_ptr.data(), s.rows.data(), s.values.data()),
          ctx);
}

std::string fmt_gamma(double g) { return std::to_string(g); }  // std::to_string as the reference

}  // namespace

extern "C" {

// scx_build_design (the device build of build_sorted_design) is in
// design_build.cu; build_sorted above prepares the CV folds' designs.

scx_status scx_default_gamma_grid(double gamma_max, int64_t size, double* out) {
    if (size < 1) return SCX_ERR_VALIDATION;  // "gamma grid size must be >= 1"
    if (!(gamma_max > 0.0)) return SCX_ERR_VALIDATION;  // "gamma_max must be positive"
    const double hi = std::log(gamma_max);
    const double lo = hi - std::log(1e4);
    for (int64_t i = 0; i < size; ++i) {
        const double t = size == 1 ? 1.0 : (double)i / (double)(size - 1);
        out[i] = std::exp(lo + t * (hi - lo));
    }
    return SCX_OK;
}

scx_status scx_fold_assignment(const scx_dataset* data, int folds, uint64_t seed, int32_t* fold_of_row) {
    if (!data) return SCX_ERR_VALIDATION;
    try {
        const auto f = folds_of(copy_in(data), folds, seed);
        std::memcpy(fold_of_row, f.data(), f.size() * sizeof(int32_t));
        return SCX_OK;
    } catch (const ScxError& e) {
        return e.status;
    }
}

scx_status scx_kfold_select_gamma(const scx_dataset* data, const double* penalty_template,
                                  const scx_cv_config* cv, const scx_fit_options* opt,
                                  const int* devices, int n_devices, scx_cv_result* res,
                                  char* error_out, int error_cap) {
    auto report = [&](scx_status st, const std::string& msg) {
        if (error_out && error_cap > 0) {
            std::strncpy(error_out, msg.c_str(), (size_t)error_cap - 1);
            error_out[error_cap - 1] = 0;
        }
        return st;
    };
    if (!data || !cv || !opt || !res) return report(SCX_ERR_VALIDATION, "null argument");
    try {
        const Data d = copy_in(data);
        const int64_t p = d.p();
        for (int64_t j = 0; j < p; ++j)  // PenaltySpec::validate (optimizer.cpp:24-30)
            if (!std::isfinite(penalty_template[j]) || penalty_template[j] < 0.0)
                throw ScxError(SCX_ERR_VALIDATION, "penalty weights must be finite and non-negative");
        const int64_t ng = cv->grid_size;
        if (ng < 1) throw ScxError(SCX_ERR_VALIDATION, "gamma grid is empty");
        for (int64_t i = 0; i < ng; ++i)
            if (!(cv->gamma_grid[i] > 0.0) || (i > 0 && cv->gamma_grid[i] <= cv->gamma_grid[i - 1]))
                throw ScxError(SCX_ERR_VALIDATION, "gamma grid must be positive and strictly increasing");
        const int folds = cv->folds;
        const std::vector<int32_t> fold_of_row = folds_of(d, folds, cv->seed);
        std::vector<int64_t> fold_events(folds, 0);
        for (int64_t r = 0; r < d.n(); ++r)
            if (d.event[r]) ++fold_events[fold_of_row[r]];
        for (int f = 0; f < folds; ++f)
            if (fold_events[f] == 0) throw ScxError(SCX_ERR_VALIDATION, "degenerate fold; reduce folds or reseed");

        std::vector<double> scores((size_t)ng * folds, 0.0);
        std::vector<std::vector<std::string>> warnings(folds);
        std::vector<std::string> failures(folds);
        std::vector<int> devs;
        for (int q = 0; q < std::max(1, n_devices); ++q) devs.push_back(devices && n_devices > 0 ? devices[q] : 0);

        auto run_fold = [&](int f, int device) {
            try {
                std::vector<int64_t> train_rows, test_rows;
                for (int64_t r = 0; r < d.n(); ++r) (fold_of_row[r] == f ? test_rows : train_rows).push_back(r);
                const Sorted train = build_sorted(subset(d, train_rows));
                const Sorted test = build_sorted(subset(d, test_rows));
                Ctx ctr(device), cte(device);
                upload_sorted(ctr.c, train, p);
                upload_sorted(cte.c, test, p);
                std::vector<double> warm(p, 0.0), gamma(p), beta(p), trace(opt->max_cycles + 1);
                for (int64_t g = ng; g-- > 0;) {  // from the sparse end, warm-started
                    for (int64_t j = 0; j < p; ++j) gamma[j] = penalty_template[j] > 0.0 ? cv->gamma_grid[g] : 0.0;
                    double score = -std::numeric_limits<double>::infinity();
                    scx_fit_result fr{};
                    fr.beta = beta.data();
                    fr.objective_trace = trace.data();
                    scx_status st = scx_ccd_fit(ctr.c, gamma.data(), opt, warm.data(), &fr);
                    std::string err;
                    if (st == SCX_OK) {
                        warm = beta;
                        st = scx_make_state(cte.c, beta.data());
                        if (st == SCX_OK) st = scx_log_partial_likelihood(cte.c, &score);
                        if (st != SCX_OK) {
                            err = scx_last_error(cte.c);
                            score = -std::numeric_limits<double>::infinity();
                        }
                    } else {
                        err = scx_last_error(ctr.c);
                    }
                    if (st == SCX_ERR_CUDA) throw ScxError(st, err);
                    if (st != SCX_OK)
                        warnings[f].push_back("fold " + std::to_string(f) + ", gamma " +
                                              fmt_gamma(cv->gamma_grid[g]) + ": " + err);
                    scores[(size_t)g * folds + f] = score;
                }
            } catch (const std::exception& e) {
                failures[f] = e.what();
            }
        };
        // folds dealt round-robin over the devices, one host thread per device
        std::vector<std::thread> pool;
        for (size_t q = 0; q < devs.size(); ++q)
            pool.emplace_back([&, q] {
                for (int f = (int)q; f < folds; f += (int)devs.size()) run_fold(f, devs[q]);
            });
        for (auto& t : pool) t.join();
        for (const auto& fl : failures)
            if (!fl.empty()) throw ScxError(SCX_ERR_NUMERIC, "cross-validation fold failed: " + fl);

        int32_t nw = 0;
        for (const auto& w : warnings) nw += (int32_t)w.size();
        res->n_warnings = nw;
        if (res->fold_scores) std::memcpy(res->fold_scores, scores.data(), scores.size() * sizeof(double));
        std::vector<double> mean(ng, 0.0);
        for (int64_t g = 0; g < ng; ++g) {
            double total = 0.0;
            for (int f = 0; f < folds; ++f) total += scores[(size_t)g * folds + f];
            mean[g] = total / (double)folds;
        }
        if (res->mean_scores) std::memcpy(res->mean_scores, mean.data(), mean.size() * sizeof(double));
        int64_t best = 0;
        for (int64_t g = 1; g < ng; ++g)
            if (mean[g] >= mean[best]) best = g;  // ties favor the larger gamma
        res->gamma_star = cv->gamma_grid[best];
        std::string all;
        for (const auto& w : warnings)
            for (const auto& s : w) all += s + "\n";
        report(SCX_OK, all);
        return SCX_OK;
    } catch (const ScxError& e) {
        return report(e.status, e.what());
    }
}

}  // extern "C"
