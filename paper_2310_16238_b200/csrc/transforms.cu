// Lowering transforms: a Cox model with time-varying
// coefficients becomes one with time-varying covariates by splitting columns
// across effect windows, and that becomes a stratified Cox model by
// augmenting each subject into one row per interval it is at risk in — the
// input layout of BASELINE configs 2 and 3. Host preprocessing, run once;
// restates proj/src/transforms.cpp:
//   event_interval / at_risk_in_interval   :25-37
//   validate_cut_points                    :39-46
//   make_time_varying (time-fixed columns) :64-96
//   split_time_varying_coefficient         :98-175
//   augment_to_strata                      :177-223
// streaming each (interval, column) pair straight into the augmented CSC
// instead of materialising the per-interval schedules; the output arrays are
// identical to the reference's lower_pipeline.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <set>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "../../include/stratcox_b200.h"

#include "lowered.h"

namespace {

struct LowerError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

int event_interval(double y, const std::vector<double>& cuts) {
    const int k_count = (int)cuts.size() - 1;
    if (y == cuts.back()) return k_count;
    return (int)(std::upper_bound(cuts.begin(), cuts.end(), y) - cuts.begin());
}

bool at_risk(double y, uint8_t event, int k, const std::vector<double>& cuts) {
    if (y > cuts[k - 1]) return true;
    return event != 0 && y == cuts[k - 1] && event_interval(y, cuts) == k;
}

std::string short_number(double v) {
    char buf[64];
    std::snprintf(buf, sizeof buf, "%.17g", v);
    // shortest round-trip form, as std::to_chars in the reference
    for (int prec = 1; prec <= 17; ++prec) {
        char t[64];
        std::snprintf(t, sizeof t, "%.*g", prec, v);
        if (std::strtod(t, nullptr) == v) return t;
    }
    return buf;
}

}  // namespace

// Validation and output-column plan of the lowering (transforms.cpp:39-175 and
// make_time_varying's coverage check), shared with the device lowering.
bool lowering_plan(const scx_dataset* subj, const double* cut_points, int64_t n_cuts,
                   const int64_t* split_covariate, const int64_t* split_ptr,
                   const double* split_times, int64_t n_splits, std::vector<LowerCol>& cols,
                   std::string& err) {
    try {
        const std::vector<double> cuts(cut_points, cut_points + n_cuts);
        // validate_cut_points (transforms.cpp:39-46)
        if (cuts.size() < 2) throw LowerError("need at least two cut points");
        if (cuts.front() != 0.0) throw LowerError("first cut point must be 0");
        for (size_t i = 1; i < cuts.size(); ++i)
            if (!std::isfinite(cuts[i]) || cuts[i] <= cuts[i - 1])
                throw LowerError("cut points must be finite and strictly increasing");
        const int64_t n = subj->n_rows, p = subj->n_covariates;
        for (int64_t i = 0; i < n; ++i)  // make_time_varying (:74-79)
            if (subj->time[i] > cuts.back())
                throw LowerError("cut points do not cover follow-up of subject " +
                                 std::to_string(subj->subject ? subj->subject[i] : i + 1));
        for (int64_t i = 0; i < n; ++i)  // validate (:48-62)
            if (!std::isfinite(subj->time[i]) || subj->time[i] < 0.0)
                throw LowerError("negative or non-finite time for subject index " + std::to_string(i));
        // split_time_varying_coefficient (:98-175): effect-window edges per covariate
        std::vector<std::vector<double>> bounds(p);
        for (int64_t sidx = 0; sidx < n_splits; ++sidx) {
            const int64_t j = split_covariate[sidx];
            if (j < 0 || j >= p) throw LowerError("split covariate index out of range");
            const std::string name = "x" + std::to_string(j + 1);
            if (split_ptr[sidx + 1] == split_ptr[sidx])
                throw LowerError("split for covariate " + name + " declares no times");
            if (!bounds[j].empty()) throw LowerError("covariate split declared twice");
            std::set<double> seen;
            for (int64_t q = split_ptr[sidx]; q < split_ptr[sidx + 1]; ++q) {
                const double t = split_times[q];
                if (!(t > 0.0) || !(t < cuts.back()))
                    throw LowerError("split time " + short_number(t) + " outside the follow-up window");
                if (!std::binary_search(cuts.begin(), cuts.end(), t))
                    throw LowerError("split time " + short_number(t) + " is not a cut point");
                if (!seen.insert(t).second) throw LowerError("duplicate split time " + short_number(t));
            }
            bounds[j].assign(seen.begin(), seen.end());
        }
        cols.clear();
        for (int64_t j = 0; j < p; ++j) {
            if (bounds[j].empty()) {
                cols.push_back({j, -1, cuts.front(), cuts.back()});
                continue;
            }
            std::vector<double> edges{cuts.front()};
            edges.insert(edges.end(), bounds[j].begin(), bounds[j].end());
            edges.push_back(cuts.back());
            for (size_t w = 0; w + 1 < edges.size(); ++w) cols.push_back({j, (int)w, edges[w], edges[w + 1]});
        }
        return true;
    } catch (const LowerError& e) {
        err = e.what();
        return false;
    }
}

extern "C" {

scx_status scx_lower_time_varying(const scx_dataset* subj, const double* cut_points, int64_t n_cuts,
                                  const int64_t* split_covariate, const int64_t* split_ptr,
                                  const double* split_times, int64_t n_splits, scx_lowered** out,
                                  char* error_out, int error_cap) {
    auto report = [&](const std::string& m) {
        if (error_out && error_cap > 0) {
            std::strncpy(error_out, m.c_str(), (size_t)error_cap - 1);
            error_out[error_cap - 1] = 0;
        }
        return SCX_ERR_VALIDATION;
    };
    if (!subj || !cut_points || !out) return report("null argument");
    *out = nullptr;
    try {
        const std::vector<double> cuts(cut_points, cut_points + n_cuts);
        std::vector<LowerCol> plan;
        std::string why;
        if (!lowering_plan(subj, cut_points, n_cuts, split_covariate, split_ptr, split_times, n_splits,
                           plan, why))
            throw LowerError(why);
        const int64_t n = subj->n_rows;
        const int k_count = (int)cuts.size() - 1;
        std::vector<int64_t> subject(n);
        for (int64_t i = 0; i < n; ++i) subject[i] = subj->subject ? subj->subject[i] : i + 1;
        auto* L = new scx_lowered();
        struct OutCol {
            int64_t src;
            int window;
            double start, end;
        };
        std::vector<OutCol> cols;
        for (const LowerCol& c : plan) cols.push_back({c.src, c.window, c.start, c.end});
        // augment_to_strata (:177-223): interval-major rows, subjects in input
        // order; rank[k-1][i] = augmented row of subject i in interval k (-1: not at risk)
        std::vector<std::vector<int64_t>> rank(k_count, std::vector<int64_t>(n, -1));
        for (int k = 1; k <= k_count; ++k) {
            const int64_t offset = (int64_t)L->time.size();
            int64_t emitted = 0;
            for (int64_t i = 0; i < n; ++i) {
                if (!at_risk(subj->time[i], subj->event[i], k, cuts)) continue;
                rank[k - 1][i] = offset + emitted++;
                L->time.push_back(std::min(subj->time[i], cuts[k]));
                L->event.push_back(subj->event[i] && event_interval(subj->time[i], cuts) == k ? 1 : 0);
                L->stratum.push_back(k);
                L->subject.push_back(subject[i]);
            }
        }
        // columns are independent: one worker per column, intervals in order
        std::vector<std::vector<std::pair<int64_t, double>>> acc(cols.size());
        {
            std::atomic<size_t> next{0};
            const unsigned nt = std::max(1u, std::min(std::thread::hardware_concurrency(), 32u));
            std::vector<std::thread> pool;
            for (unsigned w = 0; w < nt; ++w)
                pool.emplace_back([&] {
                    for (size_t c; (c = next.fetch_add(1)) < cols.size();) {
                        const OutCol& oc = cols[c];
                        const int64_t j = oc.src;
                        for (int k = 1; k <= k_count; ++k) {
                            // window w's column carries interval k iff t_{k-1} in [start, end)
                            if (oc.window >= 0 && !(cuts[k - 1] >= oc.start && cuts[k - 1] < oc.end))
                                continue;
                            const std::vector<int64_t>& rk = rank[k - 1];
                            for (int64_t t = subj->col_ptr[j]; t < subj->col_ptr[j + 1]; ++t) {
                                const int64_t i = subj->row_idx[t];
                                const double v = subj->values ? subj->values[t] : 1.0;
                                if (rk[i] >= 0 && v != 0.0) acc[c].emplace_back(rk[i], v);
                            }
                        }
                    }
                });
            for (auto& th : pool) th.join();
        }
        L->col_ptr.push_back(0);
        for (size_t c = 0; c < cols.size(); ++c) {
            for (const auto& [r, v] : acc[c]) {
                L->rows.push_back(r);
                L->values.push_back(v);
            }
            L->col_ptr.push_back((int64_t)L->rows.size());
            L->map_source.push_back(cols[c].src);
            L->map_window.push_back(cols[c].window);
            L->map_start.push_back(cols[c].start);
            L->map_end.push_back(cols[c].end);
        }
        *out = L;
        return SCX_OK;
    } catch (const LowerError& e) {
        return report(e.what());
    }
}

scx_status scx_lowered_sizes(const scx_lowered* L, int64_t* n_rows, int64_t* n_covariates, int64_t* nnz) {
    if (!L) return SCX_ERR_VALIDATION;
    if (n_rows) *n_rows = (int64_t)L->time.size();
    if (n_covariates) *n_covariates = (int64_t)L->col_ptr.size() - 1;
    if (nnz) *nnz = (int64_t)L->rows.size();
    return SCX_OK;
}

scx_status scx_lowered_dataset(const scx_lowered* L, scx_dataset* view) {
    if (!L || !view) return SCX_ERR_VALIDATION;
    view->n_rows = (int64_t)L->time.size();
    view->time = L->time.data();
    view->event = L->event.data();
    view->stratum = L->stratum.data();
    view->subject = L->subject.data();
    view->n_covariates = (int64_t)L->col_ptr.size() - 1;
    view->col_ptr = L->col_ptr.data();
    view->row_idx = L->rows.data();
    view->values = L->values.data();
    return SCX_OK;
}

scx_status scx_lowered_column_map(const scx_lowered* L, int64_t* source, int32_t* window,
                                  double* window_start, double* window_end) {
    if (!L) return SCX_ERR_VALIDATION;
    const size_t m = L->map_source.size();
    if (source) std::memcpy(source, L->map_source.data(), m * sizeof(int64_t));
    if (window) std::memcpy(window, L->map_window.data(), m * sizeof(int32_t));
    if (window_start) std::memcpy(window_start, L->map_start.data(), m * sizeof(double));
    if (window_end) std::memcpy(window_end, L->map_end.data(), m * sizeof(double));
    return SCX_OK;
}

void scx_lowered_free(scx_lowered* L) { delete L; }

}  // extern "C"
