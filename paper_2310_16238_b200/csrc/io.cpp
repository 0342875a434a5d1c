// On-disk formats and configuration, host C++ behind the
// C-ABI: the reference's proj/src/io.cpp, same formats, same canonical order
// and the same error messages, parsed in parallel.
//
//   wide CSV  subject,stratum,time,event,covariates     read_wide_csv  io.cpp:123-193
//                                                       write_wide_csv io.cpp:195-223
//   long CSV  subject,start,stop,event,covariates       read_long_csv  io.cpp:225-272
//             -> to_time_varying (io.cpp:293-345)       write_long_csv io.cpp:274-291
//             -> lower_pipeline (transforms.cpp:98-231: split + augment_to_strata)
//   config    key = value, '#' comments                 ConfigMap      io.cpp:347-444
//
// Parsing: the file is read whole, split into lines, and the lines are parsed
// by a pool of threads (fields, numbers by std::from_chars, covariate tokens);
// every line records its first error in the reference's check order, and the
// earliest failing line wins, so the message is the reference's. Assembly
// (name indices in first-appearance order, stratum relabelling, the long
// format's per-subject contiguity checks) is sequential.
#include <algorithm>
#include <atomic>
#include <charconv>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <map>
#include <numeric>
#include <set>
#include <sstream>
#include <stdexcept>
#include <string>
#include <string_view>
#include <thread>
#include <unordered_map>
#include <vector>

#include "../../include/stratcox_b200.h"
#include "lowered.h"

namespace {

struct IoError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

constexpr const char* kWideHeader = "subject,stratum,time,event,covariates";
constexpr const char* kLongHeader = "subject,start,stop,event,covariates";

std::string_view trim(std::string_view s) {
    while (!s.empty() && (s.front() == ' ' || s.front() == '\t' || s.front() == '\r')) s.remove_prefix(1);
    while (!s.empty() && (s.back() == ' ' || s.back() == '\t' || s.back() == '\r')) s.remove_suffix(1);
    return s;
}

std::string format_double(double v) {  // io.cpp:117-121 (shortest round trip)
    char buf[40];
    const auto res = std::to_chars(buf, buf + sizeof(buf), v);
    return std::string(buf, res.ptr);
}

std::string line_msg(const std::string& path, size_t line, const std::string& what) {
    return path + ":" + std::to_string(line) + ": " + what;
}

// Number parsing with the reference's messages ("cannot parse WHAT 'TEXT'").
bool parse_double(std::string_view text, double& v) {
    const std::string_view t = trim(text);
    const auto res = std::from_chars(t.data(), t.data() + t.size(), v);
    return res.ec == std::errc{} && res.ptr == t.data() + t.size();
}
bool parse_int(std::string_view text, int64_t& v) {
    const std::string_view t = trim(text);
    const auto res = std::from_chars(t.data(), t.data() + t.size(), v);
    return res.ec == std::errc{} && res.ptr == t.data() + t.size();
}
std::string cannot(const char* what, std::string_view text) {
    return std::string("cannot parse ") + what + " '" + std::string(trim(text)) + "'";
}

// One parsed data line; `err` is the first failure in the reference's order.
struct Token {
    std::string_view name;
    double value;
};
struct Line {
    size_t line_no = 0;
    bool empty = true;
    std::string err;
    int64_t subject = 0;
    std::string_view label;  // wide: stratum label
    double a = 0.0, b = 0.0; // wide: time; long: start, stop
    uint8_t event = 0;
    std::vector<Token> tokens;
};

// first `count` comma fields; the remainder (covariate names may hold commas)
// is the last (io.cpp:56-67)
bool split_fields(std::string_view s, size_t count, std::vector<std::string_view>& f) {
    f.clear();
    for (size_t i = 0; i + 1 < count; ++i) {
        const size_t pos = s.find(',');
        if (pos == std::string_view::npos) return false;
        f.push_back(s.substr(0, pos));
        s.remove_prefix(pos + 1);
    }
    f.push_back(s);
    return true;
}

bool parse_event(std::string_view t, uint8_t& ev, std::string& err) {
    int64_t v;
    if (!parse_int(t, v)) {
        err = cannot("event flag", t);
        return false;
    }
    if (v != 0 && v != 1) {
        err = "event flag must be 0 or 1";
        return false;
    }
    ev = (uint8_t)v;
    return true;
}

// name:value tokens, value split on the last ':' (io.cpp:69-89); wide lines
// also reject a name repeated in the line (io.cpp:152-154, after the token parses)
bool parse_tokens(std::string_view cell, bool wide, std::vector<Token>& out, std::string& err) {
    cell = trim(cell);
    while (!cell.empty()) {
        const size_t sp = cell.find(' ');
        std::string_view token = sp == std::string_view::npos ? cell : cell.substr(0, sp);
        cell.remove_prefix(sp == std::string_view::npos ? cell.size() : sp + 1);
        token = trim(token);
        if (token.empty()) continue;
        const size_t colon = token.rfind(':');
        if (colon == std::string_view::npos || colon == 0) {
            err = "malformed covariate token '" + std::string(token) + "'";
            return false;
        }
        const std::string_view name = token.substr(0, colon);
        double value;
        if (!parse_double(token.substr(colon + 1), value)) {
            err = cannot("covariate value", token.substr(colon + 1));
            return false;
        }
        if (!std::isfinite(value)) {
            err = "non-finite covariate value";
            return false;
        }
        if (wide)
            for (const Token& t : out)
                if (t.name == name) {
                    err = "duplicate covariate '" + std::string(name) + "'";
                    return false;
                }
        out.push_back({name, value});
    }
    return true;
}

void parse_line(std::string_view s, bool wide, Line& L) {
    if (trim(s).empty()) return;
    L.empty = false;
    std::vector<std::string_view> f;
    if (!split_fields(s, 5, f)) {
        L.err = "too few fields";
        return;
    }
    if (!parse_int(f[0], L.subject)) {
        L.err = cannot("subject", f[0]);
        return;
    }
    if (wide) {
        L.label = trim(f[1]);
        if (!parse_double(f[2], L.a)) {
            L.err = cannot("time", f[2]);
            return;
        }
        if (!std::isfinite(L.a) || L.a < 0.0) {
            L.err = "time must be finite and >= 0";
            return;
        }
        if (!parse_event(f[3], L.event, L.err)) return;
    } else {
        if (!parse_double(f[1], L.a)) {
            L.err = cannot("interval start", f[1]);
            return;
        }
        if (!parse_double(f[2], L.b)) {
            L.err = cannot("interval stop", f[2]);
            return;
        }
        if (!parse_event(f[3], L.event, L.err)) return;
        if (!std::isfinite(L.a) || !std::isfinite(L.b) || L.a < 0.0) {
            L.err = "interval bounds must be finite and non-negative";
            return;
        }
        if (!(L.a < L.b)) {
            L.err = "interval start must precede interval stop";
            return;
        }
    }
    parse_tokens(f[4], wide, L.tokens, L.err);
}

std::string slurp(const std::string& path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw IoError("cannot open " + path);
    std::ostringstream b;
    b << in.rdbuf();
    return b.str();
}

// Header check + parallel parse of the data lines (line numbers from 2).
std::vector<Line> parse_file(const std::string& path, const std::string& text, bool wide) {
    const char* hdr = wide ? kWideHeader : kLongHeader;
    std::vector<std::pair<size_t, size_t>> spans;  // [begin, end) of each line
    size_t pos = 0;
    while (pos < text.size()) {
        const size_t nl = text.find('\n', pos);
        const size_t e = nl == std::string::npos ? text.size() : nl;
        spans.push_back({pos, e});
        pos = e + 1;
    }
    if (spans.empty()) throw IoError(path + ": empty file");
    const std::string_view first(text.data() + spans[0].first, spans[0].second - spans[0].first);
    if (trim(first) != hdr)
        throw IoError(path + ":1: expected " + (wide ? "wide" : "long") + " header '" + hdr + "'");
    const size_t nl = spans.size() - 1;
    std::vector<Line> lines(nl);
    const unsigned nt = (unsigned)std::max<size_t>(
        1, std::min<size_t>({std::thread::hardware_concurrency(), 32u, nl / 4096 + 1}));
    std::atomic<size_t> next{0};
    auto work = [&] {
        constexpr size_t kBlock = 2048;
        for (size_t b; (b = next.fetch_add(kBlock)) < nl;)
            for (size_t i = b; i < std::min(nl, b + kBlock); ++i) {
                const auto& sp = spans[i + 1];
                lines[i].line_no = i + 2;
                parse_line(std::string_view(text.data() + sp.first, sp.second - sp.first), wide,
                           lines[i]);
            }
    };
    std::vector<std::thread> pool;
    for (unsigned t = 1; t < nt; ++t) pool.emplace_back(work);
    work();
    for (auto& t : pool) t.join();
    return lines;  // per-line errors are raised by the (sequential) assembly, in line order
}

// NameIndex (io.cpp:91-101): first-appearance order.
struct NameIndex {
    std::unordered_map<std::string_view, size_t> index;
    std::vector<std::string_view> names;
    size_t at(std::string_view n) {
        const auto [it, ins] = index.try_emplace(n, names.size());
        if (ins) names.push_back(n);
        return it->second;
    }
};

}  // namespace

// ---------------------------------------------------------------- library-owned objects
struct scx_table {  // SurvivalDataset with names and labels (data.hpp:31-45)
    std::vector<double> time;
    std::vector<uint8_t> event;
    std::vector<int32_t> stratum;
    std::vector<int64_t> subject;
    std::vector<int64_t> col_ptr;
    std::vector<int64_t> rows;
    std::vector<double> values;
    std::vector<std::string> names;
    std::vector<std::string> labels;
};

struct scx_long {  // LongData (io.hpp:32-43)
    struct Record {
        int64_t subject;
        double start, stop;
        uint8_t event;
        std::vector<std::pair<size_t, double>> values;
    };
    std::vector<std::vector<Record>> subjects;
    std::vector<std::string> names;
    double max_stop = 0.0;
};

struct scx_config {  // ConfigMap (io.hpp:57-76)
    std::string origin;
    std::map<std::string, std::string> values;
    std::set<std::string> consumed;
    std::vector<std::string> str_out;  // backing store of returned strings
};

namespace {

scx_status report(char* err, int cap, const std::string& m) {
    if (err && cap > 0) {
        std::strncpy(err, m.c_str(), (size_t)cap - 1);
        err[cap - 1] = 0;
    }
    return SCX_ERR_VALIDATION;
}

// read_wide_csv (io.cpp:123-193)
scx_table* read_wide(const std::string& path) {
    const std::string text = slurp(path);
    std::vector<Line> lines = parse_file(path, text, true);
    auto* T = new scx_table();
    NameIndex cov, strata;
    std::vector<std::vector<std::pair<int64_t, double>>> entries;
    std::vector<int32_t> raw;
    for (const Line& L : lines) {
        if (!L.err.empty()) {
            delete T;
            throw IoError(line_msg(path, L.line_no, L.err));
        }
        if (L.empty) continue;
        const int64_t row = (int64_t)T->time.size();
        T->subject.push_back(L.subject);
        raw.push_back((int32_t)strata.at(L.label) + 1);
        T->time.push_back(L.a);
        T->event.push_back(L.event);
        for (const Token& t : L.tokens) {
            const size_t j = cov.at(t.name);  // a zero still declares the covariate
            if (t.value == 0.0) continue;     // but is never stored
            if (entries.size() <= j) entries.resize(j + 1);
            entries[j].emplace_back(row, t.value);
        }
    }
    if (T->time.empty()) {
        delete T;
        throw IoError(path + ": no rows");
    }
    // strata relabelled 1..K by label: numeric order when every label is a number
    const size_t K = strata.names.size();
    std::vector<size_t> order(K);
    std::iota(order.begin(), order.end(), 0);
    bool numeric = true;
    std::vector<double> num(K, 0.0);
    for (size_t i = 0; i < K && numeric; ++i) {
        const std::string_view l = strata.names[i];
        const auto res = std::from_chars(l.data(), l.data() + l.size(), num[i]);
        numeric = res.ec == std::errc{} && res.ptr == l.data() + l.size();
    }
    std::sort(order.begin(), order.end(), [&](size_t a, size_t b) {
        return numeric ? num[a] < num[b] : strata.names[a] < strata.names[b];
    });
    std::vector<int32_t> remap(K);
    for (size_t r = 0; r < K; ++r) {
        remap[order[r]] = (int32_t)(r + 1);
        T->labels.emplace_back(strata.names[order[r]]);
    }
    T->stratum.reserve(raw.size());
    for (int32_t s : raw) T->stratum.push_back(remap[(size_t)(s - 1)]);
    // columns in name order (sort_columns_by_name, data.cpp:199-217)
    const size_t p = cov.names.size();
    std::vector<size_t> by(p);
    std::iota(by.begin(), by.end(), 0);
    std::sort(by.begin(), by.end(), [&](size_t a, size_t b) { return cov.names[a] < cov.names[b]; });
    T->col_ptr.push_back(0);
    for (size_t pos = 0; pos < p; ++pos) {
        const size_t j = by[pos];
        T->names.emplace_back(cov.names[j]);
        if (j < entries.size())
            for (const auto& [r, v] : entries[j]) {
                T->rows.push_back(r);
                T->values.push_back(v);
            }
        T->col_ptr.push_back((int64_t)T->rows.size());
    }
    return T;
}

std::string cov_name(const char* const* names, int64_t j) {
    if (names && names[j] && names[j][0]) return names[j];
    return "x" + std::to_string(j + 1);
}

// write_wide_csv (io.cpp:195-223): tokens per row in name order
void write_wide(const std::string& path, const scx_dataset* d, const char* const* names,
                const char* const* labels) {
    const int64_t n = d->n_rows, p = d->n_covariates;
    for (int64_t i = 0; i < n; ++i) {  // validate_invariants (data.cpp:27-66), row part
        if (!std::isfinite(d->time[i]) || d->time[i] < 0.0)
            throw IoError("negative or non-finite time at row " + std::to_string(i));
        if (d->event[i] > 1) throw IoError("event indicator must be 0 or 1 at row " + std::to_string(i));
    }
    std::ofstream out(path);
    if (!out) throw IoError("cannot write " + path);
    std::vector<std::string> nm(p);
    for (int64_t j = 0; j < p; ++j) nm[j] = cov_name(names, j);
    std::vector<int64_t> by(p);
    std::iota(by.begin(), by.end(), 0);
    std::sort(by.begin(), by.end(), [&](int64_t a, int64_t b) { return nm[a] < nm[b]; });
    std::vector<std::vector<std::pair<int64_t, double>>> by_row(n);
    for (const int64_t j : by)
        for (int64_t t = d->col_ptr[j]; t < d->col_ptr[j + 1]; ++t)
            by_row[d->row_idx[t]].emplace_back(j, d->values ? d->values[t] : 1.0);
    std::string line;
    out << kWideHeader << "\n";
    for (int64_t i = 0; i < n; ++i) {
        const int32_t s = d->stratum[i];
        const std::string label =
            (labels && labels[s - 1] && labels[s - 1][0]) ? labels[s - 1] : std::to_string(s);
        line.clear();
        line += std::to_string(d->subject ? d->subject[i] : i + 1);
        line += ',';
        line += label;
        line += ',';
        line += format_double(d->time[i]);
        line += ',';
        line += d->event[i] ? '1' : '0';
        line += ',';
        for (size_t t = 0; t < by_row[i].size(); ++t) {
            if (t) line += ' ';
            line += nm[by_row[i][t].first];
            line += ':';
            line += format_double(by_row[i][t].second);
        }
        line += '\n';
        out << line;
    }
}

// read_long_csv (io.cpp:225-272)
scx_long* read_long(const std::string& path) {
    const std::string text = slurp(path);
    std::vector<Line> lines = parse_file(path, text, false);
    auto* D = new scx_long();
    NameIndex cov;
    std::unordered_map<int64_t, size_t> slot;
    for (const Line& L : lines) {
        if (!L.err.empty()) {
            delete D;
            throw IoError(line_msg(path, L.line_no, L.err));
        }
        if (L.empty) continue;
        scx_long::Record rec{L.subject, L.a, L.b, L.event, {}};
        for (const Token& t : L.tokens)
            if (t.value != 0.0) rec.values.emplace_back(cov.at(t.name), t.value);
        const auto [it, ins] = slot.try_emplace(L.subject, D->subjects.size());
        if (ins) D->subjects.emplace_back();
        auto& recs = D->subjects[it->second];
        const std::string sid = std::to_string(L.subject);
        if (recs.empty()) {
            if (rec.start != 0.0) {
                delete D;
                throw IoError(line_msg(path, L.line_no, "first interval of subject " + sid + " must start at 0"));
            }
        } else {
            if (recs.back().event) {
                delete D;
                throw IoError(line_msg(path, L.line_no, "subject " + sid + " has records after its event"));
            }
            if (rec.start != recs.back().stop) {
                delete D;
                throw IoError(line_msg(path, L.line_no, "intervals of subject " + sid + " must be contiguous"));
            }
        }
        D->max_stop = std::max(D->max_stop, rec.stop);
        recs.push_back(std::move(rec));
    }
    if (D->subjects.empty()) {
        delete D;
        throw IoError(path + ": no rows");
    }
    for (std::string_view n : cov.names) D->names.emplace_back(n);
    return D;
}

void write_long(const std::string& path, const scx_long* D) {  // io.cpp:274-291
    std::ofstream out(path);
    if (!out) throw IoError("cannot write " + path);
    out << kLongHeader << "\n";
    for (const auto& recs : D->subjects)
        for (const auto& r : recs) {
            out << r.subject << ',' << format_double(r.start) << ',' << format_double(r.stop) << ','
                << int(r.event) << ',';
            for (size_t t = 0; t < r.values.size(); ++t) {
                if (t) out << ' ';
                out << D->names[r.values[t].first] << ':' << format_double(r.values[t].second);
            }
            out << '\n';
        }
}

int event_interval(double y, const std::vector<double>& cuts) {  // transforms.cpp:25-30
    const int k_count = (int)cuts.size() - 1;
    if (y == cuts.back()) return k_count;
    return (int)(std::upper_bound(cuts.begin(), cuts.end(), y) - cuts.begin());
}
bool at_risk(double y, uint8_t event, int k, const std::vector<double>& cuts) {  // :32-36
    if (y > cuts[k - 1]) return true;
    return event != 0 && y == cuts[k - 1] && event_interval(y, cuts) == k;
}

// to_time_varying (io.cpp:293-345) + lower_pipeline (transforms.cpp:98-231):
// per-interval schedules from the records, effect-window splits, then the
// interval-major augmentation with the reference's names and column map.
scx_lowered* lower_long(const scx_long* D, const std::vector<double>& cuts, const int64_t* split_cov,
                        const int64_t* split_ptr, const double* split_times, int64_t n_splits) {
    // validate_cut_points (transforms.cpp:39-46)
    if (cuts.size() < 2) throw IoError("need at least two cut points");
    if (cuts.front() != 0.0) throw IoError("first cut point must be 0");
    for (size_t i = 1; i < cuts.size(); ++i)
        if (!std::isfinite(cuts[i]) || cuts[i] <= cuts[i - 1])
            throw IoError("cut points must be finite and strictly increasing");
    const size_t n = D->subjects.size(), p = D->names.size();
    const int K = (int)cuts.size() - 1;
    std::vector<double> time(n);
    std::vector<uint8_t> event(n);
    std::vector<int64_t> subject(n);
    // sched[j][k] = (subject, value) entries of covariate j in interval k
    std::vector<std::vector<std::vector<std::pair<int64_t, double>>>> sched(
        p, std::vector<std::vector<std::pair<int64_t, double>>>(K));
    for (size_t i = 0; i < n; ++i) {
        const auto& recs = D->subjects[i];
        subject[i] = recs.front().subject;
        time[i] = recs.back().stop;
        event[i] = recs.back().event;
        if (time[i] > cuts.back())
            throw IoError("cut points do not cover follow-up of subject " + std::to_string(subject[i]));
        for (size_t r = 1; r < recs.size(); ++r)
            if (!std::binary_search(cuts.begin(), cuts.end(), recs[r].start))
                throw IoError("covariate change at time " + format_double(recs[r].start) + " of subject " +
                              std::to_string(subject[i]) + " does not align with a cut point");
        for (int k = 1; k <= K; ++k) {
            if (!at_risk(time[i], event[i], k, cuts)) continue;
            const double at = cuts[k - 1];
            const scx_long::Record* src = &recs.back();
            for (const auto& rec : recs)
                if (rec.start <= at && at < rec.stop) {
                    src = &rec;
                    break;
                }
            for (const auto& [j, v] : src->values) sched[j][k - 1].emplace_back((int64_t)i, v);
        }
    }
    // validate (transforms.cpp:48-62): times are finite and >= 0 by construction
    // split_time_varying_coefficient (:98-175)
    std::vector<std::vector<double>> bounds(p);
    for (int64_t sidx = 0; sidx < n_splits; ++sidx) {
        const int64_t j = split_cov[sidx];
        if (j < 0 || (size_t)j >= p) throw IoError("split covariate index out of range");
        if (split_ptr[sidx + 1] == split_ptr[sidx])
            throw IoError("split for covariate " + D->names[j] + " declares no times");
        if (!bounds[j].empty()) throw IoError("covariate split declared twice");
        std::set<double> seen;
        for (int64_t t = split_ptr[sidx]; t < split_ptr[sidx + 1]; ++t) {
            const double v = split_times[t];
            if (!(v > 0.0) || !(v < cuts.back()))
                throw IoError("split time " + format_double(v) + " outside the follow-up window");
            if (!std::binary_search(cuts.begin(), cuts.end(), v))
                throw IoError("split time " + format_double(v) + " is not a cut point");
            if (!seen.insert(v).second) throw IoError("duplicate split time " + format_double(v));
        }
        bounds[j].assign(seen.begin(), seen.end());
    }
    auto* L = new scx_lowered();
    struct OutCol {
        size_t src;
        int window;
        double start, end;
    };
    std::vector<OutCol> cols;
    for (size_t j = 0; j < p; ++j) {
        if (bounds[j].empty()) {
            cols.push_back({j, -1, cuts.front(), cuts.back()});
            L->names.push_back(D->names[j]);
            continue;
        }
        std::vector<double> edges{cuts.front()};
        edges.insert(edges.end(), bounds[j].begin(), bounds[j].end());
        edges.push_back(cuts.back());
        for (size_t w = 0; w + 1 < edges.size(); ++w) {
            cols.push_back({j, (int)w, edges[w], edges[w + 1]});
            const bool last = w + 2 == edges.size();  // window_name (transforms.cpp:18-21)
            L->names.push_back(D->names[j] + "[" + format_double(edges[w]) + "-" +
                               format_double(edges[w + 1]) + (last ? "]" : ")"));
        }
    }
    // augment_to_strata (:177-223): interval-major rows, subjects in input order
    std::vector<std::vector<int64_t>> rank(K, std::vector<int64_t>(n, -1));
    for (int k = 1; k <= K; ++k) {
        const int64_t offset = (int64_t)L->time.size();
        int64_t emitted = 0;
        for (size_t i = 0; i < n; ++i) {
            if (!at_risk(time[i], event[i], k, cuts)) continue;
            rank[k - 1][i] = offset + emitted++;
            L->time.push_back(std::min(time[i], cuts[k]));
            L->event.push_back(event[i] && event_interval(time[i], cuts) == k ? 1 : 0);
            L->stratum.push_back(k);
            L->subject.push_back(subject[i]);
        }
    }
    L->col_ptr.push_back(0);
    for (const OutCol& oc : cols) {
        for (int k = 1; k <= K; ++k) {
            if (oc.window >= 0 && !(cuts[k - 1] >= oc.start && cuts[k - 1] < oc.end)) continue;
            for (const auto& [i, v] : sched[oc.src][k - 1]) {
                const int64_t r = rank[k - 1][i];
                if (r >= 0 && v != 0.0) {
                    L->rows.push_back(r);
                    L->values.push_back(v);
                }
            }
        }
        L->col_ptr.push_back((int64_t)L->rows.size());
        L->map_source.push_back((int64_t)oc.src);
        L->map_window.push_back(oc.window);
        L->map_start.push_back(oc.start);
        L->map_end.push_back(oc.end);
    }
    return L;
}

// ConfigMap::from_string (io.cpp:353-375)
scx_config* config_parse(const std::string& text, const std::string& origin) {
    auto* c = new scx_config();
    c->origin = origin;
    std::istringstream in(text);
    std::string line;
    size_t no = 0;
    while (std::getline(in, line)) {
        ++no;
        std::string_view body(line);
        const size_t hash = body.find('#');
        if (hash != std::string_view::npos) body = body.substr(0, hash);
        body = trim(body);
        if (body.empty()) continue;
        const size_t eq = body.find('=');
        if (eq == std::string_view::npos) {
            delete c;
            throw IoError(line_msg(origin, no, "expected key = value"));
        }
        const std::string key(trim(body.substr(0, eq)));
        const std::string value(trim(body.substr(eq + 1)));
        if (key.empty()) {
            delete c;
            throw IoError(line_msg(origin, no, "empty key"));
        }
        if (!c->values.emplace(key, value).second) {
            delete c;
            throw IoError(line_msg(origin, no, "duplicate key '" + key + "'"));
        }
    }
    return c;
}

std::vector<std::string_view> list_pieces(std::string_view rest) {
    std::vector<std::string_view> out;
    while (!rest.empty()) {
        const size_t comma = rest.find(',');
        const std::string_view piece = trim(comma == std::string_view::npos ? rest : rest.substr(0, comma));
        rest.remove_prefix(comma == std::string_view::npos ? rest.size() : comma + 1);
        if (!piece.empty()) out.push_back(piece);
    }
    return out;
}

template <class F>
scx_status guarded(char* err, int cap, F&& f) {
    try {
        f();
        return SCX_OK;
    } catch (const IoError& e) {
        return report(err, cap, e.what());
    } catch (const std::bad_alloc&) {
        return report(err, cap, "out of memory");
    }
}

}  // namespace

extern "C" {

// ---------------------------------------------------------------- wide CSV
scx_status scx_read_wide_csv(const char* path, scx_table** out, char* err, int cap) {
    if (!path || !out) return report(err, cap, "null argument");
    *out = nullptr;
    return guarded(err, cap, [&] { *out = read_wide(path); });
}

scx_status scx_table_dataset(const scx_table* T, scx_dataset* v) {
    if (!T || !v) return SCX_ERR_VALIDATION;
    v->n_rows = (int64_t)T->time.size();
    v->time = T->time.data();
    v->event = T->event.data();
    v->stratum = T->stratum.data();
    v->subject = T->subject.data();
    v->n_covariates = (int64_t)T->names.size();
    v->col_ptr = T->col_ptr.data();
    v->row_idx = T->rows.data();
    v->values = T->values.data();
    return SCX_OK;
}

const char* scx_table_covariate_name(const scx_table* T, int64_t j) {
    return (T && j >= 0 && (size_t)j < T->names.size()) ? T->names[j].c_str() : nullptr;
}

int32_t scx_table_n_strata(const scx_table* T) { return T ? (int32_t)T->labels.size() : 0; }

const char* scx_table_stratum_label(const scx_table* T, int32_t k) {
    return (T && k >= 1 && (size_t)k <= T->labels.size()) ? T->labels[k - 1].c_str() : nullptr;
}

void scx_table_free(scx_table* T) { delete T; }

scx_status scx_write_wide_csv(const char* path, const scx_dataset* data,
                              const char* const* covariate_names, const char* const* stratum_labels,
                              char* err, int cap) {
    if (!path || !data) return report(err, cap, "null argument");
    return guarded(err, cap, [&] { write_wide(path, data, covariate_names, stratum_labels); });
}

// ---------------------------------------------------------------- long CSV
scx_status scx_read_long_csv(const char* path, scx_long** out, char* err, int cap) {
    if (!path || !out) return report(err, cap, "null argument");
    *out = nullptr;
    return guarded(err, cap, [&] { *out = read_long(path); });
}

scx_status scx_long_sizes(const scx_long* D, int64_t* n_subjects, int64_t* n_records,
                          int64_t* n_covariates, double* max_stop) {
    if (!D) return SCX_ERR_VALIDATION;
    int64_t r = 0;
    for (const auto& s : D->subjects) r += (int64_t)s.size();
    if (n_subjects) *n_subjects = (int64_t)D->subjects.size();
    if (n_records) *n_records = r;
    if (n_covariates) *n_covariates = (int64_t)D->names.size();
    if (max_stop) *max_stop = D->max_stop;
    return SCX_OK;
}

const char* scx_long_covariate_name(const scx_long* D, int64_t j) {
    return (D && j >= 0 && (size_t)j < D->names.size()) ? D->names[j].c_str() : nullptr;
}

scx_status scx_write_long_csv(const char* path, const scx_long* D, char* err, int cap) {
    if (!path || !D) return report(err, cap, "null argument");
    return guarded(err, cap, [&] { write_long(path, D); });
}

scx_status scx_long_lower(const scx_long* D, const double* cut_points, int64_t n_cuts,
                          const int64_t* split_covariate, const int64_t* split_ptr,
                          const double* split_times, int64_t n_splits, scx_lowered** out, char* err,
                          int cap) {
    if (!D || !cut_points || !out) return report(err, cap, "null argument");
    *out = nullptr;
    return guarded(err, cap, [&] {
        *out = lower_long(D, std::vector<double>(cut_points, cut_points + n_cuts), split_covariate,
                          split_ptr, split_times, n_splits);
    });
}

void scx_long_free(scx_long* D) { delete D; }

const char* scx_lowered_covariate_name(const scx_lowered* L, int64_t j) {
    return (L && j >= 0 && (size_t)j < L->names.size()) ? L->names[j].c_str() : nullptr;
}

// ---------------------------------------------------------------- ConfigMap
scx_status scx_config_from_string(const char* text, const char* origin, scx_config** out, char* err,
                                  int cap) {
    if (!text || !out) return report(err, cap, "null argument");
    *out = nullptr;
    return guarded(err, cap, [&] { *out = config_parse(text, origin ? origin : "<config>"); });
}

scx_status scx_config_from_file(const char* path, scx_config** out, char* err, int cap) {
    if (!path || !out) return report(err, cap, "null argument");
    *out = nullptr;
    return guarded(err, cap, [&] { *out = config_parse(slurp(path), path); });
}

int scx_config_has(const scx_config* c, const char* key) {
    return c && key && c->values.count(key) ? 1 : 0;
}

// get_string (io.cpp:379-383): the value or the fallback; the key is consumed.
const char* scx_config_get_string(scx_config* c, const char* key, const char* fallback) {
    if (!c || !key) return fallback;
    c->consumed.insert(key);
    const auto it = c->values.find(key);
    if (it == c->values.end()) return fallback;
    c->str_out.push_back(it->second);
    return c->str_out.back().c_str();
}

// get_double / get_int (io.cpp:385-397); messages "ORIGIN:0: cannot parse KEY 'TEXT'"
scx_status scx_config_get_double(scx_config* c, const char* key, double fallback, double* out,
                                 char* err, int cap) {
    if (!c || !key || !out) return report(err, cap, "null argument");
    c->consumed.insert(key);
    const auto it = c->values.find(key);
    if (it == c->values.end()) {
        *out = fallback;
        return SCX_OK;
    }
    if (!parse_double(it->second, *out)) return report(err, cap, line_msg(c->origin, 0, cannot(key, it->second)));
    return SCX_OK;
}

scx_status scx_config_get_int(scx_config* c, const char* key, int64_t fallback, int64_t* out,
                              char* err, int cap) {
    if (!c || !key || !out) return report(err, cap, "null argument");
    c->consumed.insert(key);
    const auto it = c->values.find(key);
    if (it == c->values.end()) {
        *out = fallback;
        return SCX_OK;
    }
    if (!parse_int(it->second, *out)) return report(err, cap, line_msg(c->origin, 0, cannot(key, it->second)));
    return SCX_OK;
}

// get_double_list (io.cpp:399-413): comma-separated, empty pieces skipped;
// *n = number of values (out may be NULL to query, cap_out entries written)
scx_status scx_config_get_double_list(scx_config* c, const char* key, double* out, int64_t cap_out,
                                      int64_t* n, char* err, int cap) {
    if (!c || !key || !n) return report(err, cap, "null argument");
    c->consumed.insert(key);
    *n = 0;
    const auto it = c->values.find(key);
    if (it == c->values.end()) return SCX_OK;
    int64_t m = 0;
    for (std::string_view piece : list_pieces(it->second)) {
        double v;
        if (!parse_double(piece, v)) return report(err, cap, line_msg(c->origin, 0, cannot(key, piece)));
        if (out && m < cap_out) out[m] = v;
        ++m;
    }
    *n = m;
    return SCX_OK;
}

// get_string_list (io.cpp:415-429): newline-joined pieces (valid until the next get)
const char* scx_config_get_string_list(scx_config* c, const char* key, int64_t* n) {
    if (n) *n = 0;
    if (!c || !key) return "";
    c->consumed.insert(key);
    const auto it = c->values.find(key);
    if (it == c->values.end()) return "";
    std::string joined;
    int64_t m = 0;
    for (std::string_view piece : list_pieces(it->second)) {
        if (m++) joined += '\n';
        joined += piece;
    }
    if (n) *n = m;
    c->str_out.push_back(joined);
    return c->str_out.back().c_str();
}

// finish (io.cpp:431-438): every key consumed, else "ORIGIN: unknown config key(s): a, b"
scx_status scx_config_finish(const scx_config* c, char* err, int cap) {
    if (!c) return report(err, cap, "null argument");
    std::string unknown;
    for (const auto& [key, value] : c->values)
        if (!c->consumed.count(key)) unknown += unknown.empty() ? key : ", " + key;
    if (!unknown.empty()) return report(err, cap, c->origin + ": unknown config key(s): " + unknown);
    return SCX_OK;
}

void scx_config_free(scx_config* c) { delete c; }

}  // extern "C"
