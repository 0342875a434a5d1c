#include <chrono>
// C-ABI (include/stratcox_b200.h) over the sm_100a kernels in kernels.cu.
//
// Host responsibilities only: argument validation with the reference's exact
// messages, device allocation and upload of the SortedDesign, kernel
// sequencing on the context's stream, and mapping the device error word back
// to the reference exception taxonomy (proj/include/stratcox/errors.hpp).
// No arithmetic of the hot path runs here.
#include <algorithm>
#include <array>
#include <cinttypes>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include <cudaTypedefs.h>

#include "../../include/stratcox_b200.h"
#include "internal.cuh"

using namespace scx;

namespace {

constexpr long long kNoRow = 0x7fffffffffffffffLL;

PFN_cuTensorMapEncodeTiled_v12000 tmap_encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q;
        void* p = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    return fn;
}

// [npad/16][16] f64 view, box 16 x (tile_rows/16) (one tile), 128-B swizzle.
bool make_tmap(CUtensorMap* m, double* base, int64_t npad, int tile_rows = kTileRows) {
    auto enc = tmap_encoder();
    if (!enc) return false;
    cuuint64_t dims[2] = {16, (cuuint64_t)(npad / 16)};
    cuuint64_t strides[1] = {16 * sizeof(double)};
    cuuint32_t box[2] = {16, (cuuint32_t)(tile_rows / 16)};
    cuuint32_t es[2] = {1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, base, dims, strides, box, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
               CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <class T>
cudaError_t dmalloc(T** p, size_t count) {
    return cudaMalloc((void**)p, std::max<size_t>(count, 1) * sizeof(T));
}

struct Timer {
    bool on = false;
    double ms[4] = {0, 0, 0, 0};
    int64_t launches[4] = {0, 0, 0, 0};
    std::vector<cudaEvent_t> ev;
    std::vector<int> kinds;
    size_t used = 0;
};

}  // namespace

struct scx_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    std::string err;
    bool has_design = false;
    DesignDev d{};
    DevCtl* ctl_h = nullptr;  // pinned mirror of d.ctl
    long long* warn_d = nullptr;  // [kWarnCap] fit warnings (DevCtl::warn_coord)
    // host metadata
    std::vector<ColArgs> cols;
    std::vector<int32_t> zero_cols;
    int32_t* zero_cols_d = nullptr;
    std::vector<int64_t> tie_end_h;  // for error-message row mapping only
    std::vector<uint8_t> event_h;
    int64_t nnz = 0;
    int64_t n_indicator = 0;
    double* xdense = nullptr;
    double* out2 = nullptr;
    int64_t* col_beg_d = nullptr;
    int64_t* val_off_d = nullptr;
    int64_t* offsets_d = nullptr;
    int32_t* rows_d = nullptr;
    double* vals_d = nullptr;
    int32_t* tptr_d = nullptr;
    // CCD cycle kernel: the nnz > 0 columns in ascending j (device copy) and
    // their maximal runs of one kind (indicator / value): {first, count, indicator}
    ColArgs* cols_d = nullptr;
    std::vector<std::array<int32_t, 3>> runs;
    bool per_coordinate_fit = false;  // SCX_FIT_PER_COORD=1: one K1 + K3 launch per coordinate
    int fit_path = 0;                 // 0 auto (risk-suffix cycle when eligible), 1 fused-scan cycle
    ColArgs* col1_d = nullptr;        // one column's ColArgs (risk-suffix evaluation)
    int64_t rs_stats[4] = {0, 0, 0, 0};  // last fit: risk-suffix launches, exact hand-offs,
                                         // bound hand-offs, fused-scan cycle launches
    // multi-GPU (row shards): the device exchange (XSlot pairs of every rank,
    // see internal.cuh) and the global column set
    Xchg x{};                   // x.nranks == 0 / 1: single device
    XSlot* xslots = nullptr;    // this rank's two slots
    std::vector<void*> ipc_open;  // peer slot mappings opened from IPC handles
    int nranks = 1, rank = 0;
    int sm_budget = 0;          // chunks / co-resident CTAs of the cycle kernel (0: every SM)
    std::vector<uint8_t> gnz;   // column has entries on SOME rank (the sharded loop's column set)
    std::vector<ColArgs> cycle_cols;  // host copy of cols_d
    Timer timer;
    int64_t launches = 0;  // kernels launched by this context
};

namespace {

scx_status fail(scx_ctx* c, scx_status s, const std::string& msg) {
    if (c) c->err = msg;
    return s;
}

scx_status cuda_fail(scx_ctx* c, cudaError_t e, const char* where) {
    return fail(c, SCX_ERR_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

#define CK(expr)                                                   \
    do {                                                           \
        cudaError_t _e = (expr);                                   \
        if (_e != cudaSuccess) return cuda_fail(ctx, _e, #expr);   \
    } while (0)

// kernel launch through the launch_* helpers, counted for bench.py's gpu_launches
#define KL(n, expr)              \
    do {                         \
        ctx->launches += (n);    \
        CK(expr);                \
    } while (0)

void free_design(scx_ctx* ctx) {
    DesignDev& d = ctx->d;
    void* ptrs[] = {d.code,   d.D,          d.eta,         d.beta,      d.gamma,     d.l2,
                    d.trust,  d.status,     d.slots,       d.partial,   ctx->xdense,
                    ctx->col_beg_d, ctx->val_off_d, ctx->offsets_d, ctx->rows_d,
                    ctx->vals_d, ctx->tptr_d, ctx->zero_cols_d, d.lasth1, d.ref_act,
                    d.ref_abeg, d.ref_avo, d.ref_ab, d.ref_nact, d.ref_meta,
                    d.chunk_rows, ctx->cols_d, d.rs_CR, d.rs_CQ, d.rs_R, d.rs_Q, d.chunk_k, ctx->col1_d,
                    d.rs_chunk_nk, d.rs_xagg, d.rs_aligned ? nullptr : d.rs_chunk_rows,
                    d.ell_col, d.ell_val, d.ell_base};
    for (void* p : ptrs)
        if (p) cudaFree(p);
    const DevCtl* keep_ctl = d.ctl;
    d = DesignDev{};
    d.ctl = const_cast<DevCtl*>(keep_ctl);
    ctx->xdense = nullptr;
    ctx->col1_d = nullptr;
    ctx->col_beg_d = nullptr;
    ctx->val_off_d = nullptr;
    ctx->offsets_d = nullptr;
    ctx->rows_d = nullptr;
    ctx->vals_d = nullptr;
    ctx->tptr_d = nullptr;
    ctx->zero_cols_d = nullptr;
    ctx->cols_d = nullptr;
    ctx->cycle_cols.clear();
    ctx->runs.clear();
    ctx->cols.clear();
    ctx->zero_cols.clear();
    ctx->has_design = false;
}

scx_status sync(scx_ctx* ctx) {
    CK(cudaStreamSynchronize(ctx->stream));
    return SCX_OK;
}

scx_status read_ctl(scx_ctx* ctx) {
    CK(cudaMemcpyAsync(ctx->ctl_h, ctx->d.ctl, sizeof(DevCtl), cudaMemcpyDeviceToHost,
                       ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    return SCX_OK;
}

scx_status clear_error(scx_ctx* ctx) {
    const int zero = 0;
    const long long none = kNoRow;
    CK(cudaMemcpyAsync(&ctx->d.ctl->err_kind, &zero, sizeof(int), cudaMemcpyHostToDevice,
                       ctx->stream));
    CK(cudaMemcpyAsync(&ctx->d.ctl->bad_min, &none, sizeof(long long), cudaMemcpyHostToDevice,
                       ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    return SCX_OK;
}

// First event row i (sorted order) whose tie group ends at s.
int64_t first_event_row_of_group(const scx_ctx* ctx, int64_t s) {
    int64_t best = s;
    for (int64_t r = s; r >= 0 && ctx->tie_end_h[r] == s; --r)
        if (ctx->event_h[r]) best = r;
    return best;
}

// Map a pending device error to the reference's exception text.
scx_status map_error(scx_ctx* ctx, int j_hint) {
    const DevCtl& c = *ctx->ctl_h;
    const int kind = c.err_kind;
    const long long idx = c.err_idx;
    char buf[256];
    scx_status st = SCX_ERR_INTERNAL;
    switch (kind) {
        case kErrNonFiniteD:
            snprintf(buf, sizeof buf, "non-finite input at index %lld", idx);
            st = SCX_ERR_VALIDATION;
            break;
        case kErrBadDenom:
            snprintf(buf, sizeof buf, "risk-set sum not positive at sorted row %" PRId64,
                     first_event_row_of_group(ctx, idx));
            st = SCX_ERR_INTERNAL;
            break;
        case kErrNonFiniteGH: {
            // Diagnose like likelihood.cpp:178-187: a non-positive / non-finite
            // risk-set sum at an event row is an internal error, else numeric.
            const int j = (int)idx;
            clear_error(ctx);
            const ColArgs& col = ctx->cols[j];
            launch_k1(ctx->d, col, kK1Diag, ctx->stream);
            read_ctl(ctx);
            if (ctx->ctl_h->bad_min != kNoRow) {
                snprintf(buf, sizeof buf, "risk-set sum not positive at sorted row %" PRId64,
                         first_event_row_of_group(ctx, ctx->ctl_h->bad_min));
                st = SCX_ERR_INTERNAL;
            } else {
                snprintf(buf, sizeof buf, "non-finite gradient/Hessian for covariate x%d", j + 1);
                st = SCX_ERR_NUMERIC;
            }
            break;
        }
        case kErrNonFiniteLL:
            snprintf(buf, sizeof buf, "non-finite log partial likelihood");
            st = SCX_ERR_NUMERIC;
            break;
        case kErrRuleNewton:
            snprintf(buf, sizeof buf, "non-finite gradient or Hessian in Newton step");
            st = SCX_ERR_NUMERIC;
            break;
        case kErrRuleTrust:
            snprintf(buf, sizeof buf, "non-finite trust-region inputs");
            st = SCX_ERR_NUMERIC;
            break;
        case kErrRuleBothNegative:
            snprintf(buf, sizeof buf, "both directional derivatives negative at the origin");
            st = SCX_ERR_INTERNAL;
            break;
        case kErrLPOverflow:
            snprintf(buf, sizeof buf, "linear predictor overflow at row %lld", idx);
            st = SCX_ERR_NUMERIC;
            break;
        case kErrStepOverflow:
            snprintf(buf, sizeof buf, "step overflow");
            st = SCX_ERR_NUMERIC;
            break;
        case kErrNonFiniteStep:
            snprintf(buf, sizeof buf, "non-finite coordinate step");
            st = SCX_ERR_NUMERIC;
            break;
        case kErrBadTieEnd:
            snprintf(buf, sizeof buf, "tie_group_end out of range at row %lld", idx);
            st = SCX_ERR_VALIDATION;
            break;
        case kErrBadEvent:
            snprintf(buf, sizeof buf, "event indicator must be 0 or 1 at row %lld", idx);
            st = SCX_ERR_VALIDATION;
            break;
        case kErrBadRows:
            snprintf(buf, sizeof buf, "column row indices must be strictly increasing");
            st = SCX_ERR_VALIDATION;
            break;
        case kErrXchgTimeout:
            snprintf(buf, sizeof buf,
                     "multi-GPU exchange timed out (exchange %lld, site %lld): a peer rank did "
                     "not arrive", idx / 16, idx % 16);
            st = SCX_ERR_CUDA;
            break;
        case kErrPeer:
            snprintf(buf, sizeof buf, "another rank of the sharded fit stopped with an error");
            st = SCX_ERR_CUDA;
            break;
        default:
            snprintf(buf, sizeof buf, "device error kind %d (index %lld)", kind, idx);
    }
    (void)j_hint;
    clear_error(ctx);
    return fail(ctx, st, buf);
}

scx_status check_device_error(scx_ctx* ctx, int j_hint = -1) {
    scx_status s = read_ctl(ctx);
    if (s) return s;
    if (ctx->ctl_h->err_kind != kErrNone) return map_error(ctx, j_hint);
    return SCX_OK;
}

scx_status need_design(scx_ctx* ctx) {
    if (!ctx) return SCX_ERR_VALIDATION;
    if (!ctx->has_design) return fail(ctx, SCX_ERR_VALIDATION, "no design uploaded");
    return SCX_OK;
}

// timing helpers (bench only)
void tmark(scx_ctx* ctx, int kind) {
    Timer& t = ctx->timer;
    if (!t.on) return;
    if (t.used + 2 > t.ev.size()) {
        const size_t add = 4096;
        for (size_t i = 0; i < add; ++i) {
            cudaEvent_t e;
            cudaEventCreate(&e);
            t.ev.push_back(e);
        }
        t.kinds.resize(t.ev.size() / 2);
    }
    cudaEventRecord(t.ev[t.used], ctx->stream);
    t.kinds[t.used / 2] = kind;
    t.used += 1;
}
void tend(scx_ctx* ctx) {
    Timer& t = ctx->timer;
    if (!t.on) return;
    cudaEventRecord(t.ev[t.used], ctx->stream);
    t.used += 1;
}
void tcollect(scx_ctx* ctx) {
    Timer& t = ctx->timer;
    if (!t.on || t.used == 0) return;
    cudaStreamSynchronize(ctx->stream);
    for (size_t i = 0; i + 1 < t.used; i += 2) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, t.ev[i], t.ev[i + 1]);
        const int k = t.kinds[i / 2];
        t.ms[k] += ms;
        t.launches[k] += 1;
    }
    t.used = 0;
}

struct ColStats {
    double lin;
    double xmax;
};

__global__ void k_col_stats(const int32_t* rows, const double* vals, const int64_t* col_beg,
                            const int64_t* val_off, const uint8_t* event, int64_t p,
                            ColStats* out) {
    // one warp per column; lane 0 accumulates x*delta in entry order
    // (likelihood.cpp:147), lanes gather the next 32 entries.
    const int lane = threadIdx.x & 31;
    const int64_t wid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t j = wid; j < p; j += nw) {
        const int64_t beg = col_beg[j], end = col_beg[j + 1];
        const int64_t vo = val_off[j];
        double lin = 0.0, xm = 0.0;
        for (int64_t b = beg; b < end; b += 32) {
            const int64_t t = b + lane;
            double term = 0.0, x = 0.0;
            if (t < end) {
                x = vo < 0 ? 1.0 : vals[vo + (t - beg)];
                term = x * (double)event[rows[t]];
            }
            xm = fmax(xm, fabs(x));
            const int cnt = (int)((end - b) < 32 ? (end - b) : 32);
            for (int q = 0; q < cnt; ++q) {
                const double v = __shfl_sync(0xffffffffu, term, q);
                if (lane == 0) lin += v;
            }
        }
        for (int off = 16; off > 0; off >>= 1) xm = fmax(xm, __shfl_xor_sync(0xffffffffu, xm, off));
        if (lane == 0) out[j] = ColStats{lin, xm};
    }
}

__global__ void k_check_rows(const int32_t* rows, const int64_t* col_beg, int64_t p, int64_t nnz,
                             int64_t n, DevCtl* ctl) {
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < nnz;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int32_t r = rows[t];
        if (r < 0 || r >= n) {
            set_error(ctl, kErrBadRows, t);
            continue;
        }
        if (t == 0) continue;
        // is t the first entry of its column?
        int64_t lo = 0, hi = p;  // largest j with col_beg[j] <= t
        while (hi - lo > 1) {
            const int64_t mid = (lo + hi) >> 1;
            if (col_beg[mid] <= t)
                lo = mid;
            else
                hi = mid;
        }
        if (col_beg[lo] != t && rows[t - 1] >= r) set_error(ctl, kErrBadRows, t);
    }
}

__global__ void k_narrow_checked(int32_t* dst, const int64_t* src, int64_t count, int64_t n,
                                 DevCtl* ctl) {
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < count;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = src[t];
        if (r < 0 || r >= n) set_error(ctl, kErrBadRows, t);
        dst[t] = (int32_t)r;
    }
}

__global__ void k_fill(double* p, double v, int64_t n) {
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n;
         t += (int64_t)gridDim.x * blockDim.x)
        p[t] = v;
}

__global__ void k_k3_check(const int32_t* rows, const double* vals, const double* eta,
                           const ColArgs col, DevCtl* ctl) {
    const double a = ctl->applied;
    if (a == 0.0 || ctl->err_kind) return;
    int hl = 0;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < col.nnz;
         t += (int64_t)gridDim.x * blockDim.x) {
        const double x = col.indicator ? 1.0 : vals[col.val_off + t];
        const double e = eta[rows[col.beg + t]];
        double s = a;
        int h = 0;
        for (; h <= kMaxHalvings; ++h) {
            const double next = __dadd_rn(e, __dmul_rn(x, s));
            if (isfinite(next) && fabs(next) <= kLinearPredictorBound) break;
            s *= 0.5;
        }
        hl = max(hl, h);
    }
    for (int off = 16; off > 0; off >>= 1) hl = max(hl, __shfl_xor_sync(0xffffffffu, hl, off));
    if ((threadIdx.x & 31) == 0 && hl > 0) atomicMax(&ctl->hmax, hl);
}

}  // namespace

// Record a message on a context (read back by scx_last_error); used by the
// drivers in cv.cu.
void scx_note_error(scx_ctx* ctx, const char* msg) {
    if (ctx) ctx->err = msg;
}


// =================================================================== C-ABI
extern "C" {

const char* scx_version(void) { return "stratcox_b200 0.1 (sm_100a)"; }

int scx_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
    return n;
}

scx_status scx_create(int device, scx_ctx** out) {
    static const bool per_coord = getenv("SCX_FIT_PER_COORD") && atoi(getenv("SCX_FIT_PER_COORD"));
    if (!out) return SCX_ERR_VALIDATION;
    *out = nullptr;
    auto* ctx = new scx_ctx();
    ctx->device = device;
    ctx->per_coordinate_fit = per_coord;
    cudaError_t e = cudaSetDevice(device);
    if (e != cudaSuccess) {
        delete ctx;
        return SCX_ERR_CUDA;
    }
    int major = 0, minor = 0;
    cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device);
    cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, device);
    if (major != 10) {
        delete ctx;
        return SCX_ERR_CUDA;  // sm_100a binary only
    }
    if (cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaMalloc((void**)&ctx->d.ctl, sizeof(DevCtl)) != cudaSuccess ||
        cudaMallocHost((void**)&ctx->ctl_h, sizeof(DevCtl)) != cudaSuccess ||
        cudaMalloc((void**)&ctx->warn_d, kWarnCap * sizeof(long long)) != cudaSuccess ||
        cudaMalloc((void**)&ctx->out2, 4 * sizeof(double)) != cudaSuccess) {
        delete ctx;
        return SCX_ERR_CUDA;
    }
    DevCtl init;
    memset(&init, 0, sizeof init);
    init.epoch = 1;
    init.bad_min = kNoRow;
    init.warn_coord = ctx->warn_d;
    init.warn_cap = kWarnCap;
    cudaMemcpy(ctx->d.ctl, &init, sizeof init, cudaMemcpyHostToDevice);
    *out = ctx;
    return SCX_OK;
}

void scx_destroy(scx_ctx* ctx) {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    free_design(ctx);
    for (void* q : ctx->ipc_open) cudaIpcCloseMemHandle(q);
    if (ctx->xslots) cudaFree(ctx->xslots);
    if (ctx->d.ctl) cudaFree(ctx->d.ctl);
    if (ctx->out2) cudaFree(ctx->out2);
    if (ctx->warn_d) cudaFree(ctx->warn_d);
    if (ctx->ctl_h) cudaFreeHost(ctx->ctl_h);
    for (auto e : ctx->timer.ev) cudaEventDestroy(e);
    if (ctx->stream) cudaStreamDestroy(ctx->stream);
    delete ctx;
}

const char* scx_last_error(const scx_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

void* scx_stream(scx_ctx* ctx) { return ctx ? (void*)ctx->stream : nullptr; }

// Sorted arrays already on the device (the device design build,
// design_build.cu): event and tie ends are read in place; the int32 rows and
// the compacted values pass to the context; the column classification was
// done by the builder.
struct DevSrc {
    const uint8_t* event_d;
    const int64_t* tie_d;
    int32_t* rows32_d;
    double* vals_d;
    const std::vector<int64_t>* val_off;
    int64_t n_ind;
};

// Upload phase timing (SCX_UPLOAD_TRACE=1: stream synchronised at each phase,
// durations on stderr; diagnostics only).
struct UploadClock {
    bool on;
    cudaStream_t s;
    std::chrono::steady_clock::time_point t;
    explicit UploadClock(cudaStream_t st)
        : on(getenv("SCX_UPLOAD_TRACE") != nullptr), s(st), t(std::chrono::steady_clock::now()) {}
    void mark(const char* what) {
        if (!on) return;
        cudaStreamSynchronize(s);
        const auto n = std::chrono::steady_clock::now();
        fprintf(stderr, "[scx upload] %-28s %9.2f ms\n", what,
                std::chrono::duration<double, std::milli>(n - t).count());
        t = n;
    }
};

static scx_status upload_common(scx_ctx* ctx, int64_t n, int32_t k, const int64_t* offsets,
                                const uint8_t* event, const int64_t* tie_end, int64_t p,
                                const int64_t* col_ptr, const int64_t* row64,
                                const int32_t* row32, const double* values,
                                const DevSrc* dev = nullptr) {
    if (!ctx) return SCX_ERR_VALIDATION;
    cudaSetDevice(ctx->device);
    UploadClock uc(ctx->stream);
    if (n < 1) return fail(ctx, SCX_ERR_VALIDATION, "dataset has no rows");
    if (k < 1) return fail(ctx, SCX_ERR_VALIDATION, "dataset has no strata");
    if (n > (int64_t)0x7fffffff - kTileRows)
        return fail(ctx, SCX_ERR_VALIDATION, "row count exceeds the int32 row-index range");
    if (p < 0) return fail(ctx, SCX_ERR_VALIDATION, "negative covariate count");
    if (offsets[0] != 0 || offsets[k] != n)
        return fail(ctx, SCX_ERR_VALIDATION, "stratum offsets must span [0, n_rows]");
    for (int32_t s = 0; s < k; ++s)
        if (offsets[s + 1] <= offsets[s])
            return fail(ctx, SCX_ERR_VALIDATION, "stratum offsets must be strictly increasing");
    if (col_ptr[0] != 0) return fail(ctx, SCX_ERR_VALIDATION, "col_ptr[0] must be 0");
    for (int64_t j = 0; j < p; ++j)
        if (col_ptr[j + 1] < col_ptr[j])
            return fail(ctx, SCX_ERR_VALIDATION, "col_ptr must be non-decreasing");
    const int64_t nnz = col_ptr[p];
    if (nnz > (int64_t)0x7fffffff * 64)
        return fail(ctx, SCX_ERR_VALIDATION, "too many nonzeros");

    // Column classification (host, input preprocessing): indicator columns
    // (all values 1.0) keep only row indices; others keep compacted values.
    std::vector<int64_t> val_off(p, -1);
    std::vector<double> compact;
    int64_t n_ind = 0;
    if (dev) {
        val_off = *dev->val_off;
        n_ind = dev->n_ind;
    }
    for (int64_t j = 0; j < p && !dev; ++j) {
        bool ind = true;
        if (values) {
            for (int64_t t = col_ptr[j]; t < col_ptr[j + 1]; ++t) {
                if (!std::isfinite(values[t]))
                    return fail(ctx, SCX_ERR_VALIDATION,
                                "column x" + std::to_string(j + 1) + " has a non-finite value");
                if (values[t] != 1.0) ind = false;
            }
        }
        if (ind) {
            ++n_ind;
        } else {
            val_off[j] = (int64_t)compact.size();
            compact.insert(compact.end(), values + col_ptr[j], values + col_ptr[j + 1]);
        }
    }

    free_design(ctx);
    DesignDev& d = ctx->d;
    d.n = n;
    d.k = k;
    d.p = p;
    d.ntiles = (n + kTileRows - 1) / kTileRows;
    d.npad = d.ntiles * kTileRows;
    d.ntiles1 = d.npad / kK1TileRows;
    cudaStream_t s = ctx->stream;

    uc.mark("validation + columns (host)");
    // --- event codes
    uint8_t* event_d = nullptr;
    int64_t* tie_d = nullptr;
    uint32_t* w_d = nullptr;
    unsigned int* maxw_d = nullptr;
    if (dev) {
        event_d = const_cast<uint8_t*>(dev->event_d);
        tie_d = const_cast<int64_t*>(dev->tie_d);
    } else {
        CK(dmalloc(&event_d, n));
        CK(dmalloc(&tie_d, n));
        CK(cudaMemcpyAsync(event_d, event, n, cudaMemcpyHostToDevice, s));
        CK(cudaMemcpyAsync(tie_d, tie_end, n * sizeof(int64_t), cudaMemcpyHostToDevice, s));
    }
    CK(dmalloc(&w_d, d.npad));
    CK(dmalloc(&maxw_d, 1));
    CK(dmalloc(&ctx->offsets_d, k + 1));
    CK(cudaMemcpyAsync(ctx->offsets_d, offsets, (k + 1) * sizeof(int64_t), cudaMemcpyHostToDevice,
                       s));
    CK(cudaMemsetAsync(w_d, 0, d.npad * sizeof(uint32_t), s));
    CK(cudaMemsetAsync(maxw_d, 0, sizeof(unsigned int), s));
    KL(2, launch_tie_weights(w_d, event_d, tie_d, n, d.ctl, maxw_d, s));
    unsigned int maxw = 0;
    CK(cudaMemcpyAsync(&maxw, maxw_d, sizeof maxw, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    d.code_bytes = maxw <= 0x1fu ? 1 : (maxw <= 0x1fffu ? 2 : 4);
    CK(cudaMalloc(&d.code, d.npad * d.code_bytes));
    KL(1, launch_build_codes(d.code, d.code_bytes, n, d.npad, event_d, tie_d, ctx->offsets_d, k, w_d,
                          s));
    if (dev) {  // host copies for error-message row mapping
        ctx->tie_end_h.resize(n);
        ctx->event_h.resize(n);
        CK(cudaMemcpyAsync(ctx->tie_end_h.data(), tie_d, n * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
        CK(cudaMemcpyAsync(ctx->event_h.data(), event_d, n, cudaMemcpyDeviceToHost, s));
    } else {
        ctx->tie_end_h.assign(tie_end, tie_end + n);
        ctx->event_h.assign(event, event + n);
    }

    uc.mark("event codes");
    // --- CSC
    if (dev)
        ctx->rows_d = dev->rows32_d;  // sorted on the device, nnz + 16 entries
    else
        CK(dmalloc(&ctx->rows_d, nnz + 16));  // +16: 16-B-aligned bulk copies may overhang
    CK(dmalloc(&ctx->col_beg_d, p + 1));
    CK(dmalloc(&ctx->val_off_d, p));
    CK(cudaMemcpyAsync(ctx->col_beg_d, col_ptr, (p + 1) * sizeof(int64_t), cudaMemcpyHostToDevice,
                       s));
    CK(cudaMemcpyAsync(ctx->val_off_d, val_off.data(), p * sizeof(int64_t),
                       cudaMemcpyHostToDevice, s));
    if (dev) {
    } else if (row32) {
        CK(cudaMemcpyAsync(ctx->rows_d, row32, nnz * sizeof(int32_t), cudaMemcpyHostToDevice, s));
    } else if (nnz > 0) {
        const int64_t chunk = std::min<int64_t>(nnz, (int64_t)1 << 26);
        int64_t* stage = nullptr;
        CK(dmalloc(&stage, chunk));
        for (int64_t off = 0; off < nnz; off += chunk) {
            const int64_t m = std::min(chunk, nnz - off);
            CK(cudaMemcpyAsync(stage, row64 + off, m * sizeof(int64_t), cudaMemcpyHostToDevice, s));
            k_narrow_checked<<<1184, 256, 0, s>>>(ctx->rows_d + off, stage, m, n, d.ctl);
        }
        CK(cudaStreamSynchronize(s));
        cudaFree(stage);
    }
    if (nnz > 0) k_check_rows<<<1184, 256, 0, s>>>(ctx->rows_d, ctx->col_beg_d, p, nnz, n, d.ctl);
    if (dev)
        ctx->vals_d = dev->vals_d;
    else
        CK(dmalloc(&ctx->vals_d, compact.size() + 16));
    if (!compact.empty())
        CK(cudaMemcpyAsync(ctx->vals_d, compact.data(), compact.size() * sizeof(double),
                           cudaMemcpyHostToDevice, s));
    ColStats* stats_d = nullptr;
    CK(dmalloc(&stats_d, p));
    if (p > 0)
        k_col_stats<<<1184, 256, 0, s>>>(ctx->rows_d, ctx->vals_d, ctx->col_beg_d, ctx->val_off_d,
                                          event_d, p, stats_d);
    std::vector<ColStats> stats(p);
    if (p > 0)
        CK(cudaMemcpyAsync(stats.data(), stats_d, p * sizeof(ColStats), cudaMemcpyDeviceToHost, s));
    CK(dmalloc(&ctx->tptr_d, p * (d.ntiles1 + 1)));
    if (p > 0) KL(1, launch_tile_ptr(ctx->tptr_d, ctx->rows_d, ctx->col_beg_d, p, d.ntiles1, s));
    d.ref_ps = (std::max<int64_t>(p, 1) + 31) / 32 * 32;
    CK(dmalloc(&d.ref_act, d.ref_ps));
    CK(dmalloc(&d.ref_abeg, d.ref_ps));
    CK(dmalloc(&d.ref_avo, d.ref_ps));
    CK(dmalloc(&d.ref_ab, d.ref_ps));
    CK(dmalloc(&d.ref_nact, 1));
    CK(dmalloc(&d.ref_meta, d.ref_ps * (d.ntiles1 + 1)));
    CK(cudaStreamSynchronize(s));
    if (!dev) {
        cudaFree(event_d);
        cudaFree(tie_d);
    }
    cudaFree(w_d);
    cudaFree(maxw_d);
    cudaFree(stats_d);

    uc.mark("CSC upload + column stats + tile pointers");
    // --- state + scratch
    CK(dmalloc(&d.D, d.npad));
    CK(dmalloc(&d.eta, d.npad));
    CK(dmalloc(&d.beta, p));
    CK(dmalloc(&d.gamma, p));
    CK(dmalloc(&d.l2, p));
    CK(dmalloc(&d.trust, p));
    CK(dmalloc(&d.lasth1, d.ntiles1));
    KL(1, launch_last_head(d.lasth1, ctx->offsets_d, k, d.ntiles1, s));
    // Stratum-aligned chunks, one per SM, for the chunked fused scan: strata
    // are assigned in order, a chunk closing once it reaches its share of
    // the remaining rows. Used when the largest stratum is at most a quarter
    // of a chunk (so the longest chunk exceeds n/G by <= 25%); otherwise the
    // fused scan uses the cross-CTA look-back.
    {
        int sms = 0;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device);
        if (ctx->sm_budget > 0) sms = std::min(sms, ctx->sm_budget);  // ranks sharing one GPU
        const int64_t G = sms > 0 ? sms : 148;
        int64_t maxk = 0;
        for (int32_t q = 0; q < k; ++q) maxk = std::max<int64_t>(maxk, offsets[q + 1] - offsets[q]);
        bool ok = k >= 2 * G && n >= G * 4 * (int64_t)kK1TileRows && 4 * maxk <= n / G;
        std::vector<int32_t> ch;
        if (ok) {
            ch.push_back(0);
            int32_t q = 0;
            for (int64_t c = 1; c < G && ok; ++c) {
                const int64_t target = ch.back() + (n - ch.back()) / (G - c + 1);
                while (q < k && offsets[q + 1] <= target) ++q;
                // close at the head nearest to the target
                int64_t h = offsets[q];
                if (q + 1 <= k && offsets[q + 1] - target < target - h) h = offsets[q + 1];
                if (h <= ch.back() || h >= n) ok = false;
                else ch.push_back((int32_t)h);
            }
            ch.push_back((int32_t)n);
        }
        d.chunk_rows = nullptr;
        d.nchunks = 0;
        d.rs_ok = 0;
        if (ok) {
            CK(dmalloc(&d.chunk_rows, ch.size()));
            CK(cudaMemcpyAsync(d.chunk_rows, ch.data(), ch.size() * sizeof(int32_t),
                               cudaMemcpyHostToDevice, s));
            d.nchunks = (int32_t)G;
            // first stratum of each chunk (chunks start at heads) for the
            // risk-suffix cycle, which stages a chunk's strata in shared memory
            std::vector<int32_t> ck(ch.size());
            int32_t q = 0;
            int32_t most = 0;
            int64_t most_tiles = 0;  // 2048-row tiles a chunk touches (risk-scan tile carries)
            for (size_t c = 0; c < ch.size(); ++c) {
                while (q < k && offsets[q] < ch[c]) ++q;
                ck[c] = q;
                if (c > 0) {
                    most = std::max(most, ck[c] - ck[c - 1]);
                    most_tiles = std::max<int64_t>(
                        most_tiles, (ch[c] - 1) / kK1TileRows - ch[c - 1] / kK1TileRows + 1);
                }
            }
            if (most <= kRsMaxStrata && most_tiles <= kRsTileInfo) {
                CK(dmalloc(&d.chunk_k, ck.size()));
                CK(cudaMemcpyAsync(d.chunk_k, ck.data(), ck.size() * sizeof(int32_t),
                                   cudaMemcpyHostToDevice, s));
                std::vector<int32_t> nk(ck.size() - 1);
                for (size_t c = 0; c + 1 < ck.size(); ++c) nk[c] = ck[c + 1] - ck[c];
                CK(dmalloc(&d.rs_chunk_nk, nk.size()));
                CK(cudaMemcpyAsync(d.rs_chunk_nk, nk.data(), nk.size() * sizeof(int32_t),
                                   cudaMemcpyHostToDevice, s));
                d.rs_chunk_rows = d.chunk_rows;
                d.rs_aligned = 1;
                CK(dmalloc(&d.rs_CR, d.ntiles1));
                CK(dmalloc(&d.rs_CQ, d.ntiles1));
                CK(cudaMemsetAsync(d.rs_CR, 0, d.ntiles1 * sizeof(double), s));
                CK(cudaMemsetAsync(d.rs_CQ, 0, d.ntiles1 * sizeof(double), s));
                CK(dmalloc(&d.rs_R, d.npad));
                CK(dmalloc(&d.rs_Q, d.npad));
                d.rs_ok = 1;
            }
        }
    }
    // Few large strata (no stratum-aligned chunking, e.g. the lowered configs
    // 2-3): the risk-suffix cycle on chunks of whole 2048-row tiles, strata
    // running across chunk ends (carries meet across CTAs, rs_chunk_carry_in)
    if (!d.rs_ok) {
        int sms = 0;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device);
        if (ctx->sm_budget > 0) sms = std::min(sms, ctx->sm_budget);
        const int64_t G = sms > 0 ? sms : 148;
        const int64_t tiles = (n + kK1TileRows - 1) / kK1TileRows;
        if (k >= 1 && tiles >= 4 * G && G <= 512) {
            std::vector<int32_t> ch(G + 1), ck(G + 1), nk(G);
            for (int64_t c = 0; c <= G; ++c)
                ch[c] = (int32_t)std::min<int64_t>(n, (tiles * c / G) * kK1TileRows);
            bool fits = true;
            for (int64_t c = 0; c <= G; ++c) {
                // the stratum holding row ch[c] (the last one for c = G)
                const int64_t r = std::min<int64_t>(ch[c], n - 1);
                ck[c] = (int32_t)(std::upper_bound(offsets, offsets + k + 1, r) - offsets - 1);
            }
            for (int64_t c = 0; c < G; ++c) {
                // strata overlapping the chunk: up to the first starting at or after its end
                const int32_t e = (int32_t)(std::lower_bound(offsets, offsets + k + 1, (int64_t)ch[c + 1]) - offsets);
                nk[c] = e - ck[c];
                const int64_t nt = (ch[c + 1] - 1) / kK1TileRows - ch[c] / kK1TileRows + 1;
                if (nk[c] < 1 || nk[c] > kRsMaxStrata || nt > kRsTileInfo) fits = false;
            }
            if (fits) {
                CK(dmalloc(&d.rs_chunk_rows, ch.size()));
                CK(cudaMemcpyAsync(d.rs_chunk_rows, ch.data(), ch.size() * sizeof(int32_t),
                                   cudaMemcpyHostToDevice, s));
                CK(dmalloc(&d.chunk_k, ck.size()));
                CK(cudaMemcpyAsync(d.chunk_k, ck.data(), ck.size() * sizeof(int32_t),
                                   cudaMemcpyHostToDevice, s));
                CK(dmalloc(&d.rs_chunk_nk, nk.size()));
                CK(cudaMemcpyAsync(d.rs_chunk_nk, nk.data(), nk.size() * sizeof(int32_t),
                                   cudaMemcpyHostToDevice, s));
                CK(dmalloc(&d.rs_CR, d.ntiles1));
                CK(dmalloc(&d.rs_CQ, d.ntiles1));
                CK(cudaMemsetAsync(d.rs_CR, 0, d.ntiles1 * sizeof(double), s));
                CK(cudaMemsetAsync(d.rs_CQ, 0, d.ntiles1 * sizeof(double), s));
                CK(dmalloc(&d.rs_R, d.npad));
                CK(dmalloc(&d.rs_Q, d.npad));
                d.nchunks = (int32_t)G;
                d.rs_aligned = 0;
                d.rs_ok = 1;
            }
        }
    }
    if (d.rs_ok) CK(dmalloc(&d.rs_xagg, 4 * std::max<int64_t>(d.nchunks, 1)));
    CK(dmalloc(&d.status, d.ntiles));
    CK(dmalloc(&d.slots, 2 * d.ntiles1 * 8));
    CK(cudaMemsetAsync(d.slots, 0, 2 * d.ntiles1 * 8 * sizeof(double), s));
    CK(dmalloc(&d.partial, std::max<int64_t>(2 * d.ntiles, 4 * std::max<int64_t>(d.ntiles1, 1024))));
    CK(dmalloc(&ctx->xdense, d.npad));
    CK(cudaMemsetAsync(d.D, 0, d.npad * sizeof(double), s));
    CK(cudaMemsetAsync(d.eta, 0, d.npad * sizeof(double), s));
    CK(cudaMemsetAsync(d.beta, 0, std::max<int64_t>(p, 1) * sizeof(double), s));
    CK(cudaMemsetAsync(d.gamma, 0, std::max<int64_t>(p, 1) * sizeof(double), s));
    CK(cudaMemsetAsync(d.l2, 0, std::max<int64_t>(p, 1) * sizeof(double), s));
    CK(cudaMemsetAsync(d.status, 0, d.ntiles * sizeof(unsigned int), s));
    d.rows = ctx->rows_d;
    d.vals = ctx->vals_d;
    d.tptr = ctx->tptr_d;
    d.col_beg = ctx->col_beg_d;
    d.val_off = ctx->val_off_d;
    d.offsets = ctx->offsets_d;
    if (!make_tmap(&d.tmap_D, d.D, d.npad) || !make_tmap(&d.tmap_eta, d.eta, d.npad) ||
        !make_tmap(&d.tmap_D1, d.D, d.npad, kK1TileRows) ||
        (d.rs_ok && (!make_tmap(&d.tmap_R, d.rs_R, d.npad, kRsStoreRows) ||
                     !make_tmap(&d.tmap_Q, d.rs_Q, d.npad, kRsStoreRows))))
        return fail(ctx, SCX_ERR_CUDA, "cuTensorMapEncodeTiled failed");

    // co-resident block count for the cooperative kernels
    {
        int sms = 0, b1 = 0;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device);
        if (ctx->sm_budget > 0) sms = std::min(sms, ctx->sm_budget);
        d.sm_budget = ctx->sm_budget;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b1, k3_apply_ptr(), kThreads, 0);
        const int per = std::max(1, std::min(b1, 2));
        d.coop_blocks = sms * per;
    }

    ctx->cols.resize(p);
    ctx->zero_cols.clear();
    for (int64_t j = 0; j < p; ++j) {
        ColArgs c;
        c.beg = col_ptr[j];
        c.nnz = col_ptr[j + 1] - col_ptr[j];
        c.val_off = val_off[j];
        c.lin = stats[j].lin;
        c.xmax = stats[j].xmax;
        c.j = (int32_t)j;
        c.indicator = val_off[j] < 0 ? 1 : 0;
        ctx->cols[j] = c;
        if (c.nnz == 0) ctx->zero_cols.push_back((int32_t)j);
    }
    {
        std::vector<ColArgs> nz;
        for (int64_t j = 0; j < p; ++j)
            if (ctx->cols[j].nnz > 0) {
                const int32_t ind = ctx->cols[j].indicator;
                if (ctx->runs.empty() || ctx->runs.back()[2] != ind)
                    ctx->runs.push_back({(int32_t)nz.size(), 0, ind});
                ctx->runs.back()[1] += 1;
                nz.push_back(ctx->cols[j]);
            }
        CK(dmalloc(&ctx->cols_d, nz.size()));
        if (!nz.empty())
            CK(cudaMemcpyAsync(ctx->cols_d, nz.data(), nz.size() * sizeof(ColArgs),
                               cudaMemcpyHostToDevice, s));
        CK(cudaStreamSynchronize(s));
        ctx->cycle_cols = nz;
    }
    d.x = ctx->x;  // a re-upload keeps the multi-GPU exchange
    uc.mark("chunks + cycle columns");
    CK(dmalloc(&ctx->zero_cols_d, ctx->zero_cols.size()));
    if (!ctx->zero_cols.empty())
        CK(cudaMemcpyAsync(ctx->zero_cols_d, ctx->zero_cols.data(),
                           ctx->zero_cols.size() * sizeof(int32_t), cudaMemcpyHostToDevice, s));
    uc.mark("zero columns");
    // row-slice copy of the design for the 256-update refresh (skipped, and
    // the tile refresh kept, when the re-sort's scratch does not fit)
    {
        cudaError_t e = build_refresh_ell(d, nnz, n_ind < p, s);
        if (e == cudaErrorMemoryAllocation) {
            cudaGetLastError();
            d.ell_ok = 0;
        } else {
            CK(e);
        }
    }
    uc.mark("row-slice copy (refresh)");
    ctx->nnz = nnz;
    ctx->n_indicator = n_ind;
    ctx->has_design = true;
    scx_status st = check_device_error(ctx);
    if (st) {
        free_design(ctx);
        return st;
    }
    uc.mark("checks");
    // state at beta = 0 (make_state)
    KL(refresh_launches(d), launch_refresh(d, s));
    uc.mark("initial state");
    return check_device_error(ctx);
}

}  // extern "C"

// library-internal (C++ linkage): the device design build's hand-off
scx_status scx_upload_device_design(scx_ctx* ctx, int64_t n, int32_t k, const int64_t* offsets_h,
                                    const uint8_t* event_d, const int64_t* tie_d, int64_t p,
                                    const int64_t* col_ptr_h, int32_t* rows32_d, double* vals_d,
                                    const std::vector<int64_t>& val_off, int64_t n_ind) {
    DevSrc dev{event_d, tie_d, rows32_d, vals_d, &val_off, n_ind};
    return upload_common(ctx, n, k, offsets_h, nullptr, nullptr, p, col_ptr_h, nullptr, nullptr,
                         nullptr, &dev);
}

cudaStream_t scx_ctx_stream(scx_ctx* ctx) { return ctx->stream; }
int scx_ctx_device(scx_ctx* ctx) { return ctx->device; }

extern "C" {

scx_status scx_upload_design(scx_ctx* ctx, int64_t n_rows, int32_t n_strata,
                             const int64_t* stratum_offsets, const uint8_t* event,
                             const int64_t* tie_group_end, int64_t n_covariates,
                             const int64_t* col_ptr, const int64_t* row_idx,
                             const double* values) {
    return upload_common(ctx, n_rows, n_strata, stratum_offsets, event, tie_group_end,
                         n_covariates, col_ptr, row_idx, nullptr, values);
}

scx_status scx_upload_design_i32(scx_ctx* ctx, int64_t n_rows, int32_t n_strata,
                                 const int64_t* stratum_offsets, const uint8_t* event,
                                 const int64_t* tie_group_end, int64_t n_covariates,
                                 const int64_t* col_ptr, const int32_t* row_idx,
                                 const double* values) {
    return upload_common(ctx, n_rows, n_strata, stratum_offsets, event, tie_group_end,
                         n_covariates, col_ptr, nullptr, row_idx, values);
}

scx_status scx_design_info(const scx_ctx* ctx, int64_t* n_rows, int32_t* n_strata, int64_t* p,
                           int64_t* nnz, int32_t* code_bytes, int64_t* n_tiles,
                           int64_t* n_indicator) {
    if (!ctx || !ctx->has_design) return SCX_ERR_VALIDATION;
    if (n_rows) *n_rows = ctx->d.n;
    if (n_strata) *n_strata = ctx->d.k;
    if (p) *p = ctx->d.p;
    if (nnz) *nnz = ctx->nnz;
    if (code_bytes) *code_bytes = ctx->d.code_bytes;
    if (n_tiles) *n_tiles = ctx->d.ntiles;
    if (n_indicator) *n_indicator = ctx->n_indicator;
    return SCX_OK;
}

scx_status scx_design_export(scx_ctx* ctx, int64_t* offsets, uint8_t* event, int64_t* tie_end,
                             int64_t* col_ptr, int64_t* row_idx, double* values) {
    if (scx_status s = need_design(ctx)) return s;
    cudaSetDevice(ctx->device);
    const DesignDev& d = ctx->d;
    cudaStream_t s = ctx->stream;
    const int64_t n = d.n, p = d.p, nnz = ctx->nnz;
    if (offsets)
        CK(cudaMemcpyAsync(offsets, ctx->offsets_d, (d.k + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    if (event) std::memcpy(event, ctx->event_h.data(), n);
    if (tie_end) std::memcpy(tie_end, ctx->tie_end_h.data(), n * sizeof(int64_t));
    std::vector<int64_t> cp(p + 1, 0);
    for (int64_t j = 0; j < p; ++j) cp[j + 1] = cp[j] + ctx->cols[j].nnz;
    if (col_ptr) std::memcpy(col_ptr, cp.data(), (p + 1) * sizeof(int64_t));
    if (row_idx && nnz > 0) {
        std::vector<int32_t> r32(nnz);
        CK(cudaMemcpyAsync(r32.data(), ctx->rows_d, nnz * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        for (int64_t t = 0; t < nnz; ++t) row_idx[t] = r32[t];
    }
    if (values) {
        for (int64_t j = 0; j < p; ++j) {
            const ColArgs& c = ctx->cols[j];
            if (c.nnz == 0) continue;
            if (c.indicator) {
                std::fill(values + cp[j], values + cp[j + 1], 1.0);
            } else {
                CK(cudaMemcpyAsync(values + cp[j], ctx->vals_d + c.val_off, c.nnz * sizeof(double),
                                   cudaMemcpyDeviceToHost, s));
            }
        }
    }
    CK(cudaStreamSynchronize(s));
    return SCX_OK;
}

// ---------------------------------------------------------------- state
scx_status scx_make_state(scx_ctx* ctx, const double* beta) {
    if (scx_status s = need_design(ctx)) return s;
    cudaSetDevice(ctx->device);
    DesignDev& d = ctx->d;
    if (d.p > 0) CK(cudaMemcpyAsync(d.beta, beta, d.p * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    KL(refresh_launches(d), launch_refresh(d, ctx->stream));
    return check_device_error(ctx);
}

scx_status scx_set_state(scx_ctx* ctx, const double* beta, const double* xbeta,
                         const double* exp_xbeta, uint32_t updates) {
    if (scx_status s = need_design(ctx)) return s;
    cudaSetDevice(ctx->device);
    DesignDev& d = ctx->d;
    cudaStream_t s = ctx->stream;
    if (d.p > 0) CK(cudaMemcpyAsync(d.beta, beta, d.p * sizeof(double), cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(d.eta, xbeta, d.n * sizeof(double), cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(d.D, exp_xbeta, d.n * sizeof(double), cudaMemcpyHostToDevice, s));
    double m = 0.0;
    for (int64_t i = 0; i < d.n; ++i) {
        const double a = std::fabs(xbeta[i]);
        if (!(a <= m)) m = a;  // NaN propagates as an unusable bound
    }
    if (!std::isfinite(m)) m = INFINITY;
    CK(cudaMemcpyAsync(&d.ctl->mbound, &m, sizeof m, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(&d.ctl->updates, &updates, sizeof updates, cudaMemcpyHostToDevice, s));
    return sync(ctx);
}

scx_status scx_get_state(scx_ctx* ctx, double* beta, double* xbeta, double* exp_xbeta,
                         uint32_t* updates) {
    if (scx_status s = need_design(ctx)) return s;
    cudaSetDevice(ctx->device);
    DesignDev& d = ctx->d;
    cudaStream_t s = ctx->stream;
    if (beta && d.p > 0)
        CK(cudaMemcpyAsync(beta, d.beta, d.p * sizeof(double), cudaMemcpyDeviceToHost, s));
    if (xbeta) CK(cudaMemcpyAsync(xbeta, d.eta, d.n * sizeof(double), cudaMemcpyDeviceToHost, s));
    if (exp_xbeta)
        CK(cudaMemcpyAsync(exp_xbeta, d.D, d.n * sizeof(double), cudaMemcpyDeviceToHost, s));
    if (updates)
        CK(cudaMemcpyAsync(updates, &d.ctl->updates, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
    return sync(ctx);
}

scx_status scx_refresh_xbeta(scx_ctx* ctx) {
    if (scx_status s = need_design(ctx)) return s;
    cudaSetDevice(ctx->device);
    KL(refresh_launches(ctx->d), launch_refresh(ctx->d, ctx->stream));
    return check_device_error(ctx);
}

scx_status scx_update_xbeta(scx_ctx* ctx, int64_t j, double delta) {
    if (scx_status s = need_design(ctx)) return s;
    if (j < 0 || j >= ctx->d.p) return fail(ctx, SCX_ERR_VALIDATION, "covariate index out of range");
    if (!std::isfinite(delta)) return fail(ctx, SCX_ERR_NUMERIC, "non-finite coordinate step");
    cudaSetDevice(ctx->device);
    const int zero = 0;
    CK(cudaMemcpyAsync(&ctx->d.ctl->hmax, &zero, sizeof zero, cudaMemcpyHostToDevice, ctx->stream));
    KL(1, launch_k3(ctx->d, ctx->cols[j], 1, delta, ctx->stream));
    return check_device_error(ctx);
}

// ---------------------------------------------------------------- likelihood
scx_status scx_gradient_hessian(scx_ctx* ctx, int64_t j, double* g, double* h) {
    if (scx_status s = need_design(ctx)) return s;
    if (j < 0 || j >= ctx->d.p) return fail(ctx, SCX_ERR_VALIDATION, "covariate index out of range");
    cudaSetDevice(ctx->device);
    tmark(ctx, 0);
    KL(1, launch_k1(ctx->d, ctx->cols[j], kK1Eval, ctx->stream));
    tend(ctx);
    tcollect(ctx);
    if (scx_status s = check_device_error(ctx, (int)j)) return s;
    *g = ctx->ctl_h->g;
    *h = ctx->ctl_h->h;
    return SCX_OK;
}

scx_status scx_gradient_hessian_rs(scx_ctx* ctx, int64_t j, double* g, double* h) {
    if (scx_status s = need_design(ctx)) return s;
    if (j < 0 || j >= ctx->d.p) return fail(ctx, SCX_ERR_VALIDATION, "covariate index out of range");
    if (!ctx->d.rs_ok)
        return fail(ctx, SCX_ERR_VALIDATION, "risk-suffix evaluation needs the chunked layout");
    cudaSetDevice(ctx->device);
    if (ctx->cols[j].nnz == 0) {  // no entries: (0, 0) as the fused scan gives
        *g = 0.0;
        *h = 0.0;
        return SCX_OK;
    }
    if (!ctx->col1_d) CK(dmalloc(&ctx->col1_d, 1));
    CK(cudaMemcpyAsync(ctx->col1_d, &ctx->cols[j], sizeof(ColArgs), cudaMemcpyHostToDevice,
                       ctx->stream));
    tmark(ctx, 3);
    KL(1, launch_rs_cycle(ctx->d, ctx->col1_d, 1, 1, ctx->stream));
    tend(ctx);
    tcollect(ctx);
    if (scx_status s = check_device_error(ctx, (int)j)) return s;
    *g = ctx->ctl_h->g;
    *h = ctx->ctl_h->h;
    return SCX_OK;
}

scx_status scx_risk_prefix_n(scx_ctx* ctx, int reps) {
    if (scx_status s = need_design(ctx)) return s;
    if (!ctx->d.rs_ok)
        return fail(ctx, SCX_ERR_VALIDATION, "risk-suffix evaluation needs the chunked layout");
    if (reps < 1) return fail(ctx, SCX_ERR_VALIDATION, "reps must be >= 1");
    cudaSetDevice(ctx->device);
    tmark(ctx, 3);
    KL(1, launch_rs_cycle(ctx->d, ctx->cols_d, reps, 2, ctx->stream));
    tend(ctx);
    return SCX_OK;
}

scx_status scx_risk_prefix(scx_ctx* ctx) { return scx_risk_prefix_n(ctx, 1); }

scx_status scx_debug_risk_arrays(scx_ctx* ctx, double* R, double* Q, double* CR, double* CQ,
                                 int32_t* lasth) {
    if (scx_status s = need_design(ctx)) return s;
    if (!ctx->d.rs_ok) return fail(ctx, SCX_ERR_VALIDATION, "no risk-suffix layout");
    cudaSetDevice(ctx->device);
    const DesignDev& d = ctx->d;
    cudaStream_t s = ctx->stream;
    if (R) CK(cudaMemcpyAsync(R, d.rs_R, d.n * sizeof(double), cudaMemcpyDeviceToHost, s));
    if (Q) CK(cudaMemcpyAsync(Q, d.rs_Q, d.n * sizeof(double), cudaMemcpyDeviceToHost, s));
    if (CR) CK(cudaMemcpyAsync(CR, d.rs_CR, d.ntiles1 * sizeof(double), cudaMemcpyDeviceToHost, s));
    if (CQ) CK(cudaMemcpyAsync(CQ, d.rs_CQ, d.ntiles1 * sizeof(double), cudaMemcpyDeviceToHost, s));
    if (lasth) CK(cudaMemcpyAsync(lasth, d.lasth1, d.ntiles1 * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    return SCX_OK;
}

scx_status scx_fit_path_stats(const scx_ctx* ctx, int64_t out[4]) {
    if (!ctx || !out) return SCX_ERR_VALIDATION;
    for (int q = 0; q < 4; ++q) out[q] = ctx->rs_stats[q];
    return SCX_OK;
}

scx_status scx_set_fit_path(scx_ctx* ctx, int path, int* risk_suffix) {
    if (!ctx || path < 0 || path > 1) return SCX_ERR_VALIDATION;
    ctx->fit_path = path;
    if (risk_suffix) *risk_suffix = (path == 0 && ctx->d.rs_ok && ctx->d.k1_mode != 1) ? 1 : 0;
    return SCX_OK;
}

scx_status scx_log_partial_likelihood(scx_ctx* ctx, double* ll) {
    if (scx_status s = need_design(ctx)) return s;
    cudaSetDevice(ctx->device);
    tmark(ctx, 2);
    KL(1, launch_k2(ctx->d, 0, ctx->stream));
    tend(ctx);
    tcollect(ctx);
    if (scx_status s = check_device_error(ctx)) return s;
    *ll = ctx->ctl_h->ll;
    return SCX_OK;
}

scx_status scx_naive_gradient_hessian(scx_ctx* ctx, int64_t j, double* g, double* h) {
    if (scx_status s = need_design(ctx)) return s;
    if (j < 0 || j >= ctx->d.p) return fail(ctx, SCX_ERR_VALIDATION, "covariate index out of range");
    cudaSetDevice(ctx->device);
    KL(2, launch_naive_gh(ctx->d, ctx->cols[j], ctx->xdense, ctx->out2, ctx->stream));
    double o[2];
    CK(cudaMemcpyAsync(o, ctx->out2, sizeof o, cudaMemcpyDeviceToHost, ctx->stream));
    if (scx_status s = sync(ctx)) return s;
    *g = o[0];
    *h = o[1];
    return SCX_OK;
}

scx_status scx_naive_log_partial_likelihood(scx_ctx* ctx, double* ll) {
    if (scx_status s = need_design(ctx)) return s;
    cudaSetDevice(ctx->device);
    KL(1, launch_naive_ll(ctx->d, ctx->out2, ctx->stream));
    double o[2];
    CK(cudaMemcpyAsync(o, ctx->out2, sizeof o, cudaMemcpyDeviceToHost, ctx->stream));
    if (scx_status s = sync(ctx)) return s;
    *ll = o[0];
    return SCX_OK;
}

scx_status scx_segmented_inclusive_scan(scx_ctx* ctx, int64_t n, const double* values,
                                        const uint8_t* flags, double* out) {
    if (!ctx) return SCX_ERR_VALIDATION;
    if (n < 1) return fail(ctx, SCX_ERR_VALIDATION, "empty scan input");
    if (!flags[0]) return fail(ctx, SCX_ERR_VALIDATION, "first element must head a segment");
    cudaSetDevice(ctx->device);
    cudaStream_t s = ctx->stream;
    DesignDev t{};
    t.n = n;
    t.ntiles = (n + kTileRows - 1) / kTileRows;
    t.npad = t.ntiles * kTileRows;
    t.code_bytes = 1;
    t.ctl = ctx->d.ctl;
    std::vector<uint8_t> code(t.npad, 0);
    for (int64_t i = 0; i < n; ++i) code[i] = flags[i] ? 0x80 : 0;
    double* outd = nullptr;
    CK(dmalloc(&t.D, t.npad));
    CK(cudaMalloc(&t.code, t.npad));
    CK(dmalloc(&t.status, t.ntiles));
    CK(dmalloc(&t.slots, 2 * t.ntiles * 8));
    CK(cudaMemsetAsync(t.slots, 0, 2 * t.ntiles * 8 * sizeof(double), s));
    CK(dmalloc(&t.partial, 2 * t.ntiles));
    CK(dmalloc(&outd, t.npad));
    CK(cudaMemsetAsync(t.D, 0, t.npad * sizeof(double), s));
    CK(cudaMemsetAsync(t.status, 0, t.ntiles * sizeof(unsigned int), s));
    CK(cudaMemcpyAsync(t.D, values, n * sizeof(double), cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(t.code, code.data(), t.npad, cudaMemcpyHostToDevice, s));
    scx_status st = SCX_OK;
    if (!make_tmap(&t.tmap_D, t.D, t.npad)) {
        st = fail(ctx, SCX_ERR_CUDA, "cuTensorMapEncodeTiled failed");
    } else {
        t.tmap_eta = t.tmap_D;
        cudaError_t e = launch_scan_primitive(t, outd, s);
        if (e != cudaSuccess) st = cuda_fail(ctx, e, "scan");
        if (!st) {
            cudaMemcpyAsync(out, outd, n * sizeof(double), cudaMemcpyDeviceToHost, s);
            st = read_ctl(ctx);
            if (!st && ctx->ctl_h->bad_min != kNoRow) {
                const long long bm = ctx->ctl_h->bad_min;
                clear_error(ctx);
                st = fail(ctx, SCX_ERR_VALIDATION, "non-finite input at index " + std::to_string(bm));
            }
        }
    }
    cudaFree(t.D);
    cudaFree(t.code);
    cudaFree(t.status);
    cudaFree(t.slots);
    cudaFree(t.partial);
    cudaFree(outd);
    return st;
}

// ---------------------------------------------------------------- scalar rules
static scx_status rule_status(int rc, const char** msg) {
    switch (rc) {
        case kRuleNonFiniteNewton:
            *msg = "non-finite gradient or Hessian in Newton step";
            return SCX_ERR_NUMERIC;
        case kRuleNonFiniteTrust:
            *msg = "non-finite trust-region inputs";
            return SCX_ERR_NUMERIC;
        case kRuleBothNegative:
            *msg = "both directional derivatives negative at the origin";
            return SCX_ERR_INTERNAL;
        default:
            *msg = "";
            return SCX_OK;
    }
}

static thread_local std::string g_rule_msg;

scx_status scx_newton_step(double g1, double g2, double* step, int* flat) {
    int fl = 0;
    const char* m;
    const scx_status s = rule_status(newton_step(g1, g2, step, &fl), &m);
    if (flat) *flat = fl;
    g_rule_msg = m;
    return s;
}

scx_status scx_apply_trust_region(double proposed, double trust, double* applied,
                                  double* next_trust) {
    double nt = 0.0;
    const char* m;
    const scx_status s = rule_status(apply_trust_region(proposed, trust, applied, &nt), &m);
    if (next_trust) *next_trust = nt;
    g_rule_msg = m;
    return s;
}

scx_status scx_coordinate_update(double g1, double g2, double beta_j, double gamma_j, double l2_j,
                                 double* step, int* skipped, int* flat) {
    int sk = 0, fl = 0;
    const char* m;
    const scx_status s =
        rule_status(coordinate_update(g1, g2, beta_j, gamma_j, l2_j, step, &sk, &fl), &m);
    if (skipped) *skipped = sk;
    if (flat) *flat = fl;
    g_rule_msg = m;
    return s;
}

scx_status scx_l1_coordinate_update(double g1, double g2, double beta_j, double gamma_j,
                                    double* step, int* skipped, int* flat) {
    int sk = 0, fl = 0;
    const char* m;
    const scx_status s =
        rule_status(l1_coordinate_update(g1, g2, beta_j, gamma_j, step, &sk, &fl), &m);
    if (skipped) *skipped = sk;
    if (flat) *flat = fl;
    g_rule_msg = m;
    return s;
}

const char* scx_rule_error(void) { return g_rule_msg.c_str(); }

// ---------------------------------------------------------------- fit
static scx_status run_cycle_tail(scx_ctx* ctx, bool end_of_cycle, double* ll, double* pen,
                                 double* max_step) {
    DesignDev& d = ctx->d;
    cudaStream_t s = ctx->stream;
    // zero columns: gradient (0, 0) -> flat -> applied 0 -> trust halves
    // (optimizer.cpp:103-124); batched at the end of the cycle.
    if (end_of_cycle)
        KL(1, launch_zero_cols(d, ctx->zero_cols_d, (int64_t)ctx->zero_cols.size(), s));
    tmark(ctx, 2);
    KL(1, launch_k2(d, 1, s));
    tend(ctx);
    // sharded: log L summed over the ranks' rows, max|eta| maxed (rank order)
    if (ctx->nranks > 1) KL(1, launch_xchg_ctl(d, 1, s));
    if (scx_status st = check_device_error(ctx)) return st;
    *ll = ctx->ctl_h->ll;
    *pen = ctx->ctl_h->penalty;
    *max_step = ctx->ctl_h->max_step;
    return SCX_OK;
}

// Fused-scan cycle kernel over cols[0..n). *resumed = coordinates done before a
// stop for the 256-update refresh (which is run here), 0 when it ran to the end;
// with resumed == nullptr the refresh, if due, is run and nothing is reported.
static scx_status fused_cycle(scx_ctx* ctx, const ColArgs* cols, int32_t n, bool indicator,
                              int32_t* resumed) {
    DesignDev& d = ctx->d;
    cudaStream_t s = ctx->stream;
    const int izero = 0;
    CK(cudaMemcpyAsync(&d.ctl->resume, &izero, sizeof izero, cudaMemcpyHostToDevice, s));
    ctx->rs_stats[3] += 1;
    tmark(ctx, 0);
    KL(1, launch_cycle(d, cols, n, indicator, s));
    tend(ctx);
    if (scx_status st = read_ctl(ctx)) return st;
    if (ctx->ctl_h->err_kind) return map_error(ctx, -1);
    const int32_t r = ctx->ctl_h->resume;
    if (resumed) *resumed = r;
    if (r > 0) {
        // 256 accepted updates: refresh eta/D from beta, then resume
        KL(refresh_launches(d), launch_refresh(d, s));
        if (scx_status st = check_device_error(ctx)) return st;
    }
    return SCX_OK;
}

static bool rs_usable(const scx_ctx* ctx) {
    return ctx->fit_path == 0 && ctx->d.rs_ok && ctx->d.k1_mode != 1 &&
           ctx->ctl_h->mbound <= kRsEtaBound;
}

static scx_status run_coordinate(scx_ctx* ctx, const ColArgs& col) {
    DesignDev& d = ctx->d;
    cudaStream_t s = ctx->stream;
    if (ctx->nranks == 1) {
        tmark(ctx, 0);
        KL(1, launch_k1(d, col, kK1Fit, s));
        tend(ctx);
        tmark(ctx, 1);
        KL(1, launch_k3(d, col, 0, 0.0, s));
        tend(ctx);
        return SCX_OK;
    }
    // sharded: local (ratio, variance) partials -> device exchange (rank-ordered
    // sums) + the rule -> the rank's halving level -> max over the ranks ->
    // apply (a rank without rows of the column still moves beta) -> max|eta|
    // bound maxed over the ranks (a 256-update refresh may have reset it)
    tmark(ctx, 0);
    KL(1, launch_k1(d, col, kK1Partial, s));
    tend(ctx);
    KL(1, launch_shard_step(d, col, s));
    ctx->launches += 1;
    k_k3_check<<<std::max(1, (int)std::min<int64_t>((col.nnz + 255) / 256, 1184)), 256, 0, s>>>(
        d.rows, d.vals, d.eta, col, d.ctl);
    KL(1, launch_xchg_ctl(d, 2, s));
    tmark(ctx, 1);
    KL(1, launch_k3_sharded(d, col, s));
    tend(ctx);
    KL(1, launch_xchg_ctl(d, 0, s));
    return SCX_OK;
}

scx_status scx_ccd_fit(scx_ctx* ctx, const double* gamma, const scx_fit_options* opt,
                       const double* initial_beta, scx_fit_result* res) {
    return scx_ccd_fit_prior(ctx, gamma, nullptr, opt, initial_beta, res);
}

scx_status scx_ccd_fit_prior(scx_ctx* ctx, const double* gamma, const double* l2,
                             const scx_fit_options* opt, const double* initial_beta,
                             scx_fit_result* res) {
    if (scx_status s = need_design(ctx)) return s;
    DesignDev& d = ctx->d;
    const int64_t p = d.p;
    // PenaltySpec::validate + run_ccd argument checks (optimizer.cpp:24-30, 85-88)
    for (int64_t j = 0; j < p; ++j)
        if (!std::isfinite(gamma[j]) || gamma[j] < 0.0)
            return fail(ctx, SCX_ERR_VALIDATION, "penalty weights must be finite and non-negative");
    for (int64_t j = 0; l2 && j < p; ++j)
        if (!std::isfinite(l2[j]) || l2[j] < 0.0)
            return fail(ctx, SCX_ERR_VALIDATION, "L2 prior weights must be finite and non-negative");
    if (opt->max_cycles < 1) return fail(ctx, SCX_ERR_VALIDATION, "max_cycles must be >= 1");
    if (!(opt->tolerance > 0.0)) return fail(ctx, SCX_ERR_VALIDATION, "tolerance must be positive");
    if (!(opt->initial_trust > 0.0))
        return fail(ctx, SCX_ERR_VALIDATION, "initial_trust must be positive");
    cudaSetDevice(ctx->device);
    cudaStream_t s = ctx->stream;
    res->trace_len = 0;
    res->cycles_used = 0;
    res->converged = 0;
    res->n_warnings = 0;
    res->n_evaluations = 0;

    std::vector<double> beta0(p, 0.0);
    if (initial_beta) std::copy(initial_beta, initial_beta + p, beta0.begin());
    for (auto& v : ctx->rs_stats) v = 0;
    if (p > 0) {
        CK(cudaMemcpyAsync(d.gamma, gamma, p * sizeof(double), cudaMemcpyHostToDevice, s));
        if (l2)
            CK(cudaMemcpyAsync(d.l2, l2, p * sizeof(double), cudaMemcpyHostToDevice, s));
        else
            CK(cudaMemsetAsync(d.l2, 0, p * sizeof(double), s));
        CK(cudaMemcpyAsync(d.beta, beta0.data(), p * sizeof(double), cudaMemcpyHostToDevice, s));
        k_fill<<<std::max(1, (int)std::min<int64_t>((p + 255) / 256, 1184)), 256, 0, s>>>(
            d.trust, opt->initial_trust, p);
        ctx->launches += 1;
    }
    {
        DevCtl* c = d.ctl;
        const double zero = 0.0;
        const int izero = 0;
        const long long lzero = 0;
        CK(cudaMemcpyAsync(&c->max_step, &zero, sizeof zero, cudaMemcpyHostToDevice, s));
        CK(cudaMemcpyAsync(&c->n_warn, &izero, sizeof izero, cudaMemcpyHostToDevice, s));
        CK(cudaMemcpyAsync(&c->n_eval, &lzero, sizeof lzero, cudaMemcpyHostToDevice, s));
        CK(cudaMemcpyAsync(&c->hmax, &izero, sizeof izero, cudaMemcpyHostToDevice, s));
    }
    // make_state (likelihood.cpp:19-29)
    KL(refresh_launches(d), launch_refresh(d, s));
    if (scx_status st = check_device_error(ctx)) return st;

    double ll, pen, max_step;
    if (scx_status st = run_cycle_tail(ctx, false, &ll, &pen, &max_step)) return st;
    double objective = -ll + pen;
    res->objective_trace[res->trace_len++] = objective;

    const double zero = 0.0;
    for (int cycle = 1; cycle <= opt->max_cycles; ++cycle) {
        CK(cudaMemcpyAsync(&d.ctl->max_step, &zero, sizeof zero, cudaMemcpyHostToDevice, s));
        const bool sharded = ctx->nranks > 1;
        if (!ctx->per_coordinate_fit) {
            // the whole cycle on the device: one cooperative launch per run of
            // same-kind columns (one launch for an all-indicator design)
            // (the risk-suffix cycle when the layout allows it and max|eta| is
            // within its range; the fused-scan cycle otherwise and for the
            // coordinates the risk-suffix cycle hands back)
            for (const auto& run : ctx->runs) {
                int32_t done = 0;
                while (done < run[1]) {
                    const ColArgs* cols = ctx->cols_d + run[0] + done;
                    const int32_t left = run[1] - done;
                    if (rs_usable(ctx)) {
                        ctx->rs_stats[0] += 1;
                        tmark(ctx, 3);
                        KL(1, launch_rs_cycle(d, cols, left, 0, s));
                        tend(ctx);
                        if (scx_status st = read_ctl(ctx)) return st;
                        if (ctx->ctl_h->err_kind) return map_error(ctx, -1);
                        done += ctx->ctl_h->resume;
                        const int why = ctx->ctl_h->rs_reason;
                        if (why == kRsDone) break;
                        if (why == kRsRefresh) {
                            KL(refresh_launches(d), launch_refresh(d, s));
                            if (sharded) KL(1, launch_xchg_ctl(d, 0, s));  // global max|eta|
                            if (scx_status st = check_device_error(ctx)) return st;
                        } else if (why == kRsBound) {
                            ctx->rs_stats[2] += 1;
                        } else if (why == kRsExact) {
                            // this coordinate through the exact fused scan, then resume
                            ctx->rs_stats[1] += 1;
                            if (sharded) {
                                if (scx_status st = run_coordinate(ctx, ctx->cycle_cols[run[0] + done]))
                                    return st;
                            } else if (scx_status st = fused_cycle(ctx, ctx->cols_d + run[0] + done, 1,
                                                                   run[2] != 0, nullptr)) {
                                return st;
                            }
                            done += 1;
                        }
                        continue;  // kRsBound: rs_usable() is now false
                    }
                    if (sharded) {  // the rest of the run, one coordinate at a time
                        for (; done < run[1]; ++done)
                            if (scx_status st = run_coordinate(ctx, ctx->cycle_cols[run[0] + done]))
                                return st;
                        break;
                    }
                    int32_t r = 0;
                    if (scx_status st = fused_cycle(ctx, cols, left, run[2] != 0, &r)) return st;
                    if (r <= 0) break;
                    done += r;
                }
            }
        } else {
            for (int64_t j = 0; j < p; ++j) {
                const ColArgs& col = ctx->cols[j];
                // every rank walks the same (globally non-empty) columns, so the
                // collectives of run_coordinate pair up; a rank without local
                // rows joins with zero partials
                if (ctx->nranks > 1 ? !ctx->gnz[j] : col.nnz == 0) continue;
                if (scx_status st = run_coordinate(ctx, col)) return st;
            }
        }
        if (scx_status st = run_cycle_tail(ctx, true, &ll, &pen, &max_step)) return st;
        tcollect(ctx);
        const double next = -ll + pen;
        if (next > objective + kMonotoneSlack) {
            char buf[256];
            snprintf(buf, sizeof buf, "monotonicity violated: objective rose from %f to %f",
                     objective, next);
            return fail(ctx, SCX_ERR_NUMERIC, buf);
        }
        objective = next;
        res->objective_trace[res->trace_len++] = objective;
        res->cycles_used = cycle;
        if (max_step < opt->tolerance) {
            res->converged = 1;
            break;
        }
    }
    if (p > 0) {
        CK(cudaMemcpyAsync(res->beta, d.beta, p * sizeof(double), cudaMemcpyDeviceToHost, s));
        if (res->trust)
            CK(cudaMemcpyAsync(res->trust, d.trust, p * sizeof(double), cudaMemcpyDeviceToHost, s));
    }
    if (scx_status st = read_ctl(ctx)) return st;
    res->n_warnings = ctx->ctl_h->n_warn;
    res->updates_since_refresh = ctx->ctl_h->updates;
    res->n_evaluations = ctx->ctl_h->n_eval;
    if (res->warning_coords && res->n_warnings > 0 && res->warning_cap > 0) {
        const int nw = std::min(res->n_warnings, std::min(res->warning_cap, kWarnCap));
        std::vector<long long> w(nw);
        CK(cudaMemcpy(w.data(), ctx->warn_d, nw * sizeof(long long), cudaMemcpyDeviceToHost));
        for (int q = 0; q < nw; ++q) res->warning_coords[q] = w[q];
    }
    return SCX_OK;
}

scx_status scx_gamma_max(scx_ctx* ctx, const double* gamma_template, double* out) {
    if (scx_status s = need_design(ctx)) return s;
    cudaSetDevice(ctx->device);
    DesignDev& d = ctx->d;
    std::vector<double> zero(d.p, 0.0);
    if (scx_status s = scx_make_state(ctx, zero.data())) return s;
    double best = 0.0;
    const std::vector<ColArgs>& cc = ctx->cycle_cols;  // the non-empty columns (cols_d)
    if (ctx->nranks == 1 && ctx->fit_path == 0 && d.rs_ok && d.k1_mode != 1 && !cc.empty()) {
        // risk-suffix path (eta = 0 here): one scan, then every column's
        // g' = -lin + sum a R in gradient rounds of one launch (O(nnz) gathers
        // instead of one O(N) pass per column)
        double* gout = nullptr;
        CK(dmalloc(&gout, cc.size()));
        std::vector<double> g(cc.size());
        cudaError_t e = launch_rs_cycle(d, ctx->cols_d, (int)cc.size(), 3, ctx->stream, gout);
        if (e == cudaSuccess)
            e = cudaMemcpyAsync(g.data(), gout, cc.size() * sizeof(double), cudaMemcpyDeviceToHost,
                                ctx->stream);
        if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
        cudaFree(gout);
        CK(e);
        ++ctx->launches;
        if (scx_status s = check_device_error(ctx, -1)) return s;
        for (size_t i = 0; i < cc.size(); ++i) {
            if (gamma_template && gamma_template[cc[i].j] <= 0.0) continue;
            best = dmax(best, std::fabs(g[i]));
        }
        *out = best;
        return SCX_OK;
    }
    for (int64_t j = 0; j < d.p; ++j) {
        if (gamma_template && gamma_template[j] <= 0.0) continue;
        if (ctx->cols[j].nnz == 0) continue;
        double g, h;
        if (scx_status s = scx_gradient_hessian(ctx, j, &g, &h)) return s;
        best = dmax(best, std::fabs(g));
    }
    *out = best;
    return SCX_OK;
}

// ---------------------------------------------------------------- timing
scx_status scx_set_k1_mode(scx_ctx* ctx, int mode, int* chunked) {
    if (!ctx || mode < 0 || mode > 2) return SCX_ERR_VALIDATION;
    ctx->d.k1_mode = mode;
    if (chunked) *chunked = (ctx->d.chunk_rows != nullptr && mode != 1) ? 1 : 0;
    return SCX_OK;
}

scx_status scx_debug_k1_trace(long long* out) {
    return k1_trace_copy(out) == cudaSuccess ? SCX_OK : SCX_ERR_CUDA;
}

int64_t scx_launch_count(const scx_ctx* ctx) { return ctx ? ctx->launches : 0; }

scx_status scx_timing_enable(scx_ctx* ctx, int on) {
    if (!ctx) return SCX_ERR_VALIDATION;
    ctx->timer.on = on != 0;
    return SCX_OK;
}
scx_status scx_timing_reset(scx_ctx* ctx) {
    if (!ctx) return SCX_ERR_VALIDATION;
    for (int k = 0; k < 4; ++k) {  // every timing kind (0 fused scan .. 3 risk-suffix)
        ctx->timer.ms[k] = 0;
        ctx->timer.launches[k] = 0;
    }
    ctx->timer.used = 0;
    return SCX_OK;
}
scx_status scx_timing_get(scx_ctx* ctx, int kind, double* total_ms, int64_t* launches) {
    if (!ctx || kind < 0 || kind > 3) return SCX_ERR_VALIDATION;
    tcollect(ctx);
    *total_ms = ctx->timer.ms[kind];
    *launches = ctx->timer.launches[kind];
    return SCX_OK;
}

// ---------------------------------------------------------------- multi-GPU
// ---------------------------------------------------------------- multi-GPU (row shards)
scx_status scx_set_sm_budget(scx_ctx* ctx, int sms) {
    if (!ctx || sms < 0) return SCX_ERR_VALIDATION;
    ctx->sm_budget = sms;
    return SCX_OK;
}

scx_status scx_xchg_slots(scx_ctx* ctx, void** slots) {
    if (!ctx || !slots) return SCX_ERR_VALIDATION;
    cudaSetDevice(ctx->device);
    if (!ctx->xslots) CK(cudaMalloc((void**)&ctx->xslots, 2 * sizeof(XSlot)));
    CK(cudaMemset(ctx->xslots, 0, 2 * sizeof(XSlot)));
    *slots = ctx->xslots;
    return SCX_OK;
}

scx_status scx_xchg_ipc_handle(scx_ctx* ctx, char out[64]) {
    void* sl = nullptr;
    if (scx_status st = scx_xchg_slots(ctx, &sl)) return st;
    cudaIpcMemHandle_t h;
    CK(cudaIpcGetMemHandle(&h, sl));
    static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t is 64 bytes");
    memcpy(out, &h, 64);
    return SCX_OK;
}

scx_status scx_xchg_connect(scx_ctx* ctx, int nranks, int rank, void* const* rank_slots) {
    if (!ctx || !rank_slots) return SCX_ERR_VALIDATION;
    if (nranks < 1 || nranks > kXMaxRanks || rank < 0 || rank >= nranks)
        return fail(ctx, SCX_ERR_VALIDATION, "invalid rank / world size");
    cudaSetDevice(ctx->device);
    void* own = nullptr;
    if (scx_status st = scx_xchg_slots(ctx, &own)) return st;
    if (rank_slots[rank] != own)
        return fail(ctx, SCX_ERR_VALIDATION, "rank_slots[rank] is not this context's exchange slots");
    Xchg x{};
    x.nranks = nranks;
    x.rank = rank;
    for (int r = 0; r < nranks; ++r) {
        x.slot[r] = static_cast<XSlot*>(rank_slots[r]);
        cudaPointerAttributes at{};
        if (cudaPointerGetAttributes(&at, rank_slots[r]) == cudaSuccess && at.device != ctx->device &&
            at.type == cudaMemoryTypeDevice) {
            int can = 0;
            cudaDeviceCanAccessPeer(&can, ctx->device, at.device);
            if (!can) return fail(ctx, SCX_ERR_CUDA, "peer device not accessible (no P2P)");
            const cudaError_t e = cudaDeviceEnablePeerAccess(at.device, 0);
            if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled)
                return cuda_fail(ctx, e, "cudaDeviceEnablePeerAccess");
            cudaGetLastError();
        }
    }
    ctx->x = x;
    ctx->nranks = nranks;
    ctx->rank = rank;
    ctx->d.x = x;
    const unsigned long long zero = 0;
    CK(cudaMemcpy(&ctx->d.ctl->xseq, &zero, sizeof zero, cudaMemcpyHostToDevice));
    return SCX_OK;
}

scx_status scx_xchg_connect_ipc(scx_ctx* ctx, int nranks, int rank, const char* handles) {
    if (!ctx || !handles) return SCX_ERR_VALIDATION;
    if (nranks < 1 || nranks > kXMaxRanks || rank < 0 || rank >= nranks)
        return fail(ctx, SCX_ERR_VALIDATION, "invalid rank / world size");
    cudaSetDevice(ctx->device);
    void* own = nullptr;
    if (scx_status st = scx_xchg_slots(ctx, &own)) return st;
    std::vector<void*> ptrs(nranks, nullptr);
    for (int r = 0; r < nranks; ++r) {
        if (r == rank) {
            ptrs[r] = own;
            continue;
        }
        cudaIpcMemHandle_t h;
        memcpy(&h, handles + 64 * r, 64);
        CK(cudaIpcOpenMemHandle(&ptrs[r], h, cudaIpcMemLazyEnablePeerAccess));
        ctx->ipc_open.push_back(ptrs[r]);
    }
    return scx_xchg_connect(ctx, nranks, rank, ptrs.data());
}

scx_status scx_shard_local_columns(scx_ctx* ctx, uint8_t* nonempty, double* lin, double* xmax,
                                   int* rs_ok) {
    if (scx_status s = need_design(ctx)) return s;
    for (int64_t j = 0; j < ctx->d.p; ++j) {
        if (nonempty) nonempty[j] = ctx->cols[j].nnz > 0;
        if (lin) lin[j] = ctx->cols[j].lin;
        if (xmax) xmax[j] = ctx->cols[j].xmax;
    }
    if (rs_ok) *rs_ok = ctx->d.rs_ok;
    return SCX_OK;
}

scx_status scx_shard_set_columns(scx_ctx* ctx, const uint8_t* nonempty, const double* lin,
                                 const double* xmax, int rs_ok) {
    if (scx_status s = need_design(ctx)) return s;
    cudaSetDevice(ctx->device);
    cudaStream_t s = ctx->stream;
    const int64_t p = ctx->d.p;
    ctx->gnz.assign(nonempty, nonempty + p);
    ctx->zero_cols.clear();
    for (int64_t j = 0; j < p; ++j) {
        ctx->cols[j].lin = lin[j];
        ctx->cols[j].xmax = xmax[j];
        if (!nonempty[j]) ctx->zero_cols.push_back((int32_t)j);
    }
    // the cycle's column set: every globally non-empty column, the same list on
    // every rank (a rank without rows of a column contributes zero partials)
    std::vector<ColArgs> nz;
    ctx->runs.clear();
    for (int64_t j = 0; j < p; ++j)
        if (nonempty[j]) {
            const int32_t ind = ctx->cols[j].indicator;
            if (ctx->runs.empty() || ctx->runs.back()[2] != ind)
                ctx->runs.push_back({(int32_t)nz.size(), 0, ind});
            ctx->runs.back()[1] += 1;
            nz.push_back(ctx->cols[j]);
        }
    if (ctx->cols_d) cudaFree(ctx->cols_d);
    ctx->cols_d = nullptr;
    CK(dmalloc(&ctx->cols_d, nz.size()));
    if (!nz.empty())
        CK(cudaMemcpyAsync(ctx->cols_d, nz.data(), nz.size() * sizeof(ColArgs), cudaMemcpyHostToDevice, s));
    ctx->cycle_cols = nz;
    if (ctx->zero_cols_d) cudaFree(ctx->zero_cols_d);
    ctx->zero_cols_d = nullptr;
    CK(dmalloc(&ctx->zero_cols_d, ctx->zero_cols.size()));
    if (!ctx->zero_cols.empty())
        CK(cudaMemcpyAsync(ctx->zero_cols_d, ctx->zero_cols.data(),
                           ctx->zero_cols.size() * sizeof(int32_t), cudaMemcpyHostToDevice, s));
    ctx->d.rs_ok = ctx->d.rs_ok && rs_ok;
    CK(cudaStreamSynchronize(s));
    // every kernel of the sharded fit loaded now, not lazily while a peer spins
    preload_sharded_kernels(ctx->d);
    cudaFuncAttributes fa;
    cudaFuncGetAttributes(&fa, (const void*)k_k3_check);
    cudaFuncGetAttributes(&fa, (const void*)k_fill);
    return SCX_OK;
}

}  // extern "C"
