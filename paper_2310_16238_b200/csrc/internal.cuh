// Internal declarations shared by the sm_100a kernels and the C-ABI host code.
//
// Device data layout (one scx_ctx, sorted row space, N padded to a multiple
// of the 4096-row tile so every tile is full):
//   D       f64[Npad]  exp(X beta)             (CoefficientState::exp_xbeta)
//   eta     f64[Npad]  X beta                  (CoefficientState::xbeta)
//   code    u8/u16/u32[Npad] per-row event code: bit(W-1) = stratum head,
//           bit(W-2) = event, low W-2 bits = w_s, the number of events whose
//           tie group ends at row s (sum_{i: tie_end(i)=s} delta_i). The
//           reference gathers S[tie_end(i)] per event row i
//           (likelihood.cpp:165-175); re-associating that sum onto tie-group
//           ends turns the gather into a forward stream (exact algebra).
//   rows    i32[nnz]   CSC row indices, columns concatenated (SparseColumn::rows)
//   vals    f64[nval]  values of non-indicator columns only, compacted
//   tptr    i32[p][ntiles1+1] per column, entry offset of each 2048-row K1 tile's first row
//   beta, gamma, trust  f64[p]
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "rules.cuh"

namespace scx {

constexpr int kTileRows = 4096;
constexpr int kK1TileRows = 2048;  // fused scan+reduce (K1) tile
constexpr int kThreads = 256;
constexpr int kRowsPerThread = kTileRows / kThreads;  // 16
constexpr int kWarps = kThreads / 32;
constexpr int kLookbackWindows = 16;  // smem stack depth of the look-back (512 tiles)

// look-back slot states (low 2 bits of the status word; high 30 bits = epoch)
constexpr uint32_t kStAgg = 1;
constexpr uint32_t kStInc = 2;

// Per-column metadata, passed by value to the per-coordinate kernels.
struct ColArgs {
    int64_t beg;      // first entry in rows[]
    int64_t nnz;      // entries
    int64_t val_off;  // first value in vals[] (-1 for an indicator column)
    double lin;       // sum_t x_t * delta_{row_t}, in entry order (likelihood.cpp:147)
    double xmax;      // max_t |x_t|
    int32_t j;
    int32_t indicator;
};

// Device error word: first failure wins.
enum ErrKind : int {
    kErrNone = 0,
    kErrNonFiniteD = 1,        // validation "non-finite input at index i"  (idx = row)
    kErrBadDenom = 2,          // internal "risk-set sum not positive at sorted row i" (idx = tie end)
    kErrNonFiniteGH = 3,       // numeric "non-finite gradient/Hessian for covariate NAME" (idx = j)
    kErrNonFiniteLL = 4,       // numeric "non-finite log partial likelihood"
    kErrRuleNewton = 5,        // numeric "non-finite gradient or Hessian in Newton step"
    kErrRuleTrust = 6,         // numeric "non-finite trust-region inputs"
    kErrRuleBothNegative = 7,  // internal "both directional derivatives negative at the origin"
    kErrLPOverflow = 8,        // numeric "linear predictor overflow at row s" (idx = row)
    kErrStepOverflow = 9,      // numeric "step overflow"
    kErrNonFiniteStep = 10,    // numeric "non-finite coordinate step"
    kErrBadTieEnd = 20,        // validation: tie_group_end out of range (upload)
    kErrBadEvent = 21,         // validation: event indicator must be 0 or 1 (upload)
    kErrBadRows = 22,          // validation: column rows not strictly increasing / out of range
    kErrXchgTimeout = 30,      // multi-GPU: a peer rank did not reach an exchange in time
    kErrPeer = 31,             // multi-GPU: another rank stopped with an error
};

// Control block in device memory (one per context).
struct DevCtl {
    // K1/K2 tile tickets, completion counters, look-back epoch
    unsigned int ticket;
    unsigned int done;
    unsigned int epoch;
    unsigned int pad0;
    // software grid barrier for cooperative kernels: low 32 bits arrivals,
    // high 32 bits generation (one word: the last arrival resets the count and
    // advances the generation with one atomic)
    unsigned long long bar;
    // error word
    int err_kind;
    int pad1;
    long long err_idx;
    long long bad_min;  // min offending row found by a diagnostic pass
    // last evaluation
    double g, h;
    double ll;
    double penalty;
    // coordinate scratch written by K1's last block, read by K3
    double applied;   // proposed step after the trust clip
    int fast;         // 1 = bound check proves no row can overflow
    int hmax;         // slow path: max over entries of the halvings needed
    int will_refresh; // the update counter hits 256 if this step is applied
    int pad2;
    // fit bookkeeping
    double max_step;        // sup-norm of applied steps this cycle
    double mbound;          // upper bound on max_s |eta_s|
    unsigned int updates;   // CoefficientState::updates_since_refresh
    int n_warn;             // coordinates skipped after 10 halvings
    long long n_eval;       // gradient/Hessian evaluations
    double part[4];         // multi-GPU: (local lin, ratio sum, variance sum, 0)
    long long* warn_coord;  // [warn_cap] coordinate of each warning, in order (device buffer)
    int warn_cap;
    int pad3;
    int resume;     // cycle kernel: coordinates done before it stopped for a refresh (0: ran to the end)
    int rs_reason;  // risk-suffix cycle: why it stopped (RsStop)
    unsigned long long xseq;  // multi-GPU: device exchanges done so far (the same on every rank)
    unsigned long long bar2;  // second grid-barrier word (split arrive / wait, see grid_arrive)
};

// Why a risk-suffix cycle launch returned before its last coordinate.
enum RsStop : int {
    kRsDone = 0,      // every coordinate processed
    kRsRefresh = 1,   // 256 accepted updates: refresh eta/D, then resume
    kRsExact = 2,     // coordinate `resume`'s g'' cancels against its terms (S1 ~ S0 on
                      // its risk sets): the per-coordinate fused scan decides
    kRsBound = 3,     // max|eta| bound passed kRsEtaBound: finish with the fused scan
};
constexpr double kRsEtaBound = 300.0;  // w/S0^2 and a*Q*(a+2C) stay in fp64 range below it
constexpr int kWarnCap = 1 << 16;     // warnings recorded per fit (the count is exact)
constexpr int kRsMaxStrata = 1024;     // strata of one chunk staged in shared memory
constexpr int kRsTileInfo = 384;       // 2048-row tiles of one chunk (risk-scan tile carries)
constexpr int kRsStoreRows = 512;      // rows of one risk-scan TMA store (one warp's rows)

struct Pref1 {
    double v0;
    uint32_t f;
};

// ------------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(phase)
        : "memory");
}
// Same wait with a suspend-time hint: the warp sleeps in hardware until the
// phase completes (used by the producer / look-back warps, which would
// otherwise spin and take issue slots from the compute warps).
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t phase) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAITS_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, 1000000;\n"
        "@!p bra WAITS_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(phase)
        : "memory");
}
__device__ __forceinline__ void fence_barrier_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
// this thread's generic-proxy shared-memory writes are visible to TMA stores
__device__ __forceinline__ void fence_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
// TMA: 2-D tiled tensor copy shared -> global (bulk group of the issuing thread).
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, int c0, int c1, const void* src) {
    asm volatile(
        "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(map),
        "r"(c0), "r"(c1), "r"(smem_u32(src))
        : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
// this thread's bulk groups have finished reading shared memory
__device__ __forceinline__ void bulk_wait_read() {
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
// ... and their global writes are complete
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
// TMA: 2-D tiled tensor copy global -> shared, completion on an mbarrier.
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1,
                                            uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, "
        "{%2, %3}], [%4];" ::"r"(smem_u32(dst)),
        "l"(map), "r"(c0), "r"(c1), "r"(smem_u32(bar))
        : "memory");
}
// 1-D bulk copy global -> shared (size multiple of 16, both 16-B aligned).
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes,
                                          uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, "
        "[%3];" ::"r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void prefetch_tmap(const CUtensorMap* map) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(map) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire(const unsigned int* p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(unsigned int* p, uint32_t v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Software grid barrier (kernels using it are launched cooperatively, so all
// blocks are co-resident).
__device__ __forceinline__ void grid_sync(DevCtl* ctl) {
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long* w = &ctl->bar;
        __threadfence();  // this CTA's writes before its arrival
        const unsigned long long old = atomicAdd(w, 1ull);
        if ((unsigned int)old == gridDim.x - 1) {
            // last arrival: count back to 0 and generation + 1 in one atomic, so
            // no CTA of the next barrier can arrive before the reset
            atomicAdd(w, (1ull << 32) - gridDim.x);
        } else {
            const unsigned int gen = (unsigned int)(old >> 32);
            while ((unsigned int)(*((volatile unsigned long long*)w) >> 32) == gen) {
            }
        }
        __threadfence();
    }
    __syncthreads();
}

// Split grid barrier on a word of the same layout (thread 0 only): arrive after
// the CTA's writes, returning the generation; wait until it advances. Every CTA
// arrives at every such barrier; waiting is optional, so a CTA that did not wait
// must pass a full grid_sync on another word before it arrives again (the
// arrivals of one generation then all precede it).
__device__ __forceinline__ unsigned int grid_arrive(unsigned long long* w) {
    __threadfence();
    const unsigned long long old = atomicAdd(w, 1ull);
    if ((unsigned int)old == gridDim.x - 1) atomicAdd(w, (1ull << 32) - gridDim.x);
    return (unsigned int)(old >> 32);
}
__device__ __forceinline__ void grid_wait(unsigned long long* w, unsigned int gen) {
    while ((unsigned int)(*((volatile unsigned long long*)w) >> 32) == gen) {
    }
    __threadfence();
}

__device__ __forceinline__ void set_error(DevCtl* ctl, int kind, long long idx) {
    if (atomicCAS(&ctl->err_kind, 0, kind) == 0) {
        ctl->err_idx = idx;
        __threadfence();
    }
}

// ------------------------------------------------------------------ device exchange (multi-GPU)
// Row-sharded fits exchange a few doubles per coordinate: each rank owns two
// 128-B slots (alternating by exchange number) in device memory that every
// rank can load — a peer-mapped (P2P over NVLink) or IPC-opened allocation on
// a node, the same device's memory for ranks sharing one GPU (loopback). The
// publishing thread writes its values, then the sequence word with release
// order; readers poll every rank's sequence word and sum (or max) the values
// in rank order, so every rank computes bit-identical results. Lock-step
// (every exchange needs every rank) makes two slots enough.
constexpr int kXMaxRanks = 8;
constexpr int kXVals = 12;
struct alignas(128) XSlot {
    double v[kXVals];
    int err;                  // the rank stops with an error after this exchange
    int pad;
    unsigned long long seq;   // exchange number + 1 once v / err are written
};
struct Xchg {
    XSlot* slot[kXMaxRanks];  // rank r's two slots (slot[rank] = this rank's own)
    int nranks;               // 1: no exchange
    int rank;
};

constexpr long long kXchgTimeoutCycles = 8000000000LL;  // ~4 s: a peer that never comes

// Exchange number k: `publish` (one thread per rank) writes this rank's n
// values and error flag; every calling thread waits for all ranks and gets
// the rank-ordered sum (op 0) or max (op 1) in out[] and the OR of the error
// flags. Returns false on timeout.
__device__ __forceinline__ bool xchg_values(const Xchg& x, unsigned long long k, const double* mine,
                                            int n, int op, bool publish, int err_mine, double* out,
                                            int* err_any) {
    const int s = (int)(k & 1ull);
    if (publish) {
        XSlot* own = x.slot[x.rank] + s;
#pragma unroll
        for (int i = 0; i < kXVals; ++i)  // unrolled with a guard: mine[] stays in registers
            if (i < n) own->v[i] = mine[i];
        own->err = err_mine;
        __threadfence_system();
        *((volatile unsigned long long*)&own->seq) = k + 1;
    }
    const long long t0 = clock64();
    for (int r = 0; r < x.nranks; ++r) {
        const volatile unsigned long long* sq = &x.slot[r][s].seq;
        while (*sq != k + 1) {
            if (clock64() - t0 > kXchgTimeoutCycles) return false;
            __nanosleep(64);
        }
    }
    __threadfence_system();
    int e = 0;
    for (int r = 0; r < x.nranks; ++r) {
        const XSlot* ps = x.slot[r] + s;
#pragma unroll
        for (int i = 0; i < kXVals; ++i) {
            if (i >= n) continue;
            const double v = __ldcv(&ps->v[i]);
            out[i] = op ? (r == 0 ? v : fmax(out[i], v)) : (r == 0 ? v : out[i] + v);
        }
        e |= __ldcv(&ps->err);
    }
    *err_any = e;
    return true;
}

// ------------------------------------------------------------------ launch API
// (defined in kernels.cu; all launches on `stream`)
struct DesignDev {
    int64_t n;
    int64_t npad;
    int64_t ntiles;
    int64_t ntiles1;          // K1 tiles (kK1TileRows)
    int64_t p;
    int32_t k;
    int32_t code_bytes;
    void* code;
    double* D;
    double* eta;
    const int32_t* rows;
    const double* vals;
    const int32_t* tptr;
    int32_t* lasth1;          // [ntiles1] last stratum head offset in each K1 tile (-1: none)
    int32_t* chunk_rows;      // [nchunks+1] stratum-aligned chunk starts (NULL: look-back mode)
    int32_t nchunks;
    int32_t k1_mode;          // 0 auto, 1 force look-back, 2 chunk when available
    const int64_t* col_beg;   // [p+1]
    const int64_t* val_off;   // [p] (-1 indicator)
    const int64_t* offsets;   // [k+1]
    double* beta;
    double* gamma;
    double* l2;               // [p] L2 prior weights (extension; zeros unless a prior is given)
    double* trust;
    // refresh: nonzero-beta columns compacted per refresh and their tile entry
    // offsets transposed to [tile][active column] (coalesced per tile)
    int32_t* ref_act;         // [p] active columns, ascending
    int64_t* ref_abeg;        // [p] their first CSC entry
    int64_t* ref_avo;         // [p] their value offset (-1 indicator)
    double* ref_ab;           // [p] their beta
    int32_t* ref_nact;        // [1] number of active columns
    int32_t* ref_meta;        // [ntiles1+1][ref_ps] tptr of the active columns, transposed
    int64_t ref_ps;           // row stride of ref_meta (p rounded up to 32)
    // refresh in row slices (build_refresh_ell): entry k of row 32s+l at
    // ell_base[s] + 128(k/4) + 4l + k%4; column ids u16 (u32 when ell_wide), p = padding
    void* ell_col;
    double* ell_val;          // NULL: every value 1.0
    int64_t* ell_base;        // [ell_nsl + 1]
    int64_t ell_nsl;
    int32_t ell_wide;
    int32_t ell_ok;           // the row-slice refresh is available
    // look-back scratch
    unsigned int* status;     // [ntiles]
    double* slots;            // [2][ntiles][4] agg / inc (s0, s1, s2, flag)
    double* partial;          // [ntiles][2]
    DevCtl* ctl;
    CUtensorMap tmap_D;       // box 16 x 256 (4096-row tile)
    CUtensorMap tmap_D1;      // box 16 x 128 (2048-row K1 tile)
    CUtensorMap tmap_eta;
    int coop_blocks;          // co-resident blocks for the cooperative kernels
    int sm_budget;            // SMs of a rank sharing the GPU (0: all)
    // risk-suffix CCD cycle (chunk layout only)
    double* rs_CR;            // [ntiles1] risk scan: carry of each tile's open segment (R)
    double* rs_CQ;            // [ntiles1] ... (Q)
    double* rs_R;             // [npad] within-stratum suffix sum of w/S0 from each row
    double* rs_Q;             // [npad] within-stratum suffix sum of w/S0^2 from each row
    CUtensorMap tmap_R;
    CUtensorMap tmap_Q;
    int32_t* chunk_k;         // [nchunks+1] first stratum of each chunk (holding its first row)
    int32_t* rs_chunk_nk;     // [nchunks] strata of each risk-scan chunk
    int32_t* rs_chunk_rows;   // [nchunks+1] risk-scan chunks (= chunk_rows when stratum-aligned)
    int32_t rs_aligned;       // risk-scan chunks start at heads (else whole tiles, carries cross)
    double* rs_xagg;          // [4 * nchunks] cross-chunk carries (unaligned chunks)
    int32_t rs_ok;            // chunks hold <= kRsMaxStrata strata each
    Xchg x;                   // multi-GPU exchange (x.nranks == 1: single device)
};

enum K1Mode : int { kK1Eval = 0, kK1Fit = 1, kK1Diag = 2, kK1Partial = 3 };

cudaError_t launch_k1(const DesignDev& d, const ColArgs& col, int mode, cudaStream_t s);
cudaError_t k1_trace_copy(long long* out);
// risk-suffix CCD cycle over cols_d[0..ncols): mode 0 fit, 1 evaluate cols_d[0]
// only (g, h into ctl), 2 risk scan only (ncols back-to-back scans: throughput probe),
// 3 g' of every column at the current state into gout[0..ncols) (gamma_max)
cudaError_t launch_rs_cycle(const DesignDev& d, const ColArgs* cols_d, int ncols, int mode,
                            cudaStream_t s, double* gout = nullptr);
// one CCD cycle in one cooperative launch over cols_d[0..ncols) (all of one
// kind: indicator or value columns)
cudaError_t launch_cycle(const DesignDev& d, const ColArgs* cols_d, int ncols, bool indicator,
                         cudaStream_t s);  // [2][512][8] clock64 (SCX_K1_DBG bit 8)
cudaError_t launch_k2(const DesignDev& d, int fit_mode, cudaStream_t s);
// K3: apply the step decided by K1 (mode 0 = fit with halving, 1 = standalone
// update_xbeta with delta given, no halving -> "step overflow")
cudaError_t launch_k3(const DesignDev& d, const ColArgs& col, int mode, double delta,
                      cudaStream_t s);
// refresh eta/D from beta (make_state / refresh_xbeta)
// kernels launched by launch_refresh (active columns, their tile table, the tiles, finish)
// (2 when the row-slice refresh runs: the slices, finish)
constexpr int kRefreshLaunches = 4;
int refresh_launches(const DesignDev& d);
cudaError_t launch_refresh(const DesignDev& d, cudaStream_t s);
cudaError_t launch_naive_gh(const DesignDev& d, const ColArgs& col, double* xdense,
                            double* out2, cudaStream_t s);
cudaError_t launch_naive_ll(const DesignDev& d, double* out1, cudaStream_t s);
cudaError_t launch_zero_cols(const DesignDev& d, const int32_t* cols, int64_t ncols, cudaStream_t s);
// multi-GPU: rank-summed partials + rule (k_shard_step); ctl exchanges
// (what 0: max mbound, 1: sum ll + max mbound, 2: max halving level)
void preload_sharded_kernels(const DesignDev& d);
cudaError_t build_refresh_ell(DesignDev& d, int64_t nnz, bool any_values, cudaStream_t s);
cudaError_t launch_shard_step(const DesignDev& d, const ColArgs& col, cudaStream_t s);
cudaError_t launch_xchg_ctl(const DesignDev& d, int what, cudaStream_t s);
// design preparation
cudaError_t launch_build_codes(void* code, int code_bytes, int64_t n, int64_t npad,
                               const uint8_t* event, const int64_t* tie_end,
                               const int64_t* offsets, int32_t k, uint32_t* wtmp,
                               cudaStream_t s);
cudaError_t launch_tie_weights(uint32_t* w, const uint8_t* event, const int64_t* tie_end, int64_t n,
                               DevCtl* ctl, unsigned int* maxw, cudaStream_t s);
cudaError_t launch_tile_ptr(int32_t* tptr, const int32_t* rows, const int64_t* col_beg,
                            int64_t p, int64_t ntiles, cudaStream_t s);
cudaError_t launch_last_head(int32_t* lasth, const int64_t* offsets, int32_t k, int64_t ntiles1,
                             cudaStream_t s);
cudaError_t launch_narrow_rows(int32_t* dst, const int64_t* src, int64_t count, cudaStream_t s);
cudaError_t launch_scan_primitive(const DesignDev& d, double* out, cudaStream_t s);
cudaError_t launch_k3_sharded(const DesignDev& d, const ColArgs& col, cudaStream_t s);
const void* k3_apply_ptr();

}  // namespace scx
