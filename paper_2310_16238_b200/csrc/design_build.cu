#include <mutex>
// Device build of the SortedDesign: build_sorted_design,
// proj/src/data.cpp:68-147, with validate_invariants (data.cpp:27-66) — on the
// GPU instead of the host.
//
//   validation   row checks (time, event, stratum label), empty strata, column
//                checks (strictly increasing rows, range, finite values), each
//                reduced to the FIRST failing (row | entry, check) with an
//                atomicMin on index*4 + check, so the message is the one the
//                reference's serial loops throw first.
//   row order    the reference's std::stable_sort by (stratum asc, time desc)
//                as two stable LSD radix sorts: by ~bits(time) (non-negative
//                doubles order like their bit patterns; -0.0 is folded onto
//                +0.0, which compares equal to it), then by stratum label.
//                Stable + LSD = the same permutation, bit for bit.
//   CSC          rows re-indexed through the inverse permutation and sorted
//                inside each column by a segmented LSD radix sort (tiles never
//                straddle a column), values following their rows.
//   heads, tie ends, offsets: a flag pass and a reverse min-scan; offsets from
//                the per-stratum counts of the validation pass.
//
// The radix passes: 8-bit digits, 8192-entry tiles (512 threads x 16), a per-
// tile digit histogram, a scan over (segment, digit, tile), and a stable
// scatter whose in-tile ranks come from __match_any_sync over warp rows and
// per-warp digit counters (entries keep their order inside a digit, which is
// what makes the LSD sort stable). Digits constant over all keys are skipped.
// No CUB / Thrust.
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/stratcox_b200.h"
#include "internal.cuh"
#include "lowered.h"

namespace scx {

constexpr int kRxThreads = 512;
constexpr int kRxItems = 16;
constexpr int kRxWarps = kRxThreads / 32;
constexpr int64_t kRxTile = (int64_t)kRxThreads * kRxItems;  // 8192 entries
constexpr unsigned long long kNoErr = 0xffffffffffffffffULL;

struct BuildErr {                 // device error words (first failure by index)
    unsigned long long row_err;   // row * 4 + check (0 time, 1 event, 2 label)
    unsigned long long ent_err;   // entry * 4 + check (0 order, 1 range, 2 value)
    int kmax;                     // max stratum label
    int pad;
    unsigned long long t_or, t_and;  // varying bits of the time keys
    unsigned long long k_or, k_and;  // ... of the stratum keys
    unsigned long long r_or, r_and;  // ... of the re-indexed rows
};

__device__ __forceinline__ uint64_t time_key(double t) {
    uint64_t b = (uint64_t)__double_as_longlong(t);
    if (b == 0x8000000000000000ULL) b = 0;  // -0.0 == +0.0 in the reference's comparator
    return ~b;                              // descending time = ascending key
}

// max label; row checks; time keys + identity values; per-stratum counts
// (labels 1..kcap only: with kmax > n some stratum is empty anyway)
__global__ void k_b_kmax(const int32_t* stratum, int64_t n, BuildErr* be) {
    int m = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        m = max(m, stratum[i]);
    for (int o = 16; o; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) atomicMax(&be->kmax, m);
}

__global__ void k_b_rows(const double* time, const uint8_t* event, const int32_t* stratum, int64_t n,
                         int kmax, int kcap, BuildErr* be, unsigned int* counts, uint64_t* tkey,
                         uint32_t* idx) {
    unsigned long long err = kNoErr, o = 0, a = ~0ULL;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const double t = time[i];
        const int32_t s = stratum[i];
        unsigned long long e = kNoErr;
        if (!isfinite(t) || t < 0.0)
            e = (unsigned long long)i * 4 + 0;
        else if (event[i] > 1)
            e = (unsigned long long)i * 4 + 1;
        else if (s < 1 || s > kmax)
            e = (unsigned long long)i * 4 + 2;
        err = min(err, e);
        const bool cnt_it = e == kNoErr && s <= kcap;
        const unsigned act = __activemask();
        const unsigned cm = __ballot_sync(act, cnt_it);
        if (cnt_it) {  // warp-aggregated per-stratum counts
            const unsigned peers = __match_any_sync(cm, s);
            if ((threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(counts + (s - 1), __popc(peers));
        }
        const uint64_t k = time_key(t);
        tkey[i] = k;
        idx[i] = (uint32_t)i;
        o |= k;
        a &= k;
    }
    for (int q = 16; q; q >>= 1) {
        err = min(err, (unsigned long long)__shfl_xor_sync(0xffffffffu, (long long)err, q));
        o |= (unsigned long long)__shfl_xor_sync(0xffffffffu, (long long)o, q);
        a &= (unsigned long long)__shfl_xor_sync(0xffffffffu, (long long)a, q);
    }
    if ((threadIdx.x & 31) == 0) {
        if (err != kNoErr) atomicMin(&be->row_err, err);
        atomicOr(&be->t_or, o);
        atomicAnd(&be->t_and, a);
    }
}

// ---------------------------------------------------------------- radix sort
// Tile map: tile i covers entries [tb[i], tb[i+1]) of segment tseg[i];
// segment g owns tiles [st0[g], st0[g+1]) and starts at entry sbeg[g].
struct TileMap {
    int64_t* tb = nullptr;
    int32_t* tseg = nullptr;
    int64_t* st0 = nullptr;
    int64_t* sbeg = nullptr;
    int64_t ntiles = 0, nseg = 0;
};

template <typename K>
__global__ void __launch_bounds__(kRxThreads) k_rx_hist(const K* keys, const int64_t* tb,
                                                      int64_t ntiles, int shift, uint32_t* hist) {
    __shared__ uint32_t h[256];
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        if (threadIdx.x < 256) h[threadIdx.x] = 0;
        __syncthreads();
        const int64_t b = tb[tile], e = tb[tile + 1];
        for (int64_t i = b + threadIdx.x; i < e; i += kRxThreads)
            atomicAdd(&h[(uint32_t)(keys[i] >> shift) & 0xffu], 1u);
        __syncthreads();
        if (threadIdx.x < 256) hist[tile * 256 + threadIdx.x] = h[threadIdx.x];
        __syncthreads();
    }
}

// (segment, digit) per thread: exclusive prefix over the segment's tiles (in
// place) and the segment's digit total
__global__ void k_rx_scan_tiles(uint32_t* hist, const int64_t* st0, int64_t nseg, uint32_t* segtot) {
    const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= nseg * 256) return;
    const int64_t seg = g >> 8;
    const int d = (int)(g & 255);
    uint32_t run = 0;
    int64_t t = st0[seg];
    const int64_t t1 = st0[seg + 1];
    for (; t + 8 <= t1; t += 8) {
        uint32_t c[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) c[u] = hist[(t + u) * 256 + d];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            hist[(t + u) * 256 + d] = run;
            run += c[u];
        }
    }
    for (; t < t1; ++t) {
        const uint32_t c = hist[t * 256 + d];
        hist[t * 256 + d] = run;
        run += c;
    }
    segtot[g] = run;
}

// one warp per segment: exclusive prefix of the 256 digit totals
__global__ void k_rx_scan_digits(uint32_t* segtot, int64_t nseg) {
    const int64_t seg = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (seg >= nseg) return;
    uint32_t* t = segtot + seg * 256;
    uint32_t v[8], sum = 0;
#pragma unroll
    for (int u = 0; u < 8; ++u) {
        v[u] = t[lane * 8 + u];
        sum += v[u];
    }
    uint32_t inc = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t x = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += x;
    }
    uint32_t run = inc - sum;
#pragma unroll
    for (int u = 0; u < 8; ++u) {
        t[lane * 8 + u] = run;
        run += v[u];
    }
}

// stable scatter of one tile: warp w holds entries [w*512, w*512+512) of the
// tile, row r of the warp = 32 consecutive entries
template <typename K, bool VAL>
__global__ void __launch_bounds__(kRxThreads) k_rx_scatter(const K* kin, const uint32_t* vin, K* kout,
                                                         uint32_t* vout, const int64_t* tb,
                                                         const int32_t* tseg, const int64_t* sbeg,
                                                         const uint32_t* hist, const uint32_t* segbase,
                                                         int64_t ntiles, int shift) {
    __shared__ uint16_t wc[kRxWarps][256];
    __shared__ int64_t tofs[256];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        for (int q = threadIdx.x; q < kRxWarps * 256; q += kRxThreads) (&wc[0][0])[q] = 0;
        __syncthreads();
        const int64_t b = tb[tile], e = tb[tile + 1];
        const int32_t seg = tseg[tile];
        K k[kRxItems];
        uint32_t v[kRxItems];
        uint32_t dg[kRxItems];
        uint16_t loc[kRxItems];
#pragma unroll
        for (int r = 0; r < kRxItems; ++r) {
            const int64_t i = b + w * (32 * kRxItems) + r * 32 + lane;
            if (i < e) {
                k[r] = kin[i];
                if constexpr (VAL) v[r] = vin[i];
                dg[r] = (uint32_t)(k[r] >> shift) & 0xffu;
            } else {
                dg[r] = 256;
            }
        }
#pragma unroll
        for (int r = 0; r < kRxItems; ++r) {
            const bool ok = dg[r] < 256;
            const unsigned act = __ballot_sync(0xffffffffu, ok);
            unsigned peers = 0;
            uint16_t base = 0;
            if (ok) {
                peers = __match_any_sync(act, dg[r]);
                base = wc[w][dg[r]];
                loc[r] = (uint16_t)(base + __popc(peers & ((1u << lane) - 1u)));
            }
            __syncwarp();
            if (ok && lane == __ffs(peers) - 1) wc[w][dg[r]] = (uint16_t)(base + __popc(peers));
            __syncwarp();
        }
        __syncthreads();
        if (threadIdx.x < 256) {
            const int d = threadIdx.x;
            uint16_t run = 0;
            for (int q = 0; q < kRxWarps; ++q) {
                const uint16_t c = wc[q][d];
                wc[q][d] = run;
                run = (uint16_t)(run + c);
            }
            tofs[d] = sbeg[seg] + (int64_t)segbase[(int64_t)seg * 256 + d] + hist[tile * 256 + d];
        }
        __syncthreads();
#pragma unroll
        for (int r = 0; r < kRxItems; ++r) {
            if (dg[r] < 256) {
                const int64_t pos = tofs[dg[r]] + wc[w][dg[r]] + loc[r];
                kout[pos] = k[r];
                if constexpr (VAL) vout[pos] = v[r];
            }
        }
        __syncthreads();
    }
}

static int grid_sms(int64_t work) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return (int)std::max<int64_t>(1, std::min<int64_t>(work, (int64_t)sms * 8));
}

// LSD passes over the digits of `varying`; keys/vals ping-pong (the result is
// left in keys/vals). Stable in every pass.
template <typename K>
static cudaError_t radix_sort(K*& keys, K*& kalt, uint32_t*& vals, uint32_t*& valt, bool has_val,
                              const TileMap& tm, uint64_t varying, uint32_t* hist,
                              uint32_t* segtot, cudaStream_t s) {
    if (tm.ntiles == 0) return cudaSuccess;
    for (int shift = 0; shift < (int)(8 * sizeof(K)); shift += 8) {
        if (((varying >> shift) & 0xffu) == 0) continue;
        const int g = grid_sms(tm.ntiles);
        k_rx_hist<K><<<g, kRxThreads, 0, s>>>(keys, tm.tb, tm.ntiles, shift, hist);
        const int64_t nt = tm.nseg * 256;
        k_rx_scan_tiles<<<(unsigned)((nt + 255) / 256), 256, 0, s>>>(hist, tm.st0, tm.nseg, segtot);
        k_rx_scan_digits<<<(unsigned)((tm.nseg * 32 + 255) / 256), 256, 0, s>>>(segtot, tm.nseg);
        if (has_val)
            k_rx_scatter<K, true><<<g, kRxThreads, 0, s>>>(keys, vals, kalt, valt, tm.tb, tm.tseg,
                                                          tm.sbeg, hist, segtot, tm.ntiles, shift);
        else
            k_rx_scatter<K, false><<<g, kRxThreads, 0, s>>>(keys, vals, kalt, valt, tm.tb, tm.tseg,
                                                           tm.sbeg, hist, segtot, tm.ntiles, shift);
        std::swap(keys, kalt);
        if (has_val) std::swap(vals, valt);
    }
    return cudaGetLastError();
}

// ---------------------------------------------------------------- sorted rows
// stratum key of sorted position s under the current permutation
__global__ void k_b_gather_str(const uint32_t* perm, const int32_t* stratum, int64_t n, uint32_t* key,
                               BuildErr* be) {
    unsigned long long o = 0, a = ~0ULL;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t k = (uint32_t)stratum[perm[i]];
        key[i] = k;
        o |= k;
        a &= k;
    }
    for (int q = 16; q; q >>= 1) {
        o |= (unsigned long long)__shfl_xor_sync(0xffffffffu, (long long)o, q);
        a &= (unsigned long long)__shfl_xor_sync(0xffffffffu, (long long)a, q);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicOr(&be->k_or, o);
        atomicAnd(&be->k_and, a);
    }
}

// inverse permutation, sorted event / time / stratum, tie-group-end flags
__global__ void k_b_sorted(const uint32_t* perm, const double* time, const uint8_t* event,
                           const int32_t* stratum, int64_t n, uint32_t* inv, uint8_t* ev_s,
                           int64_t* perm_out, double* time_s, int32_t* str_s) {
    for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < n;
         s += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t r = perm[s];
        inv[r] = (uint32_t)s;
        ev_s[s] = event[r];
        time_s[s] = time[r];
        str_s[s] = stratum[r];
        perm_out[s] = r;
    }
}

// tie_group_end (data.cpp:135-145): the last row of the run of equal
// (stratum, time) that holds s. Reverse min-scan of the run ends, 1024 rows
// per block; the carry across blocks comes from k_b_tie_blocks.
constexpr int kTieBlock = 1024;
__device__ __forceinline__ bool run_end(const double* t, const int32_t* k, int64_t n, int64_t s) {
    return s == n - 1 || k[s + 1] != k[s] || t[s + 1] != t[s];
}
__global__ void k_b_tie_blocks(const double* t, const int32_t* k, int64_t n, int64_t* bmin) {
    __shared__ int64_t red[32];
    const int64_t b0 = (int64_t)blockIdx.x * kTieBlock;
    const int64_t s = b0 + threadIdx.x;
    int64_t m = INT64_MAX;
    if (s < n && run_end(t, k, n, s)) m = s;
    for (int o = 16; o; o >>= 1) m = min(m, (int64_t)__shfl_xor_sync(0xffffffffu, (long long)m, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x < 32) {
        m = red[threadIdx.x];
        for (int o = 16; o; o >>= 1) m = min(m, (int64_t)__shfl_xor_sync(0xffffffffu, (long long)m, o));
        if (threadIdx.x == 0) bmin[blockIdx.x] = m;
    }
}
// carry[b] = min over blocks > b (one block of 1024 threads, serial chunks)
__global__ void k_b_tie_carry(const int64_t* bmin, int64_t nb, int64_t* carry) {
    __shared__ int64_t part[1024];
    const int64_t per = (nb + 1023) / 1024;
    const int64_t a = threadIdx.x * per, e = min(nb, a + per);
    int64_t m = INT64_MAX;
    for (int64_t b = a; b < e; ++b) m = min(m, bmin[b]);
    part[threadIdx.x] = m;
    __syncthreads();
    if (threadIdx.x == 0) {  // suffix minima of the parts, in place
        int64_t run = INT64_MAX;
        for (int q = 1023; q >= 0; --q) {
            const int64_t v = part[q];
            part[q] = run;  // exclusive: parts after q
            run = min(run, v);
        }
    }
    __syncthreads();
    int64_t run = part[threadIdx.x];
    for (int64_t b = e - 1; b >= a; --b) {
        carry[b] = run;
        run = min(run, bmin[b]);
    }
}
__global__ void k_b_tie_apply(const double* t, const int32_t* k, int64_t n, const int64_t* carry,
                              int64_t* tie_end) {
    __shared__ int64_t wmin[32];
    const int64_t s = (int64_t)blockIdx.x * kTieBlock + threadIdx.x;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    int64_t m = (s < n && run_end(t, k, n, s)) ? s : INT64_MAX;
    // inclusive suffix min inside the warp (lanes above)
    for (int o = 1; o < 32; o <<= 1) {
        const int64_t x = (int64_t)__shfl_down_sync(0xffffffffu, (long long)m, o);
        if (lane + o < 32) m = min(m, x);
    }
    if (lane == 0) wmin[w] = m;
    __syncthreads();
    int64_t c = carry[blockIdx.x];
    for (int q = w + 1; q < 32; ++q) c = min(c, wmin[q]);
    if (s < n) tie_end[s] = min(m, c);
}

// ---------------------------------------------------------------- columns
// H2D-staged int64 rows of whole tiles: column checks (data.cpp:55-64 order),
// narrowing, re-index through the inverse permutation, value-index payload.
__global__ void k_b_cols(const int64_t* rows64, int64_t chunk0, const int64_t* tb, int64_t t0,
                         int64_t t1, const int32_t* tseg, const int64_t* col_ptr, int64_t n,
                         const uint32_t* inv, uint32_t* key, uint32_t* vidx, int64_t prev_chunk_last,
                         BuildErr* be) {
    unsigned long long err = kNoErr, o = 0, a = ~0ULL;
    for (int64_t tile = t0 + blockIdx.x; tile < t1; tile += gridDim.x) {
        const int64_t b = tb[tile], e = tb[tile + 1];
        const int64_t cb = col_ptr[tseg[tile]];
        for (int64_t i = b + threadIdx.x; i < e; i += blockDim.x) {
            const int64_t r = rows64[i - chunk0];
            const int64_t prev = i == cb ? -1 : (i > chunk0 ? rows64[i - 1 - chunk0] : prev_chunk_last);
            uint32_t k = 0;
            if (r <= prev)
                err = min(err, (unsigned long long)i * 4 + 0);
            else if (r < 0 || r >= n)
                err = min(err, (unsigned long long)i * 4 + 1);
            else
                k = inv[r];
            key[i] = k;
            if (vidx) vidx[i] = (uint32_t)(i - cb);
            o |= k;
            a &= k;
        }
    }
    for (int q = 16; q; q >>= 1) {
        err = min(err, (unsigned long long)__shfl_xor_sync(0xffffffffu, (long long)err, q));
        o |= (unsigned long long)__shfl_xor_sync(0xffffffffu, (long long)o, q);
        a &= (unsigned long long)__shfl_xor_sync(0xffffffffu, (long long)a, q);
    }
    if ((threadIdx.x & 31) == 0) {
        if (err != kNoErr) atomicMin(&be->ent_err, err);
        atomicOr(&be->r_or, o);
        atomicAnd(&be->r_and, a);
    }
}

// value checks (finite) and the per-column "not all 1.0" flag
__global__ void k_b_vals(const double* vals, const int64_t* tb, int64_t ntiles, const int32_t* tseg,
                         uint32_t* nonunit, BuildErr* be) {
    unsigned long long err = kNoErr;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int64_t b = tb[tile], e = tb[tile + 1];
        bool nu = false;
        for (int64_t i = b + threadIdx.x; i < e; i += blockDim.x) {
            const double v = vals[i];
            if (!isfinite(v)) err = min(err, (unsigned long long)i * 4 + 2);
            nu |= v != 1.0;
        }
        if (__syncthreads_or(nu) && threadIdx.x == 0) nonunit[tseg[tile]] = 1;
    }
    for (int q = 16; q; q >>= 1)
        err = min(err, (unsigned long long)__shfl_xor_sync(0xffffffffu, (long long)err, q));
    if ((threadIdx.x & 31) == 0 && err != kNoErr) atomicMin(&be->ent_err, err);
}

// compacted values of the value columns, following their sorted rows
__global__ void k_b_vals_out(const uint32_t* vidx, const double* vals, const int64_t* tb,
                             int64_t ntiles, const int32_t* tseg, const int64_t* col_ptr,
                             const int64_t* val_off, double* vals_out) {
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int64_t b = tb[tile], e = tb[tile + 1];
        const int32_t j = tseg[tile];
        const int64_t cb = col_ptr[j], vo = val_off[j];
        if (vo < 0) continue;
        for (int64_t i = b + threadIdx.x; i < e; i += blockDim.x)
            vals_out[vo + (i - cb)] = vals[cb + vidx[i]];
    }
}

// ---------------------------------------------------------------- device lowering
// augment_to_strata (transforms.cpp:177-223) from the SUBJECT-level data: the
// host uploads the original (un-duplicated) subjects and the mapping subject x
// interval -> augmented row is evaluated here, so the duplicated design only
// ever exists in HBM ("mappings on the original data").
__device__ __forceinline__ int lw_event_interval(double y, const double* cuts, int K) {
    if (y == cuts[K]) return K;
    int lo = 0, hi = K + 1;  // upper_bound over cuts[0..K]
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (cuts[mid] <= y)
            lo = mid + 1;
        else
            hi = mid;
    }
    return lo;
}
__device__ __forceinline__ bool lw_at_risk(double y, uint8_t ev, int k, const double* cuts, int K) {
    if (y > cuts[k - 1]) return true;  // transforms.cpp:32-36
    return ev != 0 && y == cuts[k - 1] && lw_event_interval(y, cuts, K) == k;
}

// flag[(k-1) n + i] = subject i at risk in interval k (interval-major = output row order)
__global__ void k_lw_flags(const double* time, const uint8_t* event, int64_t n, const double* cuts,
                           int K, uint32_t* flag) {
    const int64_t m = (int64_t)K * n;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < m;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int k = (int)(t / n) + 1;
        const int64_t i = t - (int64_t)(k - 1) * n;
        flag[t] = lw_at_risk(time[i], event[i], k, cuts, K) ? 1u : 0u;
    }
}

// exclusive scan of m u32 values in place (1024 per block), block totals out
constexpr int kScanB = 1024;
__global__ void __launch_bounds__(kScanB) k_scan_blocks(uint32_t* v, int64_t m, uint32_t* tot) {
    __shared__ uint32_t ws[32];
    const int64_t i = (int64_t)blockIdx.x * kScanB + threadIdx.x;
    const uint32_t x = i < m ? v[i] : 0u;
    uint32_t inc = x;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
    }
    if (lane == 31) ws[w] = inc;
    __syncthreads();
    if (w == 0) {
        uint32_t t = ws[lane];
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, t, o);
            if (lane >= o) t += y;
        }
        ws[lane] = t;
    }
    __syncthreads();
    const uint32_t ex = inc - x + (w ? ws[w - 1] : 0u);
    if (i < m) v[i] = ex;
    if (threadIdx.x == kScanB - 1) tot[blockIdx.x] = ws[31];
}
// one block: exclusive scan of the block totals in chunks (carry between chunks)
__global__ void __launch_bounds__(kScanB) k_scan_tops(uint32_t* tot, int64_t nb, uint32_t* total) {
    __shared__ uint32_t ws[32];
    __shared__ uint32_t carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int64_t b0 = 0; b0 < nb; b0 += kScanB) {
        const int64_t i = b0 + threadIdx.x;
        const uint32_t x = i < nb ? tot[i] : 0u;
        uint32_t inc = x;
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += y;
        }
        if (lane == 31) ws[w] = inc;
        __syncthreads();
        if (w == 0) {
            uint32_t t = ws[lane];
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, t, o);
                if (lane >= o) t += y;
            }
            ws[lane] = t;
        }
        __syncthreads();
        const uint32_t c0 = carry;
        if (i < nb) tot[i] = c0 + inc - x + (w ? ws[w - 1] : 0u);
        __syncthreads();
        if (threadIdx.x == 0) carry = c0 + ws[31];
        __syncthreads();
    }
    if (threadIdx.x == 0) *total = carry;
}
__global__ void k_scan_add(uint32_t* v, int64_t m, const uint32_t* tot) {
    const int64_t i = (int64_t)blockIdx.x * kScanB + threadIdx.x;
    if (i < m) v[i] += tot[blockIdx.x];
}

// augmented rows (interval-major; subjects in input order inside an interval)
__global__ void k_lw_rows(const double* time, const uint8_t* event, const int64_t* subject,
                          int64_t n, const double* cuts, int K, const uint32_t* flag0,
                          const uint32_t* idx, double* a_time, uint8_t* a_event, int32_t* a_str,
                          int64_t* a_subj) {
    const int64_t m = (int64_t)K * n;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < m;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int k = (int)(t / n) + 1;
        const int64_t i = t - (int64_t)(k - 1) * n;
        const double y = time[i];
        if (!lw_at_risk(y, event[i], k, cuts, K)) continue;
        const uint32_t r = idx[t];
        a_time[r] = fmin(y, cuts[k]);
        a_event[r] = event[i] && lw_event_interval(y, cuts, K) == k ? 1 : 0;
        a_str[r] = k;
        a_subj[r] = subject ? subject[i] : i + 1;
    }
}

// per (output column c, interval k): the source column's entries whose subject
// is at risk in k (and value != 0), counted, then written in entry order
struct LwCol {
    int64_t beg, end;  // source entries
    double start, stop;
    int window;
    int pad;
};
__global__ void k_lw_count(const LwCol* cols, const int64_t* rows, const double* vals,
                           const uint32_t* flag0_unused, const double* cuts, int K, int64_t n,
                           const uint32_t* at_risk, uint32_t* cnt) {
    const int c = blockIdx.y, k = blockIdx.x + 1;
    const LwCol col = cols[c];
    uint32_t m = 0;
    if (col.window < 0 || (cuts[k - 1] >= col.start && cuts[k - 1] < col.stop))
        for (int64_t t = col.beg + threadIdx.x; t < col.end; t += blockDim.x) {
            const double v = vals ? vals[t] : 1.0;
            m += (v != 0.0 && at_risk[(int64_t)(k - 1) * n + rows[t]]) ? 1u : 0u;
        }
    for (int o = 16; o; o >>= 1) m += __shfl_xor_sync(0xffffffffu, m, o);
    __shared__ uint32_t ws[32];
    if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t a = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) a += ws[w];
        cnt[(int64_t)c * K + (k - 1)] = a;
    }
}
__global__ void __launch_bounds__(256) k_lw_fill(const LwCol* cols, const int64_t* rows,
                                                 const double* vals, const double* cuts, int K,
                                                 int64_t n, const uint32_t* at_risk,
                                                 const uint32_t* idx, const int64_t* off,
                                                 int64_t* out_rows, double* out_vals) {
    const int c = blockIdx.y, k = blockIdx.x + 1;
    const LwCol col = cols[c];
    if (!(col.window < 0 || (cuts[k - 1] >= col.start && cuts[k - 1] < col.stop))) return;
    __shared__ uint32_t ws[8];
    __shared__ int64_t base;
    if (threadIdx.x == 0) base = off[(int64_t)c * K + (k - 1)];
    __syncthreads();
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int64_t t0 = col.beg; t0 < col.end; t0 += 256) {
        const int64_t t = t0 + threadIdx.x;
        bool on = false;
        int64_t r = 0;
        double v = 1.0;
        if (t < col.end) {
            v = vals ? vals[t] : 1.0;
            const int64_t q = (int64_t)(k - 1) * n + rows[t];
            on = v != 0.0 && at_risk[q];
            if (on) r = idx[q];
        }
        const uint32_t bal = __ballot_sync(0xffffffffu, on);
        if (lane == 0) ws[w] = __popc(bal);
        __syncthreads();
        uint32_t before = 0, all = 0;
        for (int q = 0; q < 8; ++q) {
            before += q < w ? ws[q] : 0u;
            all += ws[q];
        }
        if (on) {
            const int64_t pos = base + before + __popc(bal & ((1u << lane) - 1u));
            out_rows[pos] = r;
            if (out_vals) out_vals[pos] = v;
        }
        __syncthreads();
        if (threadIdx.x == 0) base += all;
        __syncthreads();
    }
}

// ---------------------------------------------------------------- refresh layout (row slices)
// The 256-update refresh (likelihood.cpp:31-58) as a row-parallel pass: the
// design's entries re-sorted by row (stable, so a row's entries keep the
// ascending column order) and laid out in 32-row slices, so a warp reads 32
// rows' next entries with coalesced loads and every lane folds its own row in
// the reference's column order, without any synchronisation (k_refresh_ell in
// kernels.cu).
// Within a slice, entries come in groups of 4 per row: entry k of row l at
// base[s] + 128*(k/4) + 4l + k%4 (row lengths padded to a multiple of 4).
__global__ void k_iota_u32(uint32_t* v, int64_t m) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m;
         i += (int64_t)gridDim.x * blockDim.x)
        v[i] = (uint32_t)i;
}
// first sorted entry of each row (keys sorted ascending), rowptr[n] = nnz
__global__ void k_row_starts(const uint32_t* keys, int64_t nnz, int64_t n, int64_t* rowptr) {
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r <= n;
         r += (int64_t)gridDim.x * blockDim.x) {
        int64_t lo = 0, hi = nnz;
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if (keys[mid] < (uint32_t)r)
                lo = mid + 1;
            else
                hi = mid;
        }
        rowptr[r] = lo;
    }
}
// slice widths: max row length of each 32-row slice
__global__ void k_slice_width(const int64_t* rowptr, int64_t n, int64_t nsl, int32_t* width) {
    const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (w >= nsl) return;
    const int64_t r = w * 32 + lane;
    int len = r < n ? (int)(rowptr[r + 1] - rowptr[r]) : 0;
    for (int o = 16; o; o >>= 1) len = max(len, __shfl_xor_sync(0xffffffffu, len, o));
    if (lane == 0) width[w] = len;
}
template <typename IdT>
__global__ void k_fill_ids(IdT* v, int64_t m, IdT x) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m;
         i += (int64_t)gridDim.x * blockDim.x)
        v[i] = x;
}
template <typename IdT>
__global__ void k_ell_fill(const uint32_t* keys, const uint32_t* ent, int64_t nnz,
                           const int64_t* rowptr, const int64_t* base, const int64_t* col_beg,
                           int64_t p, const int64_t* val_off, const double* vals, IdT* ell_col,
                           double* ell_val) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nnz;
         i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t r = keys[i];
        const int64_t e = ent[i];
        int64_t lo = 0, hi = p;  // the column of entry e: col_beg[c] <= e < col_beg[c + 1]
        while (hi - lo > 1) {
            const int64_t mid = (lo + hi) >> 1;
            if (col_beg[mid] <= e)
                lo = mid;
            else
                hi = mid;
        }
        const int64_t k = i - rowptr[r];
        const int64_t pos = base[r >> 5] + (k >> 2) * 128 + (int64_t)(r & 31) * 4 + (k & 3);
        ell_col[pos] = (IdT)lo;
        if (ell_val) {
            const int64_t vo = val_off[lo];
            ell_val[pos] = vo < 0 ? 1.0 : vals[vo + (e - col_beg[lo])];
        }
    }
}

}  // namespace scx

// ---------------------------------------------------------------- host driver
using namespace scx;

namespace {

// Scratch of one build. With a stream, stream-ordered allocations from the
// device's memory pool, which keeps its memory across builds (release
// threshold raised once per device): a re-upload's multi-GB sort scratch
// costs no new page mappings.
struct DevBuf {
    std::vector<void*> ptrs;
    cudaStream_t st = nullptr;
    bool pooled = false;
    DevBuf() = default;
    explicit DevBuf(cudaStream_t s) : st(s), pooled(true) {
        int dev = 0;
        cudaGetDevice(&dev);
        static std::mutex mu;
        static bool done[64] = {};
        std::lock_guard<std::mutex> lk(mu);
        if (dev >= 0 && dev < 64 && !done[dev]) {
            cudaMemPool_t pool;
            if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
                uint64_t thr = UINT64_MAX;
                cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
            }
            done[dev] = true;
        }
    }
    template <typename T>
    cudaError_t alloc(T** p, size_t count) {
        const size_t bytes = std::max<size_t>(count, 1) * sizeof(T);
        cudaError_t e = pooled ? cudaMallocAsync((void**)p, bytes, st) : cudaMalloc((void**)p, bytes);
        if (e == cudaSuccess) ptrs.push_back(*p);
        return e;
    }
    void release(void* p) {
        auto it = std::find(ptrs.begin(), ptrs.end(), p);
        if (it != ptrs.end()) ptrs.erase(it);
    }
    ~DevBuf() {
        for (void* p : ptrs) {
            if (pooled)
                cudaFreeAsync(p, st);
            else
                cudaFree(p);
        }
    }
};

// tiles of <= kRxTile entries that never cross a segment boundary
void make_tiles(const std::vector<int64_t>& seg_ptr, std::vector<int64_t>& tb,
                std::vector<int32_t>& tseg, std::vector<int64_t>& st0) {
    const int64_t nseg = (int64_t)seg_ptr.size() - 1;
    tb.clear();
    tseg.clear();
    st0.assign(nseg + 1, 0);
    for (int64_t g = 0; g < nseg; ++g) {
        st0[g] = (int64_t)tseg.size();
        for (int64_t b = seg_ptr[g]; b < seg_ptr[g + 1]; b += kRxTile) {
            tb.push_back(b);
            tseg.push_back((int32_t)g);
        }
    }
    st0[nseg] = (int64_t)tseg.size();
    tb.push_back(seg_ptr[nseg]);
}

}  // namespace

// Implemented in capi.cu: upload of a design whose sorted arrays are already
// on the device (ownership of rows32_d / vals_d passes to the context).
scx_status scx_upload_device_design(scx_ctx* ctx, int64_t n, int32_t k, const int64_t* offsets_h,
                                    const uint8_t* event_d, const int64_t* tie_d, int64_t p,
                                    const int64_t* col_ptr_h, int32_t* rows32_d, double* vals_d,
                                    const std::vector<int64_t>& val_off, int64_t n_ind);
void scx_note_error(scx_ctx* ctx, const char* msg);
cudaStream_t scx_ctx_stream(scx_ctx* ctx);
int scx_ctx_device(scx_ctx* ctx);

#define BK(expr)                                                                   \
    do {                                                                           \
        cudaError_t e_ = (expr);                                                   \
        if (e_ != cudaSuccess) {                                                   \
            scx_note_error(ctx, (std::string("CUDA error in design build: ") +     \
                                 cudaGetErrorString(e_)).c_str());                 \
            return SCX_ERR_CUDA;                                                   \
        }                                                                          \
    } while (0)

static scx_status vfail(scx_ctx* ctx, const std::string& m) {
    scx_note_error(ctx, m.c_str());
    return SCX_ERR_VALIDATION;
}

// Input of the build: host arrays (scx_build_design) or device arrays (the
// device lowering, scx_build_lowered_design). col_ptr is always on the host.
struct BuildIn {
    int64_t n, p;
    const double* time;
    const uint8_t* event;
    const int32_t* stratum;
    const int64_t* col_ptr;
    const int64_t* rows;
    const double* values;  // NULL: every value 1.0
    bool device;           // time / event / stratum / rows / values are device pointers
};

static scx_status build_core(scx_ctx* ctx, const BuildIn& in, int64_t* perm_out);

extern "C" scx_status scx_build_design(scx_ctx* ctx, const scx_dataset* data, int64_t* perm_out) {
    if (!ctx || !data) return SCX_ERR_VALIDATION;
    const BuildIn in{data->n_rows, data->n_covariates, data->time, data->event, data->stratum,
                     data->col_ptr, data->row_idx, data->values, false};
    return build_core(ctx, in, perm_out);
}

static scx_status build_core(scx_ctx* ctx, const BuildIn& in, int64_t* perm_out) {
    BuildIn data = in;
    cudaSetDevice(scx_ctx_device(ctx));
    cudaStream_t s = scx_ctx_stream(ctx);
    const int64_t n = data.n, p = data.p;
    if (n == 0) return vfail(ctx, "dataset has no rows");
    if (n < 0 || p < 0) return vfail(ctx, "negative dataset size");
    if (n > (int64_t)0x7fffffff - kTileRows)
        return vfail(ctx, "row count exceeds the int32 row-index range");
    const int64_t* col_ptr = data.col_ptr;
    if (col_ptr[0] != 0) return vfail(ctx, "col_ptr[0] must be 0");
    for (int64_t j = 0; j < p; ++j)
        if (col_ptr[j + 1] < col_ptr[j]) return vfail(ctx, "col_ptr must be non-decreasing");
    const int64_t nnz = col_ptr[p];
    DevBuf B;

    // ---- rows: upload, label range, row checks, time keys
    double* time_d;
    uint8_t* event_d;
    int32_t* str_d;
    BuildErr* be;
    BK(B.alloc(&be, 1));
    if (data.device) {
        time_d = const_cast<double*>(data.time);
        event_d = const_cast<uint8_t*>(data.event);
        str_d = const_cast<int32_t*>(data.stratum);
    } else {
        BK(B.alloc(&time_d, n));
        BK(B.alloc(&event_d, n));
        BK(B.alloc(&str_d, n));
        BK(cudaMemcpyAsync(time_d, data.time, n * sizeof(double), cudaMemcpyHostToDevice, s));
        BK(cudaMemcpyAsync(event_d, data.event, n, cudaMemcpyHostToDevice, s));
        BK(cudaMemcpyAsync(str_d, data.stratum, n * sizeof(int32_t), cudaMemcpyHostToDevice, s));
    }
    {
        BuildErr init;
        std::memset(&init, 0, sizeof init);
        init.row_err = init.ent_err = kNoErr;
        init.t_and = init.k_and = init.r_and = ~0ULL;
        BK(cudaMemcpyAsync(be, &init, sizeof init, cudaMemcpyHostToDevice, s));
    }
    const int gr = grid_sms((n + 255) / 256);
    k_b_kmax<<<gr, 256, 0, s>>>(str_d, n, be);
    BuildErr h;
    BK(cudaMemcpyAsync(&h, be, sizeof h, cudaMemcpyDeviceToHost, s));
    BK(cudaStreamSynchronize(s));
    const int kmax = h.kmax;
    if (kmax < 1) return vfail(ctx, "dataset has no strata");  // data.cpp:32
    const int kcap = (int)std::min<int64_t>(kmax, n + 1);
    unsigned int* cnt_d;
    uint64_t *tkey, *tkey2;
    uint32_t *perm, *perm2;
    BK(B.alloc(&cnt_d, kcap));
    BK(B.alloc(&tkey, n));
    BK(B.alloc(&tkey2, n));
    BK(B.alloc(&perm, n));
    BK(B.alloc(&perm2, n));
    BK(cudaMemsetAsync(cnt_d, 0, kcap * sizeof(unsigned int), s));
    k_b_rows<<<gr, 256, 0, s>>>(time_d, event_d, str_d, n, kmax, kcap, be, cnt_d, tkey, perm);
    std::vector<unsigned int> cnt(kcap);
    BK(cudaMemcpyAsync(&h, be, sizeof h, cudaMemcpyDeviceToHost, s));
    BK(cudaMemcpyAsync(cnt.data(), cnt_d, kcap * sizeof(unsigned int), cudaMemcpyDeviceToHost, s));
    BK(cudaStreamSynchronize(s));
    if (h.row_err != kNoErr) {  // data.cpp:35-44
        const int64_t i = (int64_t)(h.row_err / 4);
        const int c = (int)(h.row_err % 4);
        const char* what = c == 0 ? "negative or non-finite time at row "
                           : c == 1 ? "event indicator must be 0 or 1 at row "
                                    : "stratum label out of range at row ";
        return vfail(ctx, what + std::to_string(i));
    }
    for (int q = 1; q <= kmax; ++q)  // data.cpp:46-49 (some q <= n + 1 is empty when kmax > n)
        if (q > kcap || cnt[q - 1] == 0)
            return vfail(ctx, "stratum " + std::to_string(q) + " has zero rows");
    const int32_t K = kmax;
    std::vector<int64_t> offsets(K + 1, 0);
    for (int q = 0; q < K; ++q) offsets[q + 1] = offsets[q] + cnt[q];

    // ---- row permutation: stable by ~time, then stable by stratum
    TileMap rows_tm;
    std::vector<int64_t> tb_h, st0_h;
    std::vector<int32_t> tseg_h;
    make_tiles({0, n}, tb_h, tseg_h, st0_h);
    const int64_t ntr = (int64_t)tseg_h.size();
    int64_t sbeg0 = 0;
    uint32_t *hist, *segtot;
    int64_t max_tiles = ntr;
    // column tiles (for the hist/segtot scratch size)
    std::vector<int64_t> ctb, cst0;
    std::vector<int32_t> ctseg;
    {
        std::vector<int64_t> sp(col_ptr, col_ptr + p + 1);
        make_tiles(sp, ctb, ctseg, cst0);
        max_tiles = std::max<int64_t>(max_tiles, (int64_t)ctseg.size());
    }
    BK(B.alloc(&hist, max_tiles * 256));
    BK(B.alloc(&segtot, std::max<int64_t>(1, p) * 256));
    BK(B.alloc(&rows_tm.tb, ntr + 1));
    BK(B.alloc(&rows_tm.tseg, ntr));
    BK(B.alloc(&rows_tm.st0, 2));
    BK(B.alloc(&rows_tm.sbeg, 1));
    BK(cudaMemcpyAsync(rows_tm.tb, tb_h.data(), (ntr + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, s));
    BK(cudaMemcpyAsync(rows_tm.tseg, tseg_h.data(), ntr * sizeof(int32_t), cudaMemcpyHostToDevice, s));
    BK(cudaMemcpyAsync(rows_tm.st0, st0_h.data(), 2 * sizeof(int64_t), cudaMemcpyHostToDevice, s));
    BK(cudaMemcpyAsync(rows_tm.sbeg, &sbeg0, sizeof(int64_t), cudaMemcpyHostToDevice, s));
    rows_tm.ntiles = ntr;
    rows_tm.nseg = 1;
    BK(radix_sort<uint64_t>(tkey, tkey2, perm, perm2, true, rows_tm, h.t_or ^ h.t_and, hist, segtot, s));
    uint32_t *skey, *skey2;
    BK(B.alloc(&skey, n));
    BK(B.alloc(&skey2, n));
    k_b_gather_str<<<gr, 256, 0, s>>>(perm, str_d, n, skey, be);
    BK(cudaMemcpyAsync(&h, be, sizeof h, cudaMemcpyDeviceToHost, s));
    BK(cudaStreamSynchronize(s));
    BK(radix_sort<uint32_t>(skey, skey2, perm, perm2, true, rows_tm, h.k_or ^ h.k_and, hist, segtot, s));

    // ---- sorted row arrays, tie ends
    uint32_t* inv;
    uint8_t* ev_s;
    int64_t* perm64;
    double* time_s;
    int32_t* str_s;
    int64_t* tie_d;
    BK(B.alloc(&inv, n));
    BK(B.alloc(&ev_s, n));
    BK(B.alloc(&perm64, n));
    BK(B.alloc(&time_s, n));
    BK(B.alloc(&str_s, n));
    BK(B.alloc(&tie_d, n));
    k_b_sorted<<<gr, 256, 0, s>>>(perm, time_d, event_d, str_d, n, inv, ev_s, perm64, time_s, str_s);
    const int64_t nb = (n + kTieBlock - 1) / kTieBlock;
    int64_t *bmin, *carry;
    BK(B.alloc(&bmin, nb));
    BK(B.alloc(&carry, nb));
    k_b_tie_blocks<<<(unsigned)nb, kTieBlock, 0, s>>>(time_s, str_s, n, bmin);
    k_b_tie_carry<<<1, 1024, 0, s>>>(bmin, nb, carry);
    k_b_tie_apply<<<(unsigned)nb, kTieBlock, 0, s>>>(time_s, str_s, n, carry, tie_d);
    if (perm_out)
        BK(cudaMemcpyAsync(perm_out, perm64, n * sizeof(int64_t), cudaMemcpyDeviceToHost, s));

    // ---- columns: staged H2D of the int64 rows (whole tiles per chunk),
    // checks, re-index; values: checks and indicator classification
    const int64_t nct = (int64_t)ctseg.size();
    TileMap col_tm;
    BK(B.alloc(&col_tm.tb, nct + 1));
    BK(B.alloc(&col_tm.tseg, std::max<int64_t>(nct, 1)));
    BK(B.alloc(&col_tm.st0, p + 1));
    BK(B.alloc(&col_tm.sbeg, std::max<int64_t>(p, 1)));
    int64_t* col_ptr_d;
    BK(B.alloc(&col_ptr_d, p + 1));
    BK(cudaMemcpyAsync(col_tm.tb, ctb.data(), (nct + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, s));
    if (nct)
        BK(cudaMemcpyAsync(col_tm.tseg, ctseg.data(), nct * sizeof(int32_t), cudaMemcpyHostToDevice, s));
    BK(cudaMemcpyAsync(col_tm.st0, cst0.data(), (p + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, s));
    BK(cudaMemcpyAsync(col_ptr_d, col_ptr, (p + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, s));
    if (p > 0)
        BK(cudaMemcpyAsync(col_tm.sbeg, col_ptr, p * sizeof(int64_t), cudaMemcpyHostToDevice, s));
    col_tm.ntiles = nct;
    col_tm.nseg = p;
    uint32_t *ckey, *ckey2, *vidx = nullptr, *vidx2 = nullptr;
    BK(B.alloc(&ckey, nnz + 16));  // +16: 16-B-aligned bulk copies of the rows may overhang
    BK(B.alloc(&ckey2, nnz + 16));
    const bool has_vals = data.values != nullptr;
    if (has_vals) {
        BK(B.alloc(&vidx, nnz));
        BK(B.alloc(&vidx2, nnz));
    }
    if (nnz > 0 && data.device) {  // device rows: one pass over every tile
        k_b_cols<<<grid_sms(nct), 256, 0, s>>>(data.rows, 0, col_tm.tb, 0, nct, col_tm.tseg, col_ptr_d,
                                              n, inv, ckey, vidx, -1, be);
    } else if (nnz > 0) {
        // chunks of whole tiles, about 64 Mi entries each
        const int64_t per = std::max<int64_t>(1, ((int64_t)1 << 26) / kRxTile);
        int64_t* stage;
        BK(B.alloc(&stage, std::min<int64_t>(nnz, per * kRxTile)));
        for (int64_t t0 = 0; t0 < nct; t0 += per) {
            const int64_t t1 = std::min(nct, t0 + per);
            const int64_t e0 = ctb[t0], e1 = ctb[t1];
            BK(cudaMemcpyAsync(stage, data.rows + e0, (e1 - e0) * sizeof(int64_t),
                               cudaMemcpyHostToDevice, s));
            const int64_t prev_last = e0 > 0 ? data.rows[e0 - 1] : -1;
            k_b_cols<<<grid_sms(t1 - t0), 256, 0, s>>>(stage, e0, col_tm.tb, t0, t1, col_tm.tseg,
                                                      col_ptr_d, n, inv, ckey, vidx, prev_last, be);
            BK(cudaStreamSynchronize(s));  // the stage is refilled next
        }
    }
    double* vals_in = nullptr;
    uint32_t* nonunit = nullptr;
    BK(B.alloc(&nonunit, std::max<int64_t>(p, 1)));
    BK(cudaMemsetAsync(nonunit, 0, std::max<int64_t>(p, 1) * sizeof(uint32_t), s));
    if (has_vals && nnz > 0) {
        if (data.device) {
            vals_in = const_cast<double*>(data.values);
        } else {
            BK(B.alloc(&vals_in, nnz));
            BK(cudaMemcpyAsync(vals_in, data.values, nnz * sizeof(double), cudaMemcpyHostToDevice, s));
        }
        k_b_vals<<<grid_sms(nct), 256, 0, s>>>(vals_in, col_tm.tb, nct, col_tm.tseg, nonunit, be);
    }
    BK(cudaMemcpyAsync(&h, be, sizeof h, cudaMemcpyDeviceToHost, s));
    std::vector<uint32_t> nonunit_h(std::max<int64_t>(p, 1));
    BK(cudaMemcpyAsync(nonunit_h.data(), nonunit, nonunit_h.size() * sizeof(uint32_t),
                       cudaMemcpyDeviceToHost, s));
    BK(cudaStreamSynchronize(s));
    if (h.ent_err != kNoErr) {  // data.cpp:55-64, first failing entry and check
        const int64_t i = (int64_t)(h.ent_err / 4);
        const int c = (int)(h.ent_err % 4);
        const int64_t j = std::upper_bound(col_ptr, col_ptr + p + 1, i) - col_ptr - 1;
        const std::string name = "x" + std::to_string(j + 1);
        return vfail(ctx, "column " + name +
                              (c == 0   ? " row indices must be strictly increasing"
                               : c == 1 ? " row index out of range"
                                        : " has a non-finite value"));
    }
    BK(radix_sort<uint32_t>(ckey, ckey2, vidx, vidx2, has_vals, col_tm, h.r_or ^ h.r_and, hist,
                            segtot, s));
    // indicator classification and value compaction (upload_common's rule)
    std::vector<int64_t> val_off(p, -1);
    int64_t n_ind = 0, nval = 0;
    for (int64_t j = 0; j < p; ++j) {
        if (has_vals && nonunit_h[j]) {
            val_off[j] = nval;
            nval += col_ptr[j + 1] - col_ptr[j];
        } else {
            ++n_ind;
        }
    }
    int64_t* val_off_d;
    BK(B.alloc(&val_off_d, std::max<int64_t>(p, 1)));
    if (p > 0)
        BK(cudaMemcpyAsync(val_off_d, val_off.data(), p * sizeof(int64_t), cudaMemcpyHostToDevice, s));
    int32_t* rows32 = reinterpret_cast<int32_t*>(ckey);  // sorted rows < 2^31: the int32 view
    double* vals_c;
    BK(B.alloc(&vals_c, nval + 16));
    if (nval > 0)
        k_b_vals_out<<<grid_sms(nct), 256, 0, s>>>(vidx, vals_in, col_tm.tb, nct, col_tm.tseg,
                                                  col_ptr_d, val_off_d, vals_c);
    BK(cudaGetLastError());
    BK(cudaStreamSynchronize(s));
    B.release(ckey);
    B.release(vals_c);
    return scx_upload_device_design(ctx, n, K, offsets.data(), ev_s, tie_d, p, col_ptr, rows32,
                                    vals_c, val_off, n_ind);
}


// ---------------------------------------------------------------- device lowering + build
extern "C" scx_status scx_build_lowered_design(scx_ctx* ctx, const scx_dataset* subjects,
                                               const double* cut_points, int64_t n_cuts,
                                               const int64_t* split_covariate,
                                               const int64_t* split_ptr, const double* split_times,
                                               int64_t n_splits, int64_t* perm_out,
                                               int64_t* map_source, int32_t* map_window,
                                               double* map_start, double* map_end) {
    if (!ctx || !subjects || !cut_points) return SCX_ERR_VALIDATION;
    std::vector<LowerCol> plan;
    std::string why;
    if (!lowering_plan(subjects, cut_points, n_cuts, split_covariate, split_ptr, split_times,
                       n_splits, plan, why))
        return vfail(ctx, why);
    cudaSetDevice(scx_ctx_device(ctx));
    cudaStream_t s = scx_ctx_stream(ctx);
    const int64_t n = subjects->n_rows, p = subjects->n_covariates;
    const int K = (int)n_cuts - 1;
    const int64_t* cp = subjects->col_ptr;
    const int64_t nnz = cp[p];
    const int64_t pc = (int64_t)plan.size();
    for (int64_t c = 0; c < pc; ++c) {
        if (map_source) map_source[c] = plan[c].src;
        if (map_window) map_window[c] = plan[c].window;
        if (map_start) map_start[c] = plan[c].start;
        if (map_end) map_end[c] = plan[c].end;
    }
    if ((int64_t)K * n >= ((int64_t)1 << 32))
        return vfail(ctx, "subjects x intervals exceeds the 32-bit row range");
    DevBuf B;
    // the subject-level (un-duplicated) data goes to the device once
    double *time_d, *cuts_d, *vals_d = nullptr;
    uint8_t* event_d;
    int64_t *subj_d = nullptr, *rows_d;
    BK(B.alloc(&time_d, n));
    BK(B.alloc(&event_d, n));
    BK(B.alloc(&cuts_d, n_cuts));
    BK(B.alloc(&rows_d, std::max<int64_t>(nnz, 1)));
    BK(cudaMemcpyAsync(time_d, subjects->time, n * sizeof(double), cudaMemcpyHostToDevice, s));
    BK(cudaMemcpyAsync(event_d, subjects->event, n, cudaMemcpyHostToDevice, s));
    BK(cudaMemcpyAsync(cuts_d, cut_points, n_cuts * sizeof(double), cudaMemcpyHostToDevice, s));
    if (nnz)
        BK(cudaMemcpyAsync(rows_d, subjects->row_idx, nnz * sizeof(int64_t), cudaMemcpyHostToDevice, s));
    if (subjects->subject) {
        BK(B.alloc(&subj_d, n));
        BK(cudaMemcpyAsync(subj_d, subjects->subject, n * sizeof(int64_t), cudaMemcpyHostToDevice, s));
    }
    if (subjects->values && nnz) {
        BK(B.alloc(&vals_d, nnz));
        BK(cudaMemcpyAsync(vals_d, subjects->values, nnz * sizeof(double), cudaMemcpyHostToDevice, s));
    }
    // mapping subject x interval -> augmented row: at-risk flags, exclusive scan
    const int64_t m = (int64_t)K * n;
    uint32_t *flag, *idx, *tot, *na_d;
    BK(B.alloc(&flag, m));
    BK(B.alloc(&idx, m));
    const int64_t nb = (m + kScanB - 1) / kScanB;
    BK(B.alloc(&tot, nb));
    BK(B.alloc(&na_d, 1));
    const int gm = grid_sms((m + 255) / 256);
    k_lw_flags<<<gm, 256, 0, s>>>(time_d, event_d, n, cuts_d, K, flag);
    BK(cudaMemcpyAsync(idx, flag, m * sizeof(uint32_t), cudaMemcpyDeviceToDevice, s));
    k_scan_blocks<<<(unsigned)nb, kScanB, 0, s>>>(idx, m, tot);
    k_scan_tops<<<1, kScanB, 0, s>>>(tot, nb, na_d);
    k_scan_add<<<(unsigned)nb, kScanB, 0, s>>>(idx, m, tot);
    uint32_t na = 0;
    BK(cudaMemcpyAsync(&na, na_d, sizeof na, cudaMemcpyDeviceToHost, s));
    BK(cudaStreamSynchronize(s));
    const int64_t N = na;
    if (N == 0) return vfail(ctx, "dataset has no rows");
    double* a_time;
    uint8_t* a_event;
    int32_t* a_str;
    int64_t* a_subj;
    BK(B.alloc(&a_time, N));
    BK(B.alloc(&a_event, N));
    BK(B.alloc(&a_str, N));
    BK(B.alloc(&a_subj, N));
    k_lw_rows<<<gm, 256, 0, s>>>(time_d, event_d, subj_d, n, cuts_d, K, flag, idx, a_time, a_event,
                                 a_str, a_subj);
    // the augmented columns: per (column, interval) counts -> offsets -> entries
    std::vector<LwCol> lc(pc);
    for (int64_t c = 0; c < pc; ++c)
        lc[c] = LwCol{cp[plan[c].src], cp[plan[c].src + 1], plan[c].start, plan[c].end,
                      plan[c].window, 0};
    LwCol* lc_d;
    uint32_t* cnt_d;
    BK(B.alloc(&lc_d, std::max<int64_t>(pc, 1)));
    BK(B.alloc(&cnt_d, std::max<int64_t>(pc * K, 1)));
    std::vector<int64_t> acp(pc + 1, 0);
    std::vector<int64_t> off(std::max<int64_t>(pc * K, 1), 0);
    if (pc > 0) {
        BK(cudaMemcpyAsync(lc_d, lc.data(), pc * sizeof(LwCol), cudaMemcpyHostToDevice, s));
        k_lw_count<<<dim3((unsigned)K, (unsigned)pc), 256, 0, s>>>(lc_d, rows_d, vals_d, nullptr, cuts_d,
                                                                  K, n, flag, cnt_d);
        std::vector<uint32_t> cnt(pc * K);
        BK(cudaMemcpyAsync(cnt.data(), cnt_d, pc * K * sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
        BK(cudaStreamSynchronize(s));
        for (int64_t c = 0; c < pc; ++c) {
            int64_t run = acp[c];
            for (int k = 0; k < K; ++k) {
                off[c * K + k] = run;
                run += cnt[c * K + k];
            }
            acp[c + 1] = run;
        }
    }
    const int64_t annz = acp[pc];
    int64_t *a_rows, *off_d;
    double* a_vals = nullptr;
    BK(B.alloc(&a_rows, std::max<int64_t>(annz, 1)));
    BK(B.alloc(&off_d, std::max<int64_t>(pc * K, 1)));
    if (vals_d) BK(B.alloc(&a_vals, std::max<int64_t>(annz, 1)));
    if (pc > 0) {
        BK(cudaMemcpyAsync(off_d, off.data(), pc * K * sizeof(int64_t), cudaMemcpyHostToDevice, s));
        k_lw_fill<<<dim3((unsigned)K, (unsigned)pc), 256, 0, s>>>(lc_d, rows_d, vals_d, cuts_d, K, n,
                                                                 flag, idx, off_d, a_rows, a_vals);
    }
    BK(cudaGetLastError());
    // ... and the device build of the augmented design (rows in input order)
    const BuildIn in{N, pc, a_time, a_event, a_str, acp.data(), a_rows, a_vals, true};
    return build_core(ctx, in, perm_out);
}


// ---------------------------------------------------------------- refresh layout builder
// Called at upload (capi.cu). Leaves d.ell_ok = 0 (the tile refresh stays in
// use) when the design is too large for the re-sort's scratch.
cudaError_t scx::build_refresh_ell(DesignDev& d, int64_t nnz, bool any_values, cudaStream_t s) {
    d.ell_ok = 0;
    const int64_t n = d.n, p = d.p;
    if (nnz <= 0 || p <= 0 || nnz >= ((int64_t)1 << 32)) return cudaSuccess;
    size_t free_b = 0, total_b = 0;
    cudaMemGetInfo(&free_b, &total_b);
    const size_t need = (size_t)nnz * (16 + 2 * 4 + (any_values ? 10 : 3)) + (size_t)n * 16;
    if (need > free_b / 2) return cudaSuccess;  // leave room for the fit's own scratch
    DevBuf B(s);
    uint32_t *keys, *keys2, *ent, *ent2;
    if (B.alloc(&keys, nnz) || B.alloc(&keys2, nnz) || B.alloc(&ent, nnz) || B.alloc(&ent2, nnz))
        return cudaGetLastError();
    cudaMemcpyAsync(keys, d.rows, nnz * sizeof(uint32_t), cudaMemcpyDeviceToDevice, s);
    k_iota_u32<<<grid_sms((nnz + 255) / 256), 256, 0, s>>>(ent, nnz);
    // stable radix by row (one segment): column order kept inside a row
    TileMap tm;
    std::vector<int64_t> tb_h, st0_h;
    std::vector<int32_t> tseg_h;
    make_tiles({0, nnz}, tb_h, tseg_h, st0_h);
    tm.ntiles = (int64_t)tseg_h.size();
    tm.nseg = 1;
    uint32_t *hist, *segtot;
    int64_t zero = 0;
    if (B.alloc(&hist, tm.ntiles * 256) || B.alloc(&segtot, 256) || B.alloc(&tm.tb, tm.ntiles + 1) ||
        B.alloc(&tm.tseg, tm.ntiles) || B.alloc(&tm.st0, 2) || B.alloc(&tm.sbeg, 1))
        return cudaGetLastError();
    cudaMemcpyAsync(tm.tb, tb_h.data(), (tm.ntiles + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, s);
    cudaMemcpyAsync(tm.tseg, tseg_h.data(), tm.ntiles * sizeof(int32_t), cudaMemcpyHostToDevice, s);
    cudaMemcpyAsync(tm.st0, st0_h.data(), 2 * sizeof(int64_t), cudaMemcpyHostToDevice, s);
    cudaMemcpyAsync(tm.sbeg, &zero, sizeof zero, cudaMemcpyHostToDevice, s);
    uint64_t varying = 0;
    for (int64_t v = n - 1; v > 0; v >>= 1) varying = (varying << 1) | 1;
    if (cudaError_t e = radix_sort<uint32_t>(keys, keys2, ent, ent2, true, tm, varying, hist, segtot, s))
        return e;
    int64_t* rowptr;
    const int64_t nsl = (n + 31) / 32;
    int32_t* width_d;
    if (B.alloc(&rowptr, n + 1) || B.alloc(&width_d, nsl)) return cudaGetLastError();
    k_row_starts<<<grid_sms((n + 256) / 256), 256, 0, s>>>(keys, nnz, n, rowptr);
    k_slice_width<<<(unsigned)((nsl * 32 + 255) / 256), 256, 0, s>>>(rowptr, n, nsl, width_d);
    std::vector<int32_t> width(nsl);
    cudaMemcpyAsync(width.data(), width_d, nsl * sizeof(int32_t), cudaMemcpyDeviceToHost, s);
    if (cudaError_t e = cudaStreamSynchronize(s)) return e;
    std::vector<int64_t> base(nsl + 1, 0);
    for (int64_t w = 0; w < nsl; ++w) base[w + 1] = base[w] + 32 * (((int64_t)width[w] + 3) & ~3LL);
    const int64_t cells = base[nsl];
    const bool wide = p >= 65535;  // u16 ids 0..p-1 plus the padding id p
    void* col = nullptr;
    double* val = nullptr;
    int64_t* base_d = nullptr;
    if (cudaMalloc(&col, std::max<int64_t>(cells, 1) * (wide ? 4 : 2)) != cudaSuccess) return cudaGetLastError();
    if (any_values && cudaMalloc((void**)&val, std::max<int64_t>(cells, 1) * sizeof(double)) != cudaSuccess) {
        cudaFree(col);
        return cudaGetLastError();
    }
    if (cudaMalloc((void**)&base_d, (nsl + 1) * sizeof(int64_t)) != cudaSuccess) {
        cudaFree(col);
        cudaFree(val);
        return cudaGetLastError();
    }
    // padding: column id p (beta_p reads as 0 in the refresh)
    if (wide)
        k_fill_ids<uint32_t><<<grid_sms((cells + 255) / 256), 256, 0, s>>>(static_cast<uint32_t*>(col), cells, (uint32_t)p);
    else
        k_fill_ids<uint16_t><<<grid_sms((cells + 255) / 256), 256, 0, s>>>(static_cast<uint16_t*>(col), cells, (uint16_t)p);
    cudaMemcpyAsync(base_d, base.data(), (nsl + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, s);
    const int g = grid_sms((nnz + 255) / 256);
    if (wide)
        k_ell_fill<uint32_t><<<g, 256, 0, s>>>(keys, ent, nnz, rowptr, base_d, d.col_beg, p, d.val_off,
                                               d.vals, static_cast<uint32_t*>(col), val);
    else
        k_ell_fill<uint16_t><<<g, 256, 0, s>>>(keys, ent, nnz, rowptr, base_d, d.col_beg, p, d.val_off,
                                               d.vals, static_cast<uint16_t*>(col), val);
    if (cudaError_t e = cudaStreamSynchronize(s)) {
        cudaFree(col);
        cudaFree(val);
        cudaFree(base_d);
        return e;
    }
    d.ell_col = col;
    d.ell_val = val;
    d.ell_base = base_d;
    d.ell_nsl = nsl;
    d.ell_wide = wide ? 1 : 0;
    d.ell_ok = 1;
    return cudaSuccess;
}
