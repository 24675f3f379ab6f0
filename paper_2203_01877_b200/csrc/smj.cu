// smj.cu -- generic many-to-many sort-merge join, Alg. 1 (
// prose :1114-1137) with readings R2 (ascending), R3 (bucketize right=True),
// R4 (div and remainder by rightHist), R5 (histograms over present keys), R6
// (output order key asc, left row asc, right row asc).
//
// Paper step -> kernel here:
//   l.2-3  sort both key columns with permutation       -> radix_sort (sort.cu); a
//          left side already in key order is not materialised (identity route)
//   l.4-8  bincount, histMul = L*R, cumsums              -> ONE bucket per sorted left
//          row instead of one per key: bucket i holds that row's R = rightBincount of
//          its key and startR = the key's first position among the sorted right keys
//          (bucket_r_kernel: a tile of sorted left keys stages its right key range in
//          shared memory and finds each key's [lower, upper) bound there). A key with
//          L left rows is L consecutive buckets of R outputs each, i.e. exactly its
//          L*R block of histMul in the same (l, r) order, so no run-length encoding,
//          no intersection and no compaction is needed (R = 0 buckets are empty);
//          cumHistMul = inclusive scan of R over the buckets (two passes: per-tile sums
//          with a 2^62 overflow guard, an add-scan, cum_write_kernel)
//   l.9    outSize = cumHistMul[-1]                       -> one 8-byte readback
//   l.10-14 arange, bucketize, in-bucket offset, div/rem -> expand_kernel: each CTA
//          owns a fixed output range, finds its first bucket with one
//          upper_bound (= bucketize right=True), and walks the buckets (the offset
//          inside bucket i is r directly: L = 1, q = 0).
#include "internal.h"

struct tqp_smj_plan {
    int64_t n_left = 0, n_right = 0, K = 0, out_size = 0;   // K = buckets = sorted left rows
    tqp::DevBuf<uint32_t> perm_l, perm_r;      // perm_l empty: the left side was already in key order
    tqp::DevBuf<uint32_t> mR, msR;             // per bucket: right count and right run start (< 2^30)
    tqp::DevBuf<int64_t> mcum;                 // cumHistMul (inclusive)
    tqp::DevBuf<uint32_t> tb;                  // per output tile of ETILE << tg_shift: bucket of its first output (+ sentinel)
    int tg_shift = 0;                          // > 0 when outSize is far larger than the keys (coarse table)
};

namespace tqp {

namespace {
constexpr int JNT = 256;
constexpr int JNW = JNT / 32;
#ifndef TQP_SMJ_JIPT
#define TQP_SMJ_JIPT 4
#endif
// left rows (buckets) per thread of the bucket / cumsum kernels; measured at SF10 (buckets +
// cumsum ms): 4 -> 0.166 + 0.070, 8 -> 0.195 + 0.073, 16 -> 0.270 + 0.105 (fewer searches per
// thread in flight matter less than more threads searching)
constexpr int JIPT = TQP_SMJ_JIPT;
static_assert(JIPT % 4 == 0, "16-byte stores");
constexpr int JTILE = JNT * JIPT;

constexpr uint32_t NOMATCH = 0xFFFFFFFFu;

// Left keys of the bucket kernel: the sort's internal keys (KL) or, for a left side
// already in key order, the caller's column converted on the fly; both mapped into the
// common key domain KO (hi | internal key).
struct LeftKeys {
    const void* p;
    int dt;           // 0 = internal KL keys; else the caller's column dtype (identity route)
    uint64_t hi;      // high bits of the internal keys (k32)
};

template <typename KL, typename KO>
__device__ __forceinline__ KO left_key(const LeftKeys& L, int64_t i) {
    if (L.dt == 0) return (KO)(L.hi | (uint64_t)__ldg((const KL*)L.p + i));
    return (KO)ordered_u64(load_as_i64(L.p, L.dt, i));
}

template <typename KR, typename KO>
__device__ __forceinline__ KO right_key(const KR* r, uint64_t hi, int64_t i) {
    return (KO)(hi | (uint64_t)__ldg(r + i));
}

// first index in [lo, hi) with key >= k (upper = false) or > k (upper = true)
template <typename KR, typename KO>
__device__ __forceinline__ int64_t bound_g(const KR* r, uint64_t hi_bits, int64_t lo, int64_t hi, KO k, bool upper) {
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        const KO v = right_key<KR, KO>(r, hi_bits, mid);
        if (upper ? v <= k : v < k) lo = mid + 1; else hi = mid;
    }
    return lo;
}

// Galloping search from lo: probe lo, lo + 1, lo + 3, lo + 7, ... then bisect the last
// gap. A sorted left tile's keys step through the right keys a few at a time (TPC-H: ~4
// lineitems per order), so a search costs a couple of probes instead of log2(range).
template <typename KR, typename KO>
__device__ __forceinline__ int64_t gallop_g(const KR* r, uint64_t hi_bits, int64_t lo, int64_t hi, KO k, bool upper) {
    int64_t step = 1, end = lo;
    while (end < hi) {
        const KO v = right_key<KR, KO>(r, hi_bits, end);
        if (!(upper ? v <= k : v < k)) break;
        lo = end + 1;
        end = lo + step;
        step <<= 1;
    }
    return bound_g<KR, KO>(r, hi_bits, lo, min(end, hi), k, upper);
}

// cumHistMul's input per bucket (= sorted left row b): R = count of right rows with the
// row's key, startR = their first sorted position. Tile of JTILE left rows, whose right
// key range comes from tile_rbounds_kernel; each thread takes JIPT consecutive rows,
// bisects the first key inside the tile's range, reuses the bounds for equal keys and
// gallops from the previous upper bound for a new key (measured: staging the tile's right
// range in shared memory held the kernel to 2 CTAs per SM, 0.29 ms at SF10; a merge path
// over the tile's left rows and right range, each thread walking its ~40 merged positions
// from global memory, 0.708 ms against 0.194 -- the per-thread walks are uncoalesced;
// with 1,024-row tiles, staging ranges of up to 2,048 / 4,096 right keys in shared memory
// and searching there: 0.193 / 0.187 ms against 0.175 from global memory).
// Per tile: the sum of R (saturated at 2^62; an fp64 running total flags larger outSize).
constexpr uint64_t SUM_CAP = 1ull << 62;

// Each tile's right key range [lower_bound(first left key), upper_bound(last left key)),
// every tile's two searches in parallel (one thread each): a search at the head of the
// bucket kernel itself put 2 x 26 dependent L2 round trips in front of every tile.
template <typename KL, typename KR, typename KO>
__global__ void tile_rbounds_kernel(LeftKeys lk, int64_t nl, const KR* __restrict__ rk, uint64_t rhi_bits, int64_t nr,
                                    int64_t tiles, int64_t* __restrict__ rb) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= 2 * tiles) return;
    const int64_t t = i >> 1;
    if (i & 1) rb[i] = bound_g<KR, KO>(rk, rhi_bits, 0, nr, left_key<KL, KO>(lk, min((t + 1) * JTILE, nl) - 1), true);
    else rb[i] = bound_g<KR, KO>(rk, rhi_bits, 0, nr, left_key<KL, KO>(lk, t * JTILE), false);
}

template <typename KL, typename KR, typename KO>
__global__ void __launch_bounds__(JNT) bucket_r_kernel(LeftKeys lk, int64_t nl, const KR* __restrict__ rk,
                                                       uint64_t rhi_bits, int64_t nr, const int64_t* __restrict__ rb,
                                                       uint32_t* __restrict__ mR,
                                                       uint32_t* __restrict__ msR, uint64_t* __restrict__ tsum,
                                                       double* dtot, int* overflow, int* unsorted) {
    __shared__ unsigned long long s_w[JNW];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t base = (int64_t)blockIdx.x * JTILE;
    const int64_t rlo = rb[2 * blockIdx.x], rhi = max(rb[2 * blockIdx.x + 1], rlo);
    const KO kfirst = left_key<KL, KO>(lk, base), klast = left_key<KL, KO>(lk, min(base + JTILE, nl) - 1);
    const int64_t r0 = base + (int64_t)tid * JIPT;
    uint64_t tot = 0;
    if (r0 < nl) {
        KO k[JIPT];
        if (r0 + JIPT <= nl && lk.dt == TQP_I64 && ((uintptr_t)lk.p & 15) == 0) {   // the caller's int64 column:
#pragma unroll                                                                      // 16-byte loads
            for (int q = 0; q < JIPT / 2; q++) {
                const longlong2 u = __ldg(reinterpret_cast<const longlong2*>((const long long*)lk.p + r0) + q);
                k[2 * q] = (KO)ordered_u64(u.x);
                k[2 * q + 1] = (KO)ordered_u64(u.y);
            }
        } else if (r0 + JIPT <= nl && lk.dt == 0 && sizeof(KL) == 4) {   // internal u32 keys
#pragma unroll
            for (int q = 0; q < JIPT / 4; q++) {
                const uint4 u = __ldg(reinterpret_cast<const uint4*>((const uint32_t*)lk.p + r0) + q);
                k[4 * q] = (KO)(lk.hi | u.x); k[4 * q + 1] = (KO)(lk.hi | u.y);
                k[4 * q + 2] = (KO)(lk.hi | u.z); k[4 * q + 3] = (KO)(lk.hi | u.w);
            }
        } else {
#pragma unroll
            for (int i = 0; i < JIPT; i++) k[i] = r0 + i < nl ? left_key<KL, KO>(lk, r0 + i) : KO(0);
        }
        if (unsorted) {   // speculative presorted left side (the caller's column, lk.dt != 0): verify
                          // the order of the full 64-bit keys, each adjacent pair once (a key outside
                          // [first, last] cannot pass as a truncated 32-bit key)
            bool bad = false;
            uint64_t up = ordered_u64(load_as_i64(lk.p, lk.dt, r0));
#pragma unroll
            for (int i = 1; i <= JIPT; i++) {
                if (r0 + i >= nl) break;
                const uint64_t u = ordered_u64(load_as_i64(lk.p, lk.dt, r0 + i));
                bad |= up > u;
                up = u;
            }
            if (bad) *unsorted = 1;
        }
        uint32_t R[JIPT], S[JIPT];
        int64_t lb = 0, ub = 0;
#pragma unroll
        for (int i = 0; i < JIPT; i++) {
            if (r0 + i >= nl) { R[i] = 0; S[i] = 0; continue; }
            if (i == 0) {   // the thread's first key: bisect the tile's right range (L1-resident top levels);
                            // the tile's first / last key has the range's own bounds (a heavy key
                            // spanning tiles costs no search at all)
                lb = k[0] == kfirst ? rlo : bound_g<KR, KO>(rk, rhi_bits, rlo, rhi, k[0], false);
                ub = k[0] == klast ? rhi : gallop_g<KR, KO>(rk, rhi_bits, lb, rhi, k[0], true);
            } else if (k[i] != k[i - 1]) {   // sorted: a new key's bounds lie at or after the previous upper
                lb = gallop_g<KR, KO>(rk, rhi_bits, ub, rhi, k[i], false);
                ub = gallop_g<KR, KO>(rk, rhi_bits, lb, rhi, k[i], true);
            }
            R[i] = (uint32_t)(ub - lb);
            S[i] = (uint32_t)lb;
            tot += R[i];
        }
        if (r0 + JIPT <= nl) {   // 16-byte stores
#pragma unroll
            for (int q = 0; q < JIPT / 4; q++) {
                reinterpret_cast<uint4*>(mR + r0)[q] = make_uint4(R[4 * q], R[4 * q + 1], R[4 * q + 2], R[4 * q + 3]);
                reinterpret_cast<uint4*>(msR + r0)[q] = make_uint4(S[4 * q], S[4 * q + 1], S[4 * q + 2], S[4 * q + 3]);
            }
        } else {
#pragma unroll
            for (int i = 0; i < JIPT; i++)
                if (r0 + i < nl) { mR[r0 + i] = R[i]; msR[r0 + i] = S[i]; }
        }
    }
    for (int o = 16; o > 0; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);   // <= 2^30 * 2048: no wrap
    if (lane == 0) s_w[warp] = tot;
    __syncthreads();
    if (tid == 0) {
        unsigned __int128 t = 0;
        for (int w = 0; w < JNW; w++) t += s_w[w];
        if (t >= SUM_CAP) {
            *overflow = 1;
            t = SUM_CAP - 1;
        }
        tsum[blockIdx.x] = (uint64_t)t;
        if (t) atomicAdd(dtot, (double)(uint64_t)t);
    }
}

// cumHistMul = inclusive scan of histMul = R over the buckets: per-tile sums from
// bucket_r_kernel, an exclusive 64-bit add-scan gives tile offsets, and cum_write_kernel
// writes cumHistMul and, in the same pass, the per-output-tile bucket table expand needs.
constexpr int64_t ETILE_C = 256 * 8;   // == ETILE (expand's outputs per CTA), defined below

__global__ void __launch_bounds__(JNT) cum_write_kernel(const uint32_t* __restrict__ mR, int64_t K,
                                                        const uint64_t* __restrict__ toff, int64_t* mcum, uint32_t* tb,
                                                        int64_t n_tb) {
    __shared__ uint64_t s_w[JNW];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t base = (int64_t)blockIdx.x * JTILE + (int64_t)tid * JIPT;
    if ((int64_t)blockIdx.x * JTILE >= K) return;
    uint64_t v[JIPT], t = 0;
    const bool fullv = base + JIPT <= K;   // whole rows: 16-byte loads / stores
    if (fullv) {
#pragma unroll
        for (int q = 0; q < JIPT / 4; q++) {
            const uint4 u = reinterpret_cast<const uint4*>(mR + base)[q];
            v[4 * q] = u.x; v[4 * q + 1] = u.y; v[4 * q + 2] = u.z; v[4 * q + 3] = u.w;
        }
    }
#pragma unroll
    for (int i = 0; i < JIPT; i++) {
        if (!fullv) v[i] = base + i < K ? (uint64_t)mR[base + i] : 0;
        t += v[i];
    }
    uint64_t x = t;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint64_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) s_w[warp] = x;
    __syncthreads();
    uint64_t run = toff[blockIdx.x] + x - t;
#pragma unroll
    for (int w = 0; w < JNW; w++)
        if (w < warp) run += s_w[w];
    if (fullv) {
        uint64_t c[JIPT];
        uint64_t r2 = run;
#pragma unroll
        for (int i = 0; i < JIPT; i++) { r2 += v[i]; c[i] = r2; }
#pragma unroll
        for (int q = 0; q < JIPT / 2; q++)
            reinterpret_cast<longlong2*>(mcum + base)[q] = make_longlong2((long long)c[2 * q], (long long)c[2 * q + 1]);
    }
#pragma unroll
    for (int i = 0; i < JIPT; i++) {
        const int64_t b = base + i;
        if (b >= K) break;
        const int64_t start = (int64_t)run;
        run += v[i];
        if (!fullv) mcum[b] = (int64_t)run;
        // output tiles whose first output falls inside this key's range [start, run)
        if (!tb) continue;   // coarse table: tb_search_kernel
        for (int64_t c = (start + ETILE_C - 1) / ETILE_C; c * ETILE_C < (int64_t)run; c++) tb[c] = (uint32_t)b;
        if (b == K - 1) tb[n_tb - 1] = (uint32_t)b;
    }
}

// Coarse tile-bucket table (outSize >> number of keys, e.g. both-Zipf joins): entry c is
// the bucket of output c * TG, found by a binary search over cumHistMul (one thread per
// entry; the filling loop of cum_write_kernel would spend one thread per heavy key).
__global__ void tb_search_kernel(const int64_t* __restrict__ mcum, int64_t K, int tg_shift_total, uint32_t* tb,
                                 int64_t n_tb) {
    for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < n_tb; c += (int64_t)gridDim.x * blockDim.x) {
        if (c == n_tb - 1) {
            tb[c] = (uint32_t)(K - 1);
            continue;
        }
        const int64_t x = c << tg_shift_total;
        int64_t lo = 0, hi = K - 1;   // first b with mcum[b] > x (mcum[K-1] = outSize > x)
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if (mcum[mid] > x) hi = mid; else lo = mid + 1;
        }
        tb[c] = (uint32_t)lo;
    }
}

// Warp-cooperative search: the first b in [lo, hi] with mcum[b] > x, given mcum[hi] > x
// (32 probes per step).
__device__ __forceinline__ int64_t warp_upper(const int64_t* __restrict__ mcum, int64_t lo, int64_t hi, int64_t x) {
    const int lane = threadIdx.x & 31;
    while (lo < hi) {
        const int64_t step = (hi - lo + 32) / 32;
        const int64_t idx = min(lo + lane * step, hi);
        const unsigned bal = __ballot_sync(0xffffffffu, mcum[idx] > x);
        if (bal == 0) {
            lo = min(lo + 31 * step, hi) + 1;
        } else {
            const int f = __ffs(bal) - 1;
            const int64_t nhi = min(lo + f * step, hi);
            lo = f == 0 ? lo : min(lo + (f - 1) * step, hi) + 1;
            hi = nhi;
        }
    }
    return lo;
}

constexpr int ENT = 256;
constexpr int EIPT = 8;
constexpr int ETILE = ENT * EIPT;
static_assert(ETILE == ETILE_C, "cum_write_kernel's tile-bucket table uses expand's tile size");


// Output offsets [begin, end): bucket b = upper_bound(cumHistMul, o) (bucketize
// right=True); o' = o - (cumHistMul[b] - histMul[b]); q = o' / R, r = o' % R;
// left = leftIdx[startL + q], right = rightIdx[startR + r]. The CTA's candidate
// buckets come from the tile-bucket table (two loads); their cumulative ends,
// clamped to the CTA's output window, are staged in shared memory where every
// thread finds its first bucket.
// Fused consumer (tqp_smj_expand_checksum): h_j = mix64(mix64((left << 32) | right) ^ j)
// over output positions j, summed mod 2^64 with the left and right indices.
__device__ __forceinline__ uint64_t mix64(uint64_t x) {
    x ^= x >> 30;
    x *= 0xbf58476d1ce4e5b9ull;
    x ^= x >> 27;
    x *= 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}

constexpr int CK_SLOTS = 1024;
__global__ void ck_final_kernel(const unsigned long long* __restrict__ slots, unsigned long long* out) {
    __shared__ unsigned long long s[3][32];
    uint64_t v[3] = {0, 0, 0};
    for (int i = threadIdx.x; i < CK_SLOTS; i += blockDim.x)
        for (int k = 0; k < 3; k++) v[k] += slots[3 * i + k];
    for (int k = 0; k < 3; k++) {
        for (int o = 16; o > 0; o >>= 1) v[k] += __shfl_xor_sync(0xffffffffu, v[k], o);
        if ((threadIdx.x & 31) == 0) s[k][threadIdx.x >> 5] = v[k];
    }
    __syncthreads();
    if (threadIdx.x < 3) {
        uint64_t t = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); w++) t += s[threadIdx.x][w];
        out[threadIdx.x] = t;
    }
}

// createOutput fused into the expansion (Alg. 1's return; SURVEY §8(f) NEXT
// 2): payload columns gathered by the pairs' left / right rows as they are written.
constexpr int SMJ_MAXPAY = 8;
struct SmjPayload {
    int nl, nr;
    const void* lsrc[SMJ_MAXPAY];
    int ldt[SMJ_MAXPAY];
    void* ldst[SMJ_MAXPAY];
    const void* rsrc[SMJ_MAXPAY];
    int rdt[SMJ_MAXPAY];
    void* rdst[SMJ_MAXPAY];
};

__device__ __forceinline__ void pay_copy(const void* src, int dt, int64_t from, void* dst, int64_t to) {
    switch (dt) {
        case TQP_U8: static_cast<uint8_t*>(dst)[to] = __ldg(static_cast<const uint8_t*>(src) + from); break;
        case TQP_I32: __stcs(static_cast<int*>(dst) + to, __ldg(static_cast<const int*>(src) + from)); break;
        default: __stcs(static_cast<long long*>(dst) + to, __ldg(static_cast<const long long*>(src) + from));
    }
}

// Occupancy: the staged bucket ends (CCAP, more: searches in global memory) and the blocks
// per SM the register budget must allow (sparse buckets -- more than ~700 per output tile,
// e.g. Zipf x uniform where most left rows have no partner -- take CC = 4098 at 4 blocks/SM). Measured, SF10 expansion: CCAP 4098 (40 KB of
// shared memory, 4 blocks/SM) 0.367 ms; CCAP 1025 (28 KB) 0.326 ms; + 6 blocks/SM (40
// registers, 16 bytes of spills) 0.301 ms; 7 / 8 blocks 0.299 / 0.299. (r01, before the
// per-row buckets: 4/5/6/8 blocks 0.435/0.443/0.439/0.494 ms.)
// (r02, with the coalesced gather and stores: 6 -> 7 blocks per SM, 0.271 -> 0.265 ms)
#ifndef TQP_EXPAND_MINB
#define TQP_EXPAND_MINB 7
#endif
#ifndef TQP_EXPAND_CCAP
#define TQP_EXPAND_CCAP 1025
#endif
// Bucket-major fill: 1 = the threads write each output's sorted right position, then the
// CTA gathers perm_r for consecutive outputs (warp-coalesced: consecutive buckets own
// consecutive sorted right rows); 0 = each thread gathers its own buckets' rows.
// Measured (SF10 orders x lineitem expansion): 0.273 -> 0.256 ms.
#ifndef TQP_EXPAND_COOP
#define TQP_EXPAND_COOP 1
#endif
template <bool CK, bool PAY = false, int CC = TQP_EXPAND_CCAP>
__global__ void __launch_bounds__(ENT, CC <= 1025 ? TQP_EXPAND_MINB : 4) expand_kernel(const uint32_t* __restrict__ mR,
                                                     const uint32_t* __restrict__ msR,
                                                     const int64_t* __restrict__ mcum, int64_t K,
                                                     const uint32_t* __restrict__ tb,
                                                     const uint32_t* __restrict__ perm_l,
                                                     const uint32_t* __restrict__ perm_r, int64_t begin, int64_t end,
                                                     void* __restrict__ lo_out, void* __restrict__ ro_out, int idx32,
                                                     unsigned long long* __restrict__ ck, int tg_shift,
                                                     SmjPayload pay) {
    // shared memory: the staged bucket ends (when the CTA spans <= CCAP buckets), plus
    // (when it spans <= MCAP) the buckets' (R, startR) so that walking across buckets
    // needs no global loads. Empty buckets (R = 0: left rows without a partner) make the
    // span unbounded, so both are optional and searches fall back to global memory.
    constexpr int MCAP = 1024, CCAP = CC;
    __shared__ __align__(16) int32_t s_cum[CCAP];
    __shared__ __align__(16) uint32_t s_m[2 * MCAP];
    __shared__ __align__(16) uint32_t s_l[ETILE], s_r[ETILE];
    const int64_t c0 = begin + (int64_t)blockIdx.x * ETILE;
    const int64_t c1 = min(c0 + ETILE, end);
    TQP_DCHECK(c0 < c1);
    // buckets of outputs c0 and c1 - 1 lie in [b0, b1]: at most two output tiles' worth
    int64_t b0, b1;
    if (tg_shift == 0) {
        b0 = tb[c0 / ETILE];
        b1 = min((int64_t)tb[(c1 - 1) / ETILE + 1], K - 1);
    } else {   // coarse table: narrow [tb[c0 / TG], tb[(c1 - 1) / TG + 1]] to this CTA's buckets
        __shared__ int64_t s_b[2];
        if (threadIdx.x < 32) {
            const int64_t lo = tb[(c0 / ETILE) >> tg_shift];
            const int64_t hi = min((int64_t)tb[(((c1 - 1) / ETILE) >> tg_shift) + 1], K - 1);
            const int64_t x0 = warp_upper(mcum, lo, hi, c0);
            const int64_t x1 = warp_upper(mcum, x0, hi, c1 - 1);
            if (threadIdx.x == 0) { s_b[0] = x0; s_b[1] = x1; }
        }
        __syncthreads();
        b0 = s_b[0];
        b1 = s_b[1];
    }
    const int64_t nb = b1 - b0 + 1;
    const bool meta = nb <= MCAP, cst = nb <= CCAP;
    for (int i = threadIdx.x; cst && i < nb; i += ENT) {
        const int64_t v = mcum[b0 + i] - c0;
        s_cum[i] = (int32_t)(v < 0 ? -1 : (v > ETILE ? ETILE + 1 : v));
        if (meta) {
            s_m[i] = mR[b0 + i];
            s_m[MCAP + i] = msR[b0 + i];
        }
    }
    __syncthreads();
    // first bucket index i >= lo (relative to b0) whose cumulative end exceeds output o
    // (bucketize right=True; empty buckets are skipped because their end equals the next's start)
    auto find = [&](int64_t o, int64_t lo) {
        int64_t hi = nb;
        if (cst) {
            const int32_t rel = (int32_t)(o - c0);
            while (lo < hi) {
                const int64_t mid = (lo + hi) >> 1;
                if (s_cum[mid] <= rel) lo = mid + 1; else hi = mid;
            }
        } else {
            while (lo < hi) {
                const int64_t mid = (lo + hi) >> 1;
                if (mcum[b0 + mid] <= o) lo = mid + 1; else hi = mid;
            }
        }
        return lo;
    };
    const int64_t o0 = c0 + (int64_t)threadIdx.x * EIPT;
    uint64_t hs = 0, sl = 0, sr = 0;   // CK: this thread's share of the consumer sums
    const int n_out = (int)(c1 - c0);
    // Bucket-major when the tile's buckets are many and small (<= 16 outputs on average,
    // e.g. a PK-FK-shaped join: ~4 lineitems per order): a thread takes whole buckets and
    // fills their outputs in the staging buffer -- a gather and two shared stores per
    // output instead of the per-output bucket walk. Few large buckets (skew) keep the
    // output-major walk, which balances by output.
    const bool bmajor = meta && cst && nb * 16 >= n_out;   // (unstaged sparse buckets measured slower: 1.15 -> 1.91 ms, Zipf x uniform)
    if (bmajor) {
        // end of bucket i relative to the tile, unclamped below (-1 / negative: before the tile)
        auto rend = [&](int64_t i) -> int64_t { return cst ? (int64_t)s_cum[i] : mcum[b0 + i] - c0; };
        for (int64_t i = threadIdx.x; i < nb; i += ENT) {
            const int64_t pe = i == 0 ? -1 : rend(i - 1);
            const int st = (int)min(max(pe, (int64_t)0), (int64_t)n_out);
            const int en = (int)min(max(rend(i), (int64_t)0), (int64_t)n_out);
            if (st >= en) continue;
            const int64_t b = b0 + i;
            const uint32_t R = meta ? s_m[i] : mR[b], sR = meta ? s_m[MCAP + i] : msR[b];
            // offset of the tile's first output of this bucket inside the bucket: 0 unless the
            // bucket started before the tile (only the first non-empty bucket)
            const int64_t r0 = (i > 0 && pe >= 0) ? 0 : c0 - (mcum[b] - (int64_t)R);
            TQP_DCHECK(r0 >= 0 && r0 + (en - st) <= (int64_t)R);
            const uint32_t lrow = perm_l ? __ldg(perm_l + b) : (uint32_t)b;
            if (TQP_EXPAND_COOP) {   // the right row's sorted position; gathered below, warp-coalesced
                const uint32_t q0 = sR + (uint32_t)r0;
                for (int p = st; p < en; p++) {
                    s_l[p] = lrow;
                    s_r[p] = q0 + (uint32_t)(p - st);
                }
            } else {
                const uint32_t* pr = perm_r + sR + r0;
                for (int p = st; p < en; p++) {
                    s_l[p] = lrow;
                    s_r[p] = __ldg(pr + (p - st));
                }
            }
        }
        if (TQP_EXPAND_COOP) {   // consecutive outputs of consecutive buckets: consecutive sorted right rows
            __syncthreads();
            for (int o = threadIdx.x; o < n_out; o += ENT) s_r[o] = __ldg(perm_r + s_r[o]);
        }
        if (CK) {
            __syncthreads();
            for (int o = threadIdx.x; o < n_out; o += ENT) {
                const uint32_t l = s_l[o], r = s_r[o];
                hs += mix64(mix64(((uint64_t)l << 32) | r) ^ (uint64_t)(c0 + o));
                sl += l;
                sr += r;
            }
        }
    } else if (o0 < c1) {   // thread: EIPT consecutive outputs, incremental offset inside the bucket
        int64_t bi = find(o0, 0);   // bucket index relative to b0 (bucket = sorted left row b0 + bi)
        TQP_DCHECK(bi < nb && b0 + bi < K);
        auto load = [&](int64_t i, int64_t& R, int64_t& sR) {
            if (meta) {
                R = s_m[i]; sR = s_m[MCAP + i];
            } else {
                R = mR[b0 + i]; sR = msR[b0 + i];
            }
        };
        int64_t R, sR;
        load(bi, R, sR);
        // o' = o - (cumHistMul[b] - histMul[b]); with L = 1 per bucket, q = 0 and r = o'
        int64_t r = o0 - (mcum[b0 + bi] - R);
        const int cnt = (int)min((int64_t)EIPT, c1 - o0);
        uint32_t vl[EIPT], vr[EIPT];
        int64_t b = b0 + bi;
        uint32_t lrow = perm_l ? __ldg(perm_l + b) : (uint32_t)b;
#pragma unroll
        for (int j = 0; j < EIPT; j++) {
            if (j >= cnt) break;
            TQP_DCHECK(r < R);
            vl[j] = lrow;
            // (COOP, stored outputs: the sorted right position, gathered below warp-coalesced)
            vr[j] = (TQP_EXPAND_COOP && !CK) ? (uint32_t)(sR + r) : __ldg(perm_r + sR + r);
            if (CK) {
                hs += mix64(mix64(((uint64_t)vl[j] << 32) | vr[j]) ^ (uint64_t)(o0 + j));
                sl += vl[j];
                sr += vr[j];
            }
            if (++r == R && j + 1 < cnt) {   // next non-empty bucket: the next one, else a search
                r = 0;
                load(++bi, R, sR);
                if (R == 0) {
                    bi = find(o0 + j + 1, bi + 1);
                    load(bi, R, sR);
                }
                TQP_DCHECK(bi < nb && R > 0);
                b = b0 + bi;
                lrow = perm_l ? __ldg(perm_l + b) : (uint32_t)b;
            }
        }
        const int o = threadIdx.x * EIPT;
        if (CK) {
        } else if (cnt == EIPT) {   // 16-byte shared stores
            reinterpret_cast<uint4*>(s_l + o)[0] = make_uint4(vl[0], vl[1], vl[2], vl[3]);
            reinterpret_cast<uint4*>(s_l + o)[1] = make_uint4(vl[4], vl[5], vl[6], vl[7]);
            reinterpret_cast<uint4*>(s_r + o)[0] = make_uint4(vr[0], vr[1], vr[2], vr[3]);
            reinterpret_cast<uint4*>(s_r + o)[1] = make_uint4(vr[4], vr[5], vr[6], vr[7]);
        } else {
#pragma unroll
            for (int j = 0; j < EIPT; j++)
                if (j < cnt) { s_l[o + j] = vl[j]; s_r[o + j] = vr[j]; }
        }
    }
    if (CK) {   // CTA sums -> one of CK_SLOTS partial slots (mod 2^64; spread so that
                // same-address atomics do not serialise), summed by ck_final_kernel
        __shared__ unsigned long long s_ck[3];
        if (threadIdx.x < 3) s_ck[threadIdx.x] = 0;
        __syncthreads();
#pragma unroll
        for (int sh = 16; sh > 0; sh >>= 1) {
            hs += __shfl_xor_sync(0xffffffffu, hs, sh);
            sl += __shfl_xor_sync(0xffffffffu, sl, sh);
            sr += __shfl_xor_sync(0xffffffffu, sr, sh);
        }
        if ((threadIdx.x & 31) == 0) {
            atomicAdd(&s_ck[0], (unsigned long long)hs);
            atomicAdd(&s_ck[1], (unsigned long long)sl);
            atomicAdd(&s_ck[2], (unsigned long long)sr);
        }
        __syncthreads();
        if (threadIdx.x < 3) atomicAdd(ck + 3 * (blockIdx.x % CK_SLOTS) + threadIdx.x, s_ck[threadIdx.x]);
        return;
    }
    __syncthreads();
    const int n = (int)(c1 - c0);
    if (TQP_EXPAND_COOP && !bmajor) {   // output-major staging holds sorted right positions
        for (int o = threadIdx.x; o < n; o += ENT) s_r[o] = __ldg(perm_r + s_r[o]);
        __syncthreads();
    }
    if (PAY) {   // index outputs optional; payload gathered per output, coalesced stores
        for (int o = threadIdx.x; o < n; o += ENT) {
            const int64_t j = c0 - begin + o;
            const uint32_t l = s_l[o], r = s_r[o];
            if (lo_out) __stcs((long long*)lo_out + j, (long long)l);
            if (ro_out) __stcs((long long*)ro_out + j, (long long)r);
            for (int c = 0; c < pay.nl; c++) pay_copy(pay.lsrc[c], pay.ldt[c], l, pay.ldst[c], j);
            for (int c = 0; c < pay.nr; c++) pay_copy(pay.rsrc[c], pay.rdt[c], r, pay.rdst[c], j);
        }
        return;
    }
    if (idx32) {   // int32 indices (tqp_smj_expand_i32)
        int* lo32 = (int*)lo_out + (c0 - begin);
        int* ro32 = (int*)ro_out + (c0 - begin);
        if (n == ETILE && (((uintptr_t)lo32 | (uintptr_t)ro32) & 15) == 0) {
            for (int o = threadIdx.x * 4; o < n; o += ENT * 4) {
                __stcs(reinterpret_cast<int4*>(lo32 + o), *reinterpret_cast<const int4*>(s_l + o));
                __stcs(reinterpret_cast<int4*>(ro32 + o), *reinterpret_cast<const int4*>(s_r + o));
            }
        } else {
            for (int o = threadIdx.x; o < n; o += ENT) {
                __stcs(lo32 + o, (int)s_l[o]);
                __stcs(ro32 + o, (int)s_r[o]);
            }
        }
        return;
    }
    int64_t* lo_p = (int64_t*)lo_out + (c0 - begin);
    int64_t* ro_p = (int64_t*)ro_out + (c0 - begin);
    const bool vec = n == ETILE && (((uintptr_t)lo_p | (uintptr_t)ro_p) & 15) == 0;
    if (vec) {   // 2 outputs per thread and store: every warp store covers 512 contiguous bytes
        for (int o = threadIdx.x * 2; o < n; o += ENT * 2) {
            const uint2 a = *reinterpret_cast<const uint2*>(s_l + o);
            const uint2 b = *reinterpret_cast<const uint2*>(s_r + o);
            __stcs(reinterpret_cast<longlong2*>(lo_p + o), make_longlong2(a.x, a.y));
            __stcs(reinterpret_cast<longlong2*>(ro_p + o), make_longlong2(b.x, b.y));
        }
    } else {
        for (int o = threadIdx.x; o < n; o += ENT) {   // coalesced, streamed (evict-first) stores
            __stcs((long long*)lo_p + o, (long long)s_l[o]);
            __stcs((long long*)ro_p + o, (long long)s_r[o]);
        }
    }
}

template <typename KL, typename KR, typename KO>
void launch_buckets(tqp_ctx* ctx, const LeftKeys& lk, int64_t nl, const KR* rk, uint64_t rhi, int64_t nr,
                    tqp_smj_plan* P, uint64_t* tsum, int64_t tiles, int64_t* scal, bool verify) {
    DevBuf<int64_t> rb(ctx, 2 * tiles);
    launch(ctx, "tqp_smj_bounds", tile_rbounds_kernel<KL, KR, KO>, dim3((unsigned)ceil_div(2 * tiles, 128)), dim3(128),
           0, lk, nl, rk, rhi, nr, tiles, rb.get());
    launch(ctx, "tqp_smj_buckets", bucket_r_kernel<KL, KR, KO>, dim3((unsigned)tiles), dim3(JNT), 0, lk, nl, rk, rhi, nr,
           (const int64_t*)rb.get(), P->mR.get(), P->msR.get(), tsum, (double*)(scal + 5), (int*)(scal + 4),
           verify ? (int*)(scal + 2) : (int*)nullptr);
}
}  // namespace

// spec: take a left side whose first / last / sampled keys are in order as sorted without
// the plan pass over it (primary-key columns are usually stored in key order); the bucket
// kernel, which reads every left key anyway, verifies the order and a left side that is
// not sorted after all is prepared again the ordinary way (returns nullptr).
static tqp_smj_plan* smj_prepare_impl(tqp_ctx* ctx, tqp_col left, int64_t nl, tqp_col right, int64_t nr,
                                      int64_t* out_size_host, bool spec) {
    auto* P = new tqp_smj_plan();
    try {
        P->n_left = nl;
        P->n_right = nr;
        if (nl == 0 || nr == 0) {
            *out_size_host = 0;
            return P;
        }
        // sort both sides (l.2-3); keep the internal sorted keys and u32 permutations
        SortOut sl, sr;
        sl.want_internal = sr.want_internal = true;
        sl.defer_identity = true;   // a left side in key order is read as it is (no identity pass)
        bool verify = false;   // the left side was taken as sorted on a sample: the bucket kernel checks it
        {   // both digit plans with one host sync
            constexpr int W = SORT_PLAN_WORDS;
            DevBuf<unsigned long long> ao(ctx, 2 * W);
            DevBuf<uint32_t> hl, hr(ctx, sort_hist0_words(nr));
            if (spec) sample_first_last(ctx, left.data, left.dtype, nl, ao.get());
            else {
                hl.alloc(ctx, sort_hist0_words(nl));
                sort_andor(ctx, left.data, left.dtype, nl, false, ao.get(), hl.get());
            }
            sort_andor(ctx, right.data, right.dtype, nr, false, ao.get() + W, hr.get());
            uint64_t h[2 * W];
            read_back(ctx, h, ao.get(), 16 * W);
            if (spec && h[2]) {   // the sample is out of order: the left side's own plan pass
                hl.alloc(ctx, sort_hist0_words(nl));
                sort_andor(ctx, left.data, left.dtype, nl, false, ao.get(), hl.get());
                read_back(ctx, h, ao.get(), 8 * W);
            } else if (spec) {   // plan words of a side in key order: its keys lie in [first, last]
                const uint64_t first = h[0], last = h[1];
                h[0] = first;    // AND / OR stand-ins whose XOR has a high word iff the keys' high words differ
                h[1] = last;
                h[2] = 0;
                h[3] = first;
                h[4] = last;
                verify = true;
            }
            radix_sort(ctx, left.data, left.dtype, nl, false, sl, h, hl.get());
            radix_sort(ctx, right.data, right.dtype, nr, false, sr, h + W, hr.get());
        }
        const bool lid = sl.identity;   // left already in key order: read the caller's keys, perm = identity
        if (!lid) P->perm_l = std::move(sl.perm32);
        P->perm_r = std::move(sr.perm32);
        DevBuf<int64_t> scal(ctx, 6);   // [3] out_size, [4] overflow flag, [5] fp64 total: one readback
        scal.zero();
        P->K = nl;
        P->mR.alloc(ctx, nl);
        P->msR.alloc(ctx, nl);
        P->mcum.alloc(ctx, nl);
        // common key domain: 32-bit when both sides vary only in one common low word
        const bool k32 = sl.k32 && sr.k32 && (sl.and_bits >> 32) == (sr.and_bits >> 32);
        LeftKeys lk{};
        if (lid) {
            lk.p = left.data;
            lk.dt = left.dtype;
        } else {
            lk.p = sl.k32 ? (const void*)sl.keys32.get() : (const void*)sl.keys64.get();
            lk.dt = 0;
            lk.hi = sl.k32 ? (sl.and_bits & 0xFFFFFFFF00000000ull) : 0;
        }
        const uint64_t rhi = sr.k32 ? (sr.and_bits & 0xFFFFFFFF00000000ull) : 0;
        const int64_t ctiles = ceil_div(nl, JTILE);
        DevBuf<uint64_t> tsum(ctx, ctiles), toff(ctx, ctiles + 1);
        auto go = [&](auto kl, auto kr) {
            using KL = decltype(kl);
            using KR = decltype(kr);
            const KR* rk = sizeof(KR) == 4 ? (const KR*)sr.keys32.get() : (const KR*)sr.keys64.get();
            if (k32) launch_buckets<KL, KR, uint32_t>(ctx, lk, nl, rk, rhi, nr, P, tsum.get(), ctiles, scal.get(), verify);
            else launch_buckets<KL, KR, uint64_t>(ctx, lk, nl, rk, rhi, nr, P, tsum.get(), ctiles, scal.get(), verify);
        };
        if (sl.k32 || lid) {
            if (sr.k32) go(uint32_t{}, uint32_t{}); else go(uint32_t{}, uint64_t{});
        } else {
            if (sr.k32) go(uint64_t{}, uint32_t{}); else go(uint64_t{}, uint64_t{});
        }
        const double kb = k32 ? 4.0 : 8.0;
        ctx->add_bytes("tqp_smj_buckets", (lid ? (double)dtype_size(left.dtype) : kb) * (double)nl + kb * (double)nr +
                                              8.0 * (double)nl);
        sl.keys32.release();
        sl.keys64.release();
        sr.keys32.release();
        sr.keys64.release();
        scan_add_u64_exclusive(ctx, tsum.get(), toff.get(), ctiles);
        TQP_CUDA(cudaMemcpyAsync(scal.get() + 3, toff.get() + ctiles, 8, cudaMemcpyDeviceToDevice, ctx->stream));
        int64_t h[6];
        read_back(ctx, h, scal.get(), 48);
        if (verify && (int)h[2]) {   // not sorted after all
            delete P;
            return nullptr;
        }
        double dt;
        memcpy(&dt, &h[5], 8);
        if (h[4] || dt >= 4.6116860184273879e18 || (uint64_t)h[3] >= SUM_CAP)   // 2^62
            fail(TQP_ERR_OVERFLOW, "smj: output size exceeds 2^62");
        P->out_size = h[3];
        if (P->out_size > 0) {   // cumHistMul + the tile -> bucket table for expand
            // a table entry per output tile while that stays small; coarser tiles (and a search
            // per entry) when outSize dwarfs the buckets. The cap is K / 8 + 2^22 entries: with
            // one bucket per left row, 4K entries (the r01 cap for keys) meant 400M binary
            // searches for the both-Zipf config (8.9 ms); a coarser table only widens the
            // range each expansion CTA narrows with its warp-cooperative search.
            const int64_t tcap = P->K / 8 + (int64_t(1) << 22);
            int sh = 0;
            while (ceil_div(P->out_size, (int64_t)ETILE << sh) + 1 > tcap) sh++;
            P->tg_shift = sh;
            const int64_t n_tb = ceil_div(P->out_size, (int64_t)ETILE << sh) + 1;
            P->tb.alloc(ctx, n_tb);
            launch(ctx, "tqp_smj_cumsum", cum_write_kernel, dim3((unsigned)ctiles), dim3(JNT), 0,
                   (const uint32_t*)P->mR.get(), P->K, (const uint64_t*)toff.get(), P->mcum.get(),
                   sh == 0 ? P->tb.get() : (uint32_t*)nullptr, n_tb);
            if (sh > 0) {
                static_assert((ETILE & (ETILE - 1)) == 0, "ETILE is a power of two");
                const int lg = __builtin_ctz(ETILE) + sh;
                const int g = (int)std::min<int64_t>(ceil_div(n_tb, 256), (int64_t)ctx->num_sms * 16);
                launch(ctx, "tqp_smj_cumsum", tb_search_kernel, dim3(g), dim3(256), 0, (const int64_t*)P->mcum.get(), P->K,
                       lg, P->tb.get(), n_tb);
            }
            ctx->add_bytes("tqp_smj_cumsum", 12.0 * (double)P->K + 4.0 * (double)n_tb);
        }
        *out_size_host = P->out_size;
        return P;
    } catch (...) {
        delete P;
        throw;
    }
}

tqp_smj_plan* smj_prepare(tqp_ctx* ctx, tqp_col left, int64_t nl, tqp_col right, int64_t nr, int64_t* out_size_host) {
    check_col(left, nl, "smj left");
    check_col(right, nr, "smj right");
    // TQP_SMJ_NO_SPEC=1 (and TQP_SORT_NO_PRESORTED, whose radix route needs the true plan)
    // always runs the left side's plan pass
    static const bool no_spec = [] {
        const char* e = std::getenv("TQP_SMJ_NO_SPEC");
        const char* f = std::getenv("TQP_SORT_NO_PRESORTED");
        return (e && std::atoi(e) != 0) || (f && std::atoi(f) != 0);
    }();
    const bool spec = !no_spec && nl >= (1 << 16) && nr > 0 && (left.dtype == TQP_I64 || left.dtype == TQP_I32);
    if (spec)
        if (tqp_smj_plan* P = smj_prepare_impl(ctx, left, nl, right, nr, out_size_host, true)) return P;
    return smj_prepare_impl(ctx, left, nl, right, nr, out_size_host, false);
}

// more than ~700 buckets per output tile on average: the larger staging of bucket ends
static bool expand_sparse(const tqp_smj_plan* P) {
    return P->out_size > 0 && (double)P->K * ETILE > 700.0 * (double)P->out_size;
}

void smj_expand(tqp_ctx* ctx, const tqp_smj_plan* P, int64_t begin, int64_t end, void* lo, void* ro, int idx32) {
    if (begin < 0 || end < begin || end > P->out_size) fail(TQP_ERR_INVALID_ARGUMENT, "smj_expand: bad window");
    if (end == begin) return;
    if (!lo || !ro) fail(TQP_ERR_INVALID_ARGUMENT, "smj_expand: null output");
    const int64_t blocks = ceil_div(end - begin, ETILE);
    if (blocks >= (int64_t(1) << 31)) fail(TQP_ERR_INVALID_ARGUMENT, "smj_expand: window too large");
    if (idx32 && (P->n_left >= (int64_t(1) << 31) || P->n_right >= (int64_t(1) << 31)))
        fail(TQP_ERR_INVALID_ARGUMENT, "smj_expand_i32: row counts must be < 2^31");
    ctx->add_bytes("tqp_smj_expand", (idx32 ? 8.0 : 16.0) * (double)(end - begin));
    auto* kf = expand_sparse(P) ? expand_kernel<false, false, 4098> : expand_kernel<false, false, TQP_EXPAND_CCAP>;
    launch(ctx, "tqp_smj_expand", kf, dim3((unsigned)blocks), dim3(ENT), 0, P->mR.get(),
           P->msR.get(), P->mcum.get(), P->K, P->tb.get(), P->perm_l.get(), P->perm_r.get(), begin, end, lo,
           ro, idx32, (unsigned long long*)nullptr, P->tg_shift, SmjPayload{});
}

void smj_expand_payload(tqp_ctx* ctx, const tqp_smj_plan* P, int64_t begin, int64_t end, const tqp_col* lp, int n_lp,
                        void* const* lp_out, const tqp_col* rp, int n_rp, void* const* rp_out, int64_t* lo,
                        int64_t* ro) {
    if (begin < 0 || end < begin || end > P->out_size) fail(TQP_ERR_INVALID_ARGUMENT, "smj_expand: bad window");
    if (n_lp < 0 || n_lp > SMJ_MAXPAY || n_rp < 0 || n_rp > SMJ_MAXPAY)
        fail(TQP_ERR_INVALID_ARGUMENT, "smj_expand_payload: at most 8 payload columns per side");
    SmjPayload pay{};
    pay.nl = n_lp;
    pay.nr = n_rp;
    double pb = 0;
    for (int c = 0; c < n_lp; c++) {
        if ((end > begin && (!lp[c].data || !lp_out[c])) || lp[c].dtype < TQP_U8 || lp[c].dtype > TQP_F64)
            fail(TQP_ERR_INVALID_ARGUMENT, "smj_expand_payload: bad left payload column");
        pay.lsrc[c] = lp[c].data;
        pay.ldt[c] = lp[c].dtype;
        pay.ldst[c] = lp_out[c];
        pb += 2.0 * (double)dtype_size(lp[c].dtype);
    }
    for (int c = 0; c < n_rp; c++) {
        if ((end > begin && (!rp[c].data || !rp_out[c])) || rp[c].dtype < TQP_U8 || rp[c].dtype > TQP_F64)
            fail(TQP_ERR_INVALID_ARGUMENT, "smj_expand_payload: bad right payload column");
        pay.rsrc[c] = rp[c].data;
        pay.rdt[c] = rp[c].dtype;
        pay.rdst[c] = rp_out[c];
        pb += 2.0 * (double)dtype_size(rp[c].dtype);
    }
    if (end == begin) return;
    const int64_t blocks = ceil_div(end - begin, ETILE);
    if (blocks >= (int64_t(1) << 31)) fail(TQP_ERR_INVALID_ARGUMENT, "smj_expand: window too large");
    ctx->add_bytes("tqp_smj_expand", ((lo ? 8.0 : 0.0) + (ro ? 8.0 : 0.0) + pb) * (double)(end - begin));
    auto* kf = expand_sparse(P) ? expand_kernel<false, true, 4098> : expand_kernel<false, true, TQP_EXPAND_CCAP>;
    launch(ctx, "tqp_smj_expand", kf, dim3((unsigned)blocks), dim3(ENT), 0,
           P->mR.get(), P->msR.get(), P->mcum.get(), P->K, P->tb.get(), P->perm_l.get(), P->perm_r.get(),
           begin, end, (void*)lo, (void*)ro, 0, (unsigned long long*)nullptr, P->tg_shift, pay);
}

// The expansion consumed in place (a fused consumer instead of
// materialising pairs that cannot be stored): out[0] = sum_j mix64(mix64((l_j << 32) |
// r_j) ^ j), out[1] = sum_j l_j, out[2] = sum_j r_j, mod 2^64, over j in [begin, end).
void smj_expand_checksum(tqp_ctx* ctx, const tqp_smj_plan* P, int64_t begin, int64_t end, uint64_t* out_host) {
    if (begin < 0 || end < begin || end > P->out_size) fail(TQP_ERR_INVALID_ARGUMENT, "smj_expand: bad window");
    out_host[0] = out_host[1] = out_host[2] = 0;
    if (end == begin) return;
    const int64_t blocks = ceil_div(end - begin, ETILE);
    if (blocks >= (int64_t(1) << 31)) fail(TQP_ERR_INVALID_ARGUMENT, "smj_expand: window too large");
    DevBuf<unsigned long long> ck(ctx, 3 * CK_SLOTS + 3);
    ck.zero();
    auto* kf = expand_sparse(P) ? expand_kernel<true, false, 4098> : expand_kernel<true, false, TQP_EXPAND_CCAP>;
    launch(ctx, "tqp_smj_expand_checksum", kf, dim3((unsigned)blocks), dim3(ENT), 0,
           P->mR.get(), P->msR.get(), P->mcum.get(), P->K, P->tb.get(), P->perm_l.get(), P->perm_r.get(),
           begin, end, (void*)nullptr, (void*)nullptr, 0, ck.get(), P->tg_shift, SmjPayload{});
    launch(ctx, "tqp_smj_expand_checksum", ck_final_kernel, dim3(1), dim3(1024), 0, (const unsigned long long*)ck.get(),
           ck.get() + 3 * CK_SLOTS);
    read_back(ctx, out_host, ck.get() + 3 * CK_SLOTS, 24);
}

void smj_release(tqp_ctx*, tqp_smj_plan* P) { delete P; }

}  // namespace tqp
