// smj.cu -- generic many-to-many sort-merge join, Alg. 1 (
// prose :1114-1137) with readings R2 (ascending), R3 (bucketize right=True),
// R4 (div and remainder by rightHist), R5 (histograms over present keys), R6
// (output order key asc, left row asc, right row asc).
//
// Paper step -> kernel here:
//   l.2-3  sort both key columns with permutation       -> radix_sort (sort.cu)
//   l.4    bincount left / right                          -> rle_kernel: run-length
//          encoding of the sorted keys (unique key, run start); counts are run
//          lengths, so no domain-sized histogram is ever materialised
//   l.5-8  histMul = L*R; cumsums                         -> intersect_kernel (each
//          left unique key located among the right unique keys by a merge walk)
//          + common_kernel (compaction of the common keys with L, R,
//          startL = cumL - L, startR = cumR - R) + cum_tiles / add-scan /
//          cum_write (inclusive scan of L*R = cumHistMul, two passes)
//   l.9    outSize = cumHistMul[-1]                       -> one 8-byte readback
//   l.10-14 arange, bucketize, in-bucket offset, div/rem -> expand_kernel: each CTA
//          owns a fixed output range, finds its first bucket with one
//          upper_bound (= bucketize right=True), and walks (q, r) incrementally
//          (o' = q*R + r) instead of a 64-bit division per output.
#include "internal.h"

struct tqp_smj_plan {
    int64_t n_left = 0, n_right = 0, K = 0, out_size = 0;
    tqp::DevBuf<uint32_t> perm_l, perm_r;
    tqp::DevBuf<uint32_t> mL, mR, msL, msR;   // per common key: counts and run starts (< 2^30)
    tqp::DevBuf<int64_t> mcum;                 // cumHistMul (inclusive)
    tqp::DevBuf<uint32_t> tb;                  // per output tile of ETILE << tg_shift: bucket of its first output (+ sentinel)
    int tg_shift = 0;                          // > 0 when outSize is far larger than the keys (coarse table)
};

namespace tqp {

namespace {
constexpr int JNT = 256;
constexpr int JNW = JNT / 32;
constexpr int JIPT = 8;
constexpr int JTILE = JNT * JIPT;

// Run-length encoding of sorted keys: heads -> (unique key, run start), in two
// passes with no inter-tile dependency (a decoupled look-back chain over 2048-key
// tiles was measured to bound this step at ~1 TB/s): rle_count_kernel counts the
// heads of every tile of RT keys, an exclusive add-scan turns counts into offsets,
// and rle_write_kernel re-reads the keys, ranks the heads inside the tile and writes
// them at their final positions (staged in shared memory, coalesced). Each thread
// owns RIPT consecutive keys (16-byte loads). Keys are read as KT (the sort's
// internal 32- or 64-bit key) and written as KO = hi | key (the common domain of
// both join sides).
constexpr int RIPT = 16;
constexpr int RT = JNT * RIPT;

template <typename KT>
__device__ __forceinline__ void rle_heads(const KT* __restrict__ u, int64_t n, int64_t r0, KT (&k)[RIPT],
                                          bool (&head)[RIPT], uint32_t& cnt) {
    const int lane = threadIdx.x & 31;
    if (r0 + RIPT <= n && (uintptr_t)u % 16 == 0) {
        constexpr int PER = 16 / sizeof(KT);
#pragma unroll
        for (int q = 0; q < RIPT / PER; q++) {
            const uint4 v = __ldg(reinterpret_cast<const uint4*>(u + r0) + q);
            memcpy(&k[q * PER], &v, 16);
        }
    } else {
#pragma unroll
        for (int j = 0; j < RIPT; j++) k[j] = r0 + j < n ? u[r0 + j] : KT(0);
    }
    // the key before this thread's first: the previous lane's last, or memory for lane 0
    KT pk = __shfl_up_sync(0xffffffffu, k[RIPT - 1], 1);
    if (lane == 0 && r0 > 0 && r0 <= n) pk = u[r0 - 1];
    cnt = 0;
#pragma unroll
    for (int j = 0; j < RIPT; j++) {
        head[j] = r0 + j < n && (j == 0 ? (r0 == 0 || k[0] != pk) : k[j] != k[j - 1]);
        cnt += head[j];
    }
}

template <typename KT>
__global__ void __launch_bounds__(JNT) rle_count_kernel(const KT* __restrict__ u, int64_t n, uint32_t* tcnt) {
    __shared__ uint32_t s_w[JNW];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t r0 = (int64_t)blockIdx.x * RT + (int64_t)tid * RIPT;
    KT k[RIPT];
    bool head[RIPT];
    uint32_t cnt;
    rle_heads(u, n, r0, k, head, cnt);
    for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    if (lane == 0) s_w[warp] = cnt;
    __syncthreads();
    if (tid == 0) {
        uint32_t t = 0;
        for (int w = 0; w < JNW; w++) t += s_w[w];
        tcnt[blockIdx.x] = t;
    }
}

template <typename KT, typename KO>
__global__ void __launch_bounds__(JNT) rle_write_kernel(const KT* __restrict__ u, uint64_t hi, int64_t n,
                                                        const uint32_t* __restrict__ toff, int64_t n_tiles, KO* ukey,
                                                        uint32_t* ustart, int64_t* U_out) {
    __shared__ uint32_t s_w[JNW];
    constexpr int SCAP = sizeof(KO) == 4 ? RT : RT / 2;   // heads staged when they fit (else written directly)
    __shared__ KO s_key[SCAP];
    __shared__ uint32_t s_pos[SCAP];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t r0 = (int64_t)blockIdx.x * RT + (int64_t)tid * RIPT;
    KT k[RIPT];
    bool head[RIPT];
    uint32_t cnt;
    rle_heads(u, n, r0, k, head, cnt);
    uint32_t x = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) s_w[warp] = x;
    __syncthreads();
    uint32_t wpre = 0, tot = 0;
#pragma unroll
    for (int w = 0; w < JNW; w++) {
        if (w < warp) wpre += s_w[w];
        tot += s_w[w];
    }
    const int64_t excl = toff[blockIdx.x];
    uint32_t lp = wpre + x - cnt;
    if (tot <= (uint32_t)SCAP) {
#pragma unroll
        for (int j = 0; j < RIPT; j++)
            if (head[j]) { s_key[lp] = (KO)(hi | (uint64_t)k[j]); s_pos[lp] = (uint32_t)(r0 + j); lp++; }
        __syncthreads();
        for (uint32_t q = tid; q < tot; q += JNT) {
            ukey[excl + q] = s_key[q];
            ustart[excl + q] = s_pos[q];
        }
    } else {
#pragma unroll
        for (int j = 0; j < RIPT; j++)
            if (head[j]) { ukey[excl + lp] = (KO)(hi | (uint64_t)k[j]); ustart[excl + lp] = (uint32_t)(r0 + j); lp++; }
    }
    if (blockIdx.x == n_tiles - 1 && tid == 0) {
        const int64_t U = excl + tot;
        *U_out = U;
        ustart[U] = (uint32_t)n;
    }
}

template <typename KO>
__device__ __forceinline__ int64_t lower_bound_k(const KO* a, int64_t lo, int64_t hi, KO k) {
    while (lo < hi) {
        int64_t mid = (lo + hi) >> 1;
        if (a[mid] < k) lo = mid + 1; else hi = mid;
    }
    return lo;
}

// For each left unique key: find it among the right unique keys (pass 1, no
// inter-tile dependency: the matching right unique index or NOMATCH per left unique
// key, and a per-tile count), then compact the common keys with (L, R, startL,
// startR) at the scanned tile offsets (pass 2). Grid covers n_left (an upper bound
// of U_l); tiles past U_l count zero.
constexpr int ICAP = 4096;   // right unique keys staged in shared memory per tile
constexpr uint32_t NOMATCH = 0xFFFFFFFFu;

// tb[t] = lower_bound(right unique keys, first left unique key of tile t), all tiles
// searched in parallel (one thread each); tb[n_tiles] = U_r.
template <typename KO>
__global__ void tile_bounds_kernel(const KO* __restrict__ ukl, const int64_t* U_l_p, const KO* __restrict__ ukr,
                                   const int64_t* U_r_p, int64_t* tb, int64_t n_tiles) {
    const int64_t U_l = *U_l_p, U_r = *U_r_p;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t <= n_tiles; t += (int64_t)gridDim.x * blockDim.x)
        tb[t] = (t < n_tiles && t * JTILE < U_l) ? lower_bound_k(ukr, 0, U_r, ukl[t * JTILE]) : U_r;
}

template <typename KO>
__global__ void __launch_bounds__(JNT) intersect_kernel(const KO* __restrict__ ukl, const int64_t* U_l_p,
                                                        const KO* __restrict__ ukr, const int64_t* U_r_p,
                                                        const int64_t* __restrict__ tb, uint32_t* __restrict__ pm,
                                                        uint32_t* __restrict__ tcnt) {
    __shared__ uint32_t s_w[JNW];
    __shared__ KO s_r[ICAP];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t U_l = *U_l_p, U_r = *U_r_p;
    const int64_t base = (int64_t)blockIdx.x * JTILE;
    if (base >= U_l) {
        if (tid == 0) tcnt[blockIdx.x] = 0;
        return;
    }
    // right unique keys <= this tile's last left key lie below tb[t + 1] + 1
    const int64_t rlo = tb[blockIdx.x], rhi = min(tb[blockIdx.x + 1] + 1, U_r);
    // the right unique keys this tile can match: staged in shared memory if they fit
    const bool staged = rhi - rlo <= ICAP;
    if (staged) {
        for (int64_t i = rlo + tid; i < rhi; i += JNT) s_r[i - rlo] = ukr[i];
        __syncthreads();
    }
    // JIPT consecutive left unique keys per thread: one lower_bound for the first,
    // then a merge walk (both lists are sorted and unique)
    const int64_t jb = base + (int64_t)tid * JIPT;
    uint32_t cnt = 0;
    if (jb < U_l) {
        KO k[JIPT];
#pragma unroll
        for (int i = 0; i < JIPT; i++) k[i] = jb + i < U_l ? ukl[jb + i] : KO(0);
        uint32_t out[JIPT];
        if (staged) {
            const int64_t nr = rhi - rlo;
            int64_t lo = 0, hi = nr;
            while (lo < hi) {
                const int64_t mid = (lo + hi) >> 1;
                if (s_r[mid] < k[0]) lo = mid + 1; else hi = mid;
            }
#pragma unroll
            for (int i = 0; i < JIPT; i++) {
                while (lo < nr && s_r[lo] < k[i]) lo++;
                const bool eq = jb + i < U_l && lo < nr && s_r[lo] == k[i];
                out[i] = eq ? (uint32_t)(lo + rlo) : NOMATCH;
                cnt += eq;
            }
        } else {
            int64_t pos = lower_bound_k(ukr, rlo, rhi, k[0]);
#pragma unroll
            for (int i = 0; i < JIPT; i++) {
                if (i > 0) pos = lower_bound_k(ukr, pos, rhi, k[i]);
                const bool eq = jb + i < U_l && pos < rhi && ukr[pos] == k[i];
                out[i] = eq ? (uint32_t)pos : NOMATCH;
                cnt += eq;
            }
        }
#pragma unroll
        for (int i = 0; i < JIPT; i++)
            if (jb + i < U_l) pm[jb + i] = out[i];
    }
    for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    if (lane == 0) s_w[warp] = cnt;
    __syncthreads();
    if (tid == 0) {
        uint32_t t = 0;
        for (int w = 0; w < JNW; w++) t += s_w[w];
        tcnt[blockIdx.x] = t;
    }
}

// pass 2: common keys in left-key order -> (L, R, startL, startR). Each thread owns
// JIPT consecutive left unique keys (16-byte loads of pm and of the run starts);
// the right run starts are gathered with all loads issued up front; outputs are
// staged in shared memory and written coalesced.
__global__ void __launch_bounds__(JNT) common_kernel(const uint32_t* __restrict__ pm, const uint32_t* __restrict__ usl,
                                                     const uint32_t* __restrict__ usr, const int64_t* U_l_p,
                                                     const uint32_t* __restrict__ toff, uint32_t* mL, uint32_t* mR,
                                                     uint32_t* msL, uint32_t* msR, int64_t* K_out, int64_t n_tiles) {
    __shared__ uint32_t s_w[JNW];
    __shared__ uint32_t s_o[4][JTILE];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t U_l = *U_l_p;
    const int64_t base = (int64_t)blockIdx.x * JTILE;
    if (blockIdx.x == n_tiles - 1 && tid == 0) *K_out = toff[n_tiles];
    const uint32_t t0 = toff[blockIdx.x];
    const uint32_t tot = toff[blockIdx.x + 1] - t0;
    if (base >= U_l || tot == 0) return;
    const int64_t r0 = base + (int64_t)tid * JIPT;   // JIPT consecutive left unique keys per thread
    uint32_t p[JIPT], ul[JIPT + 1];
    if (r0 + JIPT <= U_l) {
        const uint4 a0 = __ldcs(reinterpret_cast<const uint4*>(pm + r0));
        const uint4 a1 = __ldcs(reinterpret_cast<const uint4*>(pm + r0) + 1);
        p[0] = a0.x; p[1] = a0.y; p[2] = a0.z; p[3] = a0.w; p[4] = a1.x; p[5] = a1.y; p[6] = a1.z; p[7] = a1.w;
        const uint4 b0 = __ldg(reinterpret_cast<const uint4*>(usl + r0));
        const uint4 b1 = __ldg(reinterpret_cast<const uint4*>(usl + r0) + 1);
        ul[0] = b0.x; ul[1] = b0.y; ul[2] = b0.z; ul[3] = b0.w; ul[4] = b1.x; ul[5] = b1.y; ul[6] = b1.z; ul[7] = b1.w;
        ul[8] = usl[r0 + JIPT];
    } else {
#pragma unroll
        for (int i = 0; i < JIPT; i++) {
            p[i] = r0 + i < U_l ? pm[r0 + i] : NOMATCH;
            ul[i] = r0 + i <= U_l ? usl[r0 + i] : 0u;
        }
        ul[JIPT] = r0 + JIPT <= U_l ? usl[r0 + JIPT] : 0u;
    }
    uint32_t ur0[JIPT], ur1[JIPT], cnt = 0;
#pragma unroll
    for (int i = 0; i < JIPT; i++) {   // right run start and end of every match, loads in flight together
        const bool hit = p[i] != NOMATCH;
        ur0[i] = hit ? __ldg(usr + p[i]) : 0u;
        ur1[i] = hit ? __ldg(usr + p[i] + 1) : 0u;
        cnt += hit;
    }
    uint32_t x = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) s_w[warp] = x;
    __syncthreads();
    uint32_t m = x - cnt;
#pragma unroll
    for (int w = 0; w < JNW; w++)
        if (w < warp) m += s_w[w];
#pragma unroll
    for (int i = 0; i < JIPT; i++) {
        if (p[i] == NOMATCH) continue;
        s_o[0][m] = ul[i + 1] - ul[i];
        s_o[1][m] = ur1[i] - ur0[i];
        s_o[2][m] = ul[i];
        s_o[3][m] = ur0[i];
        m++;
    }
    __syncthreads();
    for (uint32_t k = tid; k < tot; k += JNT) {
        mL[t0 + k] = s_o[0][k];
        mR[t0 + k] = s_o[1][k];
        msL[t0 + k] = s_o[2][k];
        msR[t0 + k] = s_o[3][k];
    }
}

// cumHistMul = inclusive scan of histMul = L*R over the K common keys, in two passes
// with no inter-tile chain: cum_tiles_kernel sums L*R per tile of JTILE keys (saturated at
// 2^62, and also added into an fp64 running total that flags totals >= 2^62), an
// exclusive 64-bit add-scan gives tile offsets, and cum_write_kernel writes cumHistMul
// and, in the same pass, the per-output-tile bucket table expand needs.
constexpr uint64_t SUM_CAP = 1ull << 62;
constexpr int64_t ETILE_C = 256 * 8;   // == ETILE (expand's outputs per CTA), defined below

__global__ void __launch_bounds__(JNT) cum_tiles_kernel(const uint32_t* __restrict__ mL, const uint32_t* __restrict__ mR,
                                                        const int64_t* K_p, uint64_t* tsum, double* dtot, int* overflow) {
    __shared__ unsigned __int128 s_w[JNW];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t K = *K_p;
    const int64_t base = (int64_t)blockIdx.x * JTILE + (int64_t)tid * JIPT;
    unsigned __int128 t = 0;
#pragma unroll
    for (int i = 0; i < JIPT; i++)
        if (base + i < K) t += (uint64_t)mL[base + i] * (uint64_t)mR[base + i];
    for (int o = 16; o > 0; o >>= 1) {
        const uint64_t lo = __shfl_xor_sync(0xffffffffu, (uint64_t)t, o);
        const uint64_t hi = __shfl_xor_sync(0xffffffffu, (uint64_t)(t >> 64), o);
        t += ((unsigned __int128)hi << 64) | lo;
    }
    if (lane == 0) s_w[warp] = t;
    __syncthreads();
    if (tid == 0) {
        unsigned __int128 tot = 0;
        for (int w = 0; w < JNW; w++) tot += s_w[w];
        if (tot >= SUM_CAP) {
            *overflow = 1;
            tot = SUM_CAP - 1;
        }
        tsum[blockIdx.x] = (uint64_t)tot;
        if (tot) atomicAdd(dtot, (double)(uint64_t)tot);
    }
}

__global__ void __launch_bounds__(JNT) cum_write_kernel(const uint32_t* __restrict__ mL, const uint32_t* __restrict__ mR,
                                                        const int64_t* K_p, const uint64_t* __restrict__ toff,
                                                        int64_t* mcum, uint32_t* tb, int64_t n_tb) {
    __shared__ uint64_t s_w[JNW];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t K = *K_p;
    const int64_t base = (int64_t)blockIdx.x * JTILE + (int64_t)tid * JIPT;
    if ((int64_t)blockIdx.x * JTILE >= K) return;
    uint64_t v[JIPT], t = 0;
#pragma unroll
    for (int i = 0; i < JIPT; i++) {
        v[i] = base + i < K ? (uint64_t)mL[base + i] * (uint64_t)mR[base + i] : 0;
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
#pragma unroll
    for (int i = 0; i < JIPT; i++) {
        const int64_t b = base + i;
        if (b >= K) break;
        const int64_t start = (int64_t)run;
        run += v[i];
        mcum[b] = (int64_t)run;
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

template <bool CK, bool PAY = false>
// Blocks per SM forced by the register budget: measured no gain (SF10 expansion 0.435 ms
// at 63 registers / 4 blocks, 0.443 with 5, 0.439 with 6, 0.494 with 8 -- spills), so off.
#ifndef TQP_EXPAND_MINB
#define TQP_EXPAND_MINB 0
#endif
__global__ void __launch_bounds__(ENT, TQP_EXPAND_MINB) expand_kernel(const uint32_t* __restrict__ mL, const uint32_t* __restrict__ mR,
                                                     const uint32_t* __restrict__ msL, const uint32_t* __restrict__ msR,
                                                     const int64_t* __restrict__ mcum, int64_t K,
                                                     const uint32_t* __restrict__ tb,
                                                     const uint32_t* __restrict__ perm_l,
                                                     const uint32_t* __restrict__ perm_r, int64_t begin, int64_t end,
                                                     void* __restrict__ lo_out, void* __restrict__ ro_out, int idx32,
                                                     unsigned long long* __restrict__ ck, int tg_shift,
                                                     SmjPayload pay) {
    // shared memory: the staged bucket ends, plus (when the CTA spans <= MCAP buckets)
    // the buckets' (L, R, startL, startR) so that walking across keys needs no global loads
    constexpr int MCAP = 1024;
    __shared__ __align__(16) int32_t s_buf[2 * ETILE + 2 + 3 * MCAP];
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
    const int nb = (int)(b1 - b0 + 1);
    const bool meta = nb <= MCAP;
    int32_t* s_cum = s_buf;
    uint32_t* s_m = reinterpret_cast<uint32_t*>(s_buf + (meta ? MCAP : 0));   // [4][MCAP] when meta
    for (int i = threadIdx.x; i < nb; i += ENT) {
        const int64_t v = mcum[b0 + i] - c0;
        s_cum[i] = (int32_t)(v < 0 ? -1 : (v > ETILE ? ETILE + 1 : v));
        if (meta) {
            s_m[i] = mL[b0 + i];
            s_m[MCAP + i] = mR[b0 + i];
            s_m[2 * MCAP + i] = msL[b0 + i];
            s_m[3 * MCAP + i] = msR[b0 + i];
        }
    }
    __syncthreads();
    const int64_t o0 = c0 + (int64_t)threadIdx.x * EIPT;
    uint64_t hs = 0, sl = 0, sr = 0;   // CK: this thread's share of the consumer sums
    if (o0 < c1) {   // thread: EIPT consecutive outputs, incremental (q, r)
        const int32_t rel = threadIdx.x * EIPT;
        int lo = 0, hi = nb;
        while (lo < hi) {   // upper_bound(rel) over the staged ends
            const int mid = (lo + hi) >> 1;
            if (s_cum[mid] <= rel) lo = mid + 1; else hi = mid;
        }
        int bi = lo;   // bucket index relative to b0
        TQP_DCHECK(bi < nb && b0 + bi < K);
        auto load = [&](int i, int64_t& L, int64_t& R, int64_t& sL, int64_t& sR) {
            if (meta) {
                L = s_m[i]; R = s_m[MCAP + i]; sL = s_m[2 * MCAP + i]; sR = s_m[3 * MCAP + i];
            } else {
                L = mL[b0 + i]; R = mR[b0 + i]; sL = msL[b0 + i]; sR = msR[b0 + i];
            }
        };
        int64_t L, R, sL, sR;
        load(bi, L, R, sL, sR);
        int64_t off = o0 - (mcum[b0 + bi] - L * R);
        int64_t q, r;
        if (((uint64_t)off | (uint64_t)R) >> 32 == 0) {   // 32-bit division when it fits
            const uint32_t q32 = (uint32_t)off / (uint32_t)R;
            q = q32;
            r = (int64_t)((uint32_t)off - q32 * (uint32_t)R);
        } else {
            q = off / R;
            r = off - q * R;
        }
        const int cnt = (int)min((int64_t)EIPT, c1 - o0);
        uint32_t vl[EIPT], vr[EIPT];
#pragma unroll
        for (int j = 0; j < EIPT; j++) {
            if (j >= cnt) break;
            TQP_DCHECK(q < L && r < R);
            vl[j] = __ldg(perm_l + sL + q);
            vr[j] = __ldg(perm_r + sR + r);
            if (CK) {
                hs += mix64(mix64(((uint64_t)vl[j] << 32) | vr[j]) ^ (uint64_t)(o0 + j));
                sl += vl[j];
                sr += vr[j];
            }
            if (++r == R) {
                r = 0;
                if (++q == L) {
                    q = 0;
                    if (b0 + ++bi < K && bi < nb) load(bi, L, R, sL, sR);
                }
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
    if (vec) {   // 4 outputs per thread and step: one 16-byte shared load, two 16-byte stores per array
        for (int o = threadIdx.x * 4; o < n; o += ENT * 4) {
            const uint4 a = *reinterpret_cast<const uint4*>(s_l + o);
            const uint4 b = *reinterpret_cast<const uint4*>(s_r + o);
            __stcs(reinterpret_cast<longlong2*>(lo_p + o), make_longlong2(a.x, a.y));
            __stcs(reinterpret_cast<longlong2*>(lo_p + o) + 1, make_longlong2(a.z, a.w));
            __stcs(reinterpret_cast<longlong2*>(ro_p + o), make_longlong2(b.x, b.y));
            __stcs(reinterpret_cast<longlong2*>(ro_p + o) + 1, make_longlong2(b.z, b.w));
        }
    } else {
        for (int o = threadIdx.x; o < n; o += ENT) {   // coalesced, streamed (evict-first) stores
            __stcs((long long*)lo_p + o, (long long)s_l[o]);
            __stcs((long long*)ro_p + o, (long long)s_r[o]);
        }
    }
}

template <typename KT, typename KO>
void rle(tqp_ctx* ctx, const KT* u, uint64_t hi, int64_t n, DevBuf<KO>& ukey, DevBuf<uint32_t>& ustart,
         int64_t* U_dev) {
    ukey.alloc(ctx, n);
    ustart.alloc(ctx, n + 1);
    const int64_t tiles = ceil_div(n, RT);
    DevBuf<uint32_t> tcnt(ctx, tiles), toff(ctx, tiles + 1);
    launch(ctx, "tqp_smj_rle", rle_count_kernel<KT>, dim3((unsigned)tiles), dim3(JNT), 0, u, n, tcnt.get());
    scan_add_u32_exclusive(ctx, tcnt.get(), toff.get(), tiles);
    launch(ctx, "tqp_smj_rle", rle_write_kernel<KT, KO>, dim3((unsigned)tiles), dim3(JNT), 0, u, hi, n,
           (const uint32_t*)toff.get(), tiles, ukey.get(), ustart.get(), U_dev);
}

// Both sides' RLE in the common key domain KO, then the intersection of the unique
// keys.
template <typename KO>
void rle_intersect(tqp_ctx* ctx, tqp_smj_plan* P, SortOut& sl, SortOut& sr, int64_t* scal) {
    const int64_t nl = P->n_left, nr = P->n_right;
    DevBuf<KO> ukl, ukr;
    DevBuf<uint32_t> usl, usr;
    auto side = [&](SortOut& so, int64_t n, DevBuf<KO>& uk, DevBuf<uint32_t>& us, int64_t* U) {
        const uint64_t hi = (sizeof(KO) == 8 && so.k32) ? (so.and_bits & 0xFFFFFFFF00000000ull) : 0;
        if (so.k32) rle<uint32_t, KO>(ctx, so.keys32.get(), hi, n, uk, us, U);
        else rle<uint64_t, KO>(ctx, so.keys64.get(), 0, n, uk, us, U);
        ctx->add_bytes("tqp_smj_rle", (double)n * (so.k32 ? 4 : 8));   // compulsory: keys read once
        so.keys32.release();
        so.keys64.release();
    };
    side(sl, nl, ukl, usl, scal + 0);
    side(sr, nr, ukr, usr, scal + 1);
    const int64_t tiles = ceil_div(nl, JTILE);
    DevBuf<uint32_t> pm(ctx, nl), tcnt(ctx, tiles), toff(ctx, tiles + 1);
    DevBuf<int64_t> tb(ctx, tiles + 1);
    launch(ctx, "tqp_smj_intersect", tile_bounds_kernel<KO>, dim3((unsigned)ceil_div(tiles + 1, 128)), dim3(128), 0,
           (const KO*)ukl.get(), (const int64_t*)(scal + 0), (const KO*)ukr.get(), (const int64_t*)(scal + 1), tb.get(),
           tiles);
    launch(ctx, "tqp_smj_intersect", intersect_kernel<KO>, dim3((unsigned)tiles), dim3(JNT), 0, (const KO*)ukl.get(),
           (const int64_t*)(scal + 0), (const KO*)ukr.get(), (const int64_t*)(scal + 1), (const int64_t*)tb.get(),
           pm.get(), tcnt.get());
    scan_add_u32_exclusive(ctx, tcnt.get(), toff.get(), tiles);
    launch(ctx, "tqp_smj_intersect", common_kernel, dim3((unsigned)tiles), dim3(JNT), 0, (const uint32_t*)pm.get(),
           (const uint32_t*)usl.get(), (const uint32_t*)usr.get(), (const int64_t*)(scal + 0),
           (const uint32_t*)toff.get(), P->mL.get(), P->mR.get(), P->msL.get(), P->msR.get(), scal + 2, tiles);
}
}  // namespace

tqp_smj_plan* smj_prepare(tqp_ctx* ctx, tqp_col left, int64_t nl, tqp_col right, int64_t nr, int64_t* out_size_host) {
    check_col(left, nl, "smj left");
    check_col(right, nr, "smj right");
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
        {   // both digit plans with one host sync
            DevBuf<unsigned long long> ao(ctx, 6);
            DevBuf<uint32_t> hl(ctx, sort_hist0_words(nl)), hr(ctx, sort_hist0_words(nr));
            sort_andor(ctx, left.data, left.dtype, nl, false, ao.get(), hl.get());
            sort_andor(ctx, right.data, right.dtype, nr, false, ao.get() + 3, hr.get());
            uint64_t h[6];
            read_back(ctx, h, ao.get(), 48);
            radix_sort(ctx, left.data, left.dtype, nl, false, sl, h, hl.get());
            radix_sort(ctx, right.data, right.dtype, nr, false, sr, h + 3, hr.get());
        }
        P->perm_l = std::move(sl.perm32);
        P->perm_r = std::move(sr.perm32);
        DevBuf<int64_t> scal(ctx, 6);   // U_l, U_r, K, out_size, overflow flag, fp64 total: one readback
        scal.zero();
        const int64_t cap = std::min(nl, nr);
        P->mL.alloc(ctx, cap);
        P->mR.alloc(ctx, cap);
        P->msL.alloc(ctx, cap);
        P->msR.alloc(ctx, cap);
        P->mcum.alloc(ctx, cap);
        // 32-bit unique keys when both sides' keys differ only in one common low word
        const bool k32 = sl.k32 && sr.k32 && (sl.and_bits >> 32) == (sr.and_bits >> 32);
        const double kb = k32 ? 4.0 : 8.0;
        if (k32) rle_intersect<uint32_t>(ctx, P, sl, sr, scal.get());
        else rle_intersect<uint64_t>(ctx, P, sl, sr, scal.get());
        const int64_t ctiles = ceil_div(cap, JTILE);
        DevBuf<uint64_t> tsum(ctx, ctiles), toff(ctx, ctiles + 1);
        launch(ctx, "tqp_smj_cumsum", cum_tiles_kernel, dim3((unsigned)ctiles), dim3(JNT), 0, (const uint32_t*)P->mL.get(),
               (const uint32_t*)P->mR.get(), (const int64_t*)(scal.get() + 2), tsum.get(), (double*)(scal.get() + 5),
               (int*)(scal.get() + 4));
        scan_add_u64_exclusive(ctx, tsum.get(), toff.get(), ctiles);
        TQP_CUDA(cudaMemcpyAsync(scal.get() + 3, toff.get() + ctiles, 8, cudaMemcpyDeviceToDevice, ctx->stream));
        int64_t h[6];
        read_back(ctx, h, scal.get(), 48);
        double dt;
        memcpy(&dt, &h[5], 8);
        if (h[4] || dt >= 4.6116860184273879e18 || (uint64_t)h[3] >= SUM_CAP)   // 2^62
            fail(TQP_ERR_OVERFLOW, "smj: output size exceeds 2^62");
        ctx->add_bytes("tqp_smj_intersect", (kb + 4.0) * (double)std::min(nl, nr) + 16.0 * (double)h[2]);
        P->K = h[2];
        P->out_size = h[2] > 0 ? h[3] : 0;
        if (P->out_size > 0) {   // cumHistMul + the tile -> bucket table for expand
            // a table entry per output tile while that is comparable to the keys; coarser
            // tiles (and a search per entry) when outSize dwarfs them
            const int64_t tcap = 4 * P->K + (int64_t(1) << 22);
            int sh = 0;
            while (ceil_div(P->out_size, (int64_t)ETILE << sh) + 1 > tcap) sh++;
            P->tg_shift = sh;
            const int64_t n_tb = ceil_div(P->out_size, (int64_t)ETILE << sh) + 1;
            P->tb.alloc(ctx, n_tb);
            launch(ctx, "tqp_smj_cumsum", cum_write_kernel, dim3((unsigned)ctiles), dim3(JNT), 0,
                   (const uint32_t*)P->mL.get(), (const uint32_t*)P->mR.get(), (const int64_t*)(scal.get() + 2),
                   (const uint64_t*)toff.get(), P->mcum.get(), sh == 0 ? P->tb.get() : (uint32_t*)nullptr, n_tb);
            if (sh > 0) {
                static_assert((ETILE & (ETILE - 1)) == 0, "ETILE is a power of two");
                const int lg = __builtin_ctz(ETILE) + sh;
                const int g = (int)std::min<int64_t>(ceil_div(n_tb, 256), (int64_t)ctx->num_sms * 16);
                launch(ctx, "tqp_smj_cumsum", tb_search_kernel, dim3(g), dim3(256), 0, (const int64_t*)P->mcum.get(), P->K,
                       lg, P->tb.get(), n_tb);
            }
            ctx->add_bytes("tqp_smj_cumsum", 16.0 * (double)P->K + 4.0 * (double)n_tb);
        }
        *out_size_host = P->out_size;
        return P;
    } catch (...) {
        delete P;
        throw;
    }
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
    launch(ctx, "tqp_smj_expand", expand_kernel<false>, dim3((unsigned)blocks), dim3(ENT), 0, P->mL.get(), P->mR.get(),
           P->msL.get(), P->msR.get(), P->mcum.get(), P->K, P->tb.get(), P->perm_l.get(), P->perm_r.get(), begin, end, lo,
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
    launch(ctx, "tqp_smj_expand", expand_kernel<false, true>, dim3((unsigned)blocks), dim3(ENT), 0, P->mL.get(),
           P->mR.get(), P->msL.get(), P->msR.get(), P->mcum.get(), P->K, P->tb.get(), P->perm_l.get(), P->perm_r.get(),
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
    launch(ctx, "tqp_smj_expand_checksum", expand_kernel<true>, dim3((unsigned)blocks), dim3(ENT), 0, P->mL.get(),
           P->mR.get(), P->msL.get(), P->msR.get(), P->mcum.get(), P->K, P->tb.get(), P->perm_l.get(), P->perm_r.get(),
           begin, end, (void*)nullptr, (void*)nullptr, 0, ck.get(), P->tg_shift, SmjPayload{});
    launch(ctx, "tqp_smj_expand_checksum", ck_final_kernel, dim3(1), dim3(1024), 0, (const unsigned long long*)ck.get(),
           ck.get() + 3 * CK_SLOTS);
    read_back(ctx, out_host, ck.get() + 3 * CK_SLOTS, 24);
}

void smj_release(tqp_ctx*, tqp_smj_plan* P) { delete P; }

}  // namespace tqp
