// groupby.cu -- sort-based group-by aggregation, Alg. 2 (
// prose :1146-1152), with a fused pre-filter (Listings 1-2 predicate form).
//
// Alg. 2: cat(grpByCols) -> radix sort -> permute data -> uniqueConsecutive
// (unique keys + inverse = segment ids) -> evaluate aggregates per segment.
// The paper materialises every step as a whole-tensor op (and names
// uniqueConsecutive as a bottleneck). Here it is two
// levels of the same sort-based algorithm:
//   phase 1 (persistent kernel, one pass over the referenced columns): every
//     tile of 1024 rows is streamed into shared memory with TMA bulk copies
//     (cp.async.bulk, mbarrier completion, double-buffered so tile k+2 loads
//     while tile k is reduced). The tile's predicates are evaluated, key columns
//     packed into one 64-bit key (column 0 most significant, reading R12), the
//     passing rows radix-sorted in shared memory over the bits that vary in the
//     tile (stable LSD, peers by one warp ballot per digit bit), segment boundaries marked (the
//     uniqueConsecutive / inverse step) and every distinct (op, expression) pair
//     reduced per segment in registers, reading the values in sorted order
//     straight from the staged columns; one partial record per (tile, key);
//   phase 2: the partial records are radix-sorted by key (sort.cu), segment
//     boundaries give the final groups, and partials are added into exact
//     int128 accumulators (64-bit atomics with explicit carry; integer addition
//     is associative, so any order gives bit-identical sums), then finalised
//     (AVG = rn(sum / count), reading R15/R17).
#include <vector>

#include "internal.h"
#include "jit.h"

struct tqp_groupby_plan {
    int64_t G = 0;
    int n_keys = 0, n_aggs = 0, n_pairs = 0;
    int kdt[TQP_MAX_KEYS];
    int aop[TQP_MAX_AGGS];
    int apair[TQP_MAX_AGGS];      // aggregate -> (op, expression) pair (-1 for COUNT)
    tqp::DevBuf<unsigned long long> krange;   // per key column min (0..7) / max (8..15)
    int pop[TQP_MAX_AGGS];        // pair op: 0 sum, 1 min, 2 max
    bool empty_global = false;    // n_keys == 0 and no passing row
    tqp::DevBuf<uint64_t> gkey;
    tqp::DevBuf<int64_t> gcount;
    tqp::DevBuf<uint64_t> glo[TQP_MAX_AGGS];
    tqp::DevBuf<int64_t> ghi[TQP_MAX_AGGS];
    // fp64 aggregates (TQP_F64 factor columns): computed beside the integer plan
    bool has_f64 = false;
    int n_user_aggs = 0;
    int uop[TQP_MAX_AGGS];         // user aggregate op
    int imap[TQP_MAX_AGGS];        // user aggregate -> integer aggregate index, or -1 (fp64)
    tqp::DevBuf<double> gf[TQP_MAX_AGGS];   // fp64 aggregate per group: SUM (AVG: the sum) as double,
                                            // MIN / MAX as order-preserving int64 bit patterns
};

namespace tqp {

namespace {
constexpr int GNT = 256;
constexpr int GNW = GNT / 32;
constexpr int GPT = 4;
constexpr int GTILE = GNT * GPT;   // 1024 rows per tile
constexpr int MAXU = 16;           // distinct referenced columns
constexpr int P_SUM = 0, P_MIN = 1, P_MAX = 2;
constexpr int PCH = 8;             // (op, expression) pairs reduced per traversal
constexpr int UCAP = 64;           // runs per tile with shared-memory accumulators
constexpr int CBINS = 2048;        // key range of a tile sorted by a one-pass counting sort

struct Phase1Args {
    int n_ucols;
    const void* ucol[MAXU];
    int udt[MAXU];
    int uoff[MAXU];               // byte offset of the column inside a stage
    int stage_bytes;
    int n_stages;
    int n_keys;
    int kcol[TQP_MAX_KEYS];
    const unsigned long long* krange;   // per key column min / max (device)
    TermSet ts;                   // predicate conjunction, one interval per column (Term.col = stage slot)
    // dense small-domain path (gb_dense_kernel)
    int D;                        // distinct packed keys present; ids 0..D-1
    const uint8_t* dtab;          // packed key -> id
    const uint64_t* dkeys;        // id -> packed key
    int dense_bits;               // SUM pairs: |value| <= 2^dense_bits keeps per-thread int64 sums exact
    int poff[PCH][3];             // stage byte offset of each factor's column
    int pdtf[PCH][3];             // and its dtype
    int pext[PCH];                // leading factors shared with the previous pair (its whole list), else 0
    int direct;                   // dense / no-key paths: record blockIdx.x * D + id (fixed slots, no counter)
    int n_pairs;
    int prop[TQP_MAX_AGGS];
    int pnf[TQP_MAX_AGGS];
    int pfc[TQP_MAX_AGGS][3];
    int psign[TQP_MAX_AGGS][3];
    int64_t padd[TQP_MAX_AGGS][3];
    int64_t n;
    int64_t n_tiles;
    int bulk_ok;
    uint64_t* pkey;
    int64_t* pcount;
    uint64_t* plo[TQP_MAX_AGGS];
    int64_t* phi[TQP_MAX_AGGS];
    unsigned long long* P_counter;
    int64_t cap;
    int* overflow;                // bit 0: value overflow, bit 1: partial capacity exceeded
};

__device__ __forceinline__ uint64_t key_part(int64_t v, int dt) {
    switch (dt) {
        case TQP_U8: return (uint64_t)v & 0xFFull;
        case TQP_I32: return (uint64_t)((uint32_t)v ^ 0x80000000u);
        default: return (uint64_t)v ^ 0x8000000000000000ull;
    }
}

// Per key column: min / max of the order-preserving unsigned key value, so each
// column is packed as (value - min) in bits(max - min) bits (column 0 most
// significant). Monotone per column, so the packed order is the lexicographic
// order of the tuples (reading R12) and small-domain keys become small bins.
struct KRArgs {
    int n_keys;
    const void* kcol[TQP_MAX_KEYS];
    int kdt[TQP_MAX_KEYS];
    int64_t n;
};

__global__ void key_range_kernel(KRArgs a, unsigned long long* kr) {   // kr[k] = min, kr[8 + k] = max
    __shared__ unsigned long long smin[TQP_MAX_KEYS][GNT / 32], smax[TQP_MAX_KEYS][GNT / 32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t gt = blockIdx.x * (int64_t)blockDim.x + threadIdx.x, gs = (int64_t)gridDim.x * blockDim.x;
    for (int k = 0; k < a.n_keys; k++) {
        unsigned long long mn = ~0ull, mx = 0;
        const int dt = a.kdt[k];
        const int per = dt == TQP_U8 ? 16 : dt == TQP_I32 ? 4 : 2;   // elements per 16-byte load
        const int64_t nv = ((uintptr_t)a.kcol[k] % 16 == 0) ? a.n / per : 0;
        uint32_t mn4 = 0xFFFFFFFFu, mx4 = 0;   // u8: per-byte-lane min / max; i32: 32-bit min / max
        for (int64_t v = gt; v < nv; v += gs) {   // vectorised body: 16 bytes per load, streamed
            const uint4 q = __ldcs(reinterpret_cast<const uint4*>(a.kcol[k]) + v);
            const uint32_t wd[4] = {q.x, q.y, q.z, q.w};
            if (dt == TQP_U8) {
#pragma unroll
                for (int j = 0; j < 4; j++) {
                    mn4 = __vminu4(mn4, wd[j]);
                    mx4 = __vmaxu4(mx4, wd[j]);
                }
            } else if (dt == TQP_I32) {
#pragma unroll
                for (int j = 0; j < 4; j++) {
                    mn4 = min(mn4, wd[j] ^ 0x80000000u);
                    mx4 = max(mx4, wd[j] ^ 0x80000000u);
                }
            } else {
#pragma unroll
                for (int j = 0; j < 2; j++) {
                    const unsigned long long x = (((unsigned long long)wd[2 * j + 1] << 32) | wd[2 * j]) ^ 0x8000000000000000ull;
                    mn = min(mn, x);
                    mx = max(mx, x);
                }
            }
        }
        if (dt == TQP_U8) {
#pragma unroll
            for (int j = 0; j < 4; j++) {
                mn = min(mn, (unsigned long long)((mn4 >> (8 * j)) & 0xFFu));
                mx = max(mx, (unsigned long long)((mx4 >> (8 * j)) & 0xFFu));
            }
        } else if (dt == TQP_I32 && nv > gt) {
            mn = min(mn, (unsigned long long)mn4);
            mx = max(mx, (unsigned long long)mx4);
        }
        for (int64_t i = nv * per + gt; i < a.n; i += gs) {   // tail (or unaligned column)
            const unsigned long long x = key_part(load_as_i64(a.kcol[k], dt, i), dt);
            mn = min(mn, x);
            mx = max(mx, x);
        }
        for (int o = 16; o > 0; o >>= 1) {
            mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
            mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        }
        if (lane == 0) { smin[k][warp] = mn; smax[k][warp] = mx; }
    }
    __syncthreads();
    if (threadIdx.x < a.n_keys) {
        const int k = threadIdx.x;
        unsigned long long mn = ~0ull, mx = 0;
        for (int w = 0; w < (int)(blockDim.x / 32); w++) { mn = min(mn, smin[k][w]); mx = max(mx, smax[k][w]); }
        atomicMin(&kr[k], mn);
        atomicMax(&kr[8 + k], mx);
    }
}

// shift / width / min of every key column from the device-resident ranges
__device__ __forceinline__ void key_layout(const unsigned long long* kr, int n_keys, uint64_t* kmin, int* shift,
                                           int* width) {
    int off = 0;
    for (int k = n_keys - 1; k >= 0; k--) {
        const uint64_t mn = kr[k], mx = kr[8 + k];
        const int wdt = mx > mn ? 64 - __clzll(mx - mn) : 0;
        kmin[k] = mx >= mn ? mn : 0;
        width[k] = wdt;
        shift[k] = off;
        off += wdt;
    }
}

__device__ __forceinline__ int64_t scol(const uint8_t* stage, int off, int dt, int row) {
    switch (dt) {
        case TQP_U8: return (int64_t)stage[off + row];
        case TQP_I32: return (int64_t)reinterpret_cast<const int32_t*>(stage + off)[row];
        default: return (int64_t)reinterpret_cast<const long long*>(stage + off)[row];
    }
}

__device__ __forceinline__ uint32_t bscan256(uint32_t v, uint32_t* s_w) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t x = v;
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) s_w[warp] = x;
    __syncthreads();
    uint32_t add = 0;
    for (int w = 0; w < warp; w++) add += s_w[w];
    __syncthreads();
    return add + x - v;
}

// exact 128-bit atomic accumulation: the carry out of the low word is detected
// from the value atomicAdd returns, so the total is exact for any order.
__device__ __forceinline__ void atomic_add_i128(uint64_t* lo_p, int64_t* hi_p, unsigned __int128 v) {
    const uint64_t lo = (uint64_t)v;
    const uint64_t old = atomicAdd((unsigned long long*)lo_p, (unsigned long long)lo);
    const uint64_t h = (uint64_t)(v >> 64) + ((old + lo < old) ? 1ull : 0ull);
    if (h) atomicAdd((unsigned long long*)hi_p, (unsigned long long)h);
}

struct Work {   // shared-memory working set of one tile (after the column stages)
    uint64_t mbar[4];               // first: the no-key path allocates only these
    uint64_t skey[2][GTILE];
    uint16_t sidx[2][GTILE];
    uint16_t srun[GTILE];
    uint16_t rstart[GTILE + 2];
    union {
        uint32_t whist[GNW][256];   // in-tile sort: per-warp digit counters
        struct {
            uint64_t alo[PCH][UCAP];   // reduction: per-run split sums (low halves) / min / max
            int64_t ahi[PCH][UCAP];    //            per-run split sums (high halves)
        };
    };
    uint32_t tstart[256];
    uint32_t s_w[GNW];
    uint64_t s_min[GNW], s_max[GNW];
    uint64_t s_kmin[TQP_MAX_KEYS];
    int s_kshift[TQP_MAX_KEYS];
    int64_t s_pb;
    uint32_t s_m, s_U;
};
constexpr int WRUNS = 4;   // runs a warp may span for the warp-reduction path
// Per-warp run partials of the warp-reduction path (aliases the tile's sort key
// buffers, which are dead once the partial keys are written): combined per run
// without shared-memory atomics (64-bit ones are compare-and-swap loops).
struct WarpPart {
    uint64_t lo[PCH][GNW][WRUNS];
    int64_t hi[PCH][GNW][WRUNS];
    uint32_t r0[GNW];
    uint8_t nr[PCH][GNW];
};
static_assert(sizeof(WarpPart) <= sizeof(uint64_t) * 2 * GTILE, "WarpPart fits the sort key buffers");


// One stable LSD pass over positions [0, m) of the tile: rank by the 8-bit digit
// at `shift` (a key's peers in its warp from one ballot per digit bit), then scatter to
// the other buffer.
__device__ __forceinline__ void tile_pass(Work& w, int src, int m, int shift) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int dst = src ^ 1;
    for (int d = lane; d < 256; d += 32) w.whist[warp][d] = 0;
    __syncwarp();
    uint64_t k[GPT];
    uint16_t ix[GPT];
    uint32_t rk[GPT];
    const unsigned lt = lanemask_lt();
#pragma unroll
    for (int i = 0; i < GPT; i++) {
        const int q = warp * 32 * GPT + i * 32 + lane;
        const bool valid = q < m;
        if (valid) { k[i] = w.skey[src][q]; ix[i] = w.sidx[src][q]; }
        const unsigned vm = __ballot_sync(0xffffffffu, valid);
        const uint32_t dd = valid ? ((uint32_t)(k[i] >> shift) & 255u) : 0u;
        unsigned pe = vm;
#pragma unroll
        for (int b = 0; b < 8; b++) {   // peers by one ballot per digit bit
            const unsigned bb = __ballot_sync(0xffffffffu, (dd >> b) & 1u);
            pe &= ((dd >> b) & 1u) ? bb : ~bb;
        }
        if (valid) {
            const uint32_t d = dd;
            const unsigned peers = pe;
            const uint32_t before = w.whist[warp][d];
            rk[i] = before + __popc(peers & lt);
            __syncwarp(vm);
            if (lane == 31 - __clz(peers)) w.whist[warp][d] = before + __popc(peers);
            __syncwarp(vm);
        }
    }
    __syncthreads();
    uint32_t cnt = 0;
#pragma unroll
    for (int ww = 0; ww < GNW; ww++) {
        const uint32_t c = w.whist[ww][tid];
        w.whist[ww][tid] = cnt;
        cnt += c;
    }
    w.tstart[tid] = bscan256(cnt, w.s_w);
    __syncthreads();
#pragma unroll
    for (int i = 0; i < GPT; i++) {
        const int q = warp * 32 * GPT + i * 32 + lane;
        if (q < m) {
            const uint32_t d = (uint32_t)(k[i] >> shift) & 255u;
            const uint32_t p = w.tstart[d] + w.whist[warp][d] + rk[i];
            w.skey[dst][p] = k[i];
            w.sidx[dst][p] = ix[i];
        }
    }
    __syncthreads();
}

__device__ void process_tile(const Phase1Args& a, const uint8_t* st, Work& w, int64_t t) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t row0 = t * GTILE;
    const int nrows = (int)min((int64_t)GTILE, a.n - row0);
    // 1. predicates + packed key; rows r = i*GNT + tid
    uint64_t key[GPT];
    unsigned bal[GPT];
    uint64_t kmin = ~0ull, kmax = 0;
    if (tid == 0) w.s_m = 0;
    bool pass[GPT];
#pragma unroll
    for (int i = 0; i < GPT; i++) {
        pass[i] = !a.ts.never && i * GNT + tid < nrows;
        key[i] = 0;
    }
    // predicates: one interval term per column (common.cuh), dtype dispatch hoisted
    for (int q = 0; q < a.ts.n; q++) {
        const Term& tm = a.ts.t[q];
        const uint8_t* col = st + a.uoff[tm.col];
        const bool neg = tm.neg;
        if (tm.dt == TQP_I64) {
#pragma unroll
            for (int i = 0; i < GPT; i++)
                pass[i] &= term64(reinterpret_cast<const unsigned long long*>(col)[i * GNT + tid], tm.lo, tm.width, neg);
        } else if (tm.dt == TQP_I32) {
#pragma unroll
            for (int i = 0; i < GPT; i++)
                pass[i] &= term32(reinterpret_cast<const uint32_t*>(col)[i * GNT + tid], (uint32_t)tm.lo,
                                  (uint32_t)tm.width, neg);
        } else {
#pragma unroll
            for (int i = 0; i < GPT; i++)
                pass[i] &= term32(col[i * GNT + tid], (uint32_t)tm.lo, (uint32_t)tm.width, neg);
        }
    }
    // packed key: column 0 most significant (reading R12), each column as (value - min)
    for (int c = 0; c < a.n_keys; c++) {
        const int u = a.kcol[c];
        const uint8_t* col = st + a.uoff[u];
        const int sh = w.s_kshift[c];
        const uint64_t mn = w.s_kmin[c];
        switch (a.udt[u]) {
            case TQP_U8:
#pragma unroll
                for (int i = 0; i < GPT; i++) key[i] |= ((uint64_t)col[i * GNT + tid] - mn) << sh;
                break;
            case TQP_I32:
#pragma unroll
                for (int i = 0; i < GPT; i++)
                    key[i] |= ((uint64_t)((uint32_t)reinterpret_cast<const int32_t*>(col)[i * GNT + tid] ^ 0x80000000u) - mn)
                              << sh;
                break;
            default:
#pragma unroll
                for (int i = 0; i < GPT; i++)
                    key[i] |= (((uint64_t)reinterpret_cast<const long long*>(col)[i * GNT + tid] ^ 0x8000000000000000ull) - mn)
                              << sh;
        }
    }
#pragma unroll
    for (int i = 0; i < GPT; i++) {
        if (pass[i]) {
            kmin = min(kmin, key[i]);
            kmax = max(kmax, key[i]);
        }
        bal[i] = __ballot_sync(0xffffffffu, pass[i]);
    }
    for (int o = 16; o > 0; o >>= 1) {
        kmin = min(kmin, __shfl_xor_sync(0xffffffffu, kmin, o));
        kmax = max(kmax, __shfl_xor_sync(0xffffffffu, kmax, o));
    }
    if (lane == 0) { w.s_min[warp] = kmin; w.s_max[warp] = kmax; }
    __syncthreads();
    kmin = ~0ull;
    kmax = 0;
    for (int ww = 0; ww < GNW; ww++) { kmin = min(kmin, w.s_min[ww]); kmax = max(kmax, w.s_max[ww]); }
    const unsigned lt = lanemask_lt();
    const int p0 = tid * GPT;
    int m;
    const uint64_t* sk;
    const uint16_t* si;
    if (kmax >= kmin && kmax - kmin < (uint64_t)CBINS) {
        // 2'-4'. small key range: one-pass counting sort. Each passing row claims a
        //        rank in its key's bin (warp-aggregated shared atomics), the bin scan
        //        gives bin starts, and the non-empty bins are exactly the segments
        //        (uniqueConsecutive) -- no compaction pass, no LSD passes, no head scan.
        uint32_t* cnt = &w.whist[0][0];
        uint16_t* rid = reinterpret_cast<uint16_t*>(w.skey[1]);
        const int R = (int)(kmax - kmin) + 1;
        for (int b = tid; b < R; b += GNT) cnt[b] = 0;
        __syncthreads();
        uint32_t rk[GPT], dk[GPT];
#pragma unroll
        for (int i = 0; i < GPT; i++) {
            dk[i] = pass[i] ? (uint32_t)(key[i] - kmin) : (0x80000000u | (uint32_t)lane);
            const unsigned peers = __match_any_sync(0xffffffffu, dk[i]);
            const uint32_t leader = 31 - __clz(peers);
            uint32_t old = 0;
            if (pass[i] && lane == leader) old = atomicAdd(&cnt[dk[i]], (uint32_t)__popc(peers));
            rk[i] = old | (leader << 16) | ((uint32_t)__popc(peers & lt) << 24);
        }
#pragma unroll
        for (int i = 0; i < GPT; i++) {
            const uint32_t b = __shfl_sync(0xffffffffu, rk[i] & 0xFFFFu, (rk[i] >> 16) & 31u);
            rk[i] = b + (rk[i] >> 24);
        }
        __syncthreads();
        // bin scan: thread t owns bins [8t, 8t+8); (rows, non-empty bins) packed in one word
        constexpr int BPT = CBINS / GNT;
        uint32_t c[BPT], rows = 0, runs = 0;
#pragma unroll
        for (int j = 0; j < BPT; j++) {
            const int bidx = tid * BPT + j;
            c[j] = bidx < R ? cnt[bidx] : 0u;
            rows += c[j];
            runs += c[j] ? 1u : 0u;
        }
        const uint32_t ex = bscan256(rows | (runs << 16), w.s_w);
        uint32_t start = ex & 0xFFFFu, run = ex >> 16;
#pragma unroll
        for (int j = 0; j < BPT; j++) {
            const int bidx = tid * BPT + j;
            if (c[j]) {
                w.rstart[run] = (uint16_t)start;
                rid[bidx] = (uint16_t)run;
                run++;
            }
            if (bidx < R) cnt[bidx] = start;
            start += c[j];
        }
        if (tid == GNT - 1) {
            w.s_m = start;
            w.s_U = run;
            w.rstart[run] = (uint16_t)start;
            int64_t pb = run ? (int64_t)atomicAdd(a.P_counter, (unsigned long long)run) : 0;
            if (pb + run > a.cap) { atomicOr(a.overflow, 2); pb = -1; }
            w.s_pb = pb;
        }
        __syncthreads();
#pragma unroll
        for (int i = 0; i < GPT; i++) {
            if (pass[i]) {
                const uint32_t pos = cnt[dk[i]] + rk[i];
                w.skey[0][pos] = dk[i];
                w.sidx[0][pos] = (uint16_t)(i * GNT + tid);
                w.srun[pos] = rid[dk[i]];
            }
        }
        __syncthreads();
        m = (int)w.s_m;
        sk = w.skey[0];
        si = w.sidx[0];
    } else {
    // 2. compact passing rows into sort buffer 0 (warp-aggregated slot claims)
    #pragma unroll
    for (int i = 0; i < GPT; i++) {
        if (!bal[i]) continue;
        uint32_t base = 0;
        if (lane == 0) base = atomicAdd(&w.s_m, (uint32_t)__popc(bal[i]));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (bal[i] & (1u << lane)) {
            const uint32_t c = base + __popc(bal[i] & lt);
            w.skey[0][c] = key[i] - kmin;
            w.sidx[0][c] = (uint16_t)(i * GNT + tid);
        }
    }
    __syncthreads();
    m = (int)w.s_m;
    // 3. in-tile stable LSD radix sort over the bits that vary in this tile
    const int bits = (m > 0 && kmax != kmin) ? 64 - __clzll(kmax - kmin) : 0;
    const int passes = (bits + 7) / 8;
    for (int p = 0; p < passes; p++) tile_pass(w, p & 1, m, 8 * p);
    const int fin = passes & 1;
    sk = w.skey[fin];
    si = w.sidx[fin];
    // 4. segment boundaries (uniqueConsecutive): blocked positions p = tid*GPT + q
    uint32_t heads = 0;
#pragma unroll
    for (int q = 0; q < GPT; q++) {
        const int p = p0 + q;
        if (p < m && (p == 0 || sk[p] != sk[p - 1])) heads++;
    }
    const uint32_t hex = bscan256(heads, w.s_w);
    {
        uint32_t r = hex;
#pragma unroll
        for (int q = 0; q < GPT; q++) {
            const int p = p0 + q;
            if (p < m) {
                if (p == 0 || sk[p] != sk[p - 1]) { w.rstart[r] = (uint16_t)p; r++; }
                w.srun[p] = (uint16_t)(r - 1);
            }
        }
        if (tid == GNT - 1) {
            w.s_U = r;
            w.rstart[r] = (uint16_t)m;
            int64_t pb = r ? (int64_t)atomicAdd(a.P_counter, (unsigned long long)r) : 0;
            if (pb + r > a.cap) { atomicOr(a.overflow, 2); pb = -1; }
            w.s_pb = pb;
        }
    }
    __syncthreads();
    }
    const int U = (int)w.s_U;
    const int64_t pb = w.s_pb;
    if (U == 0 || pb < 0) return;
    // 5. partial records: key and count; per-run accumulators live in shared memory
    //    when the tile has few runs (the partial slots are private to this tile),
    //    else directly in the tile's global partial slots
    TQP_DCHECK(pb + U <= a.cap);
    for (int u = tid; u < U; u += GNT) {
        a.pkey[pb + u] = sk[w.rstart[u]] + kmin;
        a.pcount[pb + u] = (int64_t)w.rstart[u + 1] - w.rstart[u];
    }
    const bool sm_acc = U <= UCAP;
    // 6. per (op, expression) pair: (A) evaluate the expression for this thread's
    //    rows in row order into the spare sort buffer, (B) reduce it in sorted
    //    order per run. Sums are kept split (sum of low 32-bit halves, sum of high
    //    halves): exact for a tile and independent of the order of additions.
    const bool any = p0 < m;
    const int pl = min(p0 + GPT, m) - 1;
    int prow[GPT], prun[GPT];
#pragma unroll
    for (int q = 0; q < GPT; q++) {
        const int p = p0 + q;
        prow[q] = p < m ? si[p] : 0;
        prun[q] = p < m ? w.srun[p] : -1;
    }
    const int r0 = prun[0];
    const int rl = any ? w.srun[pl] : -1;
    const int wr0 = __shfl_sync(0xffffffffu, r0, 0);
    const bool uniform = __all_sync(0xffffffffu, any && r0 == rl && r0 == wr0);
    int ovf = 0;
    // the runs this warp's 128 sorted positions span
    const uint32_t rlo = __reduce_min_sync(0xffffffffu, any ? (uint32_t)r0 : 0xFFFFFFFFu);
    const uint32_t rhi = __reduce_max_sync(0xffffffffu, any ? (uint32_t)rl : 0u);
    const bool wsmall = sm_acc && rlo != 0xFFFFFFFFu && rhi == rlo;
    WarpPart& wp = *reinterpret_cast<WarpPart*>(&w.skey[0][0]);
    for (int j = 0; j < a.n_pairs; j++) {
        const int op = a.prop[j];
        const int jj = j % PCH;
        // (A) evaluate the expression at this thread's sorted positions (passing rows
        //     only; the in-tile sort is stable, so rows ascend within a run). Products
        //     wrap; overflow is excluded by magnitude bounds: with b_f = bit length of
        //     max |term f| over the thread's rows, |prod| < 2^(sum b_f), so sum b_f <= 63
        //     (and no add overflow) proves every product exact. Otherwise the rows are
        //     re-evaluated with exact per-operation checks.
        int64_t vv[GPT];
#pragma unroll
        for (int q = 0; q < GPT; q++) vv[q] = 1;
        const int nf = a.pnf[j];
        if (any) {
            int bsum = 0;
            bool addsafe = true;
            for (int f = 0; f < nf; f++) {
                const int c = a.pfc[j][f];
                const uint8_t* col = st + a.uoff[c];
                const int64_t add = a.padd[j][f];
                const bool neg = a.psign[j][f] < 0;
                int64_t x[GPT];
                switch (a.udt[c]) {
                    case TQP_U8:
#pragma unroll
                        for (int q = 0; q < GPT; q++) x[q] = (int64_t)col[prow[q]];
                        break;
                    case TQP_I32:
#pragma unroll
                        for (int q = 0; q < GPT; q++) x[q] = (int64_t)reinterpret_cast<const int32_t*>(col)[prow[q]];
                        break;
                    default:
#pragma unroll
                        for (int q = 0; q < GPT; q++) x[q] = (int64_t)reinterpret_cast<const long long*>(col)[prow[q]];
                }
                uint64_t mx = 0, mt = 0;
#pragma unroll
                for (int q = 0; q < GPT; q++) {
                    const int64_t t = neg ? add - x[q] : add + x[q];
                    mx |= (uint64_t)(x[q] ^ (x[q] >> 63));
                    mt |= (uint64_t)(t ^ (t >> 63));
                    vv[q] = f == 0 ? t : vv[q] * t;
                }
                // |x| <= mx + 1 and |add| < 2^61 keep add +- x exact
                addsafe = addsafe && (64 - __clzll(mx)) <= 61 && add < (1ll << 61) && add > -(1ll << 61);
                bsum += (64 - __clzll(mt)) + 1;
            }
            if (!addsafe || bsum > 63) {   // rare: exact re-evaluation with checks
                bool ov[GPT];
#pragma unroll
                for (int q = 0; q < GPT; q++) { vv[q] = 1; ov[q] = false; }
                for (int f = 0; f < nf; f++) {
                    const int c = a.pfc[j][f];
                    const int64_t add = a.padd[j][f];
                    const bool neg = a.psign[j][f] < 0;
#pragma unroll
                    for (int q = 0; q < GPT; q++) {
                        const int64_t x = scol(st, a.uoff[c], a.udt[c], prow[q]);
                        int64_t t;
                        if (neg) {
                            t = add - x;
                            ov[q] |= ((add ^ x) & (add ^ t)) < 0;
                        } else {
                            t = add + x;
                            ov[q] |= ((add ^ t) & (x ^ t)) < 0;
                        }
                        if (f == 0) {
                            vv[q] = t;
                        } else {
                            const int64_t lo = vv[q] * t;
                            ov[q] |= __mul64hi(vv[q], t) != (lo >> 63);
                            vv[q] = lo;
                        }
                    }
                }
#pragma unroll
                for (int q = 0; q < GPT; q++)
                    if (ov[q] && prun[q] >= 0) ovf = 1;
            }
        }
        if (jj == 0) {   // (re)initialise the accumulators of this chunk of pairs
            const int np = min(PCH, a.n_pairs - j);
            if (sm_acc) {
                for (int idx = tid; idx < np * U; idx += GNT) {
                    const int k2 = idx / U, u = idx - k2 * U;
                    const int op2 = a.prop[j + k2];
                    w.alo[k2][u] = op2 == P_SUM ? 0ull : (op2 == P_MIN ? (uint64_t)INT64_MAX : (uint64_t)INT64_MIN);
                    w.ahi[k2][u] = 0;
                }
            } else {
                for (int u = tid; u < U; u += GNT)
                    for (int k2 = 0; k2 < np; k2++) {
                        const int op2 = a.prop[j + k2];
                        a.plo[j + k2][pb + u] =
                            op2 == P_SUM ? 0ull : (op2 == P_MIN ? (uint64_t)INT64_MAX : (uint64_t)INT64_MIN);
                        if (op2 == P_SUM) a.phi[j + k2][pb + u] = 0;
                    }
            }
            __syncthreads();
        }
        // (B) reduce in sorted order
        uint64_t lo = op == P_SUM ? 0ull : (op == P_MIN ? (uint64_t)INT64_MAX : (uint64_t)INT64_MIN);
        int64_t hi = 0;
        unsigned long long* dl = sm_acc ? (unsigned long long*)&w.alo[jj][0] : (unsigned long long*)&a.plo[j][pb];
        unsigned long long* dh = sm_acc ? (unsigned long long*)&w.ahi[jj][0]
                                        : (unsigned long long*)(op == P_SUM ? &a.phi[j][pb] : nullptr);
        auto flush = [&](int run) {
            if (op == P_SUM) {
                atomicAdd(dl + run, (unsigned long long)lo);
                atomicAdd(dh + run, (unsigned long long)hi);
            } else if (op == P_MIN) {
                atomicMin((long long*)(dl + run), (long long)lo);
            } else {
                atomicMax((long long*)(dl + run), (long long)lo);
            }
        };
        // Sums over a warp whose 128 sorted positions span at most 4 runs: per run, the
        // thread's values are split into 24-bit pieces (1, 2 or 3 by the warp's magnitude
        // bound) whose warp totals fit 32 bits, summed by redux.sync and recombined exactly
        // into the split (low-half, high-half) form.
        if (op == P_SUM && wsmall && rlo == rhi) {   // one run: serial + butterfly, no atomics
            uint64_t l2 = 0;
            int64_t h2 = 0;
#pragma unroll
            for (int q = 0; q < GPT; q++) {
                if (prun[q] < 0) break;
                l2 += (uint64_t)(uint32_t)vv[q];
                h2 += vv[q] >> 32;
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                l2 += __shfl_xor_sync(0xffffffffu, l2, o);
                h2 += __shfl_xor_sync(0xffffffffu, h2, o);
            }
            if (lane == 0) {
                wp.lo[jj][warp][0] = l2;
                wp.hi[jj][warp][0] = h2;
                wp.r0[warp] = rlo;
                wp.nr[jj][warp] = 1;
            }
        } else {
        if (sm_acc && lane == 0) wp.nr[jj][warp] = 0;
        int cur = r0;
#pragma unroll
        for (int q = 0; q < GPT; q++) {
            if (prun[q] < 0) break;
            if (prun[q] != cur) {
                flush(cur);
                lo = op == P_SUM ? 0ull : (op == P_MIN ? (uint64_t)INT64_MAX : (uint64_t)INT64_MIN);
                hi = 0;
                cur = prun[q];
            }
            const int64_t v = vv[q];
            if (op == P_SUM) { lo += (uint64_t)(uint32_t)v; hi += (v >> 32); }
            else if (op == P_MIN) lo = (uint64_t)min((int64_t)lo, v);
            else lo = (uint64_t)max((int64_t)lo, v);
        }
        if (uniform) {
            for (int o = 16; o > 0; o >>= 1) {
                const uint64_t xl = __shfl_xor_sync(0xffffffffu, lo, o);
                if (op == P_SUM) {
                    lo += xl;
                    hi += __shfl_xor_sync(0xffffffffu, hi, o);
                } else if (op == P_MIN) {
                    lo = (uint64_t)min((int64_t)lo, (int64_t)xl);
                } else {
                    lo = (uint64_t)max((int64_t)lo, (int64_t)xl);
                }
            }
            if (lane == 0) flush(cur);
        } else if (any) {
            flush(cur);
        }
        }
        if (jj == PCH - 1 || j == a.n_pairs - 1) __syncthreads();
        if (sm_acc && (jj == PCH - 1 || j == a.n_pairs - 1)) {   // chunk complete: write its partials
            const int jb = j - jj, np = jj + 1;
            for (int idx = tid; idx < np * U; idx += GNT) {
                const int k2 = idx / U, u = idx - k2 * U;
                uint64_t lo2 = w.alo[k2][u];
                int64_t hi2 = w.ahi[k2][u];
                if (a.prop[jb + k2] == P_SUM) {
#pragma unroll
                    for (int ww = 0; ww < GNW; ww++) {   // warp-reduction partials of this run
                        const uint32_t d = (uint32_t)u - wp.r0[ww];
                        if (d < (uint32_t)wp.nr[k2][ww]) { lo2 += wp.lo[k2][ww][d]; hi2 += wp.hi[k2][ww][d]; }
                    }
                    a.phi[jb + k2][pb + u] = hi2;
                }
                a.plo[jb + k2][pb + u] = lo2;
            }
            __syncthreads();
        }
    }
    if (ovf) atomicOr(a.overflow, 1);
}

// No group keys (e.g. Q6's fused filter + sum): the tile sort is the identity and
// there is one segment, so every thread keeps its (op, expression) accumulators in
// registers across all the tiles of the persistent loop; one partial record per CTA.
struct NoKeyAcc {
    uint64_t lo[PCH];
    int64_t hi[PCH];
    int64_t count;
    int ovf;
};

struct NoKeyWork {   // the no-key path's shared memory after the stages (aliases Work)
    uint64_t mbar[4];
    uint64_t pad[4];
    uint16_t list[GNW][GTILE / GNW];   // per warp: the tile rows that passed the predicates
};
static_assert(offsetof(Work, mbar) == 0 && offsetof(NoKeyWork, mbar) == 0, "mbarriers lead both layouts");

// One (op, expression) pair on one row: prod_f (add_f + sign_f * x_f), 64-bit with
// overflow detection (the exact fallback re-runs on int128).
__device__ __forceinline__ int64_t pair_value(const Phase1Args& a, const uint8_t* st, int jj, int row, bool& ov) {
    int64_t vv = 1;
    const int nf = a.pnf[jj];
    for (int f = 0; f < nf; f++) {
        const int c = a.pfc[jj][f];
        const uint8_t* col = st + a.uoff[c];
        const int64_t add = a.padd[jj][f];
        int64_t x;
        switch (a.udt[c]) {
            case TQP_U8: x = (int64_t)col[row]; break;
            case TQP_I32: x = (int64_t)reinterpret_cast<const int32_t*>(col)[row]; break;
            default: x = (int64_t)reinterpret_cast<const long long*>(col)[row];
        }
        int64_t tt;
        if (a.psign[jj][f] < 0) {
            tt = add - x;
            ov |= ((add ^ x) & (add ^ tt)) < 0;
        } else {
            tt = add + x;
            ov |= ((add ^ tt) & (x ^ tt)) < 0;
        }
        if (f == 0) {
            vv = tt;
        } else if ((uint64_t)(vv + 0x80000000ll) < 0x100000000ull && (uint64_t)(tt + 0x80000000ll) < 0x100000000ull) {
            vv = (int64_t)(int32_t)vv * (int64_t)(int32_t)tt;
        } else {
            const int64_t lo = vv * tt;
            ov |= __mul64hi(vv, tt) != (lo >> 63);
            vv = lo;
        }
    }
    return vv;
}

// Each thread owns GPT consecutive rows of the stage (vector shared-memory loads);
// rows that pass are listed per warp, and the aggregate expressions are evaluated on
// the listed rows only (one lane per row), so a selective filter (Q6) pays for the
// predicates on every row and for the arithmetic on the passing ones.
__device__ __forceinline__ void process_tile_nokey(const Phase1Args& a, const uint8_t* st, int64_t t, NoKeyAcc& acc,
                                                   NoKeyWork& nw) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nrows = (int)min((int64_t)GTILE, a.n - t * GTILE);
    const int r0 = tid * GPT;
    static_assert(GPT == 4, "vector loads below assume 4 rows per thread");
    bool pass[GPT];
#pragma unroll
    for (int i = 0; i < GPT; i++) pass[i] = !a.ts.never && r0 + i < nrows;
    for (int q = 0; q < a.ts.n; q++) {
        const Term& tm = a.ts.t[q];
        const uint8_t* col = st + a.uoff[tm.col];
        const bool neg = tm.neg;
        if (tm.dt == TQP_I64) {
            const ulonglong2 u0 = reinterpret_cast<const ulonglong2*>(col)[2 * tid];
            const ulonglong2 u1 = reinterpret_cast<const ulonglong2*>(col)[2 * tid + 1];
            pass[0] &= term64(u0.x, tm.lo, tm.width, neg);
            pass[1] &= term64(u0.y, tm.lo, tm.width, neg);
            pass[2] &= term64(u1.x, tm.lo, tm.width, neg);
            pass[3] &= term64(u1.y, tm.lo, tm.width, neg);
        } else if (tm.dt == TQP_I32) {
            const uint4 u = reinterpret_cast<const uint4*>(col)[tid];
            const uint32_t lo = (uint32_t)tm.lo, wd = (uint32_t)tm.width;
            pass[0] &= term32(u.x, lo, wd, neg);
            pass[1] &= term32(u.y, lo, wd, neg);
            pass[2] &= term32(u.z, lo, wd, neg);
            pass[3] &= term32(u.w, lo, wd, neg);
        } else {
            const uint32_t u = reinterpret_cast<const uint32_t*>(col)[tid];
            const uint32_t lo = (uint32_t)tm.lo, wd = (uint32_t)tm.width;
#pragma unroll
            for (int i = 0; i < GPT; i++) pass[i] &= term32((u >> (8 * i)) & 0xFFu, lo, wd, neg);
        }
    }
    uint16_t* L = nw.list[warp];
    const unsigned lt = lanemask_lt();
    int cnt = 0;
#pragma unroll
    for (int i = 0; i < GPT; i++) {
        const unsigned b = __ballot_sync(0xffffffffu, pass[i]);
        if (pass[i]) L[cnt + __popc(b & lt)] = (uint16_t)(r0 + i);
        cnt += __popc(b);
        acc.count += pass[i] ? 1 : 0;
    }
    if (cnt == 0) return;
    __syncwarp();
    for (int k = lane; k < cnt; k += 32) {
        const int row = L[k];
        bool ov = false;
#pragma unroll
        for (int jj = 0; jj < PCH; jj++) {
            if (jj >= a.n_pairs) break;
            const int op = a.prop[jj];
            const int64_t v = pair_value(a, st, jj, row, ov);
            if (op == P_SUM) { acc.lo[jj] += (uint64_t)(uint32_t)v; acc.hi[jj] += (v >> 32); }
            else if (op == P_MIN) acc.lo[jj] = (uint64_t)min((int64_t)acc.lo[jj], v);
            else acc.lo[jj] = (uint64_t)max((int64_t)acc.lo[jj], v);
        }
        if (ov) acc.ovf = 1;
    }
}

// End of the persistent loop: reduce the CTA's register accumulators and emit one
// partial record (key 0) if any row passed.
__device__ void flush_nokey(const Phase1Args& a, NoKeyAcc& acc, Work& w) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    __shared__ int64_t s_cnt[GNW];
    __shared__ uint64_t s_lo[GNW][PCH];
    __shared__ int64_t s_hi[GNW][PCH];
    __shared__ int64_t s_pb;
    int64_t cnt = acc.count;
    for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
#pragma unroll
    for (int jj = 0; jj < PCH; jj++) {
        const int op = jj < a.n_pairs ? a.prop[jj] : P_SUM;
        for (int o = 16; o > 0; o >>= 1) {
            const uint64_t xl = __shfl_xor_sync(0xffffffffu, acc.lo[jj], o);
            const int64_t xh = __shfl_xor_sync(0xffffffffu, acc.hi[jj], o);
            if (op == P_SUM) { acc.lo[jj] += xl; acc.hi[jj] += xh; }
            else if (op == P_MIN) acc.lo[jj] = (uint64_t)min((int64_t)acc.lo[jj], (int64_t)xl);
            else acc.lo[jj] = (uint64_t)max((int64_t)acc.lo[jj], (int64_t)xl);
        }
        if (lane == 0) { s_lo[warp][jj] = acc.lo[jj]; s_hi[warp][jj] = acc.hi[jj]; }
    }
    if (lane == 0) s_cnt[warp] = cnt;
    if (acc.ovf) atomicOr(a.overflow, 1);
    __syncthreads();
    if (tid == 0) {
        int64_t c = 0;
        for (int ww = 0; ww < GNW; ww++) c += s_cnt[ww];
        int64_t pb = -1;
        if (a.direct) {
            pb = blockIdx.x;   // fixed slot (count 0 when nothing passed)
        } else if (c > 0) {
            pb = (int64_t)atomicAdd(a.P_counter, 1ull);
            if (pb + 1 > a.cap) { atomicOr(a.overflow, 2); pb = -1; }
        }
        if (pb >= 0) {
            a.pkey[pb] = 0;
            a.pcount[pb] = c;
        }
        s_pb = pb;
    }
    __syncthreads();
    const int64_t pb = s_pb;
    if (pb >= 0 && tid < a.n_pairs && tid < PCH) {
        const int jj = tid, op = a.prop[jj];
        uint64_t lo = op == P_SUM ? 0ull : (op == P_MIN ? (uint64_t)INT64_MAX : (uint64_t)INT64_MIN);
        int64_t hi = 0;
        for (int ww = 0; ww < GNW; ww++) {
            if (op == P_SUM) { lo += s_lo[ww][jj]; hi += s_hi[ww][jj]; }
            else if (op == P_MIN) lo = (uint64_t)min((int64_t)lo, (int64_t)s_lo[ww][jj]);
            else lo = (uint64_t)max((int64_t)lo, (int64_t)s_lo[ww][jj]);
        }
        a.plo[jj][pb] = lo;
        if (op == P_SUM) a.phi[jj][pb] = hi;
    }
    (void)w;
}

// The persistent tile loop shared by the phase-1 kernels: tiles t = blockIdx.x +
// k * gridDim.x are streamed into NS shared-memory stages with TMA bulk copies
// (mbarrier completion; stage s is refilled as soon as every thread is done with it);
// tail tiles and unaligned columns take plain cooperative loads.
template <int NT, bool ABORTABLE = false, int RPT = GPT, typename F>
__device__ __forceinline__ void tile_pipeline(const Phase1Args& a, uint8_t* smem, uint64_t* mbar, F&& process) {
    constexpr int TR = NT * RPT;   // rows per tile
    const int NS = a.n_stages;
    const int tid = threadIdx.x;
    auto stage_ptr = [&](int s) { return smem + (size_t)s * a.stage_bytes; };
    auto eligible = [&](int64_t t) { return a.bulk_ok && (t + 1) * TR <= a.n; };
    auto issue = [&](int64_t t, int s) {   // thread 0 only
        mbar_expect_tx(&mbar[s], (uint32_t)a.stage_bytes);
        for (int c = 0; c < a.n_ucols; c++) {
            const uint32_t es = a.udt[c] == TQP_U8 ? 1 : a.udt[c] == TQP_I32 ? 4 : 8;
            bulk_g2s(stage_ptr(s) + a.uoff[c], (const uint8_t*)a.ucol[c] + t * TR * es, TR * es, &mbar[s]);
        }
    };
    // per stage, as register bit masks (dynamically indexed arrays would live in local
    // memory): pend = a bulk copy is in flight, wpar = the phase parity of the next wait
    uint32_t pend = 0, wpar = 0;
    for (int s = 0; s < NS; s++) {
        const int64_t t = blockIdx.x + (int64_t)s * gridDim.x;
        if (t < a.n_tiles && eligible(t)) {
            if (tid == 0) issue(t, s);
            pend |= 1u << s;
        }
    }
    __shared__ int s_abort;
    for (int64_t k = 0;; k++) {
        const int64_t t = blockIdx.x + k * gridDim.x;
        if (t >= a.n_tiles) break;
        const int s = (int)(k % NS);
        if (ABORTABLE) {   // partial capacity exceeded somewhere: stop (the host takes the sort path)
            if (tid == 0) s_abort = (*reinterpret_cast<volatile int*>(a.overflow) & 2) != 0;
            __syncthreads();
            if (s_abort) {
                if (tid == 0)   // bulk copies still landing in this CTA's stages complete first
                    for (int st = 0; st < NS; st++)
                        if ((pend >> st) & 1u) mbar_wait(&mbar[st], (wpar >> st) & 1u);
                break;
            }
        }
        if (eligible(t)) {
            mbar_wait(&mbar[s], (wpar >> s) & 1u);
            wpar ^= 1u << s;
            pend &= ~(1u << s);
        } else {   // tail tile or unaligned columns: plain cooperative loads
            const int64_t row0 = t * TR;
            const int nrows = (int)min((int64_t)TR, a.n - row0);
            for (int c = 0; c < a.n_ucols; c++) {
                for (int r = tid; r < TR; r += NT) {   // rows past the end are zero-filled
                    if (r >= nrows) {
                        const uint32_t es = a.udt[c] == TQP_U8 ? 1 : a.udt[c] == TQP_I32 ? 4 : 8;
                        for (uint32_t b = 0; b < es; b++) stage_ptr(s)[a.uoff[c] + r * es + b] = 0;
                        continue;
                    }
                    switch (a.udt[c]) {
                        case TQP_U8: stage_ptr(s)[a.uoff[c] + r] = ((const uint8_t*)a.ucol[c])[row0 + r]; break;
                        case TQP_I32:
                            reinterpret_cast<int32_t*>(stage_ptr(s) + a.uoff[c])[r] = ((const int32_t*)a.ucol[c])[row0 + r];
                            break;
                        default:
                            reinterpret_cast<long long*>(stage_ptr(s) + a.uoff[c])[r] =
                                ((const long long*)a.ucol[c])[row0 + r];
                    }
                }
            }
            __syncthreads();
        }
        process(stage_ptr(s), t);
        __syncthreads();   // every thread is done with stage s
        const int64_t t2 = t + (int64_t)NS * gridDim.x;
        if (t2 < a.n_tiles && eligible(t2)) {
            if (tid == 0) {
                fence_proxy_async();
                issue(t2, s);
            }
            pend |= 1u << s;
        }
    }
}

// Blocks per SM the register budget must allow (78 registers, no spills): measured, Q6's
// fused filter + sum at SF10 (the no-key tiles), 116 registers / 2 blocks 0.337 ms, 3 blocks
// 0.277-0.281 ms, 4 blocks (64 registers) 0.308 ms; an explicit minimum of 1 let ptxas take
// 138 registers (1 block, 0.549 ms).
#ifndef TQP_PHASE1_MINB
#define TQP_PHASE1_MINB 3
#endif
__global__ void __launch_bounds__(GNT, TQP_PHASE1_MINB) gb_phase1_kernel(Phase1Args a) {
    extern __shared__ __align__(128) uint8_t smem[];
    const int NS = a.n_stages;   // 2..4 stages in flight per CTA
    Work& w = *reinterpret_cast<Work*>(smem + (size_t)NS * a.stage_bytes);
    const int tid = threadIdx.x;
    if (tid == 0) {
        for (int s = 0; s < NS; s++) mbar_init(&w.mbar[s], 1);
        fence_mbar_init();
        if (a.n_keys > 0) {
            int wd[TQP_MAX_KEYS];
            key_layout(a.krange, a.n_keys, w.s_kmin, w.s_kshift, wd);
        }
    }
    __syncthreads();
    const bool nokey = a.n_keys == 0 && a.n_pairs <= PCH;
    NoKeyAcc nacc;
#pragma unroll
    for (int jj = 0; jj < PCH; jj++) {
        const int op = jj < a.n_pairs ? a.prop[jj] : P_SUM;
        nacc.lo[jj] = op == P_SUM ? 0ull : (op == P_MIN ? (uint64_t)INT64_MAX : (uint64_t)INT64_MIN);
        nacc.hi[jj] = 0;
    }
    nacc.count = 0;
    nacc.ovf = 0;
    if (nokey)
        tile_pipeline<GNT>(a, smem, w.mbar, [&](const uint8_t* st, int64_t t) {
            process_tile_nokey(a, st, t, nacc, reinterpret_cast<NoKeyWork&>(w));
        });
    else
        tile_pipeline<GNT, true>(a, smem, w.mbar, [&](const uint8_t* st, int64_t t) { process_tile(a, st, w, t); });
    if (nokey) flush_nokey(a, nacc, w);
}

// ------------------------------------------------ dense small-domain path
// When the packed keys present in the input are few (D <= DMAX, e.g. TPC-H Q1's four
// (returnflag, linestatus) groups), the tile sort is unnecessary: a presence pass
// marks the packed keys that occur, a prefix popcount gives every present key a
// dense id, and phase 1 adds each passing row into lane-private int64 accumulators
// acc[id][pair][thread] in shared memory (no sort, no atomics, no shuffles). One
// partial record per (CTA, id) goes to the same phase 2. Values are computed with
// wrapping 64-bit arithmetic, exact because a per-thread magnitude bound on the
// inputs proves |value| <= 2^bits (the result mod 2^64 is the true value whenever
// |true value| < 2^63); per-thread sums stay below 2^62 by the host's choice of
// dense_bits. A tile that cannot be proven sets overflow bit 2 and the host re-runs
// the general path.
constexpr int PBITS = 16;   // packed key width the presence bitmap covers
constexpr int DMAX = 16;    // distinct keys of the dense path

struct PresArgs {
    int n_keys;
    const void* kcol[TQP_MAX_KEYS];
    int kdt[TQP_MAX_KEYS];
    int64_t n;
    const unsigned long long* krange;
    uint32_t* bitmap;   // 2^PBITS bits
    int64_t stride;     // > 1: a sample -- 16-row groups 0, stride, 2 * stride, ... (no tail)
};

__global__ void __launch_bounds__(GNT) gb_presence_kernel(PresArgs a) {
    __shared__ uint32_t bm[1 << (PBITS - 5)];
    __shared__ uint64_t kmin[TQP_MAX_KEYS];
    __shared__ int sh[TQP_MAX_KEYS];
    __shared__ int tw;
    const int tid = threadIdx.x;
    if (tid == 0) {
        int wd[TQP_MAX_KEYS];
        key_layout(a.krange, a.n_keys, kmin, sh, wd);
        int s = 0;
        for (int k = 0; k < a.n_keys; k++) s += wd[k];
        tw = s;
    }
    for (int w = tid; w < (1 << (PBITS - 5)); w += GNT) bm[w] = 0;
    __syncthreads();
    if (tw > PBITS) return;
    auto mark = [&](uint32_t b) {
        const uint32_t m = 1u << (b & 31);
        if (!(bm[b >> 5] & m)) atomicOr(&bm[b >> 5], m);
    };
    // body: 16 consecutive rows per thread and step, 16-byte loads (aligned columns)
    constexpr int R = 16;
    bool vec = true;
    for (int k = 0; k < a.n_keys; k++) vec = vec && (uintptr_t)a.kcol[k] % 16 == 0;
    const int64_t stride = a.stride;
    const int64_t nb = vec ? a.n / R / stride : 0;   // 16-row groups visited
    const int64_t gs = (int64_t)gridDim.x * GNT;
    // two row groups (g, g + gs) per step: their loads are in flight together
    constexpr int U = 2;
    for (int64_t g0 = blockIdx.x * (int64_t)GNT + tid; g0 < nb; g0 += U * gs) {
        uint32_t b[U][R];
        bool ok[U];
#pragma unroll
        for (int u = 0; u < U; u++) {
            ok[u] = g0 + u * gs < nb;
#pragma unroll
            for (int i = 0; i < R; i++) b[u][i] = 0;
        }
        for (int k = 0; k < a.n_keys; k++) {
            const int dt = a.kdt[k];
            const uint64_t mn = kmin[k];
            const int s = sh[k];
            if (dt == TQP_U8) {
                uint4 q[U];
#pragma unroll
                for (int u = 0; u < U; u++)
                    q[u] = ok[u] ? __ldcs(reinterpret_cast<const uint4*>(a.kcol[k]) + (g0 + u * gs) * stride) : make_uint4(0, 0, 0, 0);
#pragma unroll
                for (int u = 0; u < U; u++) {
                    const uint32_t wv[4] = {q[u].x, q[u].y, q[u].z, q[u].w};
#pragma unroll
                    for (int i = 0; i < R; i++)
                        b[u][i] |= (uint32_t)(((wv[i >> 2] >> (8 * (i & 3))) & 0xFFu) - (uint32_t)mn) << s;
                }
            } else if (dt == TQP_I32) {
#pragma unroll
                for (int u = 0; u < U; u++) {
                    if (!ok[u]) continue;
                    const int64_t g = (g0 + u * gs) * stride;
#pragma unroll
                    for (int j = 0; j < R / 4; j++) {
                        const uint4 q = __ldcs(reinterpret_cast<const uint4*>(a.kcol[k]) + g * 4 + j);
                        const uint32_t wv[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
                        for (int i = 0; i < 4; i++) b[u][4 * j + i] |= ((wv[i] ^ 0x80000000u) - (uint32_t)mn) << s;
                    }
                }
            } else {
#pragma unroll
                for (int u = 0; u < U; u++) {
                    if (!ok[u]) continue;
                    const int64_t g = (g0 + u * gs) * stride;
#pragma unroll
                    for (int j = 0; j < R / 2; j++) {
                        const ulonglong2 q = __ldcs(reinterpret_cast<const ulonglong2*>(a.kcol[k]) + g * 8 + j);
                        b[u][2 * j] |= (uint32_t)((q.x ^ 0x8000000000000000ull) - mn) << s;
                        b[u][2 * j + 1] |= (uint32_t)((q.y ^ 0x8000000000000000ull) - mn) << s;
                    }
                }
            }
        }
#pragma unroll
        for (int u = 0; u < U; u++)
            if (ok[u])
#pragma unroll
                for (int i = 0; i < R; i++) mark(b[u][i]);
    }
    for (int64_t r = nb * R + blockIdx.x * (int64_t)GNT + tid; stride == 1 && r < a.n; r += gs) {   // tail / unaligned
        uint32_t b = 0;
        for (int k = 0; k < a.n_keys; k++)
            b |= (uint32_t)(key_part(load_as_i64(a.kcol[k], a.kdt[k], r), a.kdt[k]) - kmin[k]) << sh[k];
        mark(b);
    }
    __syncthreads();
    for (int w = tid; w < (1 << (PBITS - 5)); w += GNT)
        if (bm[w]) atomicOr(&a.bitmap[w], bm[w]);
}

// one CTA of 1024 threads: D = popcount of the bitmap; if D <= DMAX, ids in key order
__global__ void __launch_bounds__(1024) gb_dense_ids_kernel(const uint32_t* bitmap, uint8_t* dtab, uint64_t* dkeys,
                                                             int* D_out) {
    __shared__ uint32_t s_w[32];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    constexpr int WPT = (1 << (PBITS - 5)) / 1024;
    uint32_t wv[WPT], c = 0;
#pragma unroll
    for (int j = 0; j < WPT; j++) { wv[j] = bitmap[tid * WPT + j]; c += __popc(wv[j]); }
    uint32_t x = c;
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) s_w[warp] = x;
    __syncthreads();
    if (warp == 0) {
        uint32_t v = s_w[lane], z = v;
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, z, o);
            if (lane >= o) z += y;
        }
        s_w[lane] = z - v;
        if (lane == 31) *D_out = (int)z;
        __syncwarp();
    }
    __syncthreads();
    uint32_t id = s_w[warp] + x - c;
    const uint32_t D = s_w[31] + 0;   // exclusive prefix of the last warp (total read below)
    (void)D;
#pragma unroll
    for (int j = 0; j < WPT; j++) {
        uint32_t m = wv[j];
        while (m) {
            const int b = __ffs(m) - 1;
            m &= m - 1;
            if (id < (uint32_t)DMAX) {
                const uint32_t bin = (uint32_t)(tid * WPT + j) * 32u + (uint32_t)b;
                dtab[bin] = (uint8_t)id;
                dkeys[id] = bin;
            }
            id++;
        }
    }
}

struct DenseHdr {
    uint64_t mbar[4];
    uint64_t kmin[TQP_MAX_KEYS];
    int kshift[TQP_MAX_KEYS];
    int64_t dcnt[DMAX];
    int64_t drec[DMAX];
    int bad;
};

// 4 consecutive rows (thread-contiguous) of a staged column, sign/zero-extended
__device__ __forceinline__ void load4(const uint8_t* col, int dt, int tid, int64_t (&x)[GPT]) {
    if (dt == TQP_I64) {
        const longlong2 u0 = reinterpret_cast<const longlong2*>(col)[2 * tid];
        const longlong2 u1 = reinterpret_cast<const longlong2*>(col)[2 * tid + 1];
        x[0] = u0.x; x[1] = u0.y; x[2] = u1.x; x[3] = u1.y;
    } else if (dt == TQP_I32) {
        const int4 u = reinterpret_cast<const int4*>(col)[tid];
        x[0] = u.x; x[1] = u.y; x[2] = u.z; x[3] = u.w;
    } else {
        const uint32_t u = reinterpret_cast<const uint32_t*>(col)[tid];
#pragma unroll
        for (int i = 0; i < GPT; i++) x[i] = (int64_t)((u >> (8 * i)) & 0xFFu);
    }
}

// DR consecutive rows (thread-contiguous) of a staged column, sign/zero-extended
template <int DR>
__device__ __forceinline__ void loadr(const uint8_t* col, int dt, int tid, int64_t (&x)[DR]) {
    if (dt == TQP_I64) {
#pragma unroll
        for (int h = 0; h < DR / 2; h++) {
            const longlong2 u = reinterpret_cast<const longlong2*>(col)[(DR / 2) * tid + h];
            x[2 * h] = u.x; x[2 * h + 1] = u.y;
        }
    } else if (dt == TQP_I32) {
#pragma unroll
        for (int h = 0; h < DR / 4; h++) {
            const int4 u = reinterpret_cast<const int4*>(col)[(DR / 4) * tid + h];
            x[4 * h] = u.x; x[4 * h + 1] = u.y; x[4 * h + 2] = u.z; x[4 * h + 3] = u.w;
        }
    } else {
#pragma unroll
        for (int h = 0; h < DR / 4; h++) {
            const uint32_t u = reinterpret_cast<const uint32_t*>(col)[(DR / 4) * tid + h];
#pragma unroll
            for (int i = 0; i < 4; i++) x[4 * h + i] = (int64_t)((u >> (8 * i)) & 0xFFu);
        }
    }
}

template <int DR>
__device__ __forceinline__ void loadr_i64(const uint8_t* col, int tid, int64_t (&x)[DR]) {
#pragma unroll
    for (int h = 0; h < DR / 2; h++) {
        const longlong2 u = reinterpret_cast<const longlong2*>(col)[(DR / 2) * tid + h];
        x[2 * h] = u.x; x[2 * h + 1] = u.y;
    }
}

// SPEC (dense kernels specialised on the column types, which removes a per-factor dtype
// switch from every row): bit 0 = every factor column is int64 (fixed-point decimals),
// bit 1 = every key column is u8 (1-character flags, reading R19).
constexpr int SPEC_VI64 = 1, SPEC_KU8 = 2;

__device__ __forceinline__ void load4_i64(const uint8_t* col, int tid, int64_t (&x)[GPT]) {
    const longlong2 u0 = reinterpret_cast<const longlong2*>(col)[2 * tid];
    const longlong2 u1 = reinterpret_cast<const longlong2*>(col)[2 * tid + 1];
    x[0] = u0.x; x[1] = u0.y; x[2] = u1.x; x[3] = u1.y;
}

// DK > 0: the D <= DK present packed keys (ascending) are held in registers and a row's
// dense id is the number of them below its key (DK compares) instead of a dependent
// global lookup in the 64K-entry table; DK = 0: the table.
template <int NT, int SPEC, int DR, int DK>
__device__ __forceinline__ void dense_tile(const Phase1Args& a, const uint8_t* st, int64_t t, const DenseHdr& h,
                                           int64_t* acc, uint32_t* cnt, uint64_t (&mt)[PCH][3],
                                           const uint32_t (&dkr)[DK > 0 ? DK : 1]) {
    const int tid = threadIdx.x;
    const int nrows = (int)min((int64_t)NT * DR, a.n - t * NT * DR);
    const int r0 = tid * DR;
    bool pass[DR];
#pragma unroll
    for (int i = 0; i < DR; i++) pass[i] = !a.ts.never && r0 + i < nrows;
    for (int q = 0; q < a.ts.n; q++) {
        const Term& tm = a.ts.t[q];
        int64_t x[DR];
        loadr<DR>(st + a.uoff[tm.col], tm.dt, tid, x);
        if (tm.dt == TQP_I64) {
#pragma unroll
            for (int i = 0; i < DR; i++) pass[i] &= term64((uint64_t)x[i], tm.lo, tm.width, tm.neg);
        } else {
#pragma unroll
            for (int i = 0; i < DR; i++) pass[i] &= term32((uint32_t)x[i], (uint32_t)tm.lo, (uint32_t)tm.width, tm.neg);
        }
    }
    bool anyp = false;
#pragma unroll
    for (int i = 0; i < DR; i++) anyp |= pass[i];
    if (!anyp) return;
    // packed key (same layout as the general path) -> dense id
    uint32_t kb[DR];
#pragma unroll
    for (int i = 0; i < DR; i++) kb[i] = 0;
    for (int c = 0; c < a.n_keys; c++) {
        const int u = a.kcol[c];
        if (SPEC & SPEC_KU8) {
            const uint32_t mn = (uint32_t)h.kmin[c];
            const int sh = h.kshift[c];
#pragma unroll
            for (int hh = 0; hh < DR / 4; hh++) {
                const uint32_t w = reinterpret_cast<const uint32_t*>(st + a.uoff[u])[(DR / 4) * tid + hh];
#pragma unroll
                for (int i = 0; i < 4; i++) kb[4 * hh + i] |= (((w >> (8 * i)) & 0xFFu) - mn) << sh;
            }
        } else {
            const int dt = a.udt[u];
            int64_t x[DR];
            loadr<DR>(st + a.uoff[u], dt, tid, x);
#pragma unroll
            for (int i = 0; i < DR; i++) kb[i] |= (uint32_t)(key_part(x[i], dt) - h.kmin[c]) << h.kshift[c];
        }
    }
    int id[DR];
    bool unseen = false;   // a key the (sampled) presence bitmap missed: the host redoes it in full
#pragma unroll
    for (int i = 0; i < DR; i++) {
        if (DK > 0) {
            int c = 0;
            bool eq = false;
#pragma unroll
            for (int j = 0; j < (DK > 0 ? DK : 1); j++) {   // unused slots hold 0xFFFFFFFF (> any 16-bit key)
                c += dkr[j] < kb[i];
                eq |= dkr[j] == kb[i];
            }
            id[i] = pass[i] ? (eq ? c : DMAX) : 0;
        } else {
            id[i] = pass[i] ? (int)__ldg(a.dtab + kb[i]) : 0;
        }
        unseen |= id[i] >= a.D;
        pass[i] &= id[i] < a.D;
    }
    if (unseen) atomicOr(a.overflow, 8);
#pragma unroll
    for (int i = 0; i < DR; i++)
        if (pass[i]) cnt[id[i] * NT + tid]++;
    const int np = a.n_pairs;
    int64_t vprev[DR];
#pragma unroll
    for (int i = 0; i < DR; i++) vprev[i] = 1;
#pragma unroll
    for (int jj = 0; jj < PCH; jj++) {
        if (jj >= np) break;
        const int fx = a.pext[jj];   // factors already multiplied into the previous pair's value
        int64_t vv[DR];
#pragma unroll
        for (int i = 0; i < DR; i++) vv[i] = fx ? vprev[i] : 1;
#pragma unroll
        for (int f = 0; f < 3; f++) {
            if (f < fx) continue;
            if (f >= a.pnf[jj]) break;
            int64_t x[DR];
            if (SPEC & SPEC_VI64) loadr_i64<DR>(st + a.poff[jj][f], tid, x);
            else loadr<DR>(st + a.poff[jj][f], a.pdtf[jj][f], tid, x);
            const uint64_t add = (uint64_t)a.padd[jj][f];
            const bool neg = a.psign[jj][f] < 0;
            uint64_t m2 = mt[jj][f];
#pragma unroll
            for (int i = 0; i < DR; i++) {
                const int64_t tt = (int64_t)(neg ? add - (uint64_t)x[i] : add + (uint64_t)x[i]);   // mod 2^64
                m2 |= (uint64_t)(tt ^ (tt >> 63));   // every staged row (tail rows are zero-filled)
                vv[i] = f == 0 ? tt : (int64_t)((uint64_t)vv[i] * (uint64_t)tt);                  // mod 2^64
            }
            mt[jj][f] = m2;
        }
#pragma unroll
        for (int i = 0; i < DR; i++) vprev[i] = vv[i];
        const int op = a.prop[jj];
#pragma unroll
        for (int i = 0; i < DR; i++) {
            if (!pass[i]) continue;
            int64_t* p = acc + ((size_t)(id[i] * np + jj) * NT + tid);
            if (op == P_SUM) *p += vv[i];
            else if (op == P_MIN) *p = min(*p, vv[i]);
            else *p = max(*p, vv[i]);
        }
    }
}

template <int NT, int SPEC, int DR, int DK>
__global__ void __launch_bounds__(NT) gb_dense_kernel(Phase1Args a) {
    constexpr int NW = NT / 32;
    extern __shared__ __align__(128) uint8_t smem[];
    const int NS = a.n_stages;
    DenseHdr& h = *reinterpret_cast<DenseHdr*>(smem + (size_t)NS * a.stage_bytes);
    int64_t* acc = reinterpret_cast<int64_t*>(smem + (size_t)NS * a.stage_bytes + ((sizeof(DenseHdr) + 15) & ~size_t(15)));
    const int D = a.D, np = a.n_pairs;
    uint32_t* cnt = reinterpret_cast<uint32_t*>(acc + (size_t)D * np * NT);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int s2 = 0; s2 < D * np; s2++) {   // own column only: no barrier needed before use
        const int op = a.prop[s2 % np];
        acc[(size_t)s2 * NT + tid] = op == P_SUM ? 0 : (op == P_MIN ? INT64_MAX : INT64_MIN);
    }
    for (int d = 0; d < D; d++) cnt[d * NT + tid] = 0;
    if (tid == 0) {
        for (int s = 0; s < NS; s++) mbar_init(&h.mbar[s], 1);
        fence_mbar_init();
        int wd[TQP_MAX_KEYS];
        key_layout(a.krange, a.n_keys, h.kmin, h.kshift, wd);
        h.bad = 0;
    }
    __syncthreads();
    // per (pair, factor): OR of |add +- x| (as computed mod 2^64) over this thread's
    // passing rows. |value| <= 2^(sum of bit lengths); a wrapped add +- x (|add| <
    // 2^61, checked on the host) has |result| > 2^62 and so fails the bound below.
    uint64_t mt[PCH][3];
#pragma unroll
    for (int jj = 0; jj < PCH; jj++)
#pragma unroll
        for (int f = 0; f < 3; f++) mt[jj][f] = 0;
    uint32_t dkr[DK > 0 ? DK : 1];
#pragma unroll
    for (int j = 0; j < (DK > 0 ? DK : 1); j++) dkr[j] = (DK > 0 && j < D) ? (uint32_t)a.dkeys[j] : 0xFFFFFFFFu;
    tile_pipeline<NT, false, DR>(a, smem, h.mbar, [&](const uint8_t* st, int64_t t) {
        dense_tile<NT, SPEC, DR, DK>(a, st, t, h, acc, cnt, mt, dkr);
    });
    bool bad = false;
#pragma unroll
    for (int jj = 0; jj < PCH; jj++) {
        if (jj >= np) break;
        int bs = 0;
#pragma unroll
        for (int f = 0; f < 3; f++) {
            if (jj > 0 && f < a.pext[jj]) mt[jj][f] = mt[jj - 1][f];   // reused factor: its bound
            if (f < a.pnf[jj]) bs += 64 - __clzll(mt[jj][f]);
        }
        bad |= bs > (a.prop[jj] == P_SUM ? a.dense_bits : 62);
    }
    if (bad) h.bad = 1;
    // flush: counts per id, one partial record per present id
    for (int d = warp; d < D; d += NW) {
        int64_t c = 0;
        for (int t2 = lane; t2 < NT; t2 += 32) c += cnt[d * NT + t2];
        for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
        if (lane == 0) h.dcnt[d] = c;
    }
    __syncthreads();
    if (tid == 0) {
        if (h.bad) atomicOr(a.overflow, 4);
        for (int d = 0; d < D; d++) h.drec[d] = (int64_t)blockIdx.x * D + d;   // fixed slots (direct merge)
    }
    __syncthreads();
    for (int s2 = warp; s2 < D * np; s2 += NW) {
        const int d = s2 / np, jj = s2 - d * np;
        const int64_t rec = h.drec[d];
        if (rec < 0) continue;
        const int op = a.prop[jj];
        const int64_t* col = acc + (size_t)s2 * NT;
        if (op == P_SUM) {   // exact: split halves of the per-thread int64 sums
            uint64_t lo = 0;
            int64_t hi = 0;
            for (int t2 = lane; t2 < NT; t2 += 32) { lo += (uint64_t)(uint32_t)col[t2]; hi += col[t2] >> 32; }
            for (int o = 16; o > 0; o >>= 1) {
                lo += __shfl_xor_sync(0xffffffffu, lo, o);
                hi += __shfl_xor_sync(0xffffffffu, hi, o);
            }
            if (lane == 0) { a.plo[jj][rec] = lo; a.phi[jj][rec] = hi; }
        } else {
            int64_t v = op == P_MIN ? INT64_MAX : INT64_MIN;
            for (int t2 = lane; t2 < NT; t2 += 32) v = op == P_MIN ? min(v, col[t2]) : max(v, col[t2]);
            for (int o = 16; o > 0; o >>= 1) {
                const int64_t y = __shfl_xor_sync(0xffffffffu, v, o);
                v = op == P_MIN ? min(v, y) : max(v, y);
            }
            if (lane == 0) a.plo[jj][rec] = (uint64_t)v;
        }
    }
    for (int d = tid; d < D; d += NT) {
        const int64_t rec = h.drec[d];
        TQP_DCHECK(rec < a.cap);
        if (rec >= 0) { a.pkey[rec] = a.dkeys[d]; a.pcount[rec] = h.dcnt[d]; }
    }
}

// f(gb_dense_kernel<nt, spec>) for runtime (nt, spec)
// f(gb_dense_kernel<nt, spec, 4 rows, dk>) for runtime (nt, spec, dk in {0, 4})
template <typename F>
static void dense_call(int nt, int spec, int dk, F&& f) {
    auto by_spec = [&](auto ntc, auto dkc) {
        constexpr int NTc = decltype(ntc)::value, DKc = decltype(dkc)::value;
        switch (spec) {
            case 0: f(gb_dense_kernel<NTc, 0, 4, DKc>); break;
            case 1: f(gb_dense_kernel<NTc, 1, 4, DKc>); break;
            case 2: f(gb_dense_kernel<NTc, 2, 4, DKc>); break;
            default: f(gb_dense_kernel<NTc, 3, 4, DKc>); break;
        }
    };
    auto by_nt = [&](auto dkc) {
        if (nt == 128) by_spec(std::integral_constant<int, 128>{}, dkc);
        else by_spec(std::integral_constant<int, 256>{}, dkc);
    };
    if (dk == 4) by_nt(std::integral_constant<int, 4>{});
    else by_nt(std::integral_constant<int, 0>{});
}

// Direct merge of fixed-slot partials (dense ids / no keys): record b * D + d holds CTA
// b's split sums for id d. One warp per id reduces over the CTAs (count, per pair the
// sums of low / high 32-bit halves -> an exact int128, or min / max); ids with rows are
// compacted in id order (= key order) into the final groups. No sort, one launch.
struct DirectArgs {
    int D, n_pairs, keep_empty;   // keep_empty: no group keys -> always one group
    int64_t nblocks;
    int pop[TQP_MAX_AGGS];
    const uint64_t* plo[TQP_MAX_AGGS];
    const int64_t* phi[TQP_MAX_AGGS];
    const int64_t* pcount;
    const uint64_t* dkeys;        // id -> packed key (dense path)
    uint64_t* gkey;
    int64_t* gcount;
    uint64_t* glo[TQP_MAX_AGGS];
    int64_t* ghi[TQP_MAX_AGGS];
    unsigned long long* G_out;    // group count (device)
};

__global__ void __launch_bounds__(1024) gb_direct_kernel(DirectArgs a) {
    __shared__ int64_t s_cnt[DMAX];
    __shared__ unsigned __int128 s_sum[DMAX][PCH];
    __shared__ int64_t s_mm[DMAX][PCH];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int per = a.n_pairs + 1;   // per id: the count and every pair, one warp each
    for (int item = warp; item < a.D * per; item += 32) {
        const int d = item / per, j = item - d * per - 1;   // j = -1: the count
        if (j < 0) {
            int64_t c = 0;
            for (int64_t b = lane; b < a.nblocks; b += 32) c += a.pcount[b * a.D + d];
            for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
            if (lane == 0) s_cnt[d] = c;
        } else if (a.pop[j] == P_SUM) {
            uint64_t lo = 0;
            int64_t hi = 0;
            for (int64_t b = lane; b < a.nblocks; b += 32) { lo += a.plo[j][b * a.D + d]; hi += a.phi[j][b * a.D + d]; }
            for (int o = 16; o > 0; o >>= 1) {
                lo += __shfl_xor_sync(0xffffffffu, lo, o);
                hi += __shfl_xor_sync(0xffffffffu, hi, o);
            }
            if (lane == 0) s_sum[d][j] = (unsigned __int128)(((__int128)hi << 32) + (__int128)lo);
        } else {
            const int op = a.pop[j];
            int64_t v = op == P_MIN ? INT64_MAX : INT64_MIN;
            for (int64_t b = lane; b < a.nblocks; b += 32) {
                const int64_t x = (int64_t)a.plo[j][b * a.D + d];
                v = op == P_MIN ? min(v, x) : max(v, x);
            }
            for (int o = 16; o > 0; o >>= 1) {
                const int64_t x = __shfl_xor_sync(0xffffffffu, v, o);
                v = op == P_MIN ? min(v, x) : max(v, x);
            }
            if (lane == 0) s_mm[d][j] = v;
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long g = 0;
        for (int dd = 0; dd < a.D; dd++) {
            if (s_cnt[dd] == 0 && !a.keep_empty) continue;
            if (a.gkey) a.gkey[g] = a.dkeys ? a.dkeys[dd] : 0;
            a.gcount[g] = s_cnt[dd];
            for (int j = 0; j < a.n_pairs; j++) {
                if (a.pop[j] == P_SUM) {
                    a.glo[j][g] = (uint64_t)s_sum[dd][j];
                    a.ghi[j][g] = (int64_t)(s_sum[dd][j] >> 64);
                } else {
                    a.glo[j][g] = (uint64_t)s_mm[dd][j];
                }
            }
            g++;
        }
        *a.G_out = g;
    }
}

// Phase 2a: group ids over the sorted partial keys (segment boundaries).
constexpr int QNT = 256;
constexpr int QNW = QNT / 32;
#ifndef TQP_GID_IPT
#define TQP_GID_IPT 8
#endif
constexpr int QIPT = TQP_GID_IPT;   // sorted keys per thread of the segment-id scan (16 / 32: 0.50 / 0.57 ms against 0.45, SF10 60M keys)
constexpr int QTILE = QNT * QIPT;

__global__ void __launch_bounds__(QNT) gb_gid_kernel(const uint64_t* __restrict__ sk, int64_t P, uint32_t* gid,
                                                     uint64_t* gkey, int64_t* G_out, uint64_t* status,
                                                     unsigned long long* counter, int64_t n_tiles) {
    __shared__ int64_t s_tile;
    __shared__ uint32_t s_cnt[QIPT * QNW];
    __shared__ uint64_t s_excl;
    __shared__ uint32_t s_tot;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t tile = take_tile(counter, &s_tile);
    const int64_t base = tile * QTILE;
    unsigned bal[QIPT];
    uint64_t k[QIPT];
#pragma unroll
    for (int i = 0; i < QIPT; i++) {
        const int64_t p = base + i * QNT + tid;
        bool head = false;
        if (p < P) { k[i] = sk[p]; head = p == 0 || sk[p - 1] != k[i]; }
        bal[i] = __ballot_sync(0xffffffffu, head);
        if (lane == 0) s_cnt[i * QNW + warp] = __popc(bal[i]);
    }
    __syncthreads();
    if (warp == 0) {
        constexpr int PER = QIPT * QNW / 32;
        uint32_t c[PER], local = 0;
#pragma unroll
        for (int j = 0; j < PER; j++) { c[j] = s_cnt[lane * PER + j]; local += c[j]; }
        uint32_t x = local;
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        const uint32_t tot = __shfl_sync(0xffffffffu, x, 31);
        uint32_t run = x - local;
#pragma unroll
        for (int j = 0; j < PER; j++) { s_cnt[lane * PER + j] = run; run += c[j]; }
        const uint64_t e = lookback_warp(status, tile, tot, OpAdd(), 0ull);
        if (lane == 0) { s_excl = e; s_tot = tot; }
    }
    __syncthreads();
    const int64_t excl = (int64_t)s_excl;
    const unsigned le = lanemask_lt() | (1u << lane);
#pragma unroll
    for (int i = 0; i < QIPT; i++) {
        const int64_t p = base + i * QNT + tid;
        if (p < P) {
            const int64_t g = excl + s_cnt[i * QNW + warp] + __popc(bal[i] & le) - 1;
            gid[p] = (uint32_t)g;
            if (bal[i] & (1u << lane)) gkey[g] = k[i];
        }
    }
    if (tile == n_tiles - 1 && tid == 0) *G_out = excl + s_tot;
}

struct AccArgs {
    int n_pairs;
    int pop[TQP_MAX_AGGS];
    const uint64_t* plo[TQP_MAX_AGGS];
    const int64_t* phi[TQP_MAX_AGGS];
    uint64_t* glo[TQP_MAX_AGGS];
    int64_t* ghi[TQP_MAX_AGGS];
    const int64_t* pcount;
    int64_t* gcount;
    const uint32_t* perm;
    const uint32_t* gid;
    int64_t P;
    int split;   // 1: phase-1 partials (sum of low / high 32-bit halves); 0: int128 (lo, hi)
};

__global__ void __launch_bounds__(QNT) gb_acc_kernel(AccArgs a) {
    const int lane = threadIdx.x & 31;
    for (int64_t p0 = blockIdx.x * (int64_t)QNT; p0 < a.P; p0 += (int64_t)gridDim.x * QNT) {
        const int64_t p = p0 + threadIdx.x;
        const bool valid = p < a.P;
        const uint32_t rec = valid ? a.perm[p] : 0;
        const uint32_t g = valid ? a.gid[p] : 0xFFFFFFFFu;
        const uint32_t g0 = __shfl_sync(0xffffffffu, g, 0);
        const bool uniform = __all_sync(0xffffffffu, valid && g == g0);
        int64_t cnt = valid ? a.pcount[rec] : 0;
        if (uniform) {
            for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
            if (lane == 0) atomicAdd((unsigned long long*)&a.gcount[g], (unsigned long long)cnt);
        } else if (valid) {
            atomicAdd((unsigned long long*)&a.gcount[g], (unsigned long long)cnt);
        }
        for (int j = 0; j < a.n_pairs; j++) {
            const int op = a.pop[j];
            if (op == P_SUM) {
                unsigned __int128 v = 0;
                if (valid) {
                    if (a.split)
                        v = (unsigned __int128)(((__int128)a.phi[j][rec] << 32) + (__int128)a.plo[j][rec]);
                    else
                        v = ((unsigned __int128)(uint64_t)a.phi[j][rec] << 64) | a.plo[j][rec];
                }
                if (uniform) {
                    for (int o = 16; o > 0; o >>= 1) {
                        const uint64_t l = __shfl_xor_sync(0xffffffffu, (uint64_t)v, o);
                        const uint64_t h = __shfl_xor_sync(0xffffffffu, (uint64_t)(v >> 64), o);
                        v += ((unsigned __int128)h << 64) | l;
                    }
                    if (lane == 0) atomic_add_i128(&a.glo[j][g], &a.ghi[j][g], v);
                } else if (valid) {
                    atomic_add_i128(&a.glo[j][g], &a.ghi[j][g], v);
                }
            } else {
                int64_t v = valid ? (int64_t)a.plo[j][rec] : (op == P_MIN ? INT64_MAX : INT64_MIN);
                if (uniform) {
                    for (int o = 16; o > 0; o >>= 1) {
                        const int64_t x = __shfl_xor_sync(0xffffffffu, v, o);
                        v = op == P_MIN ? min(v, x) : max(v, x);
                    }
                }
                if (valid && (!uniform || lane == 0)) {
                    if (op == P_MIN) atomicMin((long long*)&a.glo[j][g], (long long)v);
                    else atomicMax((long long*)&a.glo[j][g], (long long)v);
                }
            }
        }
    }
}

__global__ void gb_init_kernel(uint64_t* lo, int64_t n, uint64_t init) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        lo[i] = init;
}

// correctly rounded signed int128 -> double
__device__ __forceinline__ double i128_to_double(uint64_t lo, int64_t hi) {
    const bool neg = hi < 0;
    uint64_t mlo = lo, mhi = (uint64_t)hi;
    if (neg) {   // magnitude = -value
        mlo = ~mlo + 1;
        mhi = ~mhi + (mlo == 0 ? 1 : 0);
    }
    double d;
    if (mhi == 0) {
        d = __ull2double_rn(mlo);
    } else {
        const int nb = 128 - __clzll(mhi);    // 65..128 significant bits
        const int sh = nb - 64;               // 1..64
        uint64_t top = sh == 64 ? mhi : ((mhi << (64 - sh)) | (mlo >> sh));
        const uint64_t rest = sh == 64 ? mlo : (mlo & ((1ull << sh) - 1));
        top |= (rest != 0);                   // sticky bit below the rounding position
        d = ldexp(__ull2double_rn(top), sh);
    }
    return neg ? -d : d;
}

struct FinArgs {
    int n_keys, n_aggs;
    int kdt[TQP_MAX_KEYS];
    const unsigned long long* krange;
    void* kout[TQP_MAX_KEYS];
    int aop[TQP_MAX_AGGS];
    int apair[TQP_MAX_AGGS];
    void* rout[TQP_MAX_AGGS];
    const uint64_t* glo[TQP_MAX_AGGS];
    const int64_t* ghi[TQP_MAX_AGGS];
    const uint64_t* gkey;
    const int64_t* gcount;
    int64_t G;
    bool empty_global;
};

__global__ void gb_finalize_kernel(FinArgs a) {
    for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < a.G; g += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t key = a.empty_global ? 0 : a.gkey[g];
        if (a.n_keys > 0) {
            uint64_t kmin[TQP_MAX_KEYS];
            int shift[TQP_MAX_KEYS], width[TQP_MAX_KEYS];
            key_layout(a.krange, a.n_keys, kmin, shift, width);
            for (int k = 0; k < a.n_keys; k++) {
                if (!a.kout[k]) continue;
                const uint64_t msk = width[k] >= 64 ? ~0ull : ((1ull << width[k]) - 1);
                const uint64_t part = (width[k] ? ((key >> shift[k]) & msk) : 0ull) + kmin[k];
                switch (a.kdt[k]) {
                    case TQP_U8: ((uint8_t*)a.kout[k])[g] = (uint8_t)part; break;
                    case TQP_I32: ((int32_t*)a.kout[k])[g] = (int32_t)((uint32_t)part ^ 0x80000000u); break;
                    default: ((int64_t*)a.kout[k])[g] = (int64_t)(part ^ 0x8000000000000000ull); break;
                }
            }
        }
        const int64_t cnt = a.empty_global ? 0 : a.gcount[g];
        for (int ag = 0; ag < a.n_aggs; ag++) {
            if (!a.rout[ag]) continue;
            const int op = a.aop[ag];
            const int j = a.apair[ag];
            uint64_t lo = 0;
            int64_t hi = 0;
            if (op == TQP_MIN) lo = (uint64_t)INT64_MAX;
            if (op == TQP_MAX) lo = (uint64_t)INT64_MIN;
            if (!a.empty_global && j >= 0) {
                lo = a.glo[j][g];
                if (op == TQP_SUM || op == TQP_AVG) hi = a.ghi[j][g];
            }
            switch (op) {
                case TQP_SUM:
                    ((uint64_t*)a.rout[ag])[2 * g] = lo;
                    ((int64_t*)a.rout[ag])[2 * g + 1] = hi;
                    break;
                case TQP_COUNT: ((int64_t*)a.rout[ag])[g] = cnt; break;
                case TQP_MIN:
                case TQP_MAX: ((int64_t*)a.rout[ag])[g] = (int64_t)lo; break;
                default: {
                    const double d = cnt ? i128_to_double(lo, hi) / (double)cnt : __longlong_as_double(0x7ff8000000000000ll);
                    ((double*)a.rout[ag])[g] = d;
                }
            }
        }
    }
}

struct Partials {   // phase-1 output / phase-2 input
    DevBuf<uint64_t> pkey;
    DevBuf<int64_t> pcount;
    DevBuf<uint64_t> plo[TQP_MAX_AGGS];
    DevBuf<int64_t> phi[TQP_MAX_AGGS];
    int64_t P = 0;
};

// Phase 2: global sort of partial keys, segment ids, exact accumulation.
// ------------------------------------------------ sort path (high cardinality)
// Alg. 2 as written: when tiles do not reduce (about as many keys
// per tile as rows), the rows' packed keys are radix-sorted with their permutation,
// segment heads give the groups (uniqueConsecutive), and every (op, expression) pair
// is evaluated in sorted order from the original columns and reduced per segment.
constexpr int SPT = 8;    // consecutive sorted positions per thread in the reduction
struct SortPathArgs {
    int64_t m;                        // selected rows
    const int64_t* sel;               // selected rows (null: all rows)
    const uint32_t* perm;             // sorted position -> index into the selection
    const uint32_t* gid;              // sorted position -> group
    int n_keys;
    const void* kcol[TQP_MAX_KEYS];
    int kdt[TQP_MAX_KEYS];
    const unsigned long long* krange;
    uint64_t* pk;                     // packed keys (key kernel output)
    int n_pairs;
    int pop[TQP_MAX_AGGS];
    int pnf[TQP_MAX_AGGS];
    const void* fcol[TQP_MAX_AGGS][3];
    int fdt[TQP_MAX_AGGS][3];
    int fsign[TQP_MAX_AGGS][3];
    int64_t fadd[TQP_MAX_AGGS][3];
    int64_t* gcount;
    uint64_t* glo[TQP_MAX_AGGS];
    int64_t* ghi[TQP_MAX_AGGS];
    int* overflow;
    // nullable: the distinct factor columns interleaved per selected row (aos[q * astride + u],
    // int64), so the reduction's random gather of a row fetches one sector, not one per column
    const int64_t* aos;
    int astride;
    int fu[TQP_MAX_AGGS][3];          // factor (pair, f) -> its column's slot in a row's record
};

// the AoS copy: row q of the selection, every distinct factor column as int64
struct AosArgs {
    int64_t m;
    const int64_t* sel;
    int nu, stride;
    const void* col[4];
    int dt[4];
    int64_t* aos;
};
__global__ void sp_aos_kernel(AosArgs a) {
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < a.m; q += (int64_t)gridDim.x * blockDim.x) {
        const int64_t row = a.sel ? a.sel[q] : q;
        int64_t v[4] = {0, 0, 0, 0};
#pragma unroll
        for (int u = 0; u < 4; u++)
            if (u < a.nu) v[u] = load_as_i64(a.col[u], a.dt[u], row);
        if (a.stride == 2) {
            reinterpret_cast<longlong2*>(a.aos)[q] = make_longlong2(v[0], v[1]);
        } else {
            reinterpret_cast<longlong2*>(a.aos)[2 * q] = make_longlong2(v[0], v[1]);
            reinterpret_cast<longlong2*>(a.aos)[2 * q + 1] = make_longlong2(v[2], v[3]);
        }
    }
}

__global__ void sp_keys_kernel(SortPathArgs a) {
    __shared__ uint64_t s_kmin[TQP_MAX_KEYS];
    __shared__ int s_sh[TQP_MAX_KEYS];
    if (threadIdx.x == 0) {
        int wd[TQP_MAX_KEYS];
        key_layout(a.krange, a.n_keys, s_kmin, s_sh, wd);
    }
    __syncthreads();
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < a.m; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t row = a.sel ? a.sel[i] : i;
        uint64_t k = 0;
        for (int c = 0; c < a.n_keys; c++)
            k |= (key_part(load_as_i64(a.kcol[c], a.kdt[c], row), a.kdt[c]) - s_kmin[c]) << s_sh[c];
        a.pk[i] = k;
    }
}

// per thread: SPT consecutive sorted positions; segments wholly inside the range are
// stored directly, the (at most two) that continue into a neighbour use atomics
__global__ void __launch_bounds__(256) sp_reduce_kernel(SortPathArgs a) {
    const int64_t p0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) * SPT;
    if (p0 >= a.m) return;
    const int64_t p1 = min(p0 + (int64_t)SPT, a.m);
    const uint32_t gprev = p0 > 0 ? a.gid[p0 - 1] : 0xFFFFFFFFu;
    const uint32_t gnext = p1 < a.m ? a.gid[p1] : 0xFFFFFFFFu;
    int64_t rows[SPT];
    uint32_t g[SPT];
    const int cnt = (int)(p1 - p0);
    int64_t rec[SPT][4];   // AoS: each row's factor columns, one random sector per row
#pragma unroll
    for (int i = 0; i < SPT; i++) {
        if (i < cnt) {
            g[i] = a.gid[p0 + i];
            const uint32_t q = a.perm[p0 + i];
            if (a.aos) {
                const longlong2 u0 = __ldg(reinterpret_cast<const longlong2*>(a.aos + (int64_t)q * a.astride));
                rec[i][0] = u0.x;
                rec[i][1] = u0.y;
                if (a.astride == 4) {
                    const longlong2 u1 = __ldg(reinterpret_cast<const longlong2*>(a.aos + (int64_t)q * a.astride) + 1);
                    rec[i][2] = u1.x;
                    rec[i][3] = u1.y;
                } else {
                    rec[i][2] = rec[i][3] = 0;
                }
                rows[i] = 0;
            } else {
                rows[i] = a.sel ? a.sel[q] : (int64_t)q;
            }
        }
    }
    // a segment is shared with a neighbour iff it is this range's first (gprev equal)
    // or last (gnext equal) segment
    auto shared_seg = [&](uint32_t gg) { return gg == gprev || gg == gnext; };
    // (the loops below are unrolled to SPT so g / vv stay in registers)
    auto seg_end = [&](int i) { return i + 1 == cnt || (i + 1 < SPT && g[i + 1] != g[i]); };
    {   // counts
        int64_t c = 0;
#pragma unroll
        for (int i = 0; i < SPT; i++) {
            if (i >= cnt) break;
            c++;
            if (seg_end(i)) {
                if (shared_seg(g[i])) atomicAdd((unsigned long long*)&a.gcount[g[i]], (unsigned long long)c);
                else a.gcount[g[i]] = c;
                c = 0;
            }
        }
    }
    bool ovf = false;
    for (int j = 0; j < a.n_pairs; j++) {
        const int op = a.pop[j];
        unsigned __int128 acc = 0;
        int64_t mm = op == P_MIN ? INT64_MAX : INT64_MIN;
        // the expression for all rows of the range first: the gathers are independent and in flight together
        int64_t vv[SPT];
#pragma unroll
        for (int i = 0; i < SPT; i++) vv[i] = 1;
        for (int f = 0; f < a.pnf[j]; f++) {   // prod_f (add_f + sign_f * x_f), overflow-checked
            const int64_t add = a.fadd[j][f];
            const bool neg = a.fsign[j][f] < 0;
            const void* col = a.fcol[j][f];
            const int dt = a.fdt[j][f];
            int64_t x[SPT];
            if (a.aos) {
                const int fu = a.fu[j][f];
#pragma unroll
                for (int i = 0; i < SPT; i++) x[i] = i < cnt ? (fu == 0 ? rec[i][0] : fu == 1 ? rec[i][1] : fu == 2 ? rec[i][2] : rec[i][3]) : 0;
            } else {
#pragma unroll
                for (int i = 0; i < SPT; i++) x[i] = i < cnt ? load_as_i64(col, dt, rows[i]) : 0;
            }
#pragma unroll
            for (int i = 0; i < SPT; i++) {
                int64_t t;
                if (neg) {
                    t = (int64_t)((uint64_t)add - (uint64_t)x[i]);
                    ovf |= i < cnt && ((add ^ x[i]) & (add ^ t)) < 0;
                } else {
                    t = (int64_t)((uint64_t)add + (uint64_t)x[i]);
                    ovf |= i < cnt && ((add ^ t) & (x[i] ^ t)) < 0;
                }
                if (f == 0) {
                    vv[i] = t;
                } else {
                    const int64_t lo = (int64_t)((uint64_t)vv[i] * (uint64_t)t);
                    ovf |= i < cnt && __mul64hi(vv[i], t) != (lo >> 63);
                    vv[i] = lo;
                }
            }
        }
#pragma unroll
        for (int i = 0; i < SPT; i++) {
            if (i >= cnt) break;
            const int64_t v = vv[i];
            if (op == P_SUM) acc += (unsigned __int128)(__int128)v;
            else mm = op == P_MIN ? min(mm, v) : max(mm, v);
            if (seg_end(i)) {
                const uint32_t gg = g[i];
                if (op == P_SUM) {
                    if (shared_seg(gg)) atomic_add_i128(&a.glo[j][gg], &a.ghi[j][gg], acc);
                    else { a.glo[j][gg] = (uint64_t)acc; a.ghi[j][gg] = (int64_t)(acc >> 64); }
                    acc = 0;
                } else {
                    if (shared_seg(gg)) {
                        if (op == P_MIN) atomicMin((long long*)&a.glo[j][gg], (long long)mm);
                        else atomicMax((long long*)&a.glo[j][gg], (long long)mm);
                    } else {
                        a.glo[j][gg] = (uint64_t)mm;
                    }
                    mm = op == P_MIN ? INT64_MAX : INT64_MIN;
                }
            }
        }
    }
    if (ovf) atomicOr(a.overflow, 1);
}

void phase2(tqp_ctx* ctx, tqp_groupby_plan* PL, Partials& pr, bool split) {
    const int64_t P = pr.P;
    SortOut so;
    so.want_perm32 = true;
    DevBuf<uint64_t> sk(ctx, P);
    so.sorted_u = sk.get();
    radix_sort(ctx, pr.pkey.get(), DT_U64, P, false, so);
    DevBuf<uint32_t> gid(ctx, P);
    DevBuf<int64_t> Gd(ctx, 1);
    Gd.zero();
    PL->gkey.alloc(ctx, P);
    {
        const int64_t t2 = ceil_div(P, QTILE);
        DevBuf<uint64_t> status(ctx, t2);
        DevBuf<unsigned long long> counter(ctx, 1);
        status.zero();
        counter.zero();
        launch(ctx, "tqp_groupby_gid", gb_gid_kernel, dim3((unsigned)t2), dim3(QNT), 0, sk.get(), P, gid.get(),
               PL->gkey.get(), Gd.get(), status.get(), counter.get(), t2);
        ctx->add_bytes("tqp_groupby_gid", 12.0 * (double)P);
    }
    AccArgs c{};
    c.n_pairs = PL->n_pairs;
    PL->gcount.alloc(ctx, P);
    PL->gcount.zero();
    const int ig = (int)std::min<int64_t>(ceil_div(P, 256), (int64_t)ctx->num_sms * 8);
    double rec = 8;
    for (int j = 0; j < PL->n_pairs; j++) {
        c.pop[j] = PL->pop[j];
        c.plo[j] = pr.plo[j].get();
        c.phi[j] = pr.phi[j].get();
        PL->glo[j].alloc(ctx, P);
        c.glo[j] = PL->glo[j].get();
        if (PL->pop[j] == P_SUM) {
            PL->ghi[j].alloc(ctx, P);
            c.ghi[j] = PL->ghi[j].get();
            PL->glo[j].zero();
            PL->ghi[j].zero();
            rec += 16;
        } else {
            launch(ctx, "tqp_groupby_init", gb_init_kernel, dim3(ig), dim3(256), 0, PL->glo[j].get(), P,
                   PL->pop[j] == P_MIN ? (uint64_t)INT64_MAX : (uint64_t)INT64_MIN);
            rec += 8;
        }
    }
    c.pcount = pr.pcount.get();
    c.gcount = PL->gcount.get();
    c.perm = so.perm32.get();
    c.gid = gid.get();
    c.P = P;
    c.split = split ? 1 : 0;
    const int ag = (int)std::min<int64_t>(ceil_div(P, QNT), (int64_t)ctx->num_sms * 8);
    launch(ctx, "tqp_groupby_accumulate", gb_acc_kernel, dim3(ag), dim3(QNT), 0, c);
    ctx->add_bytes("tqp_groupby_accumulate", (rec + 8) * (double)P);
    int64_t G = 0;
    read_back(ctx, &G, Gd.get(), 8);
    PL->G = G;
}

// The sort path (see sp_reduce_kernel): selection, packed keys, global radix sort with
// the permutation, segment ids, and one reduction pass over the sorted positions.
void sort_path(tqp_ctx* ctx, tqp_groupby_plan* PL, const tqp_col* cols, int n_cols, int64_t n, const int32_t* key_idx,
               int n_keys, const tqp_pred* preds, int n_preds, const int (*pf)[3], const int (*ps)[3],
               const int64_t (*pa)[3], const int* pnf, int64_t* n_groups_host) {
    DevBuf<int64_t> sel;
    int64_t m = n;
    if (n_preds > 0) {
        sel.alloc(ctx, n);
        filter_compact(ctx, cols, n_cols, n, preds, n_preds, nullptr, sel.get(), &m);
    }
    PL->empty_global = false;
    if (m == 0) {
        PL->G = 0;
        *n_groups_host = 0;
        return;
    }
    SortPathArgs a{};
    a.m = m;
    a.sel = n_preds > 0 ? sel.get() : nullptr;
    a.n_keys = n_keys;
    double kb = 0;
    for (int k = 0; k < n_keys; k++) {
        a.kcol[k] = cols[key_idx[k]].data;
        a.kdt[k] = cols[key_idx[k]].dtype;
        kb += (double)dtype_size(a.kdt[k]);
    }
    a.krange = PL->krange.get();
    DevBuf<uint64_t> pk(ctx, m);
    a.pk = pk.get();
    const int g = (int)std::min<int64_t>(ceil_div(m, 256), (int64_t)ctx->num_sms * 8);
    launch(ctx, "tqp_groupby_keys", sp_keys_kernel, dim3(g), dim3(256), 0, a);
    ctx->add_bytes("tqp_groupby_keys", (kb + 8.0 + (a.sel ? 8.0 : 0.0)) * (double)m);
    SortOut so;
    so.want_perm32 = true;
    DevBuf<uint64_t> sk(ctx, m);
    so.sorted_u = sk.get();
    radix_sort(ctx, pk.get(), DT_U64, m, false, so);
    pk.release();
    DevBuf<uint32_t> gid(ctx, m);
    DevBuf<int64_t> hd(ctx, 2);   // [0] G, [1] overflow flag
    hd.zero();
    PL->gkey.alloc(ctx, m);
    {
        const int64_t t2 = ceil_div(m, QTILE);
        DevBuf<uint64_t> status(ctx, t2);
        DevBuf<unsigned long long> counter(ctx, 1);
        status.zero();
        counter.zero();
        launch(ctx, "tqp_groupby_gid", gb_gid_kernel, dim3((unsigned)t2), dim3(QNT), 0, (const uint64_t*)sk.get(), m,
               gid.get(), PL->gkey.get(), hd.get(), status.get(), counter.get(), t2);
        ctx->add_bytes("tqp_groupby_gid", 12.0 * (double)m);
    }
    PL->gcount.alloc(ctx, m);
    PL->gcount.zero();
    a.n_pairs = PL->n_pairs;
    const int ig = (int)std::min<int64_t>(ceil_div(m, 256), (int64_t)ctx->num_sms * 8);
    double vb = 0;
    for (int j = 0; j < PL->n_pairs; j++) {
        a.pop[j] = PL->pop[j];
        a.pnf[j] = pnf[j];
        for (int f = 0; f < pnf[j]; f++) {
            a.fcol[j][f] = cols[pf[j][f]].data;
            a.fdt[j][f] = cols[pf[j][f]].dtype;
            a.fsign[j][f] = ps[j][f];
            a.fadd[j][f] = pa[j][f];
            vb += 32.0;   // one gathered sector per value
        }
        PL->glo[j].alloc(ctx, m);
        a.glo[j] = PL->glo[j].get();
        if (PL->pop[j] == P_SUM) {
            PL->ghi[j].alloc(ctx, m);
            a.ghi[j] = PL->ghi[j].get();
            PL->glo[j].zero();
            PL->ghi[j].zero();
        } else {
            launch(ctx, "tqp_groupby_init", gb_init_kernel, dim3(ig), dim3(256), 0, PL->glo[j].get(), m,
                   PL->pop[j] == P_MIN ? (uint64_t)INT64_MAX : (uint64_t)INT64_MIN);
        }
    }
    // 2-4 distinct factor columns: interleave them per selected row first (a sequential pass),
    // so the reduction's random gather of a row fetches one sector instead of one per column
    DevBuf<int64_t> aos;
    {
        const void* uc[4];
        int ud[4], nu = 0;
        bool fits = true;
        for (int j = 0; j < PL->n_pairs && fits; j++)
            for (int f = 0; f < pnf[j]; f++) {
                int u = 0;
                while (u < nu && uc[u] != a.fcol[j][f]) u++;
                if (u == nu) {
                    if (nu == 4) { fits = false; break; }
                    uc[nu] = a.fcol[j][f];
                    ud[nu] = a.fdt[j][f];
                    nu++;
                }
                a.fu[j][f] = u;
            }
        static const bool aos_off = [] {   // TQP_SORTPATH_AOS=0: gather each column (A/B)
            const char* e = getenv("TQP_SORTPATH_AOS");
            return e && e[0] == '0';
        }();
        if (fits && nu >= 2 && m >= (int64_t(1) << 20) && !aos_off) {
            AosArgs aa{};
            aa.m = m;
            aa.sel = a.sel;
            aa.nu = nu;
            aa.stride = nu <= 2 ? 2 : 4;
            for (int u = 0; u < nu; u++) { aa.col[u] = uc[u]; aa.dt[u] = ud[u]; }
            aos.alloc(ctx, (size_t)m * aa.stride);
            aa.aos = aos.get();
            const int ag = (int)std::min<int64_t>(ceil_div(m, 256), (int64_t)ctx->num_sms * 8);
            launch(ctx, "tqp_groupby_sortpath", sp_aos_kernel, dim3(ag), dim3(256), 0, aa);
            double cb = 0;
            for (int u = 0; u < nu; u++) cb += (double)dtype_size(ud[u]);
            ctx->add_bytes("tqp_groupby_sortpath", (cb + 8.0 * aa.stride + (a.sel ? 8.0 : 0.0)) * (double)m);
            a.aos = aos.get();
            a.astride = aa.stride;
        }
    }
    a.perm = so.perm32.get();
    a.gid = gid.get();
    a.gcount = PL->gcount.get();
    a.overflow = (int*)(hd.get() + 1);
    const int rg = (int)ceil_div(ceil_div(m, SPT), 256);
    launch(ctx, "tqp_groupby_accumulate", sp_reduce_kernel, dim3(rg), dim3(256), 0, a);
    ctx->add_bytes("tqp_groupby_accumulate", (8.0 + (a.sel ? 8.0 : 0.0) + vb) * (double)m);
    int64_t h[2];
    read_back(ctx, h, hd.get(), 16);
    if (h[1]) fail(TQP_ERR_OVERFLOW, "groupby: int64 overflow in an aggregate expression");
    PL->G = h[0];
    *n_groups_host = PL->G;
}

// Key-column ranges on the device (no host sync): min in kr[0..7], max in kr[8..15].
__global__ void u8_ranges_kernel(unsigned long long* kr, int n_keys) {
    if (threadIdx.x < n_keys) {
        kr[threadIdx.x] = 0;
        kr[8 + threadIdx.x] = 255;
    }
}

void key_ranges(tqp_ctx* ctx, const void* const* kcol, const int* kdt, int n_keys, int64_t n,
                DevBuf<unsigned long long>& kr) {
    kr.alloc(ctx, 16);
    TQP_CUDA(cudaMemsetAsync(kr.get(), 0xFF, 8 * 8, ctx->stream));
    TQP_CUDA(cudaMemsetAsync(kr.get() + 8, 0, 8 * 8, ctx->stream));
    if (n_keys == 0 || n == 0) return;
    // at most two u8 key columns: their whole domains pack into 16 bits (the dense path's
    // presence bitmap), so the layout takes [0, 255] per column without a pass over the keys
    bool u8only = n_keys <= 2;
    for (int k = 0; k < n_keys; k++) u8only = u8only && kdt[k] == TQP_U8;
    if (u8only) {
        launch(ctx, "tqp_groupby_keyrange", u8_ranges_kernel, dim3(1), dim3(32), 0, kr.get(), n_keys);
        return;
    }
    KRArgs a{};
    a.n_keys = n_keys;
    a.n = n;
    double bytes = 0;
    for (int k = 0; k < n_keys; k++) {
        a.kcol[k] = kcol[k];
        a.kdt[k] = kdt[k];
        bytes += (double)dtype_size(kdt[k]) * (double)n;
    }
    const int g = (int)std::min<int64_t>(ceil_div(n, GNT * 16), (int64_t)ctx->num_sms * 8);
    launch(ctx, "tqp_groupby_keyrange", key_range_kernel, dim3(g), dim3(GNT), 0, a, kr.get());
    ctx->add_bytes("tqp_groupby_keyrange", bytes);
}

// Distinct (op, expression) pairs: SUM and AVG of the same expression share one.
void make_pairs(tqp_groupby_plan* PL, const tqp_agg* aggs, int n_aggs, int (*pf)[3], int (*ps)[3],
                int64_t (*pa)[3], int* pnf) {
    PL->n_pairs = 0;
    for (int g = 0; g < n_aggs; g++) {
        const int op = aggs[g].op;
        PL->aop[g] = op;
        if (op == TQP_COUNT) { PL->apair[g] = -1; continue; }
        const int pop = (op == TQP_SUM || op == TQP_AVG) ? P_SUM : op == TQP_MIN ? P_MIN : P_MAX;
        int found = -1;
        for (int j = 0; j < PL->n_pairs && found < 0; j++) {
            if (PL->pop[j] != pop || pnf[j] != aggs[g].n_factors) continue;
            bool same = true;
            for (int f = 0; f < pnf[j]; f++)
                same = same && pf[j][f] == aggs[g].col[f] && ps[j][f] == aggs[g].sign[f] && pa[j][f] == aggs[g].add[f];
            if (same) found = j;
        }
        if (found < 0) {
            found = PL->n_pairs++;
            PL->pop[found] = pop;
            pnf[found] = aggs[g].n_factors;
            for (int f = 0; f < pnf[found]; f++) {
                pf[found][f] = aggs[g].col[f];
                ps[found][f] = aggs[g].sign[f];
                pa[found][f] = aggs[g].add[f];
            }
        }
        PL->apair[g] = found;
    }
    // order pairs by their factor lists (lexicographic, a prefix first), so that an
    // expression extending the previous pair's (Q1: price, price*(1-disc),
    // price*(1-disc)*(1+tax)) can reuse its value (dense path)
    const int np = PL->n_pairs;
    int ord[TQP_MAX_AGGS];
    for (int j = 0; j < np; j++) ord[j] = j;
    auto less = [&](int x, int y) {
        for (int f = 0; f < 3; f++) {
            if (f >= pnf[x] || f >= pnf[y]) return pnf[x] < pnf[y] || (pnf[x] == pnf[y] && PL->pop[x] < PL->pop[y]);
            if (pf[x][f] != pf[y][f]) return pf[x][f] < pf[y][f];
            if (ps[x][f] != ps[y][f]) return ps[x][f] < ps[y][f];
            if (pa[x][f] != pa[y][f]) return pa[x][f] < pa[y][f];
        }
        return pnf[x] == pnf[y] && PL->pop[x] < PL->pop[y];
    };
    std::stable_sort(ord, ord + np, less);
    int inv[TQP_MAX_AGGS], pop2[TQP_MAX_AGGS], pnf2[TQP_MAX_AGGS], pf2[TQP_MAX_AGGS][3], ps2[TQP_MAX_AGGS][3];
    int64_t pa2[TQP_MAX_AGGS][3];
    for (int j = 0; j < np; j++) {
        const int o = ord[j];
        inv[o] = j;
        pop2[j] = PL->pop[o];
        pnf2[j] = pnf[o];
        for (int f = 0; f < 3; f++) { pf2[j][f] = pf[o][f]; ps2[j][f] = ps[o][f]; pa2[j][f] = pa[o][f]; }
    }
    for (int j = 0; j < np; j++) {
        PL->pop[j] = pop2[j];
        pnf[j] = pnf2[j];
        for (int f = 0; f < 3; f++) { pf[j][f] = pf2[j][f]; ps[j][f] = ps2[j][f]; pa[j][f] = pa2[j][f]; }
    }
    for (int g = 0; g < n_aggs; g++)
        if (PL->apair[g] >= 0) PL->apair[g] = inv[PL->apair[g]];
}
}  // namespace

static tqp_groupby_plan* groupby_prepare_int(tqp_ctx* ctx, const tqp_col* cols, int n_cols, int64_t n,
                                             const int32_t* key_idx, int n_keys, const tqp_pred* preds, int n_preds,
                                             const tqp_agg* aggs, int n_aggs, int64_t* n_groups_host) {
    if (n < 0 || n_cols < 0 || n_keys < 0 || n_keys > TQP_MAX_KEYS || n_preds < 0 || n_preds > TQP_MAX_PREDS ||
        n_aggs < 0 || n_aggs > TQP_MAX_AGGS)
        fail(TQP_ERR_INVALID_ARGUMENT, "groupby: bad sizes");
    if (n >= (int64_t(1) << 40)) fail(TQP_ERR_INVALID_ARGUMENT, "groupby: n too large");
    for (int c = 0; c < n_cols; c++) check_col(cols[c], n, "groupby column");
    for (int k = 0; k < n_keys; k++)
        if (key_idx[k] < 0 || key_idx[k] >= n_cols) fail(TQP_ERR_INVALID_ARGUMENT, "groupby: key column");
    for (int q = 0; q < n_preds; q++)
        if (preds[q].col < 0 || preds[q].col >= n_cols || preds[q].op < TQP_LT || preds[q].op > TQP_NE)
            fail(TQP_ERR_INVALID_ARGUMENT, "groupby: predicate");
    for (int g = 0; g < n_aggs; g++) {
        if (aggs[g].op < TQP_SUM || aggs[g].op > TQP_AVG || aggs[g].n_factors < 0 || aggs[g].n_factors > 3)
            fail(TQP_ERR_INVALID_ARGUMENT, "groupby: aggregate");
        if (aggs[g].op == TQP_COUNT) continue;
        for (int f = 0; f < aggs[g].n_factors; f++)
            if (aggs[g].col[f] < 0 || aggs[g].col[f] >= n_cols || (aggs[g].sign[f] != 1 && aggs[g].sign[f] != -1))
                fail(TQP_ERR_INVALID_ARGUMENT, "groupby: aggregate factor");
    }
    Phase1Args a{};
    a.n = n;
    // distinct referenced columns (one stage slot each)
    std::vector<int> ucols;
    auto uidx = [&](int c) {
        for (size_t i = 0; i < ucols.size(); i++) if (ucols[i] == c) return (int)i;
        ucols.push_back(c);
        return (int)ucols.size() - 1;
    };
    auto* PL = new tqp_groupby_plan();
    try {
        PL->n_keys = n_keys;
        PL->n_aggs = n_aggs;
        int off = 0;
        a.n_keys = n_keys;
        const void* kc[TQP_MAX_KEYS];
        int kd[TQP_MAX_KEYS];
        for (int k = n_keys - 1; k >= 0; k--) {   // column 0 most significant
            const int c = key_idx[k];
            a.kcol[k] = uidx(c);
            PL->kdt[k] = cols[c].dtype;
            kc[k] = cols[c].data;
            kd[k] = cols[c].dtype;
            off += 8 * (int)dtype_size(cols[c].dtype);
        }
        if (off > 64) fail(TQP_ERR_INVALID_ARGUMENT, "groupby: packed key wider than 64 bits");
        key_ranges(ctx, kc, kd, n_keys, n, PL->krange);
        a.krange = PL->krange.get();
        a.ts = make_terms(preds, n_preds, [&](int c) { return cols[c].dtype; });
        for (int q = 0; q < a.ts.n; q++) a.ts.t[q].col = uidx(a.ts.t[q].col);
        int pf[TQP_MAX_AGGS][3], ps[TQP_MAX_AGGS][3], pnf[TQP_MAX_AGGS];
        int64_t pa[TQP_MAX_AGGS][3];
        make_pairs(PL, aggs, n_aggs, pf, ps, pa, pnf);
        a.n_pairs = PL->n_pairs;
        for (int j = 0; j < PL->n_pairs; j++) {
            a.prop[j] = PL->pop[j];
            a.pnf[j] = pnf[j];
            for (int f = 0; f < pnf[j]; f++) {
                a.pfc[j][f] = uidx(pf[j][f]);
                a.psign[j][f] = ps[j][f];
                a.padd[j][f] = pa[j][f];
            }
        }
        if ((int)ucols.size() > MAXU) fail(TQP_ERR_INVALID_ARGUMENT, "groupby: more than 16 distinct columns");
        a.n_ucols = (int)ucols.size();
        int sb = 0;
        bool aligned = true;
        for (int i = 0; i < a.n_ucols; i++) {
            a.ucol[i] = cols[ucols[i]].data;
            a.udt[i] = cols[ucols[i]].dtype;
            a.uoff[i] = sb;
            sb += GTILE * (int)dtype_size(a.udt[i]);
            aligned = aligned && ((uintptr_t)a.ucol[i] % 16 == 0);
        }
        a.stage_bytes = std::max(sb, 16);
        a.bulk_ok = (aligned && a.n_ucols > 0) ? 1 : 0;
        const int64_t tiles = ceil_div(n, GTILE);
        a.n_tiles = tiles;
        for (int j = 0; j < PL->n_pairs && j < PCH; j++) {
            for (int f = 0; f < pnf[j]; f++) {
                a.poff[j][f] = a.uoff[a.pfc[j][f]];
                a.pdtf[j][f] = a.udt[a.pfc[j][f]];
            }
            bool pre = j > 0 && pnf[j - 1] > 0 && pnf[j - 1] <= pnf[j];
            for (int f = 0; pre && f < pnf[j - 1]; f++)
                pre = pf[j - 1][f] == pf[j][f] && ps[j - 1][f] == ps[j][f] && pa[j - 1][f] == pa[j][f];
            a.pext[j] = pre ? pnf[j - 1] : 0;
        }

        // ---- dense small-domain path (gb_dense_kernel): presence pass + dense ids
        DevBuf<uint8_t> dtab;
        DevBuf<uint64_t> dkeys;
        bool dense = false;
        size_t dense_smem = 0;
        int dense_ns = 0, dense_nt = GNT, dense_spec = 0;
        // rows per thread per tile of the dense kernel: 4 (8 measured slower, Q1: 0.665 ->
        // 0.760 ms at SF10, 6.44 -> 7.31 ms at SF100: 110 registers, fewer warps hide less
        // latency than the halved per-tile control overhead saves)
        constexpr int dense_dr = 4;
        int dense_dk = 0;   // 4: the dense ids by compares against <= 4 keys in registers
        int64_t dense_grid = 0;
        bool dense_jit = false;     // launch the kernel compiled for this plan (jit.cu)
        DenseJitSpec jit_spec;
        size_t dense_jit_smem = 0;
        const char* dz = getenv("TQP_GROUPBY_DENSE");
        bool small_add = true;   // the dense bound argument needs |add| < 2^61
        for (int j = 0; j < PL->n_pairs && j < PCH; j++)
            for (int f = 0; f < pnf[j]; f++) small_add = small_add && a.padd[j][f] < (1ll << 61) && a.padd[j][f] > -(1ll << 61);
        // presence from a sample of the rows first (~1M rows: the keys cost a few microseconds
        // instead of a pass); a row whose key the sample missed raises overflow bit 8 in the
        // dense kernel, and the presence pass is redone over every row
        bool key_cols_aligned = true;
        for (int k = 0; k < n_keys; k++) key_cols_aligned = key_cols_aligned && (uintptr_t)kc[k] % 16 == 0;
        int64_t pres_stride = key_cols_aligned ? std::max<int64_t>(1, n / (int64_t(1) << 20)) : 1;
        auto setup_dense = [&](int64_t stride) {
            dense = false;
            DevBuf<uint32_t> bitmap(ctx, 1 << (PBITS - 5));
            DevBuf<int> Dd(ctx, 1);
            bitmap.zero();
            dtab.alloc(ctx, 1 << PBITS);
            TQP_CUDA(cudaMemsetAsync(dtab.get(), 0xFF, (size_t)1 << PBITS, ctx->stream));
            dkeys.alloc(ctx, DMAX);
            PresArgs pa{};
            pa.n_keys = n_keys;
            pa.n = n;
            pa.krange = PL->krange.get();
            pa.bitmap = bitmap.get();
            pa.stride = stride;
            double kb = 0;
            for (int k = 0; k < n_keys; k++) {
                pa.kcol[k] = kc[k];
                pa.kdt[k] = kd[k];
                kb += (double)dtype_size(kd[k]);
            }
            const int g = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(n / stride, GNT * 16), (int64_t)ctx->num_sms * 8));
            launch(ctx, "tqp_groupby_presence", gb_presence_kernel, dim3(g), dim3(GNT), 0, pa);
            ctx->add_bytes("tqp_groupby_presence", kb * (double)(n / stride));
            launch(ctx, "tqp_groupby_dense_ids", gb_dense_ids_kernel, dim3(1), dim3(1024), 0, (const uint32_t*)bitmap.get(),
                   dtab.get(), dkeys.get(), Dd.get());
            int D = 0;
            read_back(ctx, &D, Dd.get(), 4);
            if (D >= 1 && D <= DMAX) {
                bool vi64 = true, ku8 = true;
                for (int j = 0; j < PL->n_pairs && j < PCH; j++)
                    for (int f = 0; f < pnf[j]; f++) vi64 = vi64 && a.pdtf[j][f] == TQP_I64;
                for (int k = 0; k < n_keys; k++) ku8 = ku8 && kd[k] == TQP_U8;
                dense_spec = (vi64 ? SPEC_VI64 : 0) | (ku8 ? SPEC_KU8 : 0);
                static const bool dk_off = [] {   // TQP_DENSE_DK=0: always the id table (A/B)
                    const char* e = getenv("TQP_DENSE_DK");
                    return e && e[0] == '0';
                }();
                dense_dk = (D <= 4 && !dk_off) ? 4 : 0;
                // (threads per CTA, stages) with the most resident warps per SM; ties go to
                // more stages per SM. Lane-private accumulators make occupancy smem-bound.
                const size_t hdr = (sizeof(DenseHdr) + 15) & ~size_t(15);
                int best_w = 0, best_st = 0;
                for (int nt : {128, 256}) {
                    const size_t stage = (size_t)a.stage_bytes * nt * dense_dr / (GNT * GPT);
                    const size_t accb = (size_t)D * PL->n_pairs * nt * 8 + (size_t)D * nt * 4;
                    for (int ns = 1; ns <= 4; ns++) {
                        const size_t sm = (size_t)ns * stage + hdr + accb;
                        if (sm > 227 * 1024) continue;
                        int occ = 0;
                        dense_call(nt, dense_spec, dense_dk, [&](auto* kfn) { occ = occupancy(kfn, nt, sm); });
                        const int wps = occ * nt / 32, st = occ * ns;
                        if (occ > 0 && (wps > best_w || (wps == best_w && st > best_st))) {
                            best_w = wps;
                            best_st = st;
                            dense_nt = nt;
                            dense_ns = ns;
                            dense_smem = sm;
                            dense_grid = (int64_t)ctx->num_sms * occ;
                        }
                    }
                }
                // the kernel compiled for this plan (jit.cu) in the chosen configuration; its
                // own occupancy sizes the grid
                dense_jit = false;
                const char* jm = getenv("TQP_JIT_MIN_ROWS");
                const int64_t jit_min = jm ? atoll(jm) : (int64_t(1) << 20);
                if (best_w > 0 && n >= jit_min && jit_enabled()) {
                    const int64_t tr = (int64_t)dense_nt * dense_dr;
                    DenseJitSpec& js = jit_spec;
                    memset(&js, 0, sizeof(js));   // padding too: the compiled-kernel cache keys on the bytes
                    js.nt = dense_nt;
                    js.ns = dense_ns;
                    js.stage_bytes = (int)((int64_t)a.stage_bytes * tr / GTILE);
                    js.n_ucols = a.n_ucols;
                    for (int c = 0; c < a.n_ucols; c++) {
                        js.udt[c] = a.udt[c];
                        js.uoff[c] = (int)((int64_t)a.uoff[c] * tr / GTILE);
                    }
                    js.n_terms = a.ts.n;
                    js.never = a.ts.never;
                    for (int q = 0; q < a.ts.n; q++) {
                        js.tcol[q] = a.ts.t[q].col;
                        js.tdt[q] = a.ts.t[q].dt;
                        js.tneg[q] = a.ts.t[q].neg;
                        js.tlo[q] = a.ts.t[q].lo;
                        js.twidth[q] = a.ts.t[q].width;
                    }
                    js.n_keys = n_keys;
                    for (int k = 0; k < n_keys; k++) js.kslot[k] = a.kcol[k];
                    js.n_pairs = PL->n_pairs;
                    for (int j = 0; j < PL->n_pairs; j++) {
                        js.prop[j] = a.prop[j];
                        js.pnf[j] = a.pnf[j];
                        js.pext[j] = a.pext[j];
                        for (int f = 0; f < a.pnf[j]; f++) {
                            js.pslot[j][f] = a.pfc[j][f];
                            js.psign[j][f] = a.psign[j][f];
                            js.padd[j][f] = a.padd[j][f];
                        }
                    }
                    js.dk = dense_dk;
                    const size_t accb = (size_t)D * PL->n_pairs * dense_nt * 8 + (size_t)D * dense_nt * 4;
                    const size_t sm = (size_t)dense_ns * js.stage_bytes + DENSE_JIT_HDR + accb;
                    const int occ = sm <= 227 * 1024 ? dense_jit_occupancy(js, sm) : 0;
                    if (occ > 0) {
                        dense_jit = true;
                        dense_jit_smem = sm;
                        dense_grid = (int64_t)ctx->num_sms * occ;
                    }
                }
                if (best_w > 0) {
                    const int64_t tr = (int64_t)dense_nt * dense_dr;
                    dense_grid = std::min<int64_t>(dense_grid, ceil_div(n, tr));
                    // rows per thread bound -> per-thread int64 sums of values <= 2^bits stay <= 2^62
                    const int64_t rpt = ceil_div(ceil_div(n, tr), dense_grid) * dense_dr;
                    int lg = 0;
                    while ((int64_t(1) << lg) < rpt) lg++;
                    a.dense_bits = 62 - lg;
                    a.D = D;
                    a.dtab = dtab.get();
                    a.dkeys = dkeys.get();
                    dense = a.dense_bits >= 1;
                }
            }
        };
        if (n_keys > 0 && n > 0 && PL->n_pairs <= PCH && small_add && !(dz && dz[0] == '0')) setup_dense(pres_stride);

        // ---- phase 1 (retried once with full capacity if the partial estimate is exceeded)
        Partials pr;
        DevBuf<unsigned long long> Pc(ctx, 2);   // [0] partial counter, [1] overflow flags: one readback
        int* ovf = reinterpret_cast<int*>(Pc.get() + 1);
        int64_t cap = std::min<int64_t>(std::max<int64_t>(n, 1), std::max<int64_t>(tiles * 64, 1 << 16));
        const char* tile_name = "tqp_groupby_tile";
        const bool nokey_path = n_keys == 0 && PL->n_pairs <= PCH;
        int64_t nokey_grid = 0;
        size_t nokey_smem = 0;
        if (nokey_path && n > 0) {
            // pipeline depth: light per-row work (no group keys) is bandwidth-bound and
            // wants more bytes in flight; keyed tiles are compute-heavy and prefer 2 CTAs/SM
#ifndef TQP_NOKEY_STAGES   // (3 stages at 3 blocks per SM: 0.349 ms; 2: 0.278)
#define TQP_NOKEY_STAGES 4
#endif
            a.n_stages = ((size_t)TQP_NOKEY_STAGES * a.stage_bytes + sizeof(NoKeyWork) <= 112 * 1024) ? TQP_NOKEY_STAGES : 2;
            nokey_smem = (size_t)a.n_stages * a.stage_bytes + sizeof(NoKeyWork);
            const int occ = occupancy(gb_phase1_kernel, GNT, nokey_smem);
            nokey_grid = std::min<int64_t>(tiles, (int64_t)ctx->num_sms * std::max(occ, 1));
        }
        for (int attempt = 0; attempt < 4; attempt++) {
            // dense ids / no keys: fixed per-CTA slots merged directly (no phase-2 sort)
            const bool direct = n > 0 && (dense || nokey_path);
            const int64_t dD = dense ? a.D : 1;
            const int64_t nblocks = dense ? dense_grid : nokey_grid;
            if (direct) cap = std::max<int64_t>(cap, nblocks * dD);
            a.direct = direct ? 1 : 0;
            pr.pkey.alloc(ctx, cap);
            pr.pcount.alloc(ctx, cap);
            for (int j = 0; j < PL->n_pairs; j++) {
                pr.plo[j].alloc(ctx, cap);
                if (PL->pop[j] == P_SUM) pr.phi[j].alloc(ctx, cap);
                a.plo[j] = pr.plo[j].get();
                a.phi[j] = pr.phi[j].get();
            }
            a.pkey = pr.pkey.get();
            a.pcount = pr.pcount.get();
            a.cap = cap;
            Pc.zero();
            a.P_counter = Pc.get();
            a.overflow = ovf;
            if (n > 0 && dense) {
                // the stage layout scaled to tiles of dense_nt * dense_dr rows
                Phase1Args ad = a;
                const int64_t tr = (int64_t)dense_nt * dense_dr;
                ad.n_stages = dense_ns;
                ad.stage_bytes = (int)((int64_t)a.stage_bytes * tr / GTILE);
                ad.n_tiles = ceil_div(n, tr);
                for (int c = 0; c < a.n_ucols; c++) ad.uoff[c] = (int)((int64_t)a.uoff[c] * tr / GTILE);
                for (int j = 0; j < PL->n_pairs && j < PCH; j++)
                    for (int f = 0; f < pnf[j]; f++) ad.poff[j][f] = ad.uoff[a.pfc[j][f]];
                tile_name = "tqp_groupby_dense";
                bool done = false;
                if (dense_jit) {
                    DenseJitArgs ja{};
                    for (int c = 0; c < a.n_ucols; c++) ja.ucol[c] = a.ucol[c];
                    ja.n = n;
                    ja.n_tiles = ad.n_tiles;
                    ja.D = a.D;
                    ja.dense_bits = a.dense_bits;
                    ja.bulk_ok = a.bulk_ok;
                    ja.krange = a.krange;
                    ja.dkeys = reinterpret_cast<const unsigned long long*>(a.dkeys);
                    ja.dtab = a.dtab;
                    ja.overflow = a.overflow;
                    for (int j = 0; j < PL->n_pairs; j++) {
                        ja.plo[j] = reinterpret_cast<unsigned long long*>(a.plo[j]);
                        ja.phi[j] = reinterpret_cast<long long*>(a.phi[j]);
                    }
                    ja.pkey = reinterpret_cast<unsigned long long*>(a.pkey);
                    ja.pcount = reinterpret_cast<long long*>(a.pcount);
                    done = dense_jit_launch(ctx, jit_spec, ja, dense_grid, dense_jit_smem, tile_name);
                }
                if (!done)
                    dense_call(dense_nt, dense_spec, dense_dk, [&](auto* kfn) {
                        set_smem(kfn, dense_smem);
                        launch(ctx, tile_name, kfn, dim3((unsigned)dense_grid), dim3(dense_nt), dense_smem, ad);
                    });
            } else if (n > 0 && nokey_path) {
                tile_name = "tqp_groupby_tile";
                if (nokey_smem > 227 * 1024) fail(TQP_ERR_INVALID_ARGUMENT, "groupby: referenced columns too wide");
                launch(ctx, "tqp_groupby_tile", gb_phase1_kernel, dim3((unsigned)nokey_grid), dim3(GNT), nokey_smem, a);
            } else if (n > 0) {
                tile_name = "tqp_groupby_tile";
                a.n_stages = 2;
                const size_t smem = (size_t)a.n_stages * a.stage_bytes + sizeof(Work);
                if (smem > 227 * 1024) fail(TQP_ERR_INVALID_ARGUMENT, "groupby: referenced columns too wide");
                const int occ = occupancy(gb_phase1_kernel, GNT, smem);
                const int64_t grid = std::min<int64_t>(tiles, (int64_t)ctx->num_sms * std::max(occ, 1));
                launch(ctx, "tqp_groupby_tile", gb_phase1_kernel, dim3((unsigned)grid), dim3(GNT), smem, a);
            }
            if (direct) {   // merge the fixed slots straight into the final groups
                PL->gkey.alloc(ctx, dD);
                PL->gcount.alloc(ctx, dD);
                DirectArgs da{};
                da.D = (int)dD;
                da.n_pairs = PL->n_pairs;
                da.keep_empty = dense ? 0 : 1;
                da.nblocks = nblocks;
                for (int j = 0; j < PL->n_pairs; j++) {
                    da.pop[j] = PL->pop[j];
                    da.plo[j] = pr.plo[j].get();
                    da.phi[j] = pr.phi[j].get();
                    PL->glo[j].alloc(ctx, dD);
                    da.glo[j] = PL->glo[j].get();
                    if (PL->pop[j] == P_SUM) {
                        PL->ghi[j].alloc(ctx, dD);
                        da.ghi[j] = PL->ghi[j].get();
                    }
                }
                da.pcount = pr.pcount.get();
                da.dkeys = dense ? a.dkeys : nullptr;
                da.gkey = PL->gkey.get();
                da.gcount = PL->gcount.get();
                da.G_out = Pc.get();
                launch(ctx, "tqp_groupby_accumulate", gb_direct_kernel, dim3(1), dim3(1024), 0, da);
                double rb = 8;
                for (int j = 0; j < PL->n_pairs; j++) rb += PL->pop[j] == P_SUM ? 16 : 8;
                ctx->add_bytes("tqp_groupby_accumulate", rb * (double)(nblocks * dD));
            }
            unsigned long long h[2] = {0, 0};
            read_back(ctx, h, Pc.get(), 16);
            const int o = (int)h[1];
            if ((o & 8) && dense && pres_stride > 1) {   // a key outside the sampled presence: full pass
                pres_stride = 1;
                setup_dense(1);
                continue;
            }
            if (o & 4) {   // dense path could not prove a tile exact: general path
                dense = false;
                continue;
            }
            if (o & 1) fail(TQP_ERR_OVERFLOW, "groupby: int64 overflow in an aggregate expression");
            if (direct) {
                pr.P = nblocks * dD;
                PL->G = (int64_t)h[0];
                PL->empty_global = false;
                double in = 0;
                for (int i = 0; i < a.n_ucols; i++) in += (double)dtype_size(a.udt[i]);
                ctx->add_bytes(tile_name, in * (double)n);
                *n_groups_host = PL->G;
                return PL;
            }
            pr.P = (int64_t)h[0];
            if (!(o & 2)) break;
            if (n_keys > 0 && n < (int64_t(1) << 30)) {
                // tiles do not reduce (more than 64 keys per 1024 rows on average):
                // Alg. 2 directly -- global sort of the packed keys + segmented reduction
                sort_path(ctx, PL, cols, n_cols, n, key_idx, n_keys, preds, n_preds, pf, ps, pa, pnf, n_groups_host);
                return PL;
            }
            cap = std::max<int64_t>(n, 1);   // more distinct keys per tile than estimated: full capacity
        }
        {   // algorithmic bytes: distinct referenced columns read once, partial records written
            double in = 0;
            for (int i = 0; i < a.n_ucols; i++) in += (double)dtype_size(a.udt[i]);
            double rec = 16;
            for (int j = 0; j < PL->n_pairs; j++) rec += PL->pop[j] == P_SUM ? 16 : 8;
            if (n > 0) ctx->add_bytes(tile_name, in * (double)n + rec * (double)pr.P);
        }
        if (pr.P == 0) {
            PL->G = n_keys == 0 ? 1 : 0;
            PL->empty_global = n_keys == 0;
            *n_groups_host = PL->G;
            return PL;
        }
        phase2(ctx, PL, pr, true);
        *n_groups_host = PL->G;
        return PL;
    } catch (...) {
        delete PL;
        throw;
    }
}

static void groupby_fetch_int(tqp_ctx* ctx, const tqp_groupby_plan* PL, void* const* keys_out,
                              void* const* results_out) {
    if (PL->G == 0) return;
    FinArgs f{};
    f.n_keys = PL->n_keys;
    f.n_aggs = PL->n_aggs;
    for (int k = 0; k < PL->n_keys; k++) {
        f.kdt[k] = PL->kdt[k];
        f.kout[k] = keys_out ? keys_out[k] : nullptr;
    }
    for (int g = 0; g < PL->n_aggs; g++) {
        f.aop[g] = PL->aop[g];
        f.apair[g] = PL->apair[g];
        f.rout[g] = results_out ? results_out[g] : nullptr;
    }
    for (int j = 0; j < PL->n_pairs; j++) {
        f.glo[j] = PL->glo[j].get();
        f.ghi[j] = PL->ghi[j].get();
    }
    f.krange = PL->krange.get();
    f.gkey = PL->gkey.get();
    f.gcount = PL->gcount.get();
    f.G = PL->G;
    f.empty_global = PL->empty_global;
    const int g = (int)std::min<int64_t>(ceil_div(PL->G, 256), (int64_t)ctx->num_sms * 8);
    launch(ctx, "tqp_groupby_finalize", gb_finalize_kernel, dim3(g), dim3(256), 0, f);
}

void groupby_release(tqp_ctx*, tqp_groupby_plan* PL) { delete PL; }

namespace {
struct MergeArgs {
    int n_keys;
    const void* kcol[TQP_MAX_KEYS];
    int kdt[TQP_MAX_KEYS];
    const unsigned long long* krange;
    int n_pairs;
    int pop[TQP_MAX_AGGS];
    const void* src[TQP_MAX_AGGS];   // SUM pair: int128 (lo, hi) rows; MIN/MAX: int64 rows
    uint64_t* plo[TQP_MAX_AGGS];
    int64_t* phi[TQP_MAX_AGGS];
    uint64_t* pkey;
    int64_t m;
};

__global__ void gb_merge_pack_kernel(MergeArgs a) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < a.m; i += (int64_t)gridDim.x * blockDim.x) {
        uint64_t kk = 0;
        if (a.n_keys > 0) {
            uint64_t kmin[TQP_MAX_KEYS];
            int shift[TQP_MAX_KEYS], width[TQP_MAX_KEYS];
            key_layout(a.krange, a.n_keys, kmin, shift, width);
            for (int c = 0; c < a.n_keys; c++)
                kk |= (key_part(load_as_i64(a.kcol[c], a.kdt[c], i), a.kdt[c]) - kmin[c]) << shift[c];
        }
        a.pkey[i] = kk;
        for (int j = 0; j < a.n_pairs; j++) {
            if (a.pop[j] == P_SUM) {
                a.plo[j][i] = ((const uint64_t*)a.src[j])[2 * i];
                a.phi[j][i] = ((const int64_t*)a.src[j])[2 * i + 1];
            } else {
                a.plo[j][i] = ((const uint64_t*)a.src[j])[i];
            }
        }
    }
}
}  // namespace

// Merge of partial group-by results (e.g. one fetch output per rank, concatenated):
// partial row i has key columns key_cols[k][i], COUNT(*) counts[i], and per
// aggregate a partial[a][i] (SUM and AVG: the int128 SUM of the aggregate's
// expression; MIN / MAX: int64; COUNT: ignored). Phase 2 of the group-by
// (global radix sort of packed keys, segment ids, exact int128 merge) is
// applied; AVG is recomputed from the merged SUM and COUNT.
tqp_groupby_plan* groupby_merge(tqp_ctx* ctx, int64_t m, const tqp_col* key_cols, int n_keys, const tqp_agg* aggs,
                                int n_aggs, const void* const* partial, const int64_t* counts, int64_t* n_groups_host) {
    if (m < 0 || n_keys < 0 || n_keys > TQP_MAX_KEYS || n_aggs < 0 || n_aggs > TQP_MAX_AGGS)
        fail(TQP_ERR_INVALID_ARGUMENT, "groupby_merge: bad sizes");
    if (m > 0 && !counts) fail(TQP_ERR_INVALID_ARGUMENT, "groupby_merge: null counts");
    for (int k = 0; k < n_keys; k++) check_col(key_cols[k], m, "groupby_merge key");
    for (int g = 0; g < n_aggs; g++)
        if (aggs[g].op < TQP_SUM || aggs[g].op > TQP_AVG || aggs[g].n_factors < 0 || aggs[g].n_factors > 3)
            fail(TQP_ERR_INVALID_ARGUMENT, "groupby_merge: aggregate");
    auto* PL = new tqp_groupby_plan();
    try {
        PL->n_keys = n_keys;
        PL->n_aggs = n_aggs;
        MergeArgs a{};
        a.n_keys = n_keys;
        a.m = m;
        int off = 0;
        int kd[TQP_MAX_KEYS];
        const void* kc[TQP_MAX_KEYS];
        for (int k = n_keys - 1; k >= 0; k--) {
            a.kcol[k] = key_cols[k].data;
            a.kdt[k] = key_cols[k].dtype;
            PL->kdt[k] = key_cols[k].dtype;
            kc[k] = key_cols[k].data;
            kd[k] = key_cols[k].dtype;
            off += 8 * (int)dtype_size(key_cols[k].dtype);
        }
        if (off > 64) fail(TQP_ERR_INVALID_ARGUMENT, "groupby_merge: packed key wider than 64 bits");
        key_ranges(ctx, kc, kd, n_keys, m, PL->krange);
        a.krange = PL->krange.get();
        int pf[TQP_MAX_AGGS][3], ps[TQP_MAX_AGGS][3], pnf[TQP_MAX_AGGS];
        int64_t pa[TQP_MAX_AGGS][3];
        make_pairs(PL, aggs, n_aggs, pf, ps, pa, pnf);
        Partials pr;
        pr.P = m;
        if (m == 0) {
            PL->G = n_keys == 0 ? 1 : 0;
            PL->empty_global = n_keys == 0;
            *n_groups_host = PL->G;
            return PL;
        }
        pr.pkey.alloc(ctx, m);
        pr.pcount.alloc(ctx, m);
        TQP_CUDA(cudaMemcpyAsync(pr.pcount.get(), counts, m * 8, cudaMemcpyDeviceToDevice, ctx->stream));
        a.pkey = pr.pkey.get();
        a.n_pairs = PL->n_pairs;
        for (int j = 0; j < PL->n_pairs; j++) {
            a.pop[j] = PL->pop[j];
            a.src[j] = nullptr;
            for (int g = 0; g < n_aggs && !a.src[j]; g++)
                if (PL->apair[g] == j) a.src[j] = partial ? partial[g] : nullptr;
            if (!a.src[j]) fail(TQP_ERR_INVALID_ARGUMENT, "groupby_merge: missing partial array");
            pr.plo[j].alloc(ctx, m);
            a.plo[j] = pr.plo[j].get();
            if (PL->pop[j] == P_SUM) { pr.phi[j].alloc(ctx, m); a.phi[j] = pr.phi[j].get(); }
        }
        const int g = (int)std::min<int64_t>(ceil_div(m, 256), (int64_t)ctx->num_sms * 8);
        launch(ctx, "tqp_groupby_merge_pack", gb_merge_pack_kernel, dim3(g), dim3(256), 0, a);
        phase2(ctx, PL, pr, false);
        *n_groups_host = PL->G;
        return PL;
    } catch (...) {
        delete PL;
        throw;
    }
}

// ------------------------------------------------------- fp64 aggregates
// SURVEY.md §8(f) NEXT 4 ("fp64 value columns"): aggregates whose factors include a
// TQP_F64 column are evaluated in fp64, value = prod_f (add_f + sign_f * x_f) left to
// right, beside the integer plan: the plan's groups (sorted packed keys) are found by a
// binary search of each passing row's packed key, and the values are reduced with
// atomics -- per CTA in shared memory when the groups x aggregates fit, then once per
// CTA into the global accumulators. SUM is therefore a float sum in an unspecified
// order (|error| <= (m - 1) u sum|v| for a group of m rows, u = 2^-53); MIN / MAX are
// exact (order-preserving int64 images of the doubles, NaN inputs unsupported).
namespace {
constexpr int F64_PRIV = 2048;   // groups x fp64 aggregates kept per CTA in shared memory

struct F64Args {
    int64_t n;
    TermSet ts;
    const void* tcol[TQP_MAX_PREDS];
    int n_keys;
    const void* kcol[TQP_MAX_KEYS];
    int kdt[TQP_MAX_KEYS];
    const unsigned long long* krange;
    const uint64_t* gkey;
    int64_t G;
    int na;
    int op[TQP_MAX_AGGS];          // P_SUM / P_MIN / P_MAX
    int nf[TQP_MAX_AGGS];
    const void* fcol[TQP_MAX_AGGS][3];
    int fdt[TQP_MAX_AGGS][3];
    double fadd[TQP_MAX_AGGS][3];
    double fsign[TQP_MAX_AGGS][3];
    unsigned long long* acc[TQP_MAX_AGGS];   // G slots each (double bits or ordered int64)
    int priv;
};

__device__ __forceinline__ long long dord(double x) {   // order-preserving int64 image
    const long long b = __double_as_longlong(x);
    return b >= 0 ? b : b ^ 0x7FFFFFFFFFFFFFFFll;
}
__device__ __forceinline__ double dunord(long long o) {
    return __longlong_as_double(o >= 0 ? o : o ^ 0x7FFFFFFFFFFFFFFFll);
}

__device__ __forceinline__ void f64_acc(unsigned long long* p, int op, double v) {
    if (op == P_SUM) atomicAdd(reinterpret_cast<double*>(p), v);
    else if (op == P_MIN) atomicMin(reinterpret_cast<long long*>(p), dord(v));
    else atomicMax(reinterpret_cast<long long*>(p), dord(v));
}

__device__ __forceinline__ unsigned long long f64_init(int op) {
    if (op == P_SUM) return 0ull;   // +0.0
    return (unsigned long long)(op == P_MIN ? dord(__longlong_as_double(0x7FF0000000000000ll))
                                            : dord(__longlong_as_double((long long)0xFFF0000000000000ull)));
}

__global__ void __launch_bounds__(256) gb_f64_init_kernel(F64Args a) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < a.G * a.na; i += (int64_t)gridDim.x * blockDim.x)
        a.acc[i % a.na][i / a.na] = f64_init(a.op[i % a.na]);
}

__global__ void __launch_bounds__(256) gb_f64_kernel(F64Args a) {
    extern __shared__ unsigned long long s_acc[];   // [G][na] when a.priv
    if (a.priv) {
        for (int i = threadIdx.x; i < a.G * a.na; i += blockDim.x) s_acc[i] = f64_init(a.op[i % a.na]);
        __syncthreads();
    }
    uint64_t kmin[TQP_MAX_KEYS];
    int sh[TQP_MAX_KEYS], wd[TQP_MAX_KEYS];
    key_layout(a.krange, a.n_keys, kmin, sh, wd);
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < a.n; r += (int64_t)gridDim.x * blockDim.x) {
        bool pass = !a.ts.never;
        for (int q = 0; q < a.ts.n && pass; q++) {
            const Term& t = a.ts.t[q];
            const int64_t x = load_as_i64(a.tcol[q], t.dt, r);
            pass = t.dt == TQP_I64 ? term64((uint64_t)x, t.lo, t.width, t.neg)
                                   : term32((uint32_t)x, (uint32_t)t.lo, (uint32_t)t.width, t.neg);
        }
        if (!pass) continue;
        uint64_t key = 0;
        for (int k = 0; k < a.n_keys; k++)
            key |= (key_part(load_as_i64(a.kcol[k], a.kdt[k], r), a.kdt[k]) - kmin[k]) << sh[k];
        int64_t lo = 0, hi = a.G - 1;   // the row's group: its packed key is one of gkey
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if (a.gkey[mid] < key) lo = mid + 1; else hi = mid;
        }
        for (int j = 0; j < a.na; j++) {
            double v = 1.0;
            for (int f = 0; f < a.nf[j]; f++) {
                const double x = a.fdt[j][f] == TQP_F64 ? reinterpret_cast<const double*>(a.fcol[j][f])[r]
                                                        : (double)load_as_i64(a.fcol[j][f], a.fdt[j][f], r);
                const double t = a.fadd[j][f] + a.fsign[j][f] * x;
                v = f == 0 ? t : v * t;
            }
            f64_acc(a.priv ? &s_acc[lo * a.na + j] : &a.acc[j][lo], a.op[j], v);
        }
    }
    if (a.priv) {
        __syncthreads();
        for (int i = threadIdx.x; i < a.G * a.na; i += blockDim.x) {
            const int j = i % a.na;
            if (s_acc[i] != f64_init(a.op[j])) {
                if (a.op[j] == P_SUM) atomicAdd(reinterpret_cast<double*>(&a.acc[j][i / a.na]), __longlong_as_double((long long)s_acc[i]));
                else if (a.op[j] == P_MIN) atomicMin(reinterpret_cast<long long*>(&a.acc[j][i / a.na]), (long long)s_acc[i]);
                else atomicMax(reinterpret_cast<long long*>(&a.acc[j][i / a.na]), (long long)s_acc[i]);
            }
        }
    }
}

struct F64Fin {
    int64_t G;
    int na;
    int uop[TQP_MAX_AGGS];
    const unsigned long long* acc[TQP_MAX_AGGS];
    const int64_t* gcount;
    double* out[TQP_MAX_AGGS];
};

__global__ void gb_f64_fetch_kernel(F64Fin f) {
    for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < f.G; g += (int64_t)gridDim.x * blockDim.x)
        for (int j = 0; j < f.na; j++) {
            if (!f.out[j]) continue;
            const long long w = (long long)f.acc[j][g];
            double v;
            if (f.uop[j] == TQP_SUM) v = __longlong_as_double(w);
            else if (f.uop[j] == TQP_AVG) v = __longlong_as_double(w) / (double)f.gcount[g];
            else v = dunord(w);
            f.out[j][g] = v;
        }
}
}  // namespace

tqp_groupby_plan* groupby_prepare(tqp_ctx* ctx, const tqp_col* cols, int n_cols, int64_t n, const int32_t* key_idx,
                                  int n_keys, const tqp_pred* preds, int n_preds, const tqp_agg* aggs, int n_aggs,
                                  int64_t* n_groups_host) {
    if (n_cols < 0 || n_aggs < 0 || n_aggs > TQP_MAX_AGGS || n_keys < 0 || n_preds < 0)
        fail(TQP_ERR_INVALID_ARGUMENT, "groupby: bad sizes");
    bool is_f64[TQP_MAX_AGGS] = {};
    bool any = false;
    for (int g = 0; g < n_aggs; g++) {
        if (aggs[g].op == TQP_COUNT || aggs[g].n_factors < 0 || aggs[g].n_factors > 3) continue;
        for (int f = 0; f < aggs[g].n_factors; f++) {
            const int c = aggs[g].col[f];
            if (c >= 0 && c < n_cols && cols[c].dtype == TQP_F64) is_f64[g] = true;
        }
        any = any || is_f64[g];
    }
    bool f64_col = false;
    for (int c = 0; c < n_cols; c++) f64_col = f64_col || cols[c].dtype == TQP_F64;
    if (!f64_col) {
        tqp_groupby_plan* P = groupby_prepare_int(ctx, cols, n_cols, n, key_idx, n_keys, preds, n_preds, aggs, n_aggs,
                                                  n_groups_host);
        P->n_user_aggs = n_aggs;
        return P;
    }
    // fp64 columns: only as aggregate factors; the integer plan sees a never-read u8 view
    for (int k = 0; k < n_keys; k++)
        if (key_idx[k] >= 0 && key_idx[k] < n_cols && cols[key_idx[k]].dtype == TQP_F64)
            fail(TQP_ERR_INVALID_ARGUMENT, "groupby: fp64 columns cannot be group keys");
    for (int q = 0; q < n_preds; q++)
        if (preds[q].col >= 0 && preds[q].col < n_cols && cols[preds[q].col].dtype == TQP_F64)
            fail(TQP_ERR_INVALID_ARGUMENT, "groupby: fp64 columns cannot carry predicates");
    std::vector<tqp_col> c2(cols, cols + n_cols);
    for (auto& c : c2)
        if (c.dtype == TQP_F64) {
            if (n > 0 && !c.data) fail(TQP_ERR_INVALID_ARGUMENT, "groupby column: null data");
            c.dtype = TQP_U8;
        }
    for (int g = 0; g < n_aggs; g++) {
        if (!is_f64[g]) continue;
        if (aggs[g].op < TQP_SUM || aggs[g].op > TQP_AVG) fail(TQP_ERR_INVALID_ARGUMENT, "groupby: aggregate");
        for (int f = 0; f < aggs[g].n_factors; f++)
            if (aggs[g].col[f] < 0 || aggs[g].col[f] >= n_cols || (aggs[g].sign[f] != 1 && aggs[g].sign[f] != -1))
                fail(TQP_ERR_INVALID_ARGUMENT, "groupby: aggregate factor");
    }
    std::vector<tqp_agg> ia;
    int imap[TQP_MAX_AGGS];
    for (int g = 0; g < n_aggs; g++) {
        imap[g] = is_f64[g] ? -1 : (int)ia.size();
        if (!is_f64[g]) ia.push_back(aggs[g]);
    }
    tqp_groupby_plan* P = groupby_prepare_int(ctx, c2.data(), n_cols, n, key_idx, n_keys, preds, n_preds,
                                              ia.empty() ? nullptr : ia.data(), (int)ia.size(), n_groups_host);
    try {
        P->n_user_aggs = n_aggs;
        P->has_f64 = any;
        for (int g = 0; g < n_aggs; g++) {
            P->uop[g] = aggs[g].op;
            P->imap[g] = imap[g];
        }
        if (!any || P->G == 0) return P;
        F64Args a{};
        a.n = n;
        a.ts = make_terms(preds, n_preds, [&](int c) { return cols[c].dtype; });
        for (int q = 0; q < a.ts.n; q++) a.tcol[q] = cols[a.ts.t[q].col].data;
        a.n_keys = n_keys;
        for (int k = 0; k < n_keys; k++) {
            a.kcol[k] = cols[key_idx[k]].data;
            a.kdt[k] = cols[key_idx[k]].dtype;
        }
        a.krange = P->krange.get();
        a.gkey = P->gkey.get();
        a.G = P->G;
        for (int g = 0; g < n_aggs; g++) {
            if (!is_f64[g]) continue;
            const int j = a.na++;
            a.op[j] = aggs[g].op == TQP_MIN ? P_MIN : (aggs[g].op == TQP_MAX ? P_MAX : P_SUM);
            a.nf[j] = aggs[g].n_factors;
            for (int f = 0; f < aggs[g].n_factors; f++) {
                const tqp_col& c = cols[aggs[g].col[f]];
                a.fcol[j][f] = c.data;
                a.fdt[j][f] = c.dtype;
                a.fadd[j][f] = (double)aggs[g].add[f];
                a.fsign[j][f] = (double)aggs[g].sign[f];
            }
            P->gf[g].alloc(ctx, P->G);
            a.acc[j] = reinterpret_cast<unsigned long long*>(P->gf[g].get());
        }
        const int gi = (int)std::min<int64_t>(ceil_div(P->G * a.na, 256), (int64_t)ctx->num_sms * 8);
        launch(ctx, "tqp_groupby_f64", gb_f64_init_kernel, dim3(gi), dim3(256), 0, a);
        if (n > 0) {
            a.priv = P->G * a.na <= F64_PRIV ? 1 : 0;
            const size_t smem = a.priv ? (size_t)P->G * a.na * 8 : 0;
            if (smem > 48 * 1024) set_smem(gb_f64_kernel, smem);
            const int occ = std::max(1, occupancy(gb_f64_kernel, 256, smem));
            const int g = (int)std::min<int64_t>(ceil_div(n, 256), (int64_t)ctx->num_sms * occ);
            launch(ctx, "tqp_groupby_f64", gb_f64_kernel, dim3(g), dim3(256), smem, a);
            double b = 0;
            for (int c = 0; c < n_cols; c++) b += (double)dtype_size(cols[c].dtype);
            ctx->add_bytes("tqp_groupby_f64", b * (double)n);
        }
        return P;
    } catch (...) {
        delete P;
        throw;
    }
}

void groupby_fetch(tqp_ctx* ctx, const tqp_groupby_plan* PL, void* const* keys_out, void* const* results_out) {
    if (!PL->has_f64) {   // integer plans (and merge plans) as they are
        groupby_fetch_int(ctx, PL, keys_out, results_out);
        return;
    }
    void* iout[TQP_MAX_AGGS] = {};
    F64Fin f{};
    f.G = PL->G;
    f.gcount = PL->gcount.get();
    for (int g = 0; g < PL->n_user_aggs; g++) {
        void* o = results_out ? results_out[g] : nullptr;
        if (PL->imap[g] >= 0) {
            iout[PL->imap[g]] = o;
        } else {
            const int j = f.na++;
            f.uop[j] = PL->uop[g];
            f.acc[j] = reinterpret_cast<const unsigned long long*>(PL->gf[g].get());
            f.out[j] = static_cast<double*>(o);
        }
    }
    groupby_fetch_int(ctx, PL, keys_out, iout);
    if (f.na > 0 && PL->G > 0) {
        const int g = (int)std::min<int64_t>(ceil_div(PL->G, 256), (int64_t)ctx->num_sms * 8);
        launch(ctx, "tqp_groupby_f64", gb_f64_fetch_kernel, dim3(g), dim3(256), 0, f);
    }
}

}  // namespace tqp
