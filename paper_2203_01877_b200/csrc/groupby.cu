// groupby.cu -- sort-based group-by aggregation, Alg. 2 (
// prose :1146-1152), with a fused pre-filter (Listings 1-2 predicate form).
//
// Alg. 2: cat(grpByCols) -> radix sort -> permute data -> uniqueConsecutive
// (unique keys + inverse = segment ids) -> evaluate aggregates per segment.
// The paper materialises every step as a whole-tensor op (and names
// uniqueConsecutive as a bottleneck). Here it is two
// levels of the same sort-based algorithm:
//   phase 1 (one kernel, one pass over the input columns): each CTA tile of
//     2048 rows evaluates the predicates, packs the key columns into one
//     64-bit key (column 0 most significant, reading R12), radix-sorts its
//     passing rows by key in shared memory (stable LSD passes with warp
//     match_any ranking), marks segment boundaries (the unique/inverse step),
//     and reduces every aggregate per segment in registers/shared memory
//     (int64 values split into 32-bit halves so partial sums are exact),
//     emitting one partial record per (tile, distinct key);
//   phase 2: the partial records are radix-sorted by key (sort.cu), segment
//     boundaries give the final groups, and partials are added into exact
//     int128 accumulators (64-bit atomics with explicit carry, order
//     independent => bit-exact), then finalised (AVG = rn(sum / count)).
#include "internal.h"

struct tqp_groupby_plan {
    int64_t G = 0;
    int n_keys = 0, n_aggs = 0;
    int kdt[TQP_MAX_KEYS];
    int kshift[TQP_MAX_KEYS];
    int aop[TQP_MAX_AGGS];
    bool empty_global = false;   // n_keys == 0 and no passing row
    tqp::DevBuf<uint64_t> gkey;
    tqp::DevBuf<int64_t> gcount;
    tqp::DevBuf<uint64_t> glo[TQP_MAX_AGGS];
    tqp::DevBuf<int64_t> ghi[TQP_MAX_AGGS];
};

namespace tqp {

namespace {
constexpr int GNT = 256;
constexpr int GNW = GNT / 32;
constexpr int GIPT = 8;
constexpr int GTILE = GNT * GIPT;   // 2048 rows per tile (fits u16 indices)

struct GBArgs {
    int n_keys;
    const void* kcol[TQP_MAX_KEYS];
    int kdt[TQP_MAX_KEYS];
    int kshift[TQP_MAX_KEYS];
    int n_preds;
    const void* pcol[TQP_MAX_PREDS];
    int pdt[TQP_MAX_PREDS];
    int pop[TQP_MAX_PREDS];
    int64_t pval[TQP_MAX_PREDS];
    int n_aggs;
    int aop[TQP_MAX_AGGS];
    int anf[TQP_MAX_AGGS];
    const void* acol[TQP_MAX_AGGS][3];
    int adt[TQP_MAX_AGGS][3];
    int asign[TQP_MAX_AGGS][3];
    int64_t aadd[TQP_MAX_AGGS][3];
    int64_t n;
    // phase-1 partial records
    uint64_t* pkey;
    int64_t* pcount;
    uint64_t* plo[TQP_MAX_AGGS];   // SUM/AVG: low 64 bits of the int128 partial; MIN/MAX: value
    int64_t* phi[TQP_MAX_AGGS];    // SUM/AVG: high 64 bits
    uint64_t* status;
    unsigned long long* counter;
    int64_t* P_out;
    int64_t n_tiles;
    int* overflow;
};

__device__ __forceinline__ bool cmp_op(int64_t x, int op, int64_t v) {
    switch (op) {
        case TQP_LT: return x < v;
        case TQP_LE: return x <= v;
        case TQP_GT: return x > v;
        case TQP_GE: return x >= v;
        case TQP_EQ: return x == v;
        default: return x != v;
    }
}

__device__ __forceinline__ uint64_t key_part(int64_t v, int dt) {
    switch (dt) {
        case TQP_U8: return (uint64_t)v & 0xFFull;
        case TQP_I32: return (uint64_t)((uint32_t)v ^ 0x80000000u);
        default: return (uint64_t)v ^ 0x8000000000000000ull;
    }
}

// value = prod_f (add_f + sign_f * col_f[row]) in int64; sets *ovf on overflow.
__device__ __forceinline__ int64_t agg_value(const GBArgs& a, int ag, int64_t row, int* ovf) {
    int64_t v = 1;
    for (int f = 0; f < a.anf[ag]; f++) {
        const int64_t x = load_as_i64(a.acol[ag][f], a.adt[ag][f], row);
        const int64_t sx = a.asign[ag][f] < 0 ? -x : x;
        if (a.asign[ag][f] < 0 && x == INT64_MIN) *ovf = 1;
        const int64_t t = a.aadd[ag][f] + sx;
        if (((a.aadd[ag][f] ^ t) & (sx ^ t)) < 0) *ovf = 1;   // signed add overflow
        const int64_t lo = v * t;
        const int64_t hi = __mul64hi(v, t);
        if (hi != (lo >> 63)) *ovf = 1;                       // signed mul overflow
        v = lo;
    }
    return v;
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

struct GBSmem {
    uint64_t skey[2][GTILE];        // 32 KB: sort ping-pong; the spare buffer holds per-row values
    uint64_t acc_lo[GTILE];         // 16 KB: per-segment accumulators
    int64_t acc_hi[GTILE];          // 16 KB
    uint16_t sidx[2][GTILE + 2];    // 8 KB: local row of each sorted element / run starts
    uint16_t inv[GTILE];            // 4 KB: local row -> sorted position
    uint16_t srun[GTILE];           // 4 KB: segment id of each sorted position
    uint32_t whist[GNW][256];       // 8 KB: per-warp digit counters
    uint32_t tstart[256];
    uint32_t s_w[GNW];
    uint32_t s_cnt[GNW * GIPT];
    uint64_t s_min[GNW], s_max[GNW];
    int64_t s_tile;
    uint64_t s_pbase;
    uint32_t s_m, s_U;
};

// One stable LSD pass over positions [0, m) of the tile: rank by the 8-bit digit
// at `shift` with warp match_any (warp-striped positions keep warp-local order
// equal to position order), then scatter to dst.
__device__ __forceinline__ void tile_pass(GBSmem& s, int src, int m, int shift) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int dst = src ^ 1;
    for (int d = lane; d < 256; d += 32) s.whist[warp][d] = 0;
    __syncwarp();
    uint64_t k[GIPT];
    uint16_t ix[GIPT];
    uint32_t rk[GIPT];
    const unsigned lt = lanemask_lt();
#pragma unroll
    for (int i = 0; i < GIPT; i++) {
        const int q = warp * 32 * GIPT + i * 32 + lane;
        const bool valid = q < m;
        if (valid) { k[i] = s.skey[src][q]; ix[i] = s.sidx[src][q]; }
        const unsigned vm = __ballot_sync(0xffffffffu, valid);
        if (valid) {
            const uint32_t d = (uint32_t)(k[i] >> shift) & 255u;
            const unsigned peers = __match_any_sync(vm, d);
            const uint32_t before = s.whist[warp][d];
            rk[i] = before + __popc(peers & lt);
            __syncwarp(vm);
            if (lane == 31 - __clz(peers)) s.whist[warp][d] = before + __popc(peers);
            __syncwarp(vm);
        }
    }
    __syncthreads();
    uint32_t cnt = 0;
#pragma unroll
    for (int w = 0; w < GNW; w++) {
        const uint32_t c = s.whist[w][tid];
        s.whist[w][tid] = cnt;
        cnt += c;
    }
    s.tstart[tid] = bscan256(cnt, s.s_w);
    __syncthreads();
#pragma unroll
    for (int i = 0; i < GIPT; i++) {
        const int q = warp * 32 * GIPT + i * 32 + lane;
        if (q < m) {
            const uint32_t d = (uint32_t)(k[i] >> shift) & 255u;
            const uint32_t p = s.tstart[d] + s.whist[warp][d] + rk[i];
            s.skey[dst][p] = k[i];
            s.sidx[dst][p] = ix[i];
        }
    }
    __syncthreads();
}

__global__ void __launch_bounds__(GNT) gb_phase1_kernel(GBArgs a) {
    extern __shared__ __align__(16) uint8_t smem_raw[];
    GBSmem& s = *reinterpret_cast<GBSmem*>(smem_raw);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) s.s_tile = (int64_t)atomicAdd(a.counter, 1ull);
    __syncthreads();
    const int64_t tile = s.s_tile;
    const int64_t base = tile * GTILE;
    const unsigned lt = lanemask_lt();

    // 1. predicates + packed key (rows are warp-striped: local row = warp*256 + i*32 + lane)
    uint64_t key[GIPT];
    unsigned bal[GIPT];
    uint64_t kmin = ~0ull, kmax = 0;
#pragma unroll
    for (int i = 0; i < GIPT; i++) {
        const int64_t row = base + warp * 32 * GIPT + i * 32 + lane;
        bool pass = row < a.n;
        key[i] = 0;
        if (pass) {
            for (int q = 0; q < a.n_preds; q++)
                pass = pass && cmp_op(load_as_i64(a.pcol[q], a.pdt[q], row), a.pop[q], a.pval[q]);
        }
        if (pass) {
            uint64_t kk = 0;
            for (int c = 0; c < a.n_keys; c++)
                kk |= key_part(load_as_i64(a.kcol[c], a.kdt[c], row), a.kdt[c]) << a.kshift[c];
            key[i] = kk;
            kmin = min(kmin, kk);
            kmax = max(kmax, kk);
        }
        bal[i] = __ballot_sync(0xffffffffu, pass);
        if (lane == 0) s.s_cnt[warp * GIPT + i] = __popc(bal[i]);
    }
    for (int o = 16; o > 0; o >>= 1) {
        kmin = min(kmin, __shfl_xor_sync(0xffffffffu, kmin, o));
        kmax = max(kmax, __shfl_xor_sync(0xffffffffu, kmax, o));
    }
    if (lane == 0) { s.s_min[warp] = kmin; s.s_max[warp] = kmax; }
    __syncthreads();
    if (warp == 0) {   // exclusive scan over the 64 (warp, item) counts in row order
        const uint32_t c0 = s.s_cnt[2 * lane], c1 = s.s_cnt[2 * lane + 1];
        uint32_t x = c0 + c1;
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        const uint32_t ex = x - c0 - c1;
        s.s_cnt[2 * lane] = ex;
        s.s_cnt[2 * lane + 1] = ex + c0;
        if (lane == 31) s.s_m = x;
    }
    kmin = ~0ull;
    kmax = 0;
    for (int w = 0; w < GNW; w++) { kmin = min(kmin, s.s_min[w]); kmax = max(kmax, s.s_max[w]); }
    __syncthreads();
    const int m = (int)s.s_m;
    // 2. compact passing rows (in row order) into sort buffer 0 as (key - kmin, local row)
#pragma unroll
    for (int i = 0; i < GIPT; i++) {
        if (bal[i] & (1u << lane)) {
            const uint32_t c = s.s_cnt[warp * GIPT + i] + __popc(bal[i] & lt);
            s.skey[0][c] = key[i] - kmin;
            s.sidx[0][c] = (uint16_t)(warp * 32 * GIPT + i * 32 + lane);
        }
    }
    __syncthreads();
    // 3. in-tile stable LSD radix sort over the bits that vary in this tile
    const int bits = (m > 0 && kmax != kmin) ? 64 - __clzll(kmax - kmin) : 0;
    const int passes = (bits + 7) / 8;
    for (int p = 0; p < passes; p++) tile_pass(s, p & 1, m, 8 * p);
    const int fin = passes & 1;
    const uint64_t* sk = s.skey[fin];
    uint64_t* sval = s.skey[fin ^ 1];           // spare buffer: per-row values in sorted order
    uint16_t* rstart = s.sidx[fin ^ 1];         // spare buffer: segment starts
    // 4. inverse map and segment boundaries (uniqueConsecutive)
    for (int p = tid; p < m; p += GNT) s.inv[s.sidx[fin][p]] = (uint16_t)p;
    uint32_t heads = 0;
#pragma unroll
    for (int j = 0; j < GIPT; j++) {
        const int p = tid * GIPT + j;
        if (p < m && (p == 0 || sk[p] != sk[p - 1])) heads++;
    }
    uint32_t hex = bscan256(heads, s.s_w);
    {
        uint32_t r = hex;
#pragma unroll
        for (int j = 0; j < GIPT; j++) {
            const int p = tid * GIPT + j;
            if (p < m) {
                if (p == 0 || sk[p] != sk[p - 1]) { rstart[r] = (uint16_t)p; r++; }
                s.srun[p] = (uint16_t)(r - 1);
            }
        }
        if (tid == GNT - 1) s.s_U = r;
    }
    __syncthreads();
    const int U = (int)s.s_U;
    if (tid == 0) rstart[U] = (uint16_t)m;
    // 5. place of this tile's partial records: decoupled look-back over U
    if (warp == 0) {
        const uint64_t e = lookback_warp(a.status, tile, (uint64_t)U, OpAdd(), 0ull);
        if (lane == 0) {
            s.s_pbase = e;
            if (tile == a.n_tiles - 1) *a.P_out = (int64_t)(e + U);
        }
    }
    __syncthreads();
    const int64_t pb = (int64_t)s.s_pbase;
    for (int u = tid; u < U; u += GNT) {
        a.pkey[pb + u] = sk[rstart[u]] + kmin;
        a.pcount[pb + u] = (int64_t)rstart[u + 1] - rstart[u];
    }
    // 6. segmented reduction of every aggregate
    int ovf = 0;
    for (int ag = 0; ag < a.n_aggs; ag++) {
        const int op = a.aop[ag];
        if (op == TQP_COUNT) continue;
        const bool is_sum = (op == TQP_SUM || op == TQP_AVG);
#pragma unroll
        for (int i = 0; i < GIPT; i++) {
            if (bal[i] & (1u << lane)) {
                const int lr = warp * 32 * GIPT + i * 32 + lane;
                const int64_t row = base + lr;
                sval[s.inv[lr]] = (uint64_t)agg_value(a, ag, row, &ovf);
            }
        }
        for (int u = tid; u < U; u += GNT) {
            s.acc_lo[u] = is_sum ? 0ull : (op == TQP_MIN ? (uint64_t)INT64_MAX : (uint64_t)INT64_MIN);
            s.acc_hi[u] = 0;
        }
        __syncthreads();
        // thread t reduces the blocked positions [t*8, t*8+8)
        const int p0 = tid * GIPT;
        const int pl = min(p0 + GIPT, m) - 1;
        const bool any = p0 < m;
        const int r0 = any ? s.srun[p0] : -1;
        const int rl = any ? s.srun[pl] : -1;
        const int wr0 = __shfl_sync(0xffffffffu, r0, 0);
        const bool uniform = __all_sync(0xffffffffu, any && r0 == rl && r0 == wr0);
        uint64_t lo = 0;
        int64_t hi = 0;
        int64_t mm = op == TQP_MIN ? INT64_MAX : INT64_MIN;
        int cur = r0;
        for (int p = p0; p <= pl; p++) {
            const int r = s.srun[p];
            if (r != cur) {
                if (is_sum) {
                    atomicAdd((unsigned long long*)&s.acc_lo[cur], (unsigned long long)lo);
                    atomicAdd((unsigned long long*)&s.acc_hi[cur], (unsigned long long)hi);
                } else if (op == TQP_MIN) atomicMin((long long*)&s.acc_lo[cur], (long long)mm);
                else atomicMax((long long*)&s.acc_lo[cur], (long long)mm);
                lo = 0; hi = 0; mm = op == TQP_MIN ? INT64_MAX : INT64_MIN;
                cur = r;
            }
            const int64_t v = (int64_t)sval[p];
            if (is_sum) { lo += (uint64_t)(uint32_t)v; hi += (v >> 32); }
            else mm = op == TQP_MIN ? min(mm, v) : max(mm, v);
        }
        if (uniform) {
            for (int o = 16; o > 0; o >>= 1) {
                if (is_sum) {
                    lo += __shfl_xor_sync(0xffffffffu, lo, o);
                    hi += __shfl_xor_sync(0xffffffffu, hi, o);
                } else {
                    const int64_t t = __shfl_xor_sync(0xffffffffu, mm, o);
                    mm = op == TQP_MIN ? min(mm, t) : max(mm, t);
                }
            }
        }
        if (any && (!uniform || lane == 0)) {
            if (is_sum) {
                atomicAdd((unsigned long long*)&s.acc_lo[cur], (unsigned long long)lo);
                atomicAdd((unsigned long long*)&s.acc_hi[cur], (unsigned long long)hi);
            } else if (op == TQP_MIN) atomicMin((long long*)&s.acc_lo[cur], (long long)mm);
            else atomicMax((long long*)&s.acc_lo[cur], (long long)mm);
        }
        __syncthreads();
        for (int u = tid; u < U; u += GNT) {
            if (is_sum) {
                // exact: value = acc_hi * 2^32 + acc_lo  (|acc_hi| < 2^43, acc_lo < 2^43)
                const __int128 t = ((__int128)s.acc_hi[u] << 32) + (__int128)s.acc_lo[u];
                a.plo[ag][pb + u] = (uint64_t)t;
                a.phi[ag][pb + u] = (int64_t)(t >> 64);
            } else {
                a.plo[ag][pb + u] = s.acc_lo[u];
            }
        }
        __syncthreads();
    }
    if (ovf) atomicOr(a.overflow, 1);
}

// Phase 2a: group ids over the sorted partial keys (segment boundaries).
__global__ void __launch_bounds__(GNT) gb_gid_kernel(const uint64_t* __restrict__ sk, int64_t P, uint32_t* gid,
                                                     uint64_t* gkey, int64_t* G_out, uint64_t* status,
                                                     unsigned long long* counter, int64_t n_tiles) {
    __shared__ int64_t s_tile;
    __shared__ uint32_t s_cnt[GIPT * GNW];
    __shared__ uint64_t s_excl;
    __shared__ uint32_t s_tot;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t tile = take_tile(counter, &s_tile);
    const int64_t base = tile * GTILE;
    unsigned bal[GIPT];
    uint64_t k[GIPT];
#pragma unroll
    for (int i = 0; i < GIPT; i++) {
        const int64_t p = base + i * GNT + tid;
        bool head = false;
        if (p < P) { k[i] = sk[p]; head = p == 0 || sk[p - 1] != k[i]; }
        bal[i] = __ballot_sync(0xffffffffu, head);
        if (lane == 0) s_cnt[i * GNW + warp] = __popc(bal[i]);
    }
    __syncthreads();
    if (warp == 0) {
        constexpr int PER = GIPT * GNW / 32;
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
    for (int i = 0; i < GIPT; i++) {
        const int64_t p = base + i * GNT + tid;
        if (p < P) {
            const int64_t g = excl + s_cnt[i * GNW + warp] + __popc(bal[i] & le) - 1;
            gid[p] = (uint32_t)g;
            if (bal[i] & (1u << lane)) gkey[g] = k[i];
        }
    }
    if (tile == n_tiles - 1 && tid == 0) *G_out = excl + s_tot;
}

struct AccArgs {
    int n_aggs;
    int aop[TQP_MAX_AGGS];
    const uint64_t* plo[TQP_MAX_AGGS];
    const int64_t* phi[TQP_MAX_AGGS];
    uint64_t* glo[TQP_MAX_AGGS];
    int64_t* ghi[TQP_MAX_AGGS];
    const int64_t* pcount;
    int64_t* gcount;
    const uint32_t* perm;
    const uint32_t* gid;
    int64_t P;
};

// exact 128-bit atomic accumulation: the carry out of the low word is detected
// from the value atomicAdd returns, so the total is exact for any order.
__device__ __forceinline__ void atomic_add_i128(uint64_t* lo_p, int64_t* hi_p, uint64_t lo, int64_t hi) {
    const uint64_t old = atomicAdd((unsigned long long*)lo_p, (unsigned long long)lo);
    const int64_t carry = (old + lo < old) ? 1 : 0;
    const int64_t h = hi + carry;
    if (h) atomicAdd((unsigned long long*)hi_p, (unsigned long long)h);
}

__global__ void __launch_bounds__(GNT) gb_acc_kernel(AccArgs a) {
    const int lane = threadIdx.x & 31;
    for (int64_t p0 = blockIdx.x * (int64_t)GNT; p0 < a.P; p0 += (int64_t)gridDim.x * GNT) {
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
        for (int ag = 0; ag < a.n_aggs; ag++) {
            const int op = a.aop[ag];
            if (op == TQP_COUNT) continue;
            if (op == TQP_SUM || op == TQP_AVG) {
                unsigned __int128 v = 0;
                if (valid) v = ((unsigned __int128)(uint64_t)a.phi[ag][rec] << 64) | a.plo[ag][rec];
                if (uniform) {
                    for (int o = 16; o > 0; o >>= 1) {
                        const uint64_t l = __shfl_xor_sync(0xffffffffu, (uint64_t)v, o);
                        const uint64_t h = __shfl_xor_sync(0xffffffffu, (uint64_t)(v >> 64), o);
                        v += ((unsigned __int128)h << 64) | l;
                    }
                    if (lane == 0) atomic_add_i128(&a.glo[ag][g], &a.ghi[ag][g], (uint64_t)v, (int64_t)(v >> 64));
                } else if (valid) {
                    atomic_add_i128(&a.glo[ag][g], &a.ghi[ag][g], (uint64_t)v, (int64_t)(v >> 64));
                }
            } else {
                int64_t v = valid ? (int64_t)a.plo[ag][rec] : (op == TQP_MIN ? INT64_MAX : INT64_MIN);
                if (uniform) {
                    for (int o = 16; o > 0; o >>= 1) {
                        const int64_t t = __shfl_xor_sync(0xffffffffu, v, o);
                        v = op == TQP_MIN ? min(v, t) : max(v, t);
                    }
                }
                if (valid && (!uniform || lane == 0)) {
                    if (op == TQP_MIN) atomicMin((long long*)&a.glo[ag][g], (long long)v);
                    else atomicMax((long long*)&a.glo[ag][g], (long long)v);
                }
            }
        }
    }
}

__global__ void gb_init_kernel(uint64_t* lo, int64_t* hi, int64_t n, uint64_t init) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        lo[i] = init;
        if (hi) hi[i] = 0;
    }
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
    int kshift[TQP_MAX_KEYS];
    void* kout[TQP_MAX_KEYS];
    int aop[TQP_MAX_AGGS];
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
        for (int k = 0; k < a.n_keys; k++) {
            if (!a.kout[k]) continue;
            switch (a.kdt[k]) {
                case TQP_U8: ((uint8_t*)a.kout[k])[g] = (uint8_t)(key >> a.kshift[k]); break;
                case TQP_I32: ((int32_t*)a.kout[k])[g] = (int32_t)((uint32_t)(key >> a.kshift[k]) ^ 0x80000000u); break;
                default: ((int64_t*)a.kout[k])[g] = (int64_t)(key ^ 0x8000000000000000ull); break;
            }
        }
        const int64_t cnt = a.empty_global ? 0 : a.gcount[g];
        for (int ag = 0; ag < a.n_aggs; ag++) {
            if (!a.rout[ag]) continue;
            const int op = a.aop[ag];
            const uint64_t lo = a.empty_global ? (op == TQP_MIN ? (uint64_t)INT64_MAX : op == TQP_MAX ? (uint64_t)INT64_MIN : 0)
                                               : (op == TQP_COUNT ? 0 : a.glo[ag][g]);
            const int64_t hi = (a.empty_global || op == TQP_COUNT || op == TQP_MIN || op == TQP_MAX) ? 0 : a.ghi[ag][g];
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
}  // namespace

tqp_groupby_plan* groupby_prepare(tqp_ctx* ctx, const tqp_col* cols, int n_cols, int64_t n, const int32_t* key_idx,
                                  int n_keys, const tqp_pred* preds, int n_preds, const tqp_agg* aggs, int n_aggs,
                                  int64_t* n_groups_host) {
    if (n < 0 || n_cols < 0 || n_keys < 0 || n_keys > TQP_MAX_KEYS || n_preds < 0 || n_preds > TQP_MAX_PREDS ||
        n_aggs < 0 || n_aggs > TQP_MAX_AGGS)
        fail(TQP_ERR_INVALID_ARGUMENT, "groupby: bad sizes");
    if (n >= (int64_t(1) << 40)) fail(TQP_ERR_INVALID_ARGUMENT, "groupby: n too large");
    for (int c = 0; c < n_cols; c++) check_col(cols[c], n, "groupby column");
    GBArgs a{};
    a.n = n;
    a.n_keys = n_keys;
    int off = 0;
    for (int k = n_keys - 1; k >= 0; k--) {   // column 0 most significant
        const int c = key_idx[k];
        if (c < 0 || c >= n_cols) fail(TQP_ERR_INVALID_ARGUMENT, "groupby: key column");
        a.kcol[k] = cols[c].data;
        a.kdt[k] = cols[c].dtype;
        a.kshift[k] = off;
        off += 8 * (int)dtype_size(cols[c].dtype);
    }
    if (off > 64) fail(TQP_ERR_INVALID_ARGUMENT, "groupby: packed key wider than 64 bits");
    a.n_preds = n_preds;
    for (int q = 0; q < n_preds; q++) {
        if (preds[q].col < 0 || preds[q].col >= n_cols || preds[q].op < TQP_LT || preds[q].op > TQP_NE)
            fail(TQP_ERR_INVALID_ARGUMENT, "groupby: predicate");
        a.pcol[q] = cols[preds[q].col].data;
        a.pdt[q] = cols[preds[q].col].dtype;
        a.pop[q] = preds[q].op;
        a.pval[q] = preds[q].value;
    }
    a.n_aggs = n_aggs;
    for (int g = 0; g < n_aggs; g++) {
        if (aggs[g].op < TQP_SUM || aggs[g].op > TQP_AVG || aggs[g].n_factors < 0 || aggs[g].n_factors > 3)
            fail(TQP_ERR_INVALID_ARGUMENT, "groupby: aggregate");
        a.aop[g] = aggs[g].op;
        a.anf[g] = aggs[g].op == TQP_COUNT ? 0 : aggs[g].n_factors;
        for (int f = 0; f < a.anf[g]; f++) {
            const int c = aggs[g].col[f];
            if (c < 0 || c >= n_cols || (aggs[g].sign[f] != 1 && aggs[g].sign[f] != -1))
                fail(TQP_ERR_INVALID_ARGUMENT, "groupby: aggregate factor");
            a.acol[g][f] = cols[c].data;
            a.adt[g][f] = cols[c].dtype;
            a.asign[g][f] = aggs[g].sign[f];
            a.aadd[g][f] = aggs[g].add[f];
        }
    }
    auto* PL = new tqp_groupby_plan();
    try {
        PL->n_keys = n_keys;
        PL->n_aggs = n_aggs;
        for (int k = 0; k < n_keys; k++) { PL->kdt[k] = a.kdt[k]; PL->kshift[k] = a.kshift[k]; }
        for (int g = 0; g < n_aggs; g++) PL->aop[g] = a.aop[g];

        // ---- phase 1: per-tile sort + segmented reduce -> partial records
        const int64_t tiles = ceil_div(n, GTILE);
        const int64_t cap = std::max<int64_t>(n, 1);
        DevBuf<uint64_t> pkey(ctx, cap);
        DevBuf<int64_t> pcount(ctx, cap);
        DevBuf<uint64_t> plo[TQP_MAX_AGGS];
        DevBuf<int64_t> phi[TQP_MAX_AGGS];
        for (int g = 0; g < n_aggs; g++) {
            if (a.aop[g] == TQP_COUNT) continue;
            plo[g].alloc(ctx, cap);
            a.plo[g] = plo[g].get();
            if (a.aop[g] == TQP_SUM || a.aop[g] == TQP_AVG) { phi[g].alloc(ctx, cap); a.phi[g] = phi[g].get(); }
        }
        DevBuf<int64_t> scal(ctx, 2);   // P, G
        DevBuf<int> ovf(ctx, 1);
        scal.zero();
        ovf.zero();
        a.pkey = pkey.get();
        a.pcount = pcount.get();
        a.P_out = scal.get();
        a.overflow = ovf.get();
        if (n > 0) {
            DevBuf<uint64_t> status(ctx, tiles);
            DevBuf<unsigned long long> counter(ctx, 1);
            status.zero();
            counter.zero();
            a.status = status.get();
            a.counter = counter.get();
            a.n_tiles = tiles;
            const size_t sm = sizeof(GBSmem);
            set_smem(gb_phase1_kernel, sm);
            launch(ctx, "tqp_groupby_tile", gb_phase1_kernel, dim3((unsigned)tiles), dim3(GNT), sm, a);
        }
        int64_t P = 0;
        {
            int64_t h[2];
            int o = 0;
            read_back(ctx, h, scal.get(), 16);
            read_back(ctx, &o, ovf.get(), 4);
            if (o) fail(TQP_ERR_OVERFLOW, "groupby: int64 overflow in an aggregate expression");
            P = h[0];
            // distinct referenced columns read once; partial records written
            double in = 0;
            std::vector<const void*> seen;
            auto note = [&](const void* d, int dt) {
                for (auto x : seen) if (x == d) return;
                seen.push_back(d);
                in += (double)dtype_size(dt);
            };
            for (int k = 0; k < n_keys; k++) note(a.kcol[k], a.kdt[k]);
            for (int q = 0; q < n_preds; q++) note(a.pcol[q], a.pdt[q]);
            for (int g = 0; g < n_aggs; g++)
                for (int f = 0; f < a.anf[g]; f++) note(a.acol[g][f], a.adt[g][f]);
            double rec = 16;
            for (int g = 0; g < n_aggs; g++)
                rec += a.aop[g] == TQP_COUNT ? 0 : (a.aop[g] == TQP_SUM || a.aop[g] == TQP_AVG) ? 16 : 8;
            if (n > 0) ctx->add_bytes("tqp_groupby_tile", in * (double)n + rec * (double)P);
        }
        // ---- phase 2: sort partial keys, segment, accumulate exactly
        if (P == 0) {
            PL->G = n_keys == 0 ? 1 : 0;
            PL->empty_global = n_keys == 0;
            *n_groups_host = PL->G;
            return PL;
        }
        SortOut so;
        so.want_perm32 = true;
        DevBuf<uint64_t> sk(ctx, P);
        so.sorted_u = sk.get();
        radix_sort(ctx, pkey.get(), DT_U64, P, false, so);
        DevBuf<uint32_t> gid(ctx, P);
        PL->gkey.alloc(ctx, P);
        {
            const int64_t t2 = ceil_div(P, GTILE);
            DevBuf<uint64_t> status(ctx, t2);
            DevBuf<unsigned long long> counter(ctx, 1);
            status.zero();
            counter.zero();
            launch(ctx, "tqp_groupby_gid", gb_gid_kernel, dim3((unsigned)t2), dim3(GNT), 0, sk.get(), P, gid.get(),
                   PL->gkey.get(), scal.get() + 1, status.get(), counter.get(), t2);
        }
        AccArgs c{};
        c.n_aggs = n_aggs;
        PL->gcount.alloc(ctx, P);
        PL->gcount.zero();
        const int ig = (int)std::min<int64_t>(ceil_div(P, 256), (int64_t)ctx->num_sms * 8);
        for (int g = 0; g < n_aggs; g++) {
            c.aop[g] = a.aop[g];
            if (a.aop[g] == TQP_COUNT) continue;
            c.plo[g] = plo[g].get();
            c.phi[g] = phi[g].get();
            PL->glo[g].alloc(ctx, P);
            c.glo[g] = PL->glo[g].get();
            if (a.aop[g] == TQP_SUM || a.aop[g] == TQP_AVG) {
                PL->ghi[g].alloc(ctx, P);
                c.ghi[g] = PL->ghi[g].get();
                PL->glo[g].zero();
                PL->ghi[g].zero();
            } else {
                launch(ctx, "tqp_groupby_init", gb_init_kernel, dim3(ig), dim3(256), 0, PL->glo[g].get(),
                       (int64_t*)nullptr, P, a.aop[g] == TQP_MIN ? (uint64_t)INT64_MAX : (uint64_t)INT64_MIN);
            }
        }
        c.pcount = pcount.get();
        c.gcount = PL->gcount.get();
        c.perm = so.perm32.get();
        c.gid = gid.get();
        c.P = P;
        const int ag = (int)std::min<int64_t>(ceil_div(P, GNT), (int64_t)ctx->num_sms * 8);
        launch(ctx, "tqp_groupby_accumulate", gb_acc_kernel, dim3(ag), dim3(GNT), 0, c);
        int64_t h[2];
        read_back(ctx, h, scal.get(), 16);
        PL->G = h[1];
        *n_groups_host = PL->G;
        return PL;
    } catch (...) {
        delete PL;
        throw;
    }
}

void groupby_fetch(tqp_ctx* ctx, const tqp_groupby_plan* PL, void* const* keys_out, void* const* results_out) {
    if (PL->G == 0) return;
    FinArgs f{};
    f.n_keys = PL->n_keys;
    f.n_aggs = PL->n_aggs;
    for (int k = 0; k < PL->n_keys; k++) {
        f.kdt[k] = PL->kdt[k];
        f.kshift[k] = PL->kshift[k];
        f.kout[k] = keys_out ? keys_out[k] : nullptr;
    }
    for (int g = 0; g < PL->n_aggs; g++) {
        f.aop[g] = PL->aop[g];
        f.rout[g] = results_out ? results_out[g] : nullptr;
        f.glo[g] = PL->glo[g].get();
        f.ghi[g] = PL->ghi[g].get();
    }
    f.gkey = PL->gkey.get();
    f.gcount = PL->gcount.get();
    f.G = PL->G;
    f.empty_global = PL->empty_global;
    const int g = (int)std::min<int64_t>(ceil_div(PL->G, 256), (int64_t)ctx->num_sms * 8);
    launch(ctx, "tqp_groupby_finalize", gb_finalize_kernel, dim3(g), dim3(256), 0, f);
}

void groupby_release(tqp_ctx*, tqp_groupby_plan* PL) { delete PL; }

}  // namespace tqp
