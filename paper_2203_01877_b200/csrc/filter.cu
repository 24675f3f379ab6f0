// filter.cu -- filter + order-preserving compaction.
//
// Listing 1 (bitmap): mask = lt(col, c) [AND-ed over predicates, PAPER.md:829];
// Listing 2 (selection vector): idx = nonzero(mask). Pass 1 evaluates the conjunction
// per row (folded to one interval term per column, common.cuh), writes the u8 mask and
// counts passing rows per tile; an exclusive add-scan gives tile offsets; pass 2 reads
// only the mask and writes passing row numbers in ascending order (warp scan of
// per-thread counts -> block scan -> staged in shared memory -> coalesced stores).
// No inter-tile chain (a decoupled look-back was measured to leave the warps of a
// tile idle at the barrier) and no atomics whose order could leak into the output.
#include "internal.h"

namespace tqp {

namespace {
constexpr int FNT = 256;
constexpr int FNW = FNT / 32;
constexpr int FIPT = 16;                // consecutive rows per thread (vector loads)
constexpr int FTILE = FNT * FIPT;

struct FilterArgs {
    TermSet ts;                          // the conjunction, folded per column (common.cuh)
    const void* tcol[TQP_MAX_PREDS];
    int vec;                             // every term column is 16-byte aligned
    int64_t n;
    uint8_t* mask;                       // the output mask, or a temporary one
    uint32_t* tcnt;                      // per tile: passing rows
};

// Rows r0 .. r0+FIPT-1 of a column; vector loads on full aligned tiles.
template <typename T, typename V>
__device__ __forceinline__ void load_rows(const T* c, int64_t r0, int64_t n, bool vec, T (&x)[FIPT]) {
    if (vec) {
        const V* v = reinterpret_cast<const V*>(c + r0);
        constexpr int PER = sizeof(V) / sizeof(T);
#pragma unroll
        for (int j = 0; j < FIPT / PER; j++) {
            const V u = __ldcs(v + j);
            memcpy(&x[j * PER], &u, sizeof(V));
        }
    } else {
#pragma unroll
        for (int i = 0; i < FIPT; i++) x[i] = r0 + i < n ? c[r0 + i] : T(0);
    }
}

// A thread owns 4 groups of 4 consecutive rows, the groups FNT * 4 rows apart, so a warp's
// vector load covers 512 contiguous bytes of an int32 column (1 KB of an int64 one in two
// loads) instead of 32 lanes each reading its own 16 consecutive rows 64-128 bytes apart.
// Measured, Q6 mask at SF10: 0.253 -> 0.200 ms (6.3 TB/s). TQP_FILTER_GROUPED=0: the
// per-thread-contiguous layout (A/B).
#ifndef TQP_FILTER_GROUPED
#define TQP_FILTER_GROUPED 1
#endif
constexpr bool FGROUPED = TQP_FILTER_GROUPED;
constexpr int FG = 4;   // rows per group
// row of item i of thread tid (grouped: group i / FG at FNT * FG rows apart)
__device__ __forceinline__ int64_t frow(int64_t base, int tid, int i) {
    return FGROUPED ? base + (int64_t)(i / FG) * (FNT * FG) + tid * FG + (i % FG) : base + (int64_t)tid * FIPT + i;
}
template <typename T>
__device__ __forceinline__ void load_grouped(const T* c, int64_t base, int tid, int64_t n, bool vec, T (&x)[FIPT]) {
    if (vec) {
#pragma unroll
        for (int g = 0; g < FIPT / FG; g++) {
            const T* p = c + base + (int64_t)g * (FNT * FG) + tid * FG;
            if (sizeof(T) == 8) {
                const ulonglong2 u0 = __ldcs(reinterpret_cast<const ulonglong2*>(p));
                const ulonglong2 u1 = __ldcs(reinterpret_cast<const ulonglong2*>(p) + 1);
                memcpy(&x[g * FG], &u0, 16);
                memcpy(&x[g * FG + 2], &u1, 16);
            } else if (sizeof(T) == 4) {
                const uint4 u = __ldcs(reinterpret_cast<const uint4*>(p));
                memcpy(&x[g * FG], &u, 16);
            } else {
                const uint32_t u = __ldcs(reinterpret_cast<const unsigned int*>(p));
                memcpy(&x[g * FG], &u, 4);
            }
        }
    } else {
#pragma unroll
        for (int i = 0; i < FIPT; i++) {
            const int64_t r = frow(base, tid, i);
            x[i] = r < n ? c[r] : T(0);
        }
    }
}

// Pass 1 (Listing 1, the bitmap): the conjunction per row -> u8 mask, and the number
// of passing rows per tile. No inter-tile dependency.
// Blocks per SM the register budget must allow (72 registers held it to 3). Measured, Q6
// mask at SF10: 0.263 ms at 72 registers, 0.253 ms with 4 blocks (56), 0.254 with 5,
// 0.256 with 6 (spills).
// (r02, with the grouped row layout: 4 -> 5 blocks per SM, 0.200 -> 0.194 ms)
#ifndef TQP_FILTER_MINB
#define TQP_FILTER_MINB 5
#endif
__global__ void __launch_bounds__(FNT, TQP_FILTER_MINB) filter_mask_kernel(FilterArgs a) {
    __shared__ uint32_t s_w[FNW];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t base = (int64_t)blockIdx.x * FTILE;
    const int64_t r0 = base + (int64_t)tid * FIPT;
    const bool full = base + FTILE <= a.n;
    const bool vec = full && a.vec;
    bool pass[FIPT];
#pragma unroll
    for (int i = 0; i < FIPT; i++) pass[i] = !a.ts.never && frow(base, tid, i) < a.n;
    // one interval term per column: one load per row, subtract + unsigned compare
    for (int q = 0; q < a.ts.n; q++) {
        const Term& tm = a.ts.t[q];
        const bool neg = tm.neg;
        if (tm.dt == TQP_I64) {
            unsigned long long x[FIPT];
            if (FGROUPED) load_grouped<unsigned long long>((const unsigned long long*)a.tcol[q], base, tid, a.n, vec, x);
            else load_rows<unsigned long long, ulonglong2>((const unsigned long long*)a.tcol[q], r0, a.n, vec, x);
#pragma unroll
            for (int i = 0; i < FIPT; i++) pass[i] &= term64(x[i], tm.lo, tm.width, neg);
        } else if (tm.dt == TQP_I32) {
            unsigned int x[FIPT];
            if (FGROUPED) load_grouped<unsigned int>((const unsigned int*)a.tcol[q], base, tid, a.n, vec, x);
            else load_rows<unsigned int, uint4>((const unsigned int*)a.tcol[q], r0, a.n, vec, x);
#pragma unroll
            for (int i = 0; i < FIPT; i++) pass[i] &= term32(x[i], (uint32_t)tm.lo, (uint32_t)tm.width, neg);
        } else {
            unsigned char x[FIPT];
            if (FGROUPED) load_grouped<unsigned char>((const unsigned char*)a.tcol[q], base, tid, a.n, vec, x);
            else load_rows<unsigned char, uint4>((const unsigned char*)a.tcol[q], r0, a.n, vec, x);
#pragma unroll
            for (int i = 0; i < FIPT; i++) pass[i] &= term32(x[i], (uint32_t)tm.lo, (uint32_t)tm.width, neg);
        }
    }
    uint32_t cnt = 0;
#pragma unroll
    for (int i = 0; i < FIPT; i++) cnt += pass[i];
    if (FGROUPED && full && (uintptr_t)a.mask % 4 == 0) {
#pragma unroll
        for (int g = 0; g < FIPT / FG; g++)
            __stcs(reinterpret_cast<unsigned int*>(a.mask + base + (int64_t)g * (FNT * FG) + tid * FG),
                   (uint32_t)pass[g * FG] | (uint32_t)pass[g * FG + 1] << 8 | (uint32_t)pass[g * FG + 2] << 16 |
                       (uint32_t)pass[g * FG + 3] << 24);
    } else if (FGROUPED) {
#pragma unroll
        for (int i = 0; i < FIPT; i++) {
            const int64_t r = frow(base, tid, i);
            if (r < a.n) a.mask[r] = (uint8_t)pass[i];
        }
    } else if (full && (uintptr_t)a.mask % 16 == 0) {
        uint32_t m[4];
#pragma unroll
        for (int w = 0; w < 4; w++)
            m[w] = (uint32_t)pass[4 * w] | (uint32_t)pass[4 * w + 1] << 8 | (uint32_t)pass[4 * w + 2] << 16 |
                   (uint32_t)pass[4 * w + 3] << 24;
        __stcs(reinterpret_cast<uint4*>(a.mask + r0), make_uint4(m[0], m[1], m[2], m[3]));
    } else {
#pragma unroll
        for (int i = 0; i < FIPT; i++)
            if (r0 + i < a.n) a.mask[r0 + i] = (uint8_t)pass[i];
    }
    for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    if (lane == 0) s_w[warp] = cnt;
    __syncthreads();
    if (tid == 0) {
        uint32_t t = 0;
        for (int w = 0; w < FNW; w++) t += s_w[w];
        a.tcnt[blockIdx.x] = t;
    }
}

// Pass 2 (Listing 2, the selection vector): passing row numbers in ascending order at
// the tile's offset; ranks by warp scan of per-thread counts + block scan; staged in
// shared memory and written coalesced.
// Tiles per CTA of the selection pass (consecutive; short tiles made the pass launch-bound).
#ifndef TQP_SEL_TPC
#define TQP_SEL_TPC 1
#endif
__global__ void __launch_bounds__(FNT) filter_sel_kernel(const uint8_t* __restrict__ mask, int64_t n,
                                                         const uint32_t* __restrict__ toff, int64_t* sel, int64_t tiles) {
    __shared__ uint32_t s_w[FNW];
    __shared__ uint16_t s_out[FTILE];   // tile-relative row numbers (8 KB instead of 32: more resident CTAs)
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int64_t tile = (int64_t)blockIdx.x * TQP_SEL_TPC; tile < min(tiles, (int64_t)(blockIdx.x + 1) * TQP_SEL_TPC); tile++) {
    const int64_t base = tile * FTILE;
    const int64_t excl = toff[tile];
    const uint32_t tot = toff[tile + 1] - (uint32_t)excl;
    if (tot == 0) continue;   // CTA-uniform
    const int64_t r0 = base + (int64_t)tid * FIPT;
    uint8_t m[FIPT];
    if (base + FTILE <= n && (uintptr_t)mask % 16 == 0) {
        const uint4 v = __ldcs(reinterpret_cast<const uint4*>(mask + r0));
        memcpy(m, &v, 16);
    } else {
#pragma unroll
        for (int i = 0; i < FIPT; i++) m[i] = r0 + i < n ? mask[r0 + i] : 0;
    }
    uint32_t cnt = 0;
#pragma unroll
    for (int i = 0; i < FIPT; i++) cnt += m[i] != 0;
    uint32_t x = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) s_w[warp] = x;
    __syncthreads();
    uint32_t lp = x - cnt;
#pragma unroll
    for (int w = 0; w < FNW; w++)
        if (w < warp) lp += s_w[w];
#pragma unroll
    for (int i = 0; i < FIPT; i++)
        if (m[i]) s_out[lp++] = (uint16_t)(r0 + i - base);
    __syncthreads();
    int64_t* dst = sel + excl;
    TQP_DCHECK(excl + (int64_t)tot <= n && lp <= (uint32_t)FTILE);
    for (uint32_t k = tid; k < tot; k += FNT) __stcs(reinterpret_cast<long long*>(dst + k), (long long)(base + s_out[k]));
    __syncthreads();   // s_w / s_out reused by the next tile
    }
}
}  // namespace

void filter_compact(tqp_ctx* ctx, const tqp_col* cols, int n_cols, int64_t n, const tqp_pred* preds, int n_preds,
                    uint8_t* mask_out, int64_t* sel_out, int64_t* n_sel_host) {
    if (n < 0 || n >= (int64_t(1) << 32) || n_cols < 0 || n_preds < 0 || n_preds > TQP_MAX_PREDS)
        fail(TQP_ERR_INVALID_ARGUMENT, "filter: bad sizes (n must be < 2^32)");
    if (n_cols > 0 && !cols) fail(TQP_ERR_INVALID_ARGUMENT, "filter: null cols");
    if (n_preds > 0 && !preds) fail(TQP_ERR_INVALID_ARGUMENT, "filter: null preds");
    if (!mask_out && !sel_out && !n_sel_host) fail(TQP_ERR_INVALID_ARGUMENT, "filter: no output requested");
    for (int c = 0; c < n_cols; c++) check_col(cols[c], n, "filter column");
    for (int q = 0; q < n_preds; q++) {
        if (preds[q].col < 0 || preds[q].col >= n_cols) fail(TQP_ERR_INVALID_ARGUMENT, "filter: predicate column");
        if (preds[q].op < TQP_LT || preds[q].op > TQP_NE) fail(TQP_ERR_INVALID_ARGUMENT, "filter: predicate op");
    }
    FilterArgs a{};
    a.ts = make_terms(preds, n_preds, [&](int c) { return cols[c].dtype; });
    a.vec = 1;
    for (int q = 0; q < a.ts.n; q++) {
        a.tcol[q] = cols[a.ts.t[q].col].data;
        a.vec = a.vec && (uintptr_t)a.tcol[q] % 16 == 0;
    }
    int64_t nsel = 0;
    if (n > 0) {
        const int64_t tiles = ceil_div(n, FTILE);
        DevBuf<uint8_t> tmask;
        if (!mask_out) tmask.alloc(ctx, n);
        DevBuf<uint32_t> tcnt(ctx, tiles), toff(ctx, tiles + 1);
        a.n = n;
        a.mask = mask_out ? mask_out : tmask.get();
        a.tcnt = tcnt.get();
        launch(ctx, "tqp_filter", filter_mask_kernel, dim3((unsigned)tiles), dim3(FNT), 0, a);
        scan_add_u32_exclusive(ctx, tcnt.get(), toff.get(), tiles);
        if (sel_out)
            launch(ctx, "tqp_filter_select", filter_sel_kernel, dim3((unsigned)ceil_div(tiles, TQP_SEL_TPC)), dim3(FNT), 0,
                   (const uint8_t*)a.mask, n, (const uint32_t*)toff.get(), sel_out, tiles);
        if (n_sel_host) {
            uint32_t t = 0;
            read_back(ctx, &t, toff.get() + tiles, 4);
            nsel = t;
            *n_sel_host = nsel;
        }
    } else if (n_sel_host) {
        *n_sel_host = 0;
    }
    {   // distinct predicate columns in; mask and selection vector out
        double in = 0;
        for (int q = 0; q < n_preds; q++) {
            bool seen = false;
            for (int r = 0; r < q; r++) seen = seen || preds[r].col == preds[q].col;
            if (!seen) in += (double)dtype_size(cols[preds[q].col].dtype);
        }
        if (n > 0) ctx->add_bytes("tqp_filter", in * (double)n + (mask_out ? (double)n : 0.0));
        if (n > 0 && sel_out) ctx->add_bytes("tqp_filter_select", 8.0 * (double)nsel + (mask_out ? (double)n : 0.0));
    }
}

}  // namespace tqp
