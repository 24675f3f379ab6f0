// filter.cu -- filter + order-preserving compaction.
//
// Listing 1 (bitmap): mask = lt(col, c) [AND-ed over predicates, PAPER.md:829];
// Listing 2 (selection vector): idx = nonzero(mask). One kernel evaluates the
// conjunction per row (folded to one interval term per column, common.cuh), writes
// the u8 mask, and compacts passing row numbers in ascending order: each thread owns
// 8 consecutive rows (vector loads) -> warp scan of per-thread counts -> block scan ->
// decoupled look-back across tiles -> rows staged in shared memory -> coalesced
// writes. No atomics whose order could leak into the output.
#include "internal.h"

namespace tqp {

namespace {
constexpr int FNT = 256;
constexpr int FNW = FNT / 32;
constexpr int FIPT = 8;                 // consecutive rows per thread (vector loads)
constexpr int FTILE = FNT * FIPT;

struct FilterArgs {
    TermSet ts;                          // the conjunction, folded per column (common.cuh)
    const void* tcol[TQP_MAX_PREDS];
    int vec;                             // every term column and the mask are 16-byte aligned
    int64_t n;
    uint8_t* mask;
    int64_t* sel;
    uint64_t* status;
    unsigned long long* counter;
    int64_t* total;
    int64_t n_tiles;
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

__global__ void __launch_bounds__(FNT) filter_kernel(FilterArgs a) {
    __shared__ int64_t s_tile;
    __shared__ uint32_t s_woff[FNW];
    __shared__ uint64_t s_excl;
    __shared__ uint32_t s_tot;
    __shared__ int64_t s_out[FTILE];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t tile = take_tile(a.counter, &s_tile);
    const int64_t base = tile * FTILE;
    const int64_t r0 = base + (int64_t)tid * FIPT;
    const bool full = base + FTILE <= a.n;
    const bool vec = full && a.vec;
    bool pass[FIPT];
#pragma unroll
    for (int i = 0; i < FIPT; i++) pass[i] = !a.ts.never && r0 + i < a.n;
    // one interval term per column: one load per row, subtract + unsigned compare
    for (int q = 0; q < a.ts.n; q++) {
        const Term& tm = a.ts.t[q];
        const bool neg = tm.neg;
        if (tm.dt == TQP_I64) {
            unsigned long long x[FIPT];
            load_rows<unsigned long long, ulonglong2>((const unsigned long long*)a.tcol[q], r0, a.n, vec, x);
#pragma unroll
            for (int i = 0; i < FIPT; i++) pass[i] &= term64(x[i], tm.lo, tm.width, neg);
        } else if (tm.dt == TQP_I32) {
            unsigned int x[FIPT];
            load_rows<unsigned int, uint4>((const unsigned int*)a.tcol[q], r0, a.n, vec, x);
#pragma unroll
            for (int i = 0; i < FIPT; i++) pass[i] &= term32(x[i], (uint32_t)tm.lo, (uint32_t)tm.width, neg);
        } else {
            unsigned char x[FIPT];
            load_rows<unsigned char, uint2>((const unsigned char*)a.tcol[q], r0, a.n, vec, x);
#pragma unroll
            for (int i = 0; i < FIPT; i++) pass[i] &= term32(x[i], (uint32_t)tm.lo, (uint32_t)tm.width, neg);
        }
    }
    uint32_t cnt = 0;
#pragma unroll
    for (int i = 0; i < FIPT; i++) cnt += pass[i];
    if (a.mask) {   // Listing 1's bitmap, one byte per row
        if (vec) {
            uint2 m;
            m.x = (uint32_t)pass[0] | (uint32_t)pass[1] << 8 | (uint32_t)pass[2] << 16 | (uint32_t)pass[3] << 24;
            m.y = (uint32_t)pass[4] | (uint32_t)pass[5] << 8 | (uint32_t)pass[6] << 16 | (uint32_t)pass[7] << 24;
            __stcs(reinterpret_cast<uint2*>(a.mask + r0), m);
        } else {
#pragma unroll
            for (int i = 0; i < FIPT; i++)
                if (r0 + i < a.n) a.mask[r0 + i] = (uint8_t)pass[i];
        }
    }
    // rank of each passing row in the tile: thread-exclusive scan within the warp
    uint32_t x = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    const uint32_t texcl = x - cnt;
    if (lane == 31) s_woff[warp] = x;
    __syncthreads();
    if (warp == 0) {
        const uint32_t wt = lane < FNW ? s_woff[lane] : 0;
        uint32_t y = wt;
#pragma unroll
        for (int o = 1; o < FNW; o <<= 1) {
            const uint32_t z = __shfl_up_sync(0xffffffffu, y, o);
            if (lane >= o) y += z;
        }
        const uint32_t tot = __shfl_sync(0xffffffffu, y, FNW - 1);
        const uint64_t e = lookback_warp(a.status, tile, tot, OpAdd(), 0ull);
        if (lane < FNW) s_woff[lane] = y - wt;
        if (lane == 0) {
            s_excl = e;
            s_tot = tot;
            if (tile == a.n_tiles - 1) *a.total = (int64_t)(e + tot);
        }
    }
    __syncthreads();
    if (!a.sel) return;
    // Listing 2's selection vector: stage the tile's passing row numbers in shared
    // memory in row order, then write them out coalesced
    uint32_t lp = s_woff[warp] + texcl;
#pragma unroll
    for (int i = 0; i < FIPT; i++)
        if (pass[i]) s_out[lp++] = r0 + i;
    __syncthreads();
    const uint32_t tot = s_tot;
    int64_t* dst = a.sel + s_excl;
    for (uint32_t k = tid; k < tot; k += FNT) __stcs(reinterpret_cast<long long*>(dst + k), (long long)s_out[k]);
}
}  // namespace

void filter_compact(tqp_ctx* ctx, const tqp_col* cols, int n_cols, int64_t n, const tqp_pred* preds, int n_preds,
                    uint8_t* mask_out, int64_t* sel_out, int64_t* n_sel_host) {
    if (n < 0 || n_cols < 0 || n_preds < 0 || n_preds > TQP_MAX_PREDS)
        fail(TQP_ERR_INVALID_ARGUMENT, "filter: bad sizes");
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
    a.vec = mask_out == nullptr || (uintptr_t)mask_out % 16 == 0;
    for (int q = 0; q < a.ts.n; q++) {
        a.tcol[q] = cols[a.ts.t[q].col].data;
        a.vec = a.vec && (uintptr_t)a.tcol[q] % 16 == 0;
    }
    DevBuf<int64_t> total(ctx, 1);
    total.zero();
    if (n > 0) {
        const int64_t tiles = ceil_div(n, FTILE);
        DevBuf<uint64_t> status(ctx, tiles);
        DevBuf<unsigned long long> counter(ctx, 1);
        status.zero();
        counter.zero();
        a.n = n;
        a.mask = mask_out;
        a.sel = sel_out;
        a.status = status.get();
        a.counter = counter.get();
        a.total = total.get();
        a.n_tiles = tiles;
        launch(ctx, "tqp_filter", filter_kernel, dim3((unsigned)tiles), dim3(FNT), 0, a);
    }
    if (n_sel_host) read_back(ctx, n_sel_host, total.get(), 8);
    {   // distinct predicate columns in; mask and selection vector out
        double in = 0;
        for (int q = 0; q < n_preds; q++) {
            bool seen = false;
            for (int r = 0; r < q; r++) seen = seen || preds[r].col == preds[q].col;
            if (!seen) in += (double)dtype_size(cols[preds[q].col].dtype);
        }
        double out = (mask_out ? 1.0 : 0.0) * (double)n + (sel_out && n_sel_host ? 8.0 * (double)*n_sel_host : 0.0);
        if (n > 0) ctx->add_bytes("tqp_filter", in * (double)n + out);
    }
}

}  // namespace tqp
