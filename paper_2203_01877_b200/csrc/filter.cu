// filter.cu -- filter + order-preserving compaction.
//
// Listing 1 (bitmap): mask = lt(col, c) [AND-ed over predicates, PAPER.md:829];
// Listing 2 (selection vector): idx = nonzero(mask). One kernel evaluates the
// conjunction per row, writes the u8 mask, and compacts passing row numbers in
// ascending order: warp ballots -> per-(item, warp) counts -> block scan ->
// decoupled look-back across tiles -> coalesced writes. No atomics whose order
// could leak into the output.
#include "internal.h"

namespace tqp {

namespace {
constexpr int FNT = 256;
constexpr int FNW = FNT / 32;
constexpr int FIPT = 8;
constexpr int FTILE = FNT * FIPT;

struct FilterArgs {
    int n_preds;
    const void* pcol[TQP_MAX_PREDS];
    int pdt[TQP_MAX_PREDS];
    int op[TQP_MAX_PREDS];
    int64_t val[TQP_MAX_PREDS];
    int64_t n;
    uint8_t* mask;
    int64_t* sel;
    uint64_t* status;
    unsigned long long* counter;
    int64_t* total;
    int64_t n_tiles;
};

__device__ __forceinline__ bool cmp(int64_t x, int op, int64_t v) {
    switch (op) {
        case TQP_LT: return x < v;
        case TQP_LE: return x <= v;
        case TQP_GT: return x > v;
        case TQP_GE: return x >= v;
        case TQP_EQ: return x == v;
        default: return x != v;
    }
}

__global__ void __launch_bounds__(FNT) filter_kernel(FilterArgs a) {
    __shared__ int64_t s_tile;
    __shared__ uint32_t s_cnt[FIPT * FNW];
    __shared__ uint64_t s_excl;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t tile = take_tile(a.counter, &s_tile);
    const int64_t base = tile * FTILE;
    unsigned bal[FIPT];
    bool pass[FIPT];
#pragma unroll
    for (int i = 0; i < FIPT; i++) pass[i] = base + i * FNT + tid < a.n;
    const bool full = base + FTILE <= a.n;
    // predicates: descriptor and dtype/op dispatch hoisted out of the row loop; all
    // loads of a predicate column are independent (no short-circuit), 8 in flight
    for (int q = 0; q < a.n_preds; q++) {
        int64_t x[FIPT];
        switch (a.pdt[q]) {
            case TQP_U8: {
                const uint8_t* c = (const uint8_t*)a.pcol[q] + base + tid;
#pragma unroll
                for (int i = 0; i < FIPT; i++) x[i] = (full || pass[i]) ? (int64_t)__ldg(c + i * FNT) : 0;
                break;
            }
            case TQP_I32: {
                const int32_t* c = (const int32_t*)a.pcol[q] + base + tid;
#pragma unroll
                for (int i = 0; i < FIPT; i++) x[i] = (full || pass[i]) ? (int64_t)__ldg(c + i * FNT) : 0;
                break;
            }
            default: {
                const long long* c = (const long long*)a.pcol[q] + base + tid;
#pragma unroll
                for (int i = 0; i < FIPT; i++) x[i] = (full || pass[i]) ? (int64_t)__ldg(c + i * FNT) : 0;
            }
        }
        const int64_t v = a.val[q];
        switch (a.op[q]) {
            case TQP_LT:
#pragma unroll
                for (int i = 0; i < FIPT; i++) pass[i] &= x[i] < v;
                break;
            case TQP_LE:
#pragma unroll
                for (int i = 0; i < FIPT; i++) pass[i] &= x[i] <= v;
                break;
            case TQP_GT:
#pragma unroll
                for (int i = 0; i < FIPT; i++) pass[i] &= x[i] > v;
                break;
            case TQP_GE:
#pragma unroll
                for (int i = 0; i < FIPT; i++) pass[i] &= x[i] >= v;
                break;
            case TQP_EQ:
#pragma unroll
                for (int i = 0; i < FIPT; i++) pass[i] &= x[i] == v;
                break;
            default:
#pragma unroll
                for (int i = 0; i < FIPT; i++) pass[i] &= x[i] != v;
        }
    }
#pragma unroll
    for (int i = 0; i < FIPT; i++) {
        const int64_t row = base + i * FNT + tid;
        if (a.mask && row < a.n) a.mask[row] = (uint8_t)pass[i];
        bal[i] = __ballot_sync(0xffffffffu, pass[i]);
        if (lane == 0) s_cnt[i * FNW + warp] = __popc(bal[i]);
    }
    __syncthreads();
    if (warp == 0) {
        constexpr int PER = FIPT * FNW / 32;
        uint32_t c[PER], local = 0;
#pragma unroll
        for (int j = 0; j < PER; j++) { c[j] = s_cnt[lane * PER + j]; local += c[j]; }
        uint32_t x = local;
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        const uint32_t tot = __shfl_sync(0xffffffffu, x, 31);
        uint32_t run = x - local;
#pragma unroll
        for (int j = 0; j < PER; j++) { s_cnt[lane * PER + j] = run; run += c[j]; }
        const uint64_t e = lookback_warp(a.status, tile, tot, OpAdd(), 0ull);
        if (lane == 0) {
            s_excl = e;
            if (tile == a.n_tiles - 1) *a.total = (int64_t)(e + tot);
        }
    }
    __syncthreads();
    if (!a.sel) return;
    const int64_t excl = (int64_t)s_excl;
    const unsigned lt = lanemask_lt();
#pragma unroll
    for (int i = 0; i < FIPT; i++) {
        if (bal[i] & (1u << lane)) {
            const int64_t row = base + i * FNT + tid;
            a.sel[excl + s_cnt[i * FNW + warp] + __popc(bal[i] & lt)] = row;
        }
    }
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
    FilterArgs a{};
    a.n_preds = n_preds;
    for (int q = 0; q < n_preds; q++) {
        if (preds[q].col < 0 || preds[q].col >= n_cols) fail(TQP_ERR_INVALID_ARGUMENT, "filter: predicate column");
        if (preds[q].op < TQP_LT || preds[q].op > TQP_NE) fail(TQP_ERR_INVALID_ARGUMENT, "filter: predicate op");
        a.pcol[q] = cols[preds[q].col].data;
        a.pdt[q] = cols[preds[q].col].dtype;
        a.op[q] = preds[q].op;
        a.val[q] = preds[q].value;
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
