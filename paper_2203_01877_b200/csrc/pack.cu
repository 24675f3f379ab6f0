// pack.cu -- multi-column join keys packed into one 63-bit key.
//
// The paper concatenates group-key columns into one sortable key ("key
// preparation ... packing of group-key columns, column 0 most significant"); the same
// packing makes a composite join key a single column for tqp_pkfk_join / tqp_smj_*:
//   packed(row) = sum_c (u_c(row) - min_c) << shift_c,
// u_c = the order-preserving unsigned image of column c, min_c / max_c over BOTH sides,
// width_c = bits(max_c - min_c), shift_c = sum of the widths of the columns after c.
// Equal tuples pack equal and different tuples differently on both sides, and the
// packed order is the tuples' lexicographic order, so joins on the packed column are
// the joins on the tuples (including the SMJ's (key, l, r) output order).
#include "internal.h"

namespace tqp {

namespace {

constexpr int PKNT = 256;

struct PackCols {
    const void* data[TQP_MAX_KEYS];
    int dt[TQP_MAX_KEYS];
    int n_cols;
};

__device__ __forceinline__ uint64_t load_ord(const void* p, int dt, int64_t i) {
    int64_t v;
    if (dt == TQP_I64) v = __ldg((const long long*)p + i);
    else if (dt == TQP_I32) v = __ldg((const int*)p + i);
    else v = __ldg((const unsigned char*)p + i);
    return ordered_u64(v);
}

// per column: min / max of the ordered images (mm[2c] = min, mm[2c+1] = max)
__global__ void __launch_bounds__(PKNT) pack_minmax_kernel(PackCols a, int64_t n, unsigned long long* mm) {
    for (int c = 0; c < a.n_cols; c++) {
        uint64_t lo = ~0ull, hi = 0;
        for (int64_t i = blockIdx.x * (int64_t)PKNT + threadIdx.x; i < n; i += (int64_t)gridDim.x * PKNT) {
            const uint64_t u = load_ord(a.data[c], a.dt[c], i);
            lo = min(lo, u);
            hi = max(hi, u);
        }
        for (int o = 16; o > 0; o >>= 1) {
            lo = min(lo, (uint64_t)__shfl_xor_sync(0xffffffffu, lo, o));
            hi = max(hi, (uint64_t)__shfl_xor_sync(0xffffffffu, hi, o));
        }
        if ((threadIdx.x & 31) == 0) {
            atomicMin(mm + 2 * c, (unsigned long long)lo);
            atomicMax(mm + 2 * c + 1, (unsigned long long)hi);
        }
    }
}

__global__ void pack_mm_init_kernel(unsigned long long* mm, int n_cols) {
    const int i = threadIdx.x;
    if (i < 2 * n_cols) mm[i] = (i & 1) ? 0ull : ~0ull;
}

struct PackLayout {
    uint64_t min[TQP_MAX_KEYS];
    int shift[TQP_MAX_KEYS];
};

__global__ void __launch_bounds__(PKNT) pack_kernel(PackCols a, PackLayout L, int64_t n, int64_t* out) {
    for (int64_t i = blockIdx.x * (int64_t)PKNT + threadIdx.x; i < n; i += (int64_t)gridDim.x * PKNT) {
        uint64_t k = 0;
        for (int c = 0; c < a.n_cols; c++) k |= (load_ord(a.data[c], a.dt[c], i) - L.min[c]) << L.shift[c];
        __stcs((long long*)out + i, (long long)k);
    }
}

PackCols pack_cols(const tqp_col* cols, int n_cols, int64_t n, const char* what) {
    PackCols a{};
    a.n_cols = n_cols;
    for (int c = 0; c < n_cols; c++) {
        check_col(cols[c], n, what);
        a.data[c] = cols[c].data;
        a.dt[c] = cols[c].dtype;
    }
    return a;
}

}  // namespace

int pack_keys(tqp_ctx* ctx, const tqp_col* a_cols, int64_t na, const tqp_col* b_cols, int64_t nb, int n_cols,
              int64_t* a_out, int64_t* b_out) {
    if (n_cols < 1 || n_cols > TQP_MAX_KEYS) fail(TQP_ERR_INVALID_ARGUMENT, "pack_keys: 1..8 key columns");
    if ((na > 0 && !a_out) || (nb > 0 && !b_out)) fail(TQP_ERR_INVALID_ARGUMENT, "pack_keys: null output");
    const PackCols A = pack_cols(a_cols, n_cols, na, "pack_keys side a");
    const PackCols B = nb > 0 || b_cols ? pack_cols(b_cols, n_cols, nb, "pack_keys side b") : PackCols{};
    DevBuf<unsigned long long> mm(ctx, 2 * n_cols);
    launch(ctx, "tqp_pack_minmax", pack_mm_init_kernel, dim3(1), dim3(32), 0, mm.get(), n_cols);
    auto grid = [&](int64_t n) { return (int)std::min<int64_t>(ceil_div(n, PKNT), (int64_t)ctx->num_sms * 8); };
    if (na > 0) launch(ctx, "tqp_pack_minmax", pack_minmax_kernel, dim3(grid(na)), dim3(PKNT), 0, A, na, mm.get());
    if (nb > 0) launch(ctx, "tqp_pack_minmax", pack_minmax_kernel, dim3(grid(nb)), dim3(PKNT), 0, B, nb, mm.get());
    uint64_t h[2 * TQP_MAX_KEYS];
    read_back(ctx, h, mm.get(), 16 * (size_t)n_cols);
    if (na + nb == 0) return 0;
    PackLayout L{};
    int width[TQP_MAX_KEYS], total = 0;
    for (int c = 0; c < n_cols; c++) {
        const uint64_t span = h[2 * c + 1] - h[2 * c];
        width[c] = span ? 64 - __builtin_clzll(span) : 0;
        total += width[c];
        L.min[c] = h[2 * c];
    }
    if (total > 63) fail(TQP_ERR_INVALID_ARGUMENT, "pack_keys: the key columns' ranges need more than 63 bits");
    int sh = 0;
    for (int c = n_cols - 1; c >= 0; c--) {   // column 0 most significant
        L.shift[c] = sh;
        sh += width[c];
    }
    auto row_bytes = [&](const tqp_col* cols) {
        double b = 8.0;   // the packed key written
        for (int c = 0; c < n_cols; c++) b += (double)dtype_size(cols[c].dtype);
        return b;
    };
    if (na > 0) {
        launch(ctx, "tqp_pack", pack_kernel, dim3(grid(na)), dim3(PKNT), 0, A, L, na, a_out);
        ctx->add_bytes("tqp_pack", row_bytes(a_cols) * (double)na);
    }
    if (nb > 0) {
        launch(ctx, "tqp_pack", pack_kernel, dim3(grid(nb)), dim3(PKNT), 0, B, L, nb, b_out);
        ctx->add_bytes("tqp_pack", row_bytes(b_cols) * (double)nb);
    }
    return total;
}

}  // namespace tqp
