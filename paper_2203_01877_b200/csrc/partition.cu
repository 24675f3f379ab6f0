// partition.cu -- the data-parallel exchange's on-GPU steps (the paper
// names data-parallel execution as future work):
//   tqp_partition  stable partition of (key, global row) by destination rank, the
//                  destination of a key being the number of splitters <= key (a key
//                  range per rank); output grouped by destination, input order kept
//                  within a destination, plus the per-destination counts -- the send
//                  buffer and split sizes of one all_to_all;
//   tqp_minmax     device min / max of a key column (all-reduced across ranks by the
//                  caller to form equal-width key ranges, no host round trip);
//   tqp_range_splitters  equal-width splitters from a device [min, max];
//   tqp_gather     out[i] = src[idx[i]] (createOutput of PAPER.md:333: received global
//                  row numbers mapped through local join indices).
// One partition pass = a per-tile destination histogram, one exclusive scan over the
// destination-major (dest, tile) counts (= each tile's offset inside each destination's
// block), and a scatter that ranks each row stably among its tile's rows with the same
// destination (warp match_any peers + per-warp counters) and writes keys and rows
// coalesced per destination run. Destinations <= 256.
#include "internal.h"

namespace tqp {

namespace {

constexpr int QNT = 256;
constexpr int QNW = QNT / 32;
constexpr int QSTEPS = 16;                       // rows per lane: warp w owns 512 contiguous rows
constexpr int QTILE = QNT * QSTEPS;              // 4096 rows per tile
constexpr int QMAXP = 256;

// destination = number of splitters <= k (upper_bound over the sorted splitters)
__device__ __forceinline__ int dest_of(const int64_t* spl, int ns, int64_t k) {
    int lo = 0, hi = ns;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (spl[mid] <= k) lo = mid + 1; else hi = mid;
    }
    return lo;
}

__device__ __forceinline__ int64_t tile_row(int64_t t, int warp, int s, int lane) {
    return t * QTILE + (int64_t)warp * (QSTEPS * 32) + s * 32 + lane;
}

__global__ void __launch_bounds__(QNT) part_hist_kernel(const void* __restrict__ keys, int dt, int64_t n,
                                                        const int64_t* __restrict__ splitters, int parts,
                                                        int64_t tiles, uint32_t* __restrict__ cnt) {
    __shared__ int64_t s_spl[QMAXP];
    __shared__ uint32_t s_cnt[QMAXP];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int j = tid; j < parts; j += QNT) {
        if (j < parts - 1) s_spl[j] = splitters[j];
        s_cnt[j] = 0;
    }
    __syncthreads();
    const int64_t t = blockIdx.x;
#pragma unroll 4
    for (int s = 0; s < QSTEPS; s++) {
        const int64_t row = tile_row(t, warp, s, lane);
        const bool valid = row < n;
        const int d = valid ? dest_of(s_spl, parts - 1, load_as_i64(keys, dt, row)) : QMAXP;
        const unsigned peers = __match_any_sync(0xffffffffu, d);
        if (valid && lane == 31 - __clz(peers)) atomicAdd(&s_cnt[d], (uint32_t)__popc(peers));
    }
    __syncthreads();
    for (int j = tid; j < parts; j += QNT) cnt[(int64_t)j * tiles + t] = s_cnt[j];
}

template <int DT>
__device__ __forceinline__ int64_t ld_key(const void* keys, int64_t row) {
    if (DT == TQP_I64) return (int64_t)__ldcs((const long long*)keys + row);
    if (DT == TQP_I32) return (int64_t)__ldcs((const int*)keys + row);
    return (int64_t)__ldcs((const unsigned char*)keys + row);
}

template <int DT>
__device__ __forceinline__ void st_key(void* out, int64_t pos, int64_t k) {
    if (DT == TQP_I64) __stcs((long long*)out + pos, (long long)k);
    else if (DT == TQP_I32) __stcs((int*)out + pos, (int)k);
    else ((unsigned char*)out)[pos] = (unsigned char)k;
}

// Per-destination output (the fused exchange): destination d's block is written at
// keys[d] + base[d] / rows[d] + base[d] -- device pointers that may be a peer GPU's
// receive buffer (CUDA IPC / NVLink P2P), so the partition's stores ARE the all-to-all.
struct PartDest {
    void* keys[QMAXP];
    int64_t* rows[QMAXP];
    int64_t base[QMAXP];
};

template <int DT>
__global__ void __launch_bounds__(QNT) part_scatter_kernel(const void* __restrict__ keys, int64_t n,
                                                           const int64_t* __restrict__ splitters, int parts,
                                                           int64_t tiles, const uint64_t* __restrict__ off,
                                                           int64_t row_base, void* keys_out, int64_t* rows_out,
                                                           const PartDest* __restrict__ dest) {
    __shared__ int64_t s_spl[QMAXP];
    __shared__ uint64_t s_off[QMAXP];
    __shared__ int64_t s_dbase[QMAXP];   // dest: base[d] - start of d's block in the local layout
    __shared__ uint32_t s_wc[QNW][QMAXP];   // per-warp counts -> per-warp offsets per destination
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t t = blockIdx.x;
    for (int j = tid; j < parts; j += QNT) {
        if (j < parts - 1) s_spl[j] = splitters[j];
        s_off[j] = off[(int64_t)j * tiles + t];
        if (dest) s_dbase[j] = dest->base[j] - (int64_t)off[(int64_t)j * tiles];
#pragma unroll
        for (int w = 0; w < QNW; w++) s_wc[w][j] = 0;
    }
    __syncthreads();
    int64_t k[QSTEPS];
    int dd[QSTEPS];
    uint32_t pos[QSTEPS];
#pragma unroll
    for (int s = 0; s < QSTEPS; s++) {
        const int64_t row = tile_row(t, warp, s, lane);
        const bool valid = row < n;
        k[s] = valid ? ld_key<DT>(keys, row) : 0;
        const int d = valid ? dest_of(s_spl, parts - 1, k[s]) : QMAXP;
        dd[s] = d;
        const unsigned peers = __match_any_sync(0xffffffffu, d);
        const uint32_t before = valid ? s_wc[warp][d] : 0;   // the warp's rows of d in earlier steps
        pos[s] = before + (uint32_t)__popc(peers & ((1u << lane) - 1u));
        __syncwarp();
        if (valid && lane == 31 - __clz(peers)) s_wc[warp][d] = before + (uint32_t)__popc(peers);
        __syncwarp();
    }
    __syncthreads();
    for (int j = tid; j < parts; j += QNT) {   // per-warp exclusive offsets, warps in row order
        uint32_t run = 0;
#pragma unroll
        for (int w = 0; w < QNW; w++) {
            const uint32_t c = s_wc[w][j];
            s_wc[w][j] = run;
            run += c;
        }
    }
    __syncthreads();
#pragma unroll
    for (int s = 0; s < QSTEPS; s++) {
        const int64_t row = tile_row(t, warp, s, lane);
        if (row >= n) continue;
        const int d = dd[s];
        const int64_t p = (int64_t)s_off[d] + s_wc[warp][d] + pos[s];
        TQP_DCHECK(d < parts && p >= 0 && p < n);
        if (dest) {   // straight into destination d's (possibly remote) receive buffer
            const int64_t q = s_dbase[d] + p;
            st_key<DT>(dest->keys[d], q, k[s]);
            if (dest->rows[d]) __stcs((long long*)dest->rows[d] + q, (long long)(row_base + row));
        } else {
            st_key<DT>(keys_out, p, k[s]);
            if (rows_out) __stcs((long long*)rows_out + p, (long long)(row_base + row));
        }
    }
}

__global__ void part_counts_kernel(const uint64_t* __restrict__ off, int64_t tiles, int parts, int64_t* counts) {
    for (int j = threadIdx.x; j < parts; j += blockDim.x)
        counts[j] = (int64_t)(off[(int64_t)(j + 1) * tiles] - off[(int64_t)j * tiles]);
}

__global__ void __launch_bounds__(QNT) minmax_kernel(const void* __restrict__ keys, int dt, int64_t n,
                                                     unsigned long long* mm) {
    uint64_t lo = ~0ull, hi = 0;
    for (int64_t i = blockIdx.x * (int64_t)QNT + threadIdx.x; i < n; i += (int64_t)gridDim.x * QNT) {
        const uint64_t u = ordered_u64(load_as_i64(keys, dt, i));
        lo = min(lo, u);
        hi = max(hi, u);
    }
    for (int o = 16; o > 0; o >>= 1) {
        lo = min(lo, (uint64_t)__shfl_xor_sync(0xffffffffu, lo, o));
        hi = max(hi, (uint64_t)__shfl_xor_sync(0xffffffffu, hi, o));
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMin(mm, (unsigned long long)lo);
        atomicMax(mm + 1, (unsigned long long)hi);
    }
}

__global__ void minmax_init_kernel(unsigned long long* mm) {
    mm[0] = ~0ull;
    mm[1] = 0ull;
}

// ordered images -> signed values; empty input: [INT64_MAX, INT64_MIN]
__global__ void minmax_final_kernel(const unsigned long long* mm, int64_t* lohi) {
    lohi[0] = unordered_i64(mm[0]);
    lohi[1] = unordered_i64(mm[1]);
}

// spl[j] = lo + (j + 1) * width, width = (hi - lo) / parts + 1 (key k -> rank (k - lo) / width);
// saturates at INT64_MAX; an empty range (lo > hi) gives INT64_MAX everywhere
__global__ void range_splitters_kernel(const int64_t* lohi, int parts, int64_t* spl) {
    const int64_t lo = lohi[0], hi = lohi[1];
    const int j = threadIdx.x;
    if (j >= parts - 1) return;
    if (lo > hi) { spl[j] = INT64_MAX; return; }
    const __int128 width = ((__int128)hi - lo) / parts + 1;
    const __int128 v = (__int128)lo + (__int128)(j + 1) * width;
    spl[j] = v > (__int128)INT64_MAX ? INT64_MAX : (int64_t)v;
}

template <int DT>
__global__ void gather_kernel(const void* __restrict__ src, const int64_t* __restrict__ idx, int64_t n, void* out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t j = __ldcs((const long long*)idx + i);
        if (DT == TQP_I64 || DT == TQP_F64) __stcs((long long*)out + i, __ldg((const long long*)src + j));
        else if (DT == TQP_I32) __stcs((int*)out + i, __ldg((const int*)src + j));
        else ((unsigned char*)out)[i] = __ldg((const unsigned char*)src + j);
    }
}

}  // namespace

void partition(tqp_ctx* ctx, tqp_col keys, int64_t n, const int64_t* splitters, int parts, int64_t row_base,
               void* keys_out, int64_t* rows_out, int64_t* counts) {
    check_col(keys, n, "partition keys");
    if (keys.dtype == TQP_F64) fail(TQP_ERR_INVALID_ARGUMENT, "partition: keys must be integer columns");
    if (parts < 1 || parts > QMAXP) fail(TQP_ERR_INVALID_ARGUMENT, "partition: parts must be in [1, 256]");
    if (!counts || (parts > 1 && !splitters)) fail(TQP_ERR_INVALID_ARGUMENT, "partition: null splitters / counts");
    if (n > 0 && !keys_out) fail(TQP_ERR_INVALID_ARGUMENT, "partition: null keys_out");
    if (n == 0) {
        TQP_CUDA(cudaMemsetAsync(counts, 0, (size_t)parts * 8, ctx->stream));
        return;
    }
    const int64_t tiles = ceil_div(n, QTILE);
    const int64_t ncnt = tiles * parts;
    DevBuf<uint32_t> cnt(ctx, ncnt);
    DevBuf<uint64_t> off(ctx, ncnt + 1);
    launch(ctx, "tqp_partition_hist", part_hist_kernel, dim3((unsigned)tiles), dim3(QNT), 0, keys.data, (int)keys.dtype,
           n, splitters, parts, tiles, cnt.get());
    ctx->add_bytes("tqp_partition_hist", (double)n * dtype_size(keys.dtype) + 4.0 * (double)ncnt);
    scan_add_u32_to_u64_exclusive(ctx, cnt.get(), off.get(), ncnt);
    switch (keys.dtype) {
        case TQP_I64: launch(ctx, "tqp_partition", part_scatter_kernel<TQP_I64>, dim3((unsigned)tiles), dim3(QNT), 0, keys.data, n, splitters, parts, tiles, (const uint64_t*)off.get(), row_base, keys_out, rows_out, (const PartDest*)nullptr); break;
        case TQP_I32: launch(ctx, "tqp_partition", part_scatter_kernel<TQP_I32>, dim3((unsigned)tiles), dim3(QNT), 0, keys.data, n, splitters, parts, tiles, (const uint64_t*)off.get(), row_base, keys_out, rows_out, (const PartDest*)nullptr); break;
        default: launch(ctx, "tqp_partition", part_scatter_kernel<TQP_U8>, dim3((unsigned)tiles), dim3(QNT), 0, keys.data, n, splitters, parts, tiles, (const uint64_t*)off.get(), row_base, keys_out, rows_out, (const PartDest*)nullptr); break;
    }
    ctx->add_bytes("tqp_partition", (double)n * (2.0 * dtype_size(keys.dtype) + (rows_out ? 8.0 : 0.0)));
    launch(ctx, "tqp_partition_hist", part_counts_kernel, dim3(1), dim3(256), 0, (const uint64_t*)off.get(), tiles, parts,
           counts);
}

}  // namespace tqp

struct tqp_partition_plan {
    tqp_col keys{};
    int64_t n = 0, tiles = 0;
    int parts = 1;
    const int64_t* splitters = nullptr;
    tqp::DevBuf<uint64_t> off;
    tqp::DevBuf<tqp::PartDest> dest;
};

namespace tqp {

// Pass 1 of the fused exchange: the destination histogram and its scan (counts_out: device
// int64 per destination); the caller exchanges the counts, then scatters into the
// destinations' buffers with partition_scatter.
tqp_partition_plan* partition_plan(tqp_ctx* ctx, tqp_col keys, int64_t n, const int64_t* splitters, int parts,
                                   int64_t* counts) {
    check_col(keys, n, "partition keys");
    if (keys.dtype == TQP_F64) fail(TQP_ERR_INVALID_ARGUMENT, "partition: keys must be integer columns");
    if (parts < 1 || parts > QMAXP) fail(TQP_ERR_INVALID_ARGUMENT, "partition: parts must be in [1, 256]");
    if (!counts || (parts > 1 && !splitters)) fail(TQP_ERR_INVALID_ARGUMENT, "partition: null splitters / counts");
    auto* P = new tqp_partition_plan();
    try {
        P->keys = keys;
        P->n = n;
        P->parts = parts;
        P->splitters = splitters;
        P->tiles = ceil_div(n, QTILE);
        if (n == 0) {
            TQP_CUDA(cudaMemsetAsync(counts, 0, (size_t)parts * 8, ctx->stream));
            return P;
        }
        const int64_t ncnt = P->tiles * parts;
        DevBuf<uint32_t> cnt(ctx, ncnt);
        P->off.alloc(ctx, ncnt + 1);
        launch(ctx, "tqp_partition_hist", part_hist_kernel, dim3((unsigned)P->tiles), dim3(QNT), 0, keys.data,
               (int)keys.dtype, n, splitters, parts, P->tiles, cnt.get());
        ctx->add_bytes("tqp_partition_hist", (double)n * dtype_size(keys.dtype) + 4.0 * (double)ncnt);
        scan_add_u32_to_u64_exclusive(ctx, cnt.get(), P->off.get(), ncnt);
        launch(ctx, "tqp_partition_hist", part_counts_kernel, dim3(1), dim3(256), 0, (const uint64_t*)P->off.get(),
               P->tiles, parts, counts);
        return P;
    } catch (...) {
        delete P;
        throw;
    }
}

void partition_scatter(tqp_ctx* ctx, tqp_partition_plan* P, int64_t row_base, void* const* dkeys, int64_t* const* drows,
                       const int64_t* dbase) {
    if (P->n == 0) return;
    if (!dkeys || !dbase) fail(TQP_ERR_INVALID_ARGUMENT, "partition_scatter: null destination arrays");
    PartDest h{};
    for (int d = 0; d < P->parts; d++) {
        h.keys[d] = dkeys[d];
        h.rows[d] = drows ? drows[d] : nullptr;
        h.base[d] = dbase[d];
    }
    // the table (6 KB) in device memory: a pageable-source copy returns once the source is
    // staged, and the buffer's reuse by the next call is stream-ordered after this kernel
    P->dest.alloc(ctx, 1);
    TQP_CUDA(cudaMemcpyAsync(P->dest.get(), &h, sizeof(PartDest), cudaMemcpyHostToDevice, ctx->stream));
    const PartDest* dp = P->dest.get();
    switch (P->keys.dtype) {
        case TQP_I64: launch(ctx, "tqp_partition", part_scatter_kernel<TQP_I64>, dim3((unsigned)P->tiles), dim3(QNT), 0, P->keys.data, P->n, P->splitters, P->parts, P->tiles, (const uint64_t*)P->off.get(), row_base, (void*)nullptr, (int64_t*)nullptr, dp); break;
        case TQP_I32: launch(ctx, "tqp_partition", part_scatter_kernel<TQP_I32>, dim3((unsigned)P->tiles), dim3(QNT), 0, P->keys.data, P->n, P->splitters, P->parts, P->tiles, (const uint64_t*)P->off.get(), row_base, (void*)nullptr, (int64_t*)nullptr, dp); break;
        default: launch(ctx, "tqp_partition", part_scatter_kernel<TQP_U8>, dim3((unsigned)P->tiles), dim3(QNT), 0, P->keys.data, P->n, P->splitters, P->parts, P->tiles, (const uint64_t*)P->off.get(), row_base, (void*)nullptr, (int64_t*)nullptr, dp); break;
    }
    ctx->add_bytes("tqp_partition", (double)P->n * (2.0 * dtype_size(P->keys.dtype) + (drows ? 8.0 : 0.0)));
}

void partition_release(tqp_ctx*, tqp_partition_plan* P) { delete P; }

// Receive buffers shared across processes (CUDA IPC; peers on NVLink map them over P2P):
// an exact cudaMalloc (an IPC handle names a whole allocation), its handle, and the
// importer's mapping of a peer's handle.
void* ipc_alloc(size_t bytes, void* handle) {
    void* p = nullptr;
    TQP_CUDA(cudaMalloc(&p, std::max<size_t>(bytes, 256)));
    cudaIpcMemHandle_t h;
    TQP_CUDA(cudaIpcGetMemHandle(&h, p));
    memcpy(handle, &h, sizeof(h));
    return p;
}

void* ipc_open(const void* handle) {
    cudaIpcMemHandle_t h;
    memcpy(&h, handle, sizeof(h));
    void* p = nullptr;
    TQP_CUDA(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
    return p;
}

void minmax(tqp_ctx* ctx, tqp_col keys, int64_t n, int64_t* lohi) {
    check_col(keys, n, "minmax keys");
    if (keys.dtype == TQP_F64) fail(TQP_ERR_INVALID_ARGUMENT, "minmax: keys must be integer columns");
    if (!lohi) fail(TQP_ERR_INVALID_ARGUMENT, "minmax: null output");
    DevBuf<unsigned long long> mm(ctx, 2);
    launch(ctx, "tqp_minmax", minmax_init_kernel, dim3(1), dim3(1), 0, mm.get());
    if (n > 0) {
        const int g = (int)std::min<int64_t>(ceil_div(n, QNT * 4), (int64_t)ctx->num_sms * 8);
        launch(ctx, "tqp_minmax", minmax_kernel, dim3(g), dim3(QNT), 0, keys.data, (int)keys.dtype, n, mm.get());
        ctx->add_bytes("tqp_minmax", (double)n * dtype_size(keys.dtype));
    }
    launch(ctx, "tqp_minmax", minmax_final_kernel, dim3(1), dim3(1), 0, (const unsigned long long*)mm.get(), lohi);
}

void range_splitters(tqp_ctx* ctx, const int64_t* lohi, int parts, int64_t* splitters) {
    if (parts < 1 || parts > QMAXP) fail(TQP_ERR_INVALID_ARGUMENT, "range_splitters: parts must be in [1, 256]");
    if (!lohi || (parts > 1 && !splitters)) fail(TQP_ERR_INVALID_ARGUMENT, "range_splitters: null pointer");
    if (parts > 1)
        launch(ctx, "tqp_range_splitters", range_splitters_kernel, dim3(1), dim3(QMAXP), 0, lohi, parts, splitters);
}

void gather(tqp_ctx* ctx, tqp_col src, const int64_t* idx, int64_t n, void* out) {
    if (n < 0 || (n > 0 && (!src.data || !idx || !out))) fail(TQP_ERR_INVALID_ARGUMENT, "gather: null pointer");
    if (n == 0) return;
    const int g = (int)std::min<int64_t>(ceil_div(n, 256), (int64_t)ctx->num_sms * 8);
    switch (src.dtype) {
        case TQP_I64: launch(ctx, "tqp_gather", gather_kernel<TQP_I64>, dim3(g), dim3(256), 0, src.data, idx, n, out); break;
        case TQP_F64: launch(ctx, "tqp_gather", gather_kernel<TQP_F64>, dim3(g), dim3(256), 0, src.data, idx, n, out); break;
        case TQP_I32: launch(ctx, "tqp_gather", gather_kernel<TQP_I32>, dim3(g), dim3(256), 0, src.data, idx, n, out); break;
        case TQP_U8: launch(ctx, "tqp_gather", gather_kernel<TQP_U8>, dim3(g), dim3(256), 0, src.data, idx, n, out); break;
        default: fail(TQP_ERR_INVALID_ARGUMENT, "gather: unsupported dtype");
    }
    ctx->add_bytes("tqp_gather", (double)n * (8.0 + 2.0 * dtype_size(src.dtype)));
}

}  // namespace tqp
