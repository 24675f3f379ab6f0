// scan.cu -- single-pass device-wide scans by decoupled look-back (sm_100a).
#include "internal.h"

namespace tqp {

namespace {
constexpr int SNT = 256;
constexpr int SIPT = 8;   // 8 consecutive u32 per thread = two 16-byte loads
constexpr int STILE = SNT * SIPT;

// Exclusive scan of u32 values under max (out[i] = max(in[0..i-1])) or add
// (out[i] = sum(in[0..i-1]), and out[n] = the total). out[0] = 0.
template <bool ADD, typename OT, typename IT = uint32_t>
__global__ void __launch_bounds__(SNT) scan_u32_kernel(const IT* __restrict__ in, OT* __restrict__ out,
                                                       int64_t n, uint64_t* status, unsigned long long* counter) {
    __shared__ int64_t s_tile;
    __shared__ OT s_w[SNT / 32];
    __shared__ uint64_t s_excl;
    const int64_t tile = take_tile(counter, &s_tile);
    const int64_t base = tile * STILE + (int64_t)threadIdx.x * SIPT;
    IT v[SIPT];
    if (sizeof(IT) == 4 && base + SIPT <= n && (((uintptr_t)(in + base)) & 15) == 0) {
        uint4 a = *reinterpret_cast<const uint4*>(in + base);
        uint4 b = *reinterpret_cast<const uint4*>(in + base + 4);
        v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
    } else {
#pragma unroll
        for (int i = 0; i < SIPT; i++) v[i] = (base + i < n) ? in[base + i] : IT(0);
    }
    auto op = [](OT a, OT b) -> OT { return ADD ? a + b : max(a, b); };
    OT t = 0;
#pragma unroll
    for (int i = 0; i < SIPT; i++) t = op(t, v[i]);
    // block exclusive max over threads
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    OT x = t;
    for (int o = 1; o < 32; o <<= 1) {
        OT y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x = op(x, y);
    }
    if (lane == 31) s_w[warp] = x;
    __syncthreads();
    OT wpre = 0, tot = 0;
    for (int w = 0; w < SNT / 32; w++) {
        if (w < warp) wpre = op(wpre, s_w[w]);
        tot = op(tot, s_w[w]);
    }
    const OT xp = __shfl_up_sync(0xffffffffu, x, 1);
    OT texcl = op(wpre, lane > 0 ? xp : OT(0));
    if (warp == 0) {
        uint64_t e = ADD ? lookback_warp(status, tile, (uint64_t)tot, OpAdd(), 0ull)
                         : lookback_warp(status, tile, (uint64_t)tot, OpMax(), 0ull);
        if (lane == 0) s_excl = e;
    }
    __syncthreads();
    OT run = op((OT)s_excl, texcl);
#pragma unroll
    for (int i = 0; i < SIPT; i++) {
        if (base + i < n) out[base + i] = run;
        run = op(run, v[i]);
    }
    if (ADD && base < n && base + SIPT >= n) out[n] = run;
}
__global__ void iota_i64_kernel(int64_t* p, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        p[i] = i;
}
}  // namespace

void iota_i64(tqp_ctx* ctx, int64_t* p, int64_t n) {
    if (n <= 0) return;
    const int g = (int)std::min<int64_t>(ceil_div(n, 256), (int64_t)ctx->num_sms * 8);
    ctx->add_bytes("tqp_iota", 8.0 * (double)n);
    launch(ctx, "tqp_iota", iota_i64_kernel, dim3(g), dim3(256), 0, p, n);
}

void scan_max_u32_exclusive(tqp_ctx* ctx, const uint32_t* in, uint32_t* out, int64_t n) {
    if (n <= 0) return;
    const int64_t tiles = ceil_div(n, STILE);
    DevBuf<uint64_t> status(ctx, tiles);
    DevBuf<unsigned long long> counter(ctx, 1);
    status.zero();
    counter.zero();
    ctx->add_bytes("tqp_scan_max", 8.0 * (double)n);
    launch(ctx, "tqp_scan_max", scan_u32_kernel<false, uint32_t>, dim3((unsigned)tiles), dim3(SNT), 0, in, out, n, status.get(),
           counter.get());
}

void scan_add_u32_exclusive(tqp_ctx* ctx, const uint32_t* in, uint32_t* out, int64_t n) {
    if (n <= 0) return;
    const int64_t tiles = ceil_div(n, STILE);
    DevBuf<uint64_t> status(ctx, tiles);
    DevBuf<unsigned long long> counter(ctx, 1);
    status.zero();
    counter.zero();
    ctx->add_bytes("tqp_scan_add", 8.0 * (double)n);
    launch(ctx, "tqp_scan_add", scan_u32_kernel<true, uint32_t>, dim3((unsigned)tiles), dim3(SNT), 0, in, out, n, status.get(),
           counter.get());
}

void scan_add_u32_to_u64_exclusive(tqp_ctx* ctx, const uint32_t* in, uint64_t* out, int64_t n) {
    if (n <= 0) return;
    const int64_t tiles = ceil_div(n, STILE);
    DevBuf<uint64_t> status(ctx, tiles);
    DevBuf<unsigned long long> counter(ctx, 1);
    status.zero();
    counter.zero();
    ctx->add_bytes("tqp_scan_add", 12.0 * (double)n);
    launch(ctx, "tqp_scan_add", scan_u32_kernel<true, uint64_t>, dim3((unsigned)tiles), dim3(SNT), 0, in, out, n,
           status.get(), counter.get());
}

// 64-bit values (< 2^62 each and in total; the caller checks the total separately)
void scan_add_u64_exclusive(tqp_ctx* ctx, const uint64_t* in, uint64_t* out, int64_t n) {
    if (n <= 0) return;
    const int64_t tiles = ceil_div(n, STILE);
    DevBuf<uint64_t> status(ctx, tiles);
    DevBuf<unsigned long long> counter(ctx, 1);
    status.zero();
    counter.zero();
    ctx->add_bytes("tqp_scan_add", 16.0 * (double)n);
    launch(ctx, "tqp_scan_add", scan_u32_kernel<true, uint64_t, uint64_t>, dim3((unsigned)tiles), dim3(SNT), 0, in, out,
           n, status.get(), counter.get());
}

}  // namespace tqp
