// sort.cu -- onesweep LSD radix sort with permutation (stable), sm_100a.
//
// Paper: the join sorts its keys (Alg. 1 l.2-3) and the
// aggregation sorts the concatenated group keys with "radix sort" (PAPER.md:256,
// prose :1148). The paper composes torch.sort; here the sort is one upfront
// AND/OR pass (which digits vary), one digit-histogram pass, and one onesweep
// pass per varying 8-bit digit:
//   - each CTA takes a dynamic tile id, ranks its tile by digit with warp-level
//     __match_any_sync (stable within the warp's contiguous slice),
//   - per-warp digit counters give the tile-local stable order,
//   - the tile's 256-bin histogram is chained across tiles by decoupled
//     look-back (one thread per digit) to get global output offsets,
//   - keys and permutation are staged in shared memory in sorted order and
//     written out so that consecutive threads write consecutive addresses.
// Digits that are constant across all keys are skipped; when every varying bit
// lies in the low 32 bits the passes carry 32-bit keys (half the traffic).
#include "internal.h"

namespace tqp {

constexpr int NT = 256;                 // threads per CTA in the sort kernels
constexpr int NW = NT / 32;
constexpr uint32_t SLB_AGG = 1u << 30;  // 32-bit look-back words for the digit chains
constexpr uint32_t SLB_PRE = 2u << 30;
constexpr uint32_t SLB_VAL = (1u << 30) - 1;

enum InMode { IN_INTERNAL = 0, IN_I64 = 1, IN_I32 = 2, IN_U8 = 3, IN_U64 = 4 };

template <int IN>
__device__ __forceinline__ uint64_t load_u(const void* p, int64_t i, bool desc) {
    uint64_t u;
    if (IN == IN_I64) u = ordered_u64((int64_t)__ldg((const long long*)p + i));
    else if (IN == IN_I32) u = ordered_u64((int64_t)__ldg((const int*)p + i));
    else if (IN == IN_U8) u = ordered_u64((int64_t)__ldg((const unsigned char*)p + i));
    else u = (uint64_t)__ldg((const unsigned long long*)p + i);
    return desc ? ~u : u;
}

template <int IN>
__global__ void __launch_bounds__(NT) andor_kernel(const void* keys, int64_t n, bool desc,
                                                   unsigned long long* out) {
    uint64_t a = ~0ull, o = 0;
    for (int64_t i = blockIdx.x * (int64_t)NT + threadIdx.x; i < n; i += (int64_t)gridDim.x * NT) {
        uint64_t u = load_u<IN>(keys, i, desc);
        a &= u;
        o |= u;
    }
    for (int s = 16; s > 0; s >>= 1) {
        a &= __shfl_xor_sync(0xffffffffu, a, s);
        o |= __shfl_xor_sync(0xffffffffu, o, s);
    }
    __shared__ uint64_t sa[NW], so[NW];
    if ((threadIdx.x & 31) == 0) { sa[threadIdx.x >> 5] = a; so[threadIdx.x >> 5] = o; }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < NW; w++) { a &= sa[w]; o |= so[w]; }
        atomicAnd(&out[0], (unsigned long long)a);
        atomicOr(&out[1], (unsigned long long)o);
    }
}

struct PassPlan {
    int n;
    int shift[8];
};

template <int IN>
__global__ void __launch_bounds__(NT) hist_kernel(const void* keys, int64_t n, bool desc, PassPlan pp,
                                                  uint32_t* ghist) {
    __shared__ uint32_t h[8][256];
    for (int i = threadIdx.x; i < 8 * 256; i += NT) (&h[0][0])[i] = 0;
    __syncthreads();
    for (int64_t i = blockIdx.x * (int64_t)NT + threadIdx.x; i < n; i += (int64_t)gridDim.x * NT) {
        uint64_t u = load_u<IN>(keys, i, desc);
#pragma unroll
        for (int p = 0; p < 8; p++)
            if (p < pp.n) atomicAdd(&h[p][(u >> pp.shift[p]) & 255], 1u);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < pp.n * 256; i += NT) {
        uint32_t c = (&h[0][0])[i];
        if (c) atomicAdd(&ghist[i], c);
    }
}

// Exclusive scan of one value per thread across a 256-thread block.
__device__ __forceinline__ uint32_t block_excl_scan256(uint32_t v, uint32_t* s_w) {
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

struct OnesweepArgs {
    const void* in_keys;
    const uint32_t* in_perm;      // IN_INTERNAL only
    void* out_keys;               // internal KT (nullable on the last pass)
    uint32_t* out_perm;           // nullable on the last pass
    void* out_orig;               // last pass: keys in the input dtype
    int orig_dtype;
    int64_t* out_perm64;          // last pass
    uint64_t* out_u;              // last pass: sort-domain values
    const uint32_t* ghist;        // this pass's 256 global digit counts
    uint32_t* lb;                 // tiles x 256 look-back words (zeroed)
    unsigned long long* counter;  // dynamic tile counter (zeroed)
    int64_t n;
    int shift;
    bool desc;
    uint64_t hi_bits;             // u's constant high 32 bits (k32 reconstruction)
};

template <typename KT>
__device__ __forceinline__ uint64_t to_u(KT k, uint64_t hi_bits) {
    if (sizeof(KT) == 4) return hi_bits | (uint64_t)k;
    return (uint64_t)k;
}

template <typename KT, int IN, int IPT>
__global__ void __launch_bounds__(NT, 3) onesweep_kernel(OnesweepArgs a) {
    constexpr int TILE = NT * IPT;
    __shared__ union {
        uint32_t whist[NW][256];
        struct {
            KT keys[TILE];
            uint32_t perm[TILE];
        } stage;
    } s;
    __shared__ uint32_t s_tstart[256], s_gstart[256], s_base[256], s_w[NW];
    __shared__ int64_t s_tile;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t tile = take_tile(a.counter, &s_tile);
    const int64_t base = tile * TILE;

    for (int d = lane; d < 256; d += 32) s.whist[warp][d] = 0;
    // global start of each digit's bin = exclusive scan of the pass histogram
    s_base[tid] = block_excl_scan256(a.ghist[tid], s_w);

    KT key[IPT];
    uint32_t pm[IPT], rk[IPT];
#pragma unroll
    for (int i = 0; i < IPT; i++) {
        int64_t pos = base + warp * 32 * IPT + i * 32 + lane;
        if (pos < a.n) {
            if (IN == IN_INTERNAL) {
                key[i] = ((const KT*)a.in_keys)[pos];
                pm[i] = a.in_perm[pos];
            } else {
                key[i] = (KT)load_u<IN>(a.in_keys, pos, a.desc);
                pm[i] = (uint32_t)pos;
            }
        } else {
            key[i] = 0;
            pm[i] = 0;
        }
    }
    __syncwarp();
    // Stable warp-level ranking: the leader of each match_any peer group claims
    // popc(peers) slots of its warp's digit counter with a shared-memory atomicAdd
    // (items are issued in order, so the claimed ranges follow item order); the
    // 16 atomics pipeline without waiting on each other. rk packs the claimed
    // base (bits 0-15), the leader lane (16-20) and the lane's rank among its
    // peers (24-28) until the bases are broadcast.
    const unsigned lt = lanemask_lt();
#pragma unroll
    for (int i = 0; i < IPT; i++) {
        const int64_t pos = base + warp * 32 * IPT + i * 32 + lane;
        const bool valid = pos < a.n;
        const uint32_t d = (uint32_t)(key[i] >> a.shift) & 255u;
        // peers = lanes with the same digit: one ballot per digit bit (cheaper than MATCH.ANY)
        unsigned peers = __ballot_sync(0xffffffffu, valid);
#pragma unroll
        for (int b = 0; b < 8; b++) {
            const unsigned bb = __ballot_sync(0xffffffffu, (d >> b) & 1u);
            peers &= ((d >> b) & 1u) ? bb : ~bb;
        }
        const uint32_t leader = 31 - __clz(peers);
        uint32_t old = 0;
        if (valid && lane == leader) old = atomicAdd(&s.whist[warp][d], (uint32_t)__popc(peers));
        rk[i] = old | (leader << 16) | ((uint32_t)__popc(peers & lt) << 24);
    }
#pragma unroll
    for (int i = 0; i < IPT; i++) {
        const uint32_t b = __shfl_sync(0xffffffffu, rk[i] & 0xFFFFu, (rk[i] >> 16) & 31u);
        rk[i] = b + (rk[i] >> 24);
    }
    __syncthreads();
    // per digit (thread d): exclusive prefix over warps and the tile count
    uint32_t cnt = 0;
    {
        const int d = tid;
#pragma unroll
        for (int w = 0; w < NW; w++) {
            uint32_t c = s.whist[w][d];
            s.whist[w][d] = cnt;
            cnt += c;
        }
    }
    s_tstart[tid] = block_excl_scan256(cnt, s_w);
    // publish this tile's digit counts as early as possible (successors sum them)
    {
        const int d = tid;
        uint32_t* st = a.lb + d;
        if (tile == 0)
            asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(st), "r"(SLB_PRE | (s_base[d] + cnt)) : "memory");
        else
            asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(st + tile * 256), "r"(SLB_AGG | cnt) : "memory");
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < IPT; i++) {
        int64_t pos = base + warp * 32 * IPT + i * 32 + lane;
        if (pos < a.n) {
            uint32_t d = (uint32_t)(key[i] >> a.shift) & 255u;
            rk[i] = s_tstart[d] + s.whist[warp][d] + rk[i];
        }
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < IPT; i++) {
        int64_t pos = base + warp * 32 * IPT + i * 32 + lane;
        if (pos < a.n) {
            s.stage.keys[rk[i]] = key[i];
            s.stage.perm[rk[i]] = pm[i];
        }
    }
    // decoupled look-back along this digit's chain of tiles, after the keys are
    // staged (their registers are free): LBW independent loads per round
    {
        const int d = tid;
        uint32_t* st = a.lb + d;
        uint32_t g;
        if (tile == 0) {
            g = s_base[d];
        } else {
            constexpr int LBW = 8;
            uint32_t excl = 0;
            int64_t t = tile - 1;
            while (true) {
                uint32_t wv[LBW];
#pragma unroll
                for (int i = 0; i < LBW; i++) {
                    const int64_t ti = t - i;
                    if (ti >= 0)
                        asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(wv[i]) : "l"(st + ti * 256) : "memory");
                    else
                        wv[i] = SLB_PRE;
                }
                uint32_t sum = 0;
                bool done = false, stall = false;
#pragma unroll
                for (int i = 0; i < LBW; i++) {
                    if (!done && !stall) {
                        const uint32_t f = wv[i] >> 30;
                        if (f == 0) stall = true;
                        else {
                            sum += wv[i] & SLB_VAL;
                            done = f == 2;
                        }
                    }
                }
                if (stall) continue;
                excl += sum;
                if (done) break;
                t -= LBW;
            }
            asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(st + tile * 256), "r"(SLB_PRE | (excl + cnt)) : "memory");
            g = excl;
        }
        s_gstart[d] = g;
    }
    __syncthreads();
    const int tile_n = (int)min((int64_t)TILE, a.n - base);
    for (int j = tid; j < tile_n; j += NT) {
        KT k = s.stage.keys[j];
        uint32_t p = s.stage.perm[j];
        uint32_t d = (uint32_t)(k >> a.shift) & 255u;
        int64_t dst = (int64_t)s_gstart[d] + (j - (int64_t)s_tstart[d]);
        if (a.out_keys) ((KT*)a.out_keys)[dst] = k;
        if (a.out_perm) a.out_perm[dst] = p;
        if (a.out_perm64) a.out_perm64[dst] = (int64_t)p;
        if (a.out_u || a.out_orig) {
            uint64_t u = to_u<KT>(k, a.hi_bits);
            if (a.out_u) a.out_u[dst] = u;
            if (a.out_orig) {
                uint64_t v = a.desc ? ~u : u;
                switch (a.orig_dtype) {
                    case TQP_U8: ((uint8_t*)a.out_orig)[dst] = (uint8_t)unordered_i64(v); break;
                    case TQP_I32: ((int32_t*)a.out_orig)[dst] = (int32_t)unordered_i64(v); break;
                    case TQP_I64: ((int64_t*)a.out_orig)[dst] = unordered_i64(v); break;
                    default: ((uint64_t*)a.out_orig)[dst] = v; break;
                }
            }
        }
    }
}

// All keys equal (or n <= 1): the stable order is the identity.
template <typename KT, int IN>
__global__ void trivial_sort_kernel(const void* in, int64_t n, bool desc, int orig_dtype, void* out_orig,
                                    int64_t* perm64, uint64_t* out_u, KT* keys_int, uint32_t* perm32) {
    for (int64_t i = blockIdx.x * (int64_t)NT + threadIdx.x; i < n; i += (int64_t)gridDim.x * NT) {
        uint64_t u = load_u<IN>(in, i, desc);
        if (perm64) perm64[i] = i;
        if (perm32) perm32[i] = (uint32_t)i;
        if (keys_int) keys_int[i] = (KT)u;
        if (out_u) out_u[i] = u;
        if (out_orig) {
            uint64_t v = desc ? ~u : u;
            switch (orig_dtype) {
                case TQP_U8: ((uint8_t*)out_orig)[i] = (uint8_t)unordered_i64(v); break;
                case TQP_I32: ((int32_t*)out_orig)[i] = (int32_t)unordered_i64(v); break;
                case TQP_I64: ((int64_t*)out_orig)[i] = unordered_i64(v); break;
                default: ((uint64_t*)out_orig)[i] = v; break;
            }
        }
    }
}

static int in_mode(int dtype) {
    switch (dtype) {
        case TQP_I64: return IN_I64;
        case TQP_I32: return IN_I32;
        case TQP_U8: return IN_U8;
        case DT_U64: return IN_U64;
    }
    fail(TQP_ERR_INVALID_ARGUMENT, "sort: unsupported key dtype");
}

template <typename F>
static void dispatch_in(int mode, F&& f) {
    switch (mode) {
        case IN_I64: f(std::integral_constant<int, IN_I64>()); break;
        case IN_I32: f(std::integral_constant<int, IN_I32>()); break;
        case IN_U8: f(std::integral_constant<int, IN_U8>()); break;
        default: f(std::integral_constant<int, IN_U64>()); break;
    }
}

template <typename KT>
static void run_passes(tqp_ctx* ctx, const void* keys, int dtype, int64_t n, bool desc, SortOut& o,
                       const PassPlan& pp, const uint32_t* ghist) {
    constexpr int IPT = sizeof(KT) == 4 ? 16 : 12;
    constexpr int TILE = NT * IPT;
    const int64_t tiles = ceil_div(n, TILE);
    const int P = pp.n;
    DevBuf<KT> kb[2];
    DevBuf<uint32_t> pb[2];
    const bool need_key_final = o.want_internal;
    const bool need_perm_final = o.want_internal || o.want_perm32;
    for (int b = 0; b < 2; b++) {
        // buffer b is written by passes p with p % 2 == b
        bool kused = false, pused = false;
        for (int p = 0; p < P; p++)
            if (p % 2 == b) {
                if (p < P - 1 || need_key_final) kused = true;
                if (p < P - 1 || need_perm_final) pused = true;
            }
        if (kused) kb[b].alloc(ctx, n);
        if (pused) pb[b].alloc(ctx, n);
    }
    DevBuf<uint32_t> lb(ctx, (size_t)P * tiles * 256);
    DevBuf<unsigned long long> counters(ctx, P);
    lb.zero();
    counters.zero();
    const int mode = in_mode(dtype);
    for (int p = 0; p < P; p++) {
        OnesweepArgs a{};
        a.in_keys = p == 0 ? keys : kb[(p - 1) % 2].get();
        a.in_perm = p == 0 ? nullptr : pb[(p - 1) % 2].get();
        const bool last = p == P - 1;
        a.out_keys = (!last || need_key_final) ? kb[p % 2].get() : nullptr;
        a.out_perm = (!last || need_perm_final) ? pb[p % 2].get() : nullptr;
        if (last) {
            a.out_orig = o.sorted_orig;
            a.orig_dtype = dtype;
            a.out_perm64 = o.perm64;
            a.out_u = o.sorted_u;
        }
        a.ghist = ghist + p * 256;
        a.lb = lb.get() + (size_t)p * tiles * 256;
        a.counter = counters.get() + p;
        a.n = n;
        a.shift = pp.shift[p];
        a.desc = desc;
        a.hi_bits = o.and_bits & 0xFFFFFFFF00000000ull;
        {   // algorithmic bytes of this pass: keys + permutation in, requested outputs out
            double rd = p == 0 ? (double)dtype_size(dtype) : (double)(sizeof(KT) + 4);
            double wr = (a.out_keys ? sizeof(KT) : 0) + (a.out_perm ? 4 : 0) + (a.out_orig ? dtype_size(dtype) : 0) +
                        (a.out_perm64 ? 8 : 0) + (a.out_u ? 8 : 0);
            ctx->add_bytes("tqp_onesweep", (rd + wr) * (double)n);
        }
        if (p == 0) {
            dispatch_in(mode, [&](auto m) {
                launch(ctx, "tqp_onesweep", onesweep_kernel<KT, decltype(m)::value, IPT>, dim3((unsigned)tiles),
                       dim3(NT), 0, a);
            });
        } else {
            launch(ctx, "tqp_onesweep", onesweep_kernel<KT, IN_INTERNAL, IPT>, dim3((unsigned)tiles), dim3(NT), 0,
                   a);
        }
    }
    const int fb = (P - 1) % 2;
    if (need_key_final) {
        if constexpr (sizeof(KT) == 4) o.keys32 = std::move(kb[fb]);
        else o.keys64 = std::move(kb[fb]);
    }
    if (need_perm_final) o.perm32 = std::move(pb[fb]);
}

void radix_sort(tqp_ctx* ctx, const void* keys, int dtype, int64_t n, bool desc, SortOut& o) {
    if (n < 0 || n >= (int64_t(1) << 30)) fail(TQP_ERR_INVALID_ARGUMENT, "sort: n must be in [0, 2^30)");
    if (n == 0) return;
    const int mode = in_mode(dtype);
    const int grid = (int)std::min<int64_t>(ceil_div(n, NT * 8), (int64_t)ctx->num_sms * 4);
    DevBuf<unsigned long long> ao(ctx, 2);
    TQP_CUDA(cudaMemsetAsync(ao.get(), 0xFF, 8, ctx->stream));
    TQP_CUDA(cudaMemsetAsync(ao.get() + 1, 0, 8, ctx->stream));
    dispatch_in(mode, [&](auto m) {
        launch(ctx, "tqp_sort_andor", andor_kernel<decltype(m)::value>, dim3(grid), dim3(NT), 0, keys, n, desc,
               ao.get());
    });
    ctx->add_bytes("tqp_sort_andor", (double)n * dtype_size(dtype));
    uint64_t h[2];
    read_back(ctx, h, ao.get(), 16);
    o.and_bits = h[0];
    o.or_bits = h[1];
    const uint64_t diff = h[0] ^ h[1];
    o.k32 = (diff >> 32) == 0;
    PassPlan pp{};
    for (int b = 0; b < 8; b++)
        if ((diff >> (8 * b)) & 0xFF) pp.shift[pp.n++] = 8 * b;
    o.passes = pp.n;
    if (pp.n == 0) {
        if (o.want_internal || o.want_perm32) o.perm32.alloc(ctx, n);
        if (o.want_internal) {
            if (o.k32) o.keys32.alloc(ctx, n); else o.keys64.alloc(ctx, n);
        }
        const int g = (int)std::min<int64_t>(ceil_div(n, NT), (int64_t)ctx->num_sms * 8);
        ctx->add_bytes("tqp_sort_trivial",
                       (double)n * (dtype_size(dtype) + (o.sorted_orig ? dtype_size(dtype) : 0) + (o.perm64 ? 8 : 0) +
                                    (o.sorted_u ? 8 : 0) + (o.perm32.n ? 4 : 0) + (o.want_internal ? (o.k32 ? 4 : 8) : 0)));
        dispatch_in(mode, [&](auto m) {
            if (o.k32)
                launch(ctx, "tqp_sort_trivial", trivial_sort_kernel<uint32_t, decltype(m)::value>, dim3(g), dim3(NT),
                       0, keys, n, desc, dtype, o.sorted_orig, o.perm64, o.sorted_u, o.keys32.get(), o.perm32.get());
            else
                launch(ctx, "tqp_sort_trivial", trivial_sort_kernel<uint64_t, decltype(m)::value>, dim3(g), dim3(NT),
                       0, keys, n, desc, dtype, o.sorted_orig, o.perm64, o.sorted_u, o.keys64.get(), o.perm32.get());
        });
        return;
    }
    DevBuf<uint32_t> ghist(ctx, (size_t)pp.n * 256);
    ghist.zero();
    dispatch_in(mode, [&](auto m) {
        launch(ctx, "tqp_sort_hist", hist_kernel<decltype(m)::value>, dim3(grid), dim3(NT), 0, keys, n, desc, pp,
               ghist.get());
    });
    ctx->add_bytes("tqp_sort_hist", (double)n * dtype_size(dtype));
    if (o.k32) run_passes<uint32_t>(ctx, keys, dtype, n, desc, o, pp, ghist.get());
    else run_passes<uint64_t>(ctx, keys, dtype, n, desc, o, pp, ghist.get());
}

}  // namespace tqp
