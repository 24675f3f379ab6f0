// pkfk.cu -- primary-key / foreign-key join ("Find matches
// using binary search"), plus left-semi / left-anti.
//
// The paper sorts both sides descending, pads the build side to a power of two
// and runs log2(n') rounds of a branch-free binary search as whole-tensor ops,
// then masks and compacts with maskedSelect. On B200 the same result (reading
// R8: lower_bound on the unpadded sorted build keys; position n = no match) is
// computed in one pass over the probe keys:
//   1. radix-sort the build keys with their permutation (sort.cu), keeping the
//      compressed internal keys (32-bit when the key range allows: the sorted
//      build side then fits in L2),
//   2. a radix bracket table T over the top B bits of (key - base):
//      T[b] = first sorted position whose bucket is >= b, built from the bucket
//      end positions by an exclusive max-scan (no domain-sized bincount),
//   3. per probe key: bucket -> [T[b], T[b+1]) -> lower_bound inside the bucket
//      -> equality test (the paper's match mask) ->
//      order-preserving compaction (ballot + block scan + decoupled look-back)
//      writing leftOutputIndex = perm[pos], rightOutputIndex = probe row
//       in ascending probe-row order (reading R7).
// Duplicate build keys (adjacent equal sorted keys) -> TQP_ERR_DUPLICATE_BUILD_KEY.
#include "internal.h"

namespace tqp {

namespace {
constexpr int PNT = 256;
constexpr int PNW = PNT / 32;
constexpr int PIPT = 8;
constexpr int PTILE = PNT * PIPT;

template <typename KT>
__global__ void bucket_ends_kernel(const KT* __restrict__ keys, int64_t n, KT base, int shift,
                                   uint32_t* __restrict__ H, int* __restrict__ dup) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        KT k = keys[i];
        uint64_t b = (uint64_t)(KT)(k - base) >> shift;
        if (i + 1 == n) {
            H[b] = (uint32_t)n;
        } else {
            KT k2 = keys[i + 1];
            if (((uint64_t)(KT)(k2 - base) >> shift) != b) H[b] = (uint32_t)(i + 1);
            if (k2 == k) *dup = 1;
        }
    }
}

// Packed build records: rec = ((key - base) mod 2^shift) << pbits | source row. The
// bracket bucket supplies the key bits above `shift`, so one u32 per build row
// carries both the residual key and the permutation (keeps the build side
// L2-resident: 15M orders -> 60 MB of records + an 8 MB bracket table).
template <typename KT>
__global__ void pack_records_kernel(const KT* __restrict__ keys, const uint32_t* __restrict__ perm, int64_t n,
                                    KT base, uint32_t lowmask, int pbits, uint32_t* __restrict__ rec) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        rec[i] = (((uint32_t)(KT)(keys[i] - base) & lowmask) << pbits) | perm[i];
}

struct ProbeArgs {
    const void* probe;
    int64_t n_probe;
    const void* bkeys;        // sorted internal build keys (KT)
    const uint32_t* bperm;    // their source rows
    const uint32_t* T;        // bracket table, 2^B + 1 entries
    const uint32_t* rec;      // packed records (PACKED)
    uint32_t lowmask;         // 2^shift - 1
    int pbits;                // bits of the row number in a record
    uint64_t base;            // internal-domain base (= AND of all build keys)
    int vbits;                // (k - base) must be < 2^vbits
    uint64_t hi_bits;         // k32: required high 32 bits of u
    int shift;
    int mode;                 // 0 = join pairs, 1 = semi/anti
    int anti;
    int64_t* left_out;
    int64_t* right_out;       // join: probe rows; semi: selected rows
    uint8_t* match_out;       // semi: per-row mask (nullable)
    uint64_t* status;
    unsigned long long* counter;
    int64_t* total;           // written by the last tile
    int64_t n_tiles;
};

template <typename KT, int PDT, bool PACKED>
__device__ __forceinline__ bool probe_one(const ProbeArgs& a, int64_t row, uint32_t& left) {
    int64_t v;   // probe keys are streamed once: evict-first
    if (PDT == TQP_I64) v = (int64_t)__ldcs((const long long*)a.probe + row);
    else if (PDT == TQP_I32) v = (int64_t)__ldcs((const int*)a.probe + row);
    else v = (int64_t)__ldcs((const unsigned char*)a.probe + row);
    uint64_t u = ordered_u64(v);
    KT k;
    if (sizeof(KT) == 4) {
        if ((u & 0xFFFFFFFF00000000ull) != a.hi_bits) return false;
        k = (KT)u;
    } else {
        k = (KT)u;
    }
    KT rel = (KT)(k - (KT)a.base);
    if (k < (KT)a.base || (a.vbits < 64 && ((uint64_t)rel >> a.vbits) != 0)) return false;
    uint64_t b = (uint64_t)rel >> a.shift;
    uint32_t lo = __ldg(a.T + b), hi = __ldg(a.T + b + 1);
    if (PACKED) {
        const uint32_t low = (uint32_t)rel & a.lowmask;
        const uint32_t target = low << a.pbits;
        const uint32_t end = hi;
        const uint32_t s0 = lo & ~7u;   // the bucket's records from one aligned 64-byte fetch
        if (hi <= s0 + 16u) {
            const uint4* p4 = reinterpret_cast<const uint4*>(a.rec + s0);
            const uint4 q0 = __ldg(p4), q1 = __ldg(p4 + 1), q2 = __ldg(p4 + 2), q3 = __ldg(p4 + 3);
            const uint32_t r16[16] = {q0.x, q0.y, q0.z, q0.w, q1.x, q1.y, q1.z, q1.w,
                                      q2.x, q2.y, q2.z, q2.w, q3.x, q3.y, q3.z, q3.w};
            bool hit = false;
#pragma unroll
            for (int j = 0; j < 16; j++) {   // residuals are distinct: at most one match
                const uint32_t pos = s0 + (uint32_t)j;
                if (pos >= lo && pos < end && (r16[j] >> a.pbits) == low) {
                    left = r16[j] & ((1u << a.pbits) - 1u);
                    hit = true;
                }
            }
            return hit;
        }
        while (lo < hi) {   // long bucket: lower_bound of the residual
            uint32_t mid = (lo + hi) >> 1;
            if (__ldg(a.rec + mid) < target) lo = mid + 1; else hi = mid;
        }
        if (lo < end) {
            const uint32_t r = __ldg(a.rec + lo);
            if ((r >> a.pbits) == low) {
                left = r & ((1u << a.pbits) - 1u);
                return true;
            }
        }
        return false;
    }
    const KT* keys = (const KT*)a.bkeys;
    const uint32_t end = hi;
    while (lo < hi) {   // lower_bound inside the bucket (a few elements)
        uint32_t mid = (lo + hi) >> 1;
        if (__ldg(keys + mid) < k) lo = mid + 1; else hi = mid;
    }
    if (lo < end && __ldg(keys + lo) == k) {
        left = __ldg(a.bperm + lo);
        return true;
    }
    return false;
}

template <typename KT, int PDT, bool PACKED>
__global__ void __launch_bounds__(PNT) probe_kernel(ProbeArgs a) {
    __shared__ int64_t s_tile;
    __shared__ uint32_t s_cnt[PIPT * PNW];
    __shared__ uint64_t s_excl;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t tile = take_tile(a.counter, &s_tile);
    const int64_t base = tile * PTILE;
    bool m[PIPT];
    uint32_t left[PIPT];
    unsigned bal[PIPT];
#pragma unroll
    for (int i = 0; i < PIPT; i++) {
        int64_t row = base + i * PNT + tid;
        m[i] = false;
        if (row < a.n_probe) m[i] = probe_one<KT, PDT, PACKED>(a, row, left[i]);
    }
#pragma unroll
    for (int i = 0; i < PIPT; i++) {
        int64_t row = base + i * PNT + tid;
        bool sel = a.mode == 0 ? m[i] : (row < a.n_probe && (m[i] != (a.anti != 0)));
        if (a.mode == 1 && a.match_out && row < a.n_probe) a.match_out[row] = (uint8_t)m[i];
        bal[i] = __ballot_sync(0xffffffffu, sel);
        if (lane == 0) s_cnt[i * PNW + warp] = __popc(bal[i]);
    }
    __syncthreads();
    if (warp == 0) {
        // exclusive scan over the PIPT*PNW (item, warp) counts, in tile order
        uint32_t c[PIPT * PNW / 32];
        uint32_t local = 0;
#pragma unroll
        for (int j = 0; j < PIPT * PNW / 32; j++) { c[j] = s_cnt[lane * (PIPT * PNW / 32) + j]; local += c[j]; }
        uint32_t x = local;
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        uint32_t tot = __shfl_sync(0xffffffffu, x, 31);
        uint32_t run = x - local;
#pragma unroll
        for (int j = 0; j < PIPT * PNW / 32; j++) { s_cnt[lane * (PIPT * PNW / 32) + j] = run; run += c[j]; }
        uint64_t e = lookback_warp(a.status, tile, tot, OpAdd(), 0ull);
        if (lane == 0) {
            s_excl = e;
            if (tile == a.n_tiles - 1) *a.total = (int64_t)(e + tot);
        }
    }
    __syncthreads();
    const int64_t excl = (int64_t)s_excl;
    const unsigned lt = lanemask_lt();
#pragma unroll
    for (int i = 0; i < PIPT; i++) {
        if (bal[i] & (1u << lane)) {
            int64_t row = base + i * PNT + tid;
            int64_t j = excl + s_cnt[i * PNW + warp] + __popc(bal[i] & lt);
            if (a.mode == 0) {   // outputs are streamed: evict-first stores
                __stcs((long long*)a.left_out + j, (long long)left[i]);
                __stcs((long long*)a.right_out + j, (long long)row);
            } else if (a.right_out) {
                __stcs((long long*)a.right_out + j, (long long)row);
            }
        }
    }
}

struct Built {
    SortOut so;
    DevBuf<uint32_t> TR;      // bracket table T, then (packed) the records, one allocation
    uint32_t* T = nullptr;
    uint32_t* rec = nullptr;
    size_t tr_bytes = 0;
    DevBuf<int> dup;
    uint64_t base = 0, hi_bits = 0;
    int shift = 0, vbits = 0, pbits = 0;
    bool packed = false;
    int64_t nb = 0;
};

void build_side(tqp_ctx* ctx, const tqp_col& bk, int64_t nb, Built& B) {
    B.so.want_internal = true;
    radix_sort(ctx, bk.data, bk.dtype, nb, false, B.so);
    B.dup.alloc(ctx, 1);
    B.dup.zero();
    if (nb == 0) return;
    const uint64_t diff = B.so.and_bits ^ B.so.or_bits;
    const int vbits = diff ? 64 - __builtin_clzll(diff) : 0;
    int lg = 0;
    while ((int64_t(1) << (lg + 1)) <= nb) lg++;
    int pbits = 1;
    while ((int64_t(1) << pbits) < nb) pbits++;
    // packed records need shift = vbits - B <= 32 - pbits; aim at ~4 keys per bucket
    const int bmax = std::min(vbits, 26);
    const int bmin_packed = vbits - (32 - pbits);
    int Bbits;
    if (vbits > 0 && bmin_packed <= bmax) {
        Bbits = std::max(std::max(std::min(bmax, std::max(lg - 2, 1)), bmin_packed), 1);
        B.packed = true;
        B.pbits = pbits;
    } else {
        Bbits = std::max(0, std::min(vbits, lg - 1));
        Bbits = std::min(Bbits, 26);
        if (vbits > 0) Bbits = std::max(Bbits, 1);   // keeps shift <= 63
    }
    B.nb = nb;
    B.shift = vbits - Bbits;
    B.vbits = vbits;
    if (B.so.k32) {
        B.base = B.so.and_bits & 0xFFFFFFFFull;
        B.hi_bits = B.so.and_bits & 0xFFFFFFFF00000000ull;
    } else {
        B.base = B.so.and_bits;
    }
    const int64_t nbk = int64_t(1) << Bbits;
    DevBuf<uint32_t> H(ctx, nbk + 1);
    H.zero();
    const int64_t toff = (nbk + 1 + 15) & ~int64_t(15);   // records start 64-byte aligned
    B.TR.alloc(ctx, toff + (B.packed ? nb + 16 : 0));     // +16: the probe reads whole aligned 64-byte groups
    B.T = B.TR.get();
    B.rec = B.packed ? B.TR.get() + toff : nullptr;
    B.tr_bytes = (size_t)(toff + (B.packed ? nb + 16 : 0)) * 4;
    const int g = (int)std::min<int64_t>(ceil_div(nb, 256), (int64_t)ctx->num_sms * 8);
    if (B.so.k32)
        launch(ctx, "tqp_pkfk_bucket_ends", bucket_ends_kernel<uint32_t>, dim3(g), dim3(256), 0, B.so.keys32.get(),
               nb, (uint32_t)B.base, B.shift, H.get(), B.dup.get());
    else
        launch(ctx, "tqp_pkfk_bucket_ends", bucket_ends_kernel<uint64_t>, dim3(g), dim3(256), 0, B.so.keys64.get(),
               nb, (uint64_t)B.base, B.shift, H.get(), B.dup.get());
    ctx->add_bytes("tqp_pkfk_bucket_ends", (double)nb * (B.so.k32 ? 4 : 8) + 4.0 * (double)std::min<int64_t>(nb, nbk));
    scan_max_u32_exclusive(ctx, H.get(), B.T, nbk + 1);
    if (B.packed) {
        const uint32_t lowmask = B.shift >= 32 ? 0xFFFFFFFFu : ((1u << B.shift) - 1u);
        if (B.so.k32)
            launch(ctx, "tqp_pkfk_records", pack_records_kernel<uint32_t>, dim3(g), dim3(256), 0, B.so.keys32.get(),
                   B.so.perm32.get(), nb, (uint32_t)B.base, lowmask, B.pbits, B.rec);
        else
            launch(ctx, "tqp_pkfk_records", pack_records_kernel<uint64_t>, dim3(g), dim3(256), 0, B.so.keys64.get(),
                   B.so.perm32.get(), nb, (uint64_t)B.base, lowmask, B.pbits, B.rec);
        ctx->add_bytes("tqp_pkfk_records", (double)nb * ((B.so.k32 ? 4 : 8) + 8));
        B.so.keys32.release();
        B.so.keys64.release();
        B.so.perm32.release();
    }
}

void run_probe(tqp_ctx* ctx, Built& B, const tqp_col& pk, int64_t np, int mode, int anti, int64_t* left_out,
               int64_t* right_out, uint8_t* match_out, int64_t* n_out_host) {
    DevBuf<int64_t> total(ctx, 1);
    total.zero();
    const int64_t nb = B.nb;
    if (np > 0 && nb > 0) {
        const int64_t tiles = ceil_div(np, PTILE);
        DevBuf<uint64_t> status(ctx, tiles);
        DevBuf<unsigned long long> counter(ctx, 1);
        status.zero();
        counter.zero();
        ProbeArgs a{};
        a.probe = pk.data;
        a.n_probe = np;
        a.bkeys = B.so.k32 ? (const void*)B.so.keys32.get() : (const void*)B.so.keys64.get();
        a.bperm = B.so.perm32.get();
        a.T = B.T;
        a.rec = B.rec;
        a.pbits = B.pbits;
        a.lowmask = B.shift >= 32 ? 0xFFFFFFFFu : ((1u << B.shift) - 1u);
        a.base = B.base;
        a.vbits = B.vbits;
        a.hi_bits = B.hi_bits;
        a.shift = B.shift;
        a.mode = mode;
        a.anti = anti;
        a.left_out = left_out;
        a.right_out = right_out;
        a.match_out = match_out;
        a.status = status.get();
        a.counter = counter.get();
        a.total = total.get();
        a.n_tiles = tiles;
        auto go = [&](auto kt, auto pk_) {
            using KT = decltype(kt);
            constexpr bool PK = decltype(pk_)::value;
            switch (pk.dtype) {
                case TQP_I64: launch(ctx, "tqp_pkfk_probe", probe_kernel<KT, TQP_I64, PK>, dim3((unsigned)tiles), dim3(PNT), 0, a); break;
                case TQP_I32: launch(ctx, "tqp_pkfk_probe", probe_kernel<KT, TQP_I32, PK>, dim3((unsigned)tiles), dim3(PNT), 0, a); break;
                default: launch(ctx, "tqp_pkfk_probe", probe_kernel<KT, TQP_U8, PK>, dim3((unsigned)tiles), dim3(PNT), 0, a); break;
            }
        };
        if (B.so.k32) {
            if (B.packed) go(uint32_t{}, std::true_type{}); else go(uint32_t{}, std::false_type{});
        } else {
            if (B.packed) go(uint64_t{}, std::true_type{}); else go(uint64_t{}, std::false_type{});
        }
    } else if (np > 0 && mode == 1) {
        // empty build side: nothing matches
        if (match_out) TQP_CUDA(cudaMemsetAsync(match_out, 0, np, ctx->stream));
        if (anti) {
            // every probe row is selected: sel = 0..np-1
            if (right_out) iota_i64(ctx, right_out, np);
            int64_t h = np;
            TQP_CUDA(cudaMemcpyAsync(total.get(), &h, 8, cudaMemcpyHostToDevice, ctx->stream));
        }
    }
    int64_t h[2];
    DevBuf<int64_t> pack(ctx, 2);
    TQP_CUDA(cudaMemcpyAsync(pack.get(), total.get(), 8, cudaMemcpyDeviceToDevice, ctx->stream));
    TQP_CUDA(cudaMemsetAsync(pack.get() + 1, 0, 8, ctx->stream));
    TQP_CUDA(cudaMemcpyAsync(pack.get() + 1, B.dup.get(), 4, cudaMemcpyDeviceToDevice, ctx->stream));
    read_back(ctx, h, pack.get(), 16);
    if (h[1] && mode == 0) fail(TQP_ERR_DUPLICATE_BUILD_KEY, "pkfk: duplicate key on the build side");
    if (n_out_host) *n_out_host = h[0];
    if (np > 0 && nb > 0)   // probe keys in; pairs (join) or mask + selection vector (semi) out
        ctx->add_bytes("tqp_pkfk_probe", (double)np * dtype_size(pk.dtype) +
                                         (mode == 0 ? 16.0 * (double)h[0]
                                                    : (match_out ? (double)np : 0.0) + (right_out ? 8.0 * (double)h[0] : 0.0)));
}
}  // namespace

void pkfk_join(tqp_ctx* ctx, tqp_col bk, int64_t nb, tqp_col pk, int64_t np, int64_t* left_out, int64_t* right_out,
               int64_t* n_out_host) {
    check_col(bk, nb, "pkfk build");
    check_col(pk, np, "pkfk probe");
    if (np > 0 && (!left_out || !right_out)) fail(TQP_ERR_INVALID_ARGUMENT, "pkfk: null output");
    if (np >= (int64_t(1) << 40)) fail(TQP_ERR_INVALID_ARGUMENT, "pkfk: probe too large");
    Built B;
    build_side(ctx, bk, nb, B);
    run_probe(ctx, B, pk, np, 0, 0, left_out, right_out, nullptr, n_out_host);
}

void pkfk_semi(tqp_ctx* ctx, tqp_col bk, int64_t nb, tqp_col pk, int64_t np, int anti, uint8_t* match_out,
               int64_t* sel_out, int64_t* n_sel_host) {
    check_col(bk, nb, "semi build");
    check_col(pk, np, "semi probe");
    Built B;
    build_side(ctx, bk, nb, B);
    run_probe(ctx, B, pk, np, 1, anti, nullptr, sel_out, match_out, n_sel_host);
}

}  // namespace tqp
