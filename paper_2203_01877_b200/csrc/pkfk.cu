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
//      -> equality test (the paper's match mask); the matching
//      build row (or a no-match sentinel) is written per probe row as u32 with a
//      per-tile count, an exclusive add-scan gives tile offsets, and an
//      order-preserving compaction pass writes leftOutputIndex = perm[pos],
//      rightOutputIndex = probe row in ascending probe-row order
//      (reading R7). Two passes instead of one with a decoupled look-back: the
//      look-back left a tile's warps idle at the barrier (measured).
//   4. direct output: when every probe row matches (a foreign key always has its
//      primary key: lineitem -> orders), the compacted pairs ARE the per-row pairs, so
//      the probe writes (build row, probe row) straight into the outputs and the u32
//      intermediate, the scan and the compaction pass disappear. A 2,048-row sample
//      probed first (probe_sample_kernel) picks the layout on the device; the one
//      readback (matched rows) tells the host whether a compaction is needed after all.
// Duplicate build keys (adjacent equal sorted keys) -> TQP_ERR_DUPLICATE_BUILD_KEY.
#include "internal.h"
#include <cmath>
#include <cstdlib>

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

// Slot table: 8 u32 per bucket holding its packed records inline (unused entries
// 0xFFFFFFFF), or, for a bucket of more than 8 records, 0x80000000 | its first record
// index. Valid records have the top bit clear (residual + row bits <= 31).
__global__ void fill_slots_kernel(const uint32_t* __restrict__ T, const uint32_t* __restrict__ rec, int64_t nbk,
                                  uint32_t* __restrict__ slots) {
    for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < nbk; b += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t lo = T[b], hi = T[b + 1], cnt = hi - lo;
        uint32_t w[8];
#pragma unroll
        for (int j = 0; j < 8; j++) w[j] = (uint32_t)j < cnt ? rec[lo + j] : 0xFFFFFFFFu;
        if (cnt > 8) w[0] = 0x80000000u | lo;
        uint4* p4 = reinterpret_cast<uint4*>(slots + b * 8);
        p4[0] = make_uint4(w[0], w[1], w[2], w[3]);
        p4[1] = make_uint4(w[4], w[5], w[6], w[7]);
    }
}

// Rank bitmap for a build side already in key order (the sort's identity route: build
// row = sorted position). Over rel = key - base, each aligned 32-byte block holds the
// number of build keys below the block and the next RB_BITS = 224 presence bits, so a
// probe is one sector: hit = the key's bit, build row = rank + popcount of the bits
// below it. 224 domain values per 32 bytes: SF10 order keys (26 bits) -> 9.6 MB.
constexpr uint32_t RB_BITS = 224;

// Each thread takes RBK consecutive sorted keys: bits of the same 32-bit word are OR-ed in a
// register and written with one atomic per word change (sorted keys: TPC-H order keys put
// ~8 keys in a word, so about a quarter of the atomics of one per key); the first key of a
// block writes the block's rank (its sorted position); equal neighbours flag a duplicate.
// Reads the caller's build keys directly (the sort's identity route writes nothing): the
// low 32 bits of the order-preserving key (all varying bits are there, k32).
// keys per thread of rank_bitmap_kernel and its grid (CTAs per SM at most); measured, SF10
// orders: 8 keys / 8 per SM 0.047 ms, 16 / 8 0.079, 4 / 8 0.042, 8 / 32 0.048, 4 / 32 0.039
#ifndef TQP_RBK
#define TQP_RBK 4
#endif
#ifndef TQP_RB_GRID
#define TQP_RB_GRID 32
#endif
constexpr int RBK = TQP_RBK;
// Speculative route (unsorted != null): the caller only knows the first and the last key;
// a key out of order, outside [first, last] or with another high word sets *unsorted and
// the host rebuilds the build side by the sort (the bitmap is then garbage, never used).
__global__ void rank_bitmap_kernel(const void* __restrict__ keys, int dt, int64_t n, uint32_t base, int64_t nblk,
                                   uint32_t* __restrict__ bm, int* __restrict__ dup, int* __restrict__ unsorted,
                                   uint32_t hi32, uint32_t span) {
    const int64_t nth = (n + RBK - 1) / RBK;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < nth; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i0 = t * RBK;
        uint32_t prev = i0 > 0 ? (uint32_t)ordered_u64(load_as_i64(keys, dt, i0 - 1)) - base : 0xFFFFFFFFu;
        uint32_t cw = 0xFFFFFFFFu, cv = 0;   // current word index and its pending bits
        uint64_t uk[RBK];   // this thread's keys (order-preserving): 16-byte loads when whole and aligned
        if (dt == TQP_I64 && RBK % 2 == 0 && i0 + RBK <= n && ((uintptr_t)keys & 15) == 0) {
#pragma unroll
            for (int q = 0; q < RBK / 2; q++) {
                const longlong2 v = __ldg(reinterpret_cast<const longlong2*>((const long long*)keys + i0) + q);
                uk[2 * q] = ordered_u64(v.x);
                uk[2 * q + 1] = ordered_u64(v.y);
            }
        } else if (dt == TQP_I32 && RBK % 4 == 0 && i0 + RBK <= n && ((uintptr_t)keys & 15) == 0) {
#pragma unroll
            for (int q = 0; q < RBK / 4; q++) {
                const int4 v = __ldg(reinterpret_cast<const int4*>((const int*)keys + i0) + q);
                uk[4 * q] = ordered_u64(v.x); uk[4 * q + 1] = ordered_u64(v.y);
                uk[4 * q + 2] = ordered_u64(v.z); uk[4 * q + 3] = ordered_u64(v.w);
            }
        } else {
#pragma unroll
            for (int j = 0; j < RBK; j++) uk[j] = i0 + j < n ? ordered_u64(load_as_i64(keys, dt, i0 + j)) : 0;
        }
#pragma unroll
        for (int j = 0; j < RBK; j++) {
            const int64_t i = i0 + j;
            if (i >= n) break;
            const uint64_t u = uk[j];
            const uint32_t rel = (uint32_t)u - base;
            if (unsorted && ((uint32_t)(u >> 32) != hi32 || rel > span || (i > 0 && rel < prev))) {
                *unsorted = 1;
                return;
            }
            const uint32_t blk = rel / RB_BITS, bit = rel % RB_BITS;
            const uint32_t w = blk * 8 + 1 + (bit >> 5);   // word index (nblk * 8 < 2^32)
            if (w != cw) {
                if (cv) atomicOr(bm + cw, cv);
                cw = w;
                cv = 0;
            }
            cv |= 1u << (bit & 31);
            if (i > 0 && prev == rel) *dup = 1;
            if (i == 0 || prev / RB_BITS != blk) bm[(int64_t)blk * 8] = (uint32_t)i;   // blocks without keys: rank unused
            prev = rel;
        }
        if (cv) atomicOr(bm + cw, cv);
    }
}

// One 256-bit load per lookup (LDG.256, new on sm_100; L1 not allocated: the bitmap
// lives in L2 and random 16-byte pairs made the probe L1-wavefront bound).
#ifndef TQP_RANK_LD256
#define TQP_RANK_LD256 1
#endif
__device__ __forceinline__ bool lookup_rank(const uint4* rb, uint32_t rel, uint32_t& left) {
    const uint32_t blk = rel / RB_BITS, bit = rel % RB_BITS, w = bit >> 5;
#if TQP_RANK_LD256
    uint32_t v[8];
    asm volatile("ld.global.nc.L1::no_allocate.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                 : "l"(rb + 2 * (int64_t)blk));
    uint32_t cnt = v[0], word = v[1];
#pragma unroll
    for (int j = 1; j < 7; j++)
        if (w >= (uint32_t)j) { cnt += __popc(v[j]); word = v[j + 1]; }
    const uint32_t m1 = 1u << (bit & 31);
    if (!(word & m1)) return false;
    left = cnt + __popc(word & (m1 - 1u));
    return true;
#else
    const uint4 q0 = __ldg(rb + 2 * (int64_t)blk);
    const uint32_t words[3] = {q0.y, q0.z, q0.w};
    uint32_t cnt = q0.x, word;
    if (w < 3) {
        word = words[0];
        if (w >= 1) { cnt += __popc(words[0]); word = words[1]; }
        if (w >= 2) { cnt += __popc(words[1]); word = words[2]; }
    } else {
        const uint4 q1 = __ldg(rb + 2 * (int64_t)blk + 1);
        cnt += __popc(words[0]) + __popc(words[1]) + __popc(words[2]);
        const uint32_t hi[4] = {q1.x, q1.y, q1.z, q1.w};
        word = hi[0];
#pragma unroll
        for (int j = 1; j < 4; j++)
            if (w >= 3 + (uint32_t)j) { cnt += __popc(hi[j - 1]); word = hi[j]; }
    }
    const uint32_t m = 1u << (bit & 31);
    if (!(word & m)) return false;
    left = cnt + __popc(word & (m - 1u));
    return true;
#endif
}

struct ProbeArgs {
    const void* probe;
    int64_t n_probe;
    const void* bkeys;        // sorted internal build keys (KT)
    const uint32_t* bperm;    // their source rows
    const uint32_t* T;        // bracket table, 2^B + 1 entries
    const uint32_t* rec;      // packed records (PACKED)
    const uint32_t* slots;    // PACKED, nullable: 8 u32 per bucket (records inline, or a pointer)
    uint32_t lowmask;         // 2^shift - 1
    int pbits;                // bits of the row number in a record
    uint64_t base;            // internal-domain base (= AND of all build keys)
    int vbits;                // (k - base) must be < 2^vbits
    uint64_t hi_bits;         // k32: required high 32 bits of u
    int shift;
    int mode;                 // 0 = join pairs, 1 = semi/anti, 2 = probe-side outer join
    int anti;
    uint32_t* lft;            // join: per probe row, the build row or NOMATCH
    int64_t* left64;          // outer: per probe row, the build row or -1
    uint8_t* mask;            // semi: per probe row, 1 = the key is on the build side
    uint32_t* tcnt;           // per tile: rows selected (join: matches; semi: match != anti)
    uint64_t blo, bhi;        // multi-pass probe: the bucket range this pass resolves
    const uint4* rank_bm;     // nullable: rank bitmap of a presorted build side (RB_BITS bits per 32-byte block)
    int64_t n_build;          // build rows (bounds checks of the checked build)
    const int* unsorted;      // nullable: the speculative build side turned out unsorted -> do nothing
    uint32_t rank_span;       // rank bitmap route: rel must be <= rank_span
    // join mode, direct output: when *direct == 0 (no sampled miss, probe_sample_kernel)
    // the probe writes the final pairs at their probe row -- left = build row (or -1),
    // right = row -- instead of the u32 build row for the compaction pass; exact when every
    // probe row matches (then no compaction runs), else the host compacts afterwards
    const int* direct;        // nullable: never direct; else the sample's miss flag
    unsigned long long* total;   // direct-capable launches: matched rows (one atomic per tile)
    void* out_l;              // int64 (or int32 when idx32) pairs, capacity n_probe
    void* out_r;
    int idx32;
};

// L2 evict-last policy on the slot-table loads: measured no change at SF10
// (probe 0.473 -> 0.477 ms), kept off.
#ifndef TQP_PROBE_EVICT_LAST
#define TQP_PROBE_EVICT_LAST 0
#endif
constexpr bool PROBE_EVICT_LAST = TQP_PROBE_EVICT_LAST;
__device__ __forceinline__ uint64_t l2_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint4 ldg_hint(const uint4* ptr, uint64_t pol) {
    uint4 v;
    asm volatile("ld.global.nc.L2::cache_hint.v4.u32 {%0, %1, %2, %3}, [%4], %5;"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(ptr), "l"(pol));
    return v;
}

// Packed route: the bucket's records [T[b], T[b+1]) from the aligned 32-byte sector(s)
// holding them (a few records), else a lower_bound over the residuals.
__device__ __forceinline__ bool lookup_packed(const ProbeArgs& a, uint32_t rel_low, uint64_t b, uint32_t& left) {
    uint32_t lo = __ldg(a.T + b), hi = __ldg(a.T + b + 1);
    const uint32_t low = rel_low & a.lowmask;
    const uint32_t target = low << a.pbits;
    const uint32_t end = hi;
    const uint32_t s0 = lo & ~7u;   // the bucket's records from the aligned 32-byte sector(s) holding it
    if (hi <= s0 + 16u) {
        const uint4* p4 = reinterpret_cast<const uint4*>(a.rec + s0);
        const uint4 q0 = __ldg(p4), q1 = __ldg(p4 + 1);
        uint4 q2 = make_uint4(0, 0, 0, 0), q3 = q2;
        if (hi > s0 + 8u) { q2 = __ldg(p4 + 2); q3 = __ldg(p4 + 3); }   // second sector only when needed
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

template <int PDT>
__device__ __forceinline__ int64_t load_probe_key(const void* probe, int64_t row) {
    // probe keys are streamed once: evict-first
    if (PDT == TQP_I64) return (int64_t)__ldcs((const long long*)probe + row);
    if (PDT == TQP_I32) return (int64_t)__ldcs((const int*)probe + row);
    return (int64_t)__ldcs((const unsigned char*)probe + row);
}

// The probe key's offset rel = k - base in the internal key domain, if the key can be on
// the build side at all (its high word and its varying-bit span match).
template <typename KT>
__device__ __forceinline__ bool probe_rel(const ProbeArgs& a, int64_t v, KT& rel) {
    const uint64_t u = ordered_u64(v);
    if (sizeof(KT) == 4 && (u & 0xFFFFFFFF00000000ull) != a.hi_bits) return false;
    const KT k = (KT)u;
    rel = (KT)(k - (KT)a.base);
    return k >= (KT)a.base && !(a.vbits < 64 && ((uint64_t)rel >> a.vbits) != 0);
}

__device__ __forceinline__ void ld256(const void* p, uint32_t (&v)[8]) {
    asm volatile("ld.global.nc.L1::no_allocate.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                 : "l"(p));
}

// rank bitmap block (already loaded) -> hit and build row
__device__ __forceinline__ bool rank_eval(const uint32_t (&v)[8], uint32_t rel, uint32_t& left) {
    const uint32_t bit = rel % RB_BITS, w = bit >> 5;
    uint32_t cnt = v[0], word = v[1];
#pragma unroll
    for (int j = 1; j < 7; j++)
        if (w >= (uint32_t)j) { cnt += __popc(v[j]); word = v[j + 1]; }
    const uint32_t m1 = 1u << (bit & 31);
    if (!(word & m1)) return false;
    left = cnt + __popc(word & (m1 - 1u));
    return true;
}

template <typename KT, int PDT, bool PACKED>
__device__ __forceinline__ bool probe_one(const ProbeArgs& a, int64_t row, uint32_t& left) {
    const int64_t v = load_probe_key<PDT>(a.probe, row);
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
    if (sizeof(KT) == 4 && a.rank_bm) return (uint32_t)rel <= a.rank_span && lookup_rank(a.rank_bm, (uint32_t)rel, left);
    uint64_t b = (uint64_t)rel >> a.shift;
    if (PACKED && a.slots) {   // one aligned 32-byte sector: the bucket's records inline
        const uint32_t low = (uint32_t)rel & a.lowmask;
        const uint4* p4 = reinterpret_cast<const uint4*>(a.slots + b * 8);
        uint4 q0, q1;
        if (PROBE_EVICT_LAST) {   // the table stays in L2 while probe keys stream past it
            const uint64_t pol = l2_evict_last();
            q0 = ldg_hint(p4, pol);
            q1 = ldg_hint(p4 + 1, pol);
        } else if (TQP_RANK_LD256) {   // the bucket's sector in one 256-bit load
            asm volatile("ld.global.nc.L1::no_allocate.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                         : "=r"(q0.x), "=r"(q0.y), "=r"(q0.z), "=r"(q0.w), "=r"(q1.x), "=r"(q1.y), "=r"(q1.z),
                           "=r"(q1.w)
                         : "l"(p4));
        } else {
            q0 = __ldg(p4);
            q1 = __ldg(p4 + 1);
        }
        const uint32_t w[8] = {q0.x, q0.y, q0.z, q0.w, q1.x, q1.y, q1.z, q1.w};
        if (!(w[0] >> 31) || w[0] == 0xFFFFFFFFu) {   // else: more than 8 records, w[0] points into rec
            bool hit = false;
#pragma unroll
            for (int j = 0; j < 8; j++) {   // empty entries have the top bit set; residuals are distinct
                if (!(w[j] >> 31) && (w[j] >> a.pbits) == low) {
                    left = w[j] & ((1u << a.pbits) - 1u);
                    hit = true;
                }
            }
            return hit;
        }
    }
    if (PACKED) return lookup_packed(a, (uint32_t)rel, b, left);
    uint32_t lo = __ldg(a.T + b), hi = __ldg(a.T + b + 1);
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

constexpr uint32_t NOMATCH = 0xFFFFFFFFu;   // build rows are < 2^30

// Pass 1: every probe row is looked up (no inter-tile dependency): join mode writes
// the matching build row (or NOMATCH) as u32, semi mode the match byte; each tile
// counts its selected rows.
template <typename KT, int PDT, bool PACKED>
// Blocks per SM forced by the register budget: measured slower at full occupancy (SF10
// probe 0.327 ms at 40 registers / 6 blocks, 0.340 ms at 32 registers / 8 blocks), so off.
#ifndef TQP_PROBE_MINB
#define TQP_PROBE_MINB 0
#endif
__global__ void __launch_bounds__(PNT, TQP_PROBE_MINB) probe_kernel(ProbeArgs a) {
    __shared__ uint32_t s_w[PNW];
    if (a.unsorted && *a.unsorted) return;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t base = (int64_t)blockIdx.x * PTILE;
    const bool direct = a.mode == 0 && a.direct && *a.direct == 0;
    bool m[PIPT];
    uint32_t left[PIPT];
#pragma unroll
    for (int i = 0; i < PIPT; i++) {
        const int64_t row = base + i * PNT + tid;
        m[i] = false;
        left[i] = NOMATCH;
        if (row < a.n_probe) m[i] = probe_one<KT, PDT, PACKED>(a, row, left[i]);
    }
    uint32_t cnt = 0;
#pragma unroll
    for (int i = 0; i < PIPT; i++) {
        const int64_t row = base + i * PNT + tid;
        if (row >= a.n_probe) continue;
        if (direct) {   // final pairs in place (streamed stores, coalesced across the warp)
            if (a.idx32) {
                __stcs((int*)a.out_l + row, m[i] ? (int)left[i] : -1);
                __stcs((int*)a.out_r + row, (int)row);
            } else {
                __stcs((long long*)a.out_l + row, m[i] ? (long long)left[i] : -1ll);
                __stcs((long long*)a.out_r + row, (long long)row);
            }
            cnt += m[i];
        } else if (a.mode == 0) {
            __stcs(a.lft + row, m[i] ? left[i] : NOMATCH);
            cnt += m[i];
        } else if (a.mode == 2) {
            __stcs((long long*)a.left64 + row, m[i] ? (long long)left[i] : -1ll);
            if (a.mask) a.mask[row] = (uint8_t)m[i];
            cnt += m[i];
        } else {
            a.mask[row] = (uint8_t)m[i];
            cnt += m[i] != (a.anti != 0);
        }
    }
    for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    if (lane == 0) s_w[warp] = cnt;
    __syncthreads();
    if (tid == 0) {
        uint32_t t = 0;
        for (int w = 0; w < PNW; w++) t += s_w[w];
        a.tcnt[blockIdx.x] = t;
        if (a.total) atomicAdd(a.total, (unsigned long long)t);
    }
}

// One-sector routes (rank bitmap, slot table), straight-line per route: the PIPT probe
// keys are loaded first (all in flight), then the 32-byte sectors (LDG.256 each) in
// batches of SECTOR_BATCH, then evaluated. Measured at SF10 (probe ms, full / half
// match): the per-row probe_one 0.418 / 0.326; batches of 1 / 2 / 4 sectors at the
// natural register count (3 blocks/SM) 0.437 / 0.441 / 0.476 and 0.298 / 0.335 / 0.428;
// batch 1 at 6 blocks/SM 0.409 / 0.309 (default); batch 2 at 4 blocks 0.417 / 0.310 --
// occupancy counts, not per-thread batching. All of a thread's sectors fetched at once
// with cp.async into shared memory (64 KB per CTA, 3 CTAs/SM) measured 0.417 -> 0.660 ms;
// an L2 evict-last policy on the sector loads left SF10 / SF100 unchanged (0.418 / 5.354
// -> 0.411 / 5.360 ms). What bounds it is the random 32-byte
// sector per probe row on top of the stream: a plain read-8 / write-16 bytes per row
// kernel takes 0.236 ms for the same 60M rows (tools/membench.cu). ROUTE: 0 = rank
// bitmap, 1 = slots. Same outputs as probe_kernel (join direct / u32 build row, semi, outer).
#ifndef TQP_SECTOR_BATCH
#define TQP_SECTOR_BATCH 1
#endif
constexpr int SECTOR_BATCH = TQP_SECTOR_BATCH;
#ifndef TQP_SECTOR_MINB
#define TQP_SECTOR_MINB 6
#endif
template <int PDT, int ROUTE>
__global__ void __launch_bounds__(PNT, TQP_SECTOR_MINB) probe_sector_kernel(ProbeArgs a) {
    __shared__ uint32_t s_w[PNW];
    if (a.unsorted && *a.unsorted) return;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t base = (int64_t)blockIdx.x * PTILE;
    const bool direct = a.mode == 0 && a.direct && *a.direct == 0;
    int64_t v[PIPT];
#pragma unroll
    for (int i = 0; i < PIPT; i++) {
        const int64_t row = base + i * PNT + tid;
        v[i] = row < a.n_probe ? load_probe_key<PDT>(a.probe, row) : 0;
    }
    uint32_t rel[PIPT];
    bool ok[PIPT];
#pragma unroll
    for (int i = 0; i < PIPT; i++) {
        const int64_t row = base + i * PNT + tid;
        uint32_t r = 0;
        ok[i] = row < a.n_probe && probe_rel<uint32_t>(a, v[i], r) && (ROUTE != 0 || r <= a.rank_span);
        rel[i] = r;
    }
    bool m[PIPT];
    uint32_t left[PIPT];
#pragma unroll
    for (int b = 0; b < PIPT; b += SECTOR_BATCH) {   // SECTOR_BATCH sectors in flight per thread
        uint32_t w[SECTOR_BATCH][8];
#pragma unroll
        for (int ii = 0; ii < SECTOR_BATCH; ii++) {
            const int i = b + ii;
            if (ok[i]) {
                const void* p = ROUTE == 0 ? (const void*)(a.rank_bm + 2 * (int64_t)(rel[i] / RB_BITS))
                                           : (const void*)(a.slots + (int64_t)(rel[i] >> a.shift) * 8);
                ld256(p, w[ii]);
            } else {
#pragma unroll
                for (int j = 0; j < 8; j++) w[ii][j] = 0;
            }
        }
#pragma unroll
        for (int ii = 0; ii < SECTOR_BATCH; ii++) {
            const int i = b + ii;
            left[i] = NOMATCH;
            m[i] = false;
            if (!ok[i]) continue;
            if (ROUTE == 0) {
                m[i] = rank_eval(w[ii], rel[i], left[i]);
            } else if (!(w[ii][0] >> 31) || w[ii][0] == 0xFFFFFFFFu) {   // records inline (residuals distinct)
                const uint32_t low = rel[i] & a.lowmask;
#pragma unroll
                for (int j = 0; j < 8; j++)
                    if (!(w[ii][j] >> 31) && (w[ii][j] >> a.pbits) == low) { left[i] = w[ii][j] & ((1u << a.pbits) - 1u); m[i] = true; }
            } else {   // more than 8 records in the bucket: the bracket + record route
                m[i] = lookup_packed(a, rel[i], (uint64_t)(rel[i] >> a.shift), left[i]);
            }
        }
    }
    uint32_t cnt = 0;
#pragma unroll
    for (int i = 0; i < PIPT; i++) {
        const int64_t row = base + i * PNT + tid;
        if (row >= a.n_probe) continue;
        TQP_DCHECK(!m[i] || (int64_t)left[i] < a.n_build);
        if (direct) {
            if (a.idx32) {
                __stcs((int*)a.out_l + row, m[i] ? (int)left[i] : -1);
                __stcs((int*)a.out_r + row, (int)row);
            } else {
                __stcs((long long*)a.out_l + row, m[i] ? (long long)left[i] : -1ll);
                __stcs((long long*)a.out_r + row, (long long)row);
            }
            cnt += m[i];
        } else if (a.mode == 0) {
            __stcs(a.lft + row, m[i] ? left[i] : NOMATCH);
            cnt += m[i];
        } else if (a.mode == 2) {
            __stcs((long long*)a.left64 + row, m[i] ? (long long)left[i] : -1ll);
            if (a.mask) a.mask[row] = (uint8_t)m[i];
            cnt += m[i];
        } else {
            a.mask[row] = (uint8_t)m[i];
            cnt += m[i] != (a.anti != 0);
        }
    }
    for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    if (lane == 0) s_w[warp] = cnt;
    __syncthreads();
    if (tid == 0) {
        uint32_t t = 0;
        for (int w2 = 0; w2 < PNW; w2++) t += s_w[w2];
        a.tcnt[blockIdx.x] = t;
        if (a.total) atomicAdd(a.total, (unsigned long long)t);
    }
}

// Direct-output decision: one CTA looks up PSAMPLE probe rows spread over the column;
// *direct = 1 iff all of them match (the full-match case -- every lineitem row has its
// order -- writes final pairs in the probe pass and skips the compaction). A wrong guess
// (a miss outside the sample) costs a host-side compaction afterwards, never a wrong result.
constexpr int PSAMPLE = 2048;   // one row per thread of PSAMPLE / PNT CTAs
template <typename KT, int PDT, bool PACKED>
__global__ void __launch_bounds__(PNT) probe_sample_kernel(ProbeArgs a, int* miss) {
    const int j = blockIdx.x * PNT + threadIdx.x;
    const int64_t row = (int64_t)(((__int128)j * a.n_probe) / PSAMPLE);
    uint32_t l;
    const bool hit = probe_one<KT, PDT, PACKED>(a, row, l);
    if (!__syncthreads_and(hit) && threadIdx.x == 0) atomicOr(miss, 1);
}

// Misprediction fallback of the direct output: the in-place pairs (left = -1 for a miss)
// back to the per-row u32 build row that emit_kernel compacts.
__global__ void direct_to_lft_kernel(const void* out_l, int idx32, int64_t n, uint32_t* __restrict__ lft) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t l = idx32 ? (int64_t)((const int*)out_l)[i] : ((const long long*)out_l)[i];
        lft[i] = l < 0 ? NOMATCH : (uint32_t)l;
    }
}

// Multi-pass probe (join mode, packed records) for build sides much larger than L2
// (SF100: 150M orders -> 868 MB of bracket table + records). A single pass makes every
// probe row a random HBM access into that structure (measured: 21.8 ms for 600M probes,
// 3.7 TB/s of DRAM reads at ~131 B per probe). Instead the bucket range is split into P
// slices of about one L2's worth of T + records; pass p resolves only the rows whose
// bucket lies in slice p, so its lookups hit L2. The first pass turns each probe key
// into a u32 code (0x80000000 | (key - base); keys outside the build domain resolve to
// NOMATCH at once) stored in `lft`; later passes stream the codes (4 B per row) and
// overwrite resolved rows in place with the build row (top bit clear) or NOMATCH; the
// last pass also counts each tile's matches for the compaction. Needs vbits <= 30.
// Thread t owns rows {t*4 .. t*4+3} and {1024 + t*4 .. +3} of its 2,048-row tile (two
// 16-byte code vectors); the slice test is one subtract + compare per row on the code.
__device__ __forceinline__ int64_t pass_row(int64_t base, int tid, int i) {
    return base + (int64_t)(i >> 2) * (PTILE / 2) + (int64_t)tid * 4 + (i & 3);
}

template <typename KT, int PDT, bool FIRST, bool LAST>
__global__ void __launch_bounds__(PNT) probe_pass_kernel(ProbeArgs a) {
    static_assert(PIPT == 8 && PTILE == 2 * 4 * PNT, "two 4-row vectors per thread");
    __shared__ uint32_t s_w[PNW];
    __shared__ uint32_t s_c[PTILE];
    __shared__ uint16_t s_q[PTILE];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t base = (int64_t)blockIdx.x * PTILE;
    const bool full = base + PTILE <= a.n_probe;
    uint32_t c[PIPT];
    if (FIRST) {
#pragma unroll
        for (int i = 0; i < PIPT; i++) {
            const int64_t row = pass_row(base, tid, i);
            c[i] = NOMATCH;
            if (row >= a.n_probe) continue;
            int64_t v;
            if (PDT == TQP_I64) v = (int64_t)__ldcs((const long long*)a.probe + row);
            else if (PDT == TQP_I32) v = (int64_t)__ldcs((const int*)a.probe + row);
            else v = (int64_t)__ldcs((const unsigned char*)a.probe + row);
            const uint64_t u = ordered_u64(v);
            bool ok = sizeof(KT) == 4 ? (u & 0xFFFFFFFF00000000ull) == a.hi_bits : true;
            const KT k = (KT)u;
            const KT rel = (KT)(k - (KT)a.base);
            ok = ok && k >= (KT)a.base && ((uint64_t)rel >> a.vbits) == 0;
            c[i] = ok ? (0x80000000u | (uint32_t)rel) : NOMATCH;
        }
    } else if (full) {
        const uint4 v0 = __ldcs(reinterpret_cast<const uint4*>(a.lft + pass_row(base, tid, 0)));
        const uint4 v1 = __ldcs(reinterpret_cast<const uint4*>(a.lft + pass_row(base, tid, 4)));
        c[0] = v0.x; c[1] = v0.y; c[2] = v0.z; c[3] = v0.w;
        c[4] = v1.x; c[5] = v1.y; c[6] = v1.z; c[7] = v1.w;
    } else {
#pragma unroll
        for (int i = 0; i < PIPT; i++) {
            const int64_t row = pass_row(base, tid, i);
            c[i] = row < a.n_probe ? __ldcs(a.lft + row) : NOMATCH;
        }
    }
    // codes of this slice: [0x80000000 + (blo << shift), 0x80000000 + (bhi << shift));
    // resolved rows (top bit clear) and NOMATCH fall outside
    const uint32_t clo = 0x80000000u + ((uint32_t)a.blo << a.shift);
    const uint32_t cspan = (uint32_t)(a.bhi - a.blo) << a.shift;
    uint32_t m = 0;
#pragma unroll
    for (int i = 0; i < PIPT; i++) m |= (uint32_t)(c[i] - clo < cspan) << i;
    if (__any_sync(0xffffffffu, m)) {
        // rows in the slice join a per-warp queue (local row indices) and the warp's
        // lanes look them up densely: a few independent L2 lookups per lane instead of
        // PIPT sparse rounds across the whole warp
        uint32_t qn = 0;
#pragma unroll
        for (int i = 0; i < PIPT; i++) {
            const bool in = (m >> i) & 1u;
            const uint32_t li = (uint32_t)((i >> 2) * (PTILE / 2) + tid * 4 + (i & 3));
            if (in) s_c[li] = c[i];
            const uint32_t bal = __ballot_sync(0xffffffffu, in);
            if (in) s_q[warp * 32 * PIPT + qn + __popc(bal & ((1u << lane) - 1u))] = (uint16_t)li;
            qn += __popc(bal);
        }
        __syncwarp();
        for (uint32_t j = lane; j < qn; j += 32) {
            const uint32_t li = s_q[warp * 32 * PIPT + j];
            const uint32_t rel = s_c[li] & 0x7FFFFFFFu;
            uint32_t l = NOMATCH;
            s_c[li] = lookup_packed(a, rel, (uint64_t)(rel >> a.shift), l) ? l : NOMATCH;
        }
        __syncwarp();
#pragma unroll
        for (int i = 0; i < PIPT; i++)
            if ((m >> i) & 1u) c[i] = s_c[(i >> 2) * (PTILE / 2) + tid * 4 + (i & 3)];
    }
    if (full) {
        if (FIRST || (m & 0xFu))
            __stcs(reinterpret_cast<uint4*>(a.lft + pass_row(base, tid, 0)), make_uint4(c[0], c[1], c[2], c[3]));
        if (FIRST || (m >> 4))
            __stcs(reinterpret_cast<uint4*>(a.lft + pass_row(base, tid, 4)), make_uint4(c[4], c[5], c[6], c[7]));
    } else {
#pragma unroll
        for (int i = 0; i < PIPT; i++) {
            const int64_t row = pass_row(base, tid, i);
            if (row < a.n_probe && (FIRST || ((m >> i) & 1u))) __stcs(a.lft + row, c[i]);
        }
    }
    if (!LAST) return;
    uint32_t cnt = 0;
#pragma unroll
    for (int i = 0; i < PIPT; i++) cnt += c[i] != NOMATCH;   // rows past the end hold NOMATCH
    for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    if (lane == 0) s_w[warp] = cnt;
    __syncthreads();
    if (tid == 0) {
        uint32_t t = 0;
        for (int w = 0; w < PNW; w++) t += s_w[w];
        a.tcnt[blockIdx.x] = t;
    }
}

// Payload columns gathered into the join output by the emit pass (SURVEY §8(f) NEXT 2:
// GenerateOutput / createOutput of PAPER.md:89, :333 fused with the compaction).
constexpr int MAXPAY = 8;
struct Payload {
    int idx32;                      // index outputs as int32 (tqp_pkfk_join_i32) instead of int64
    int nb, np;                     // build-side / probe-side payload columns
    const void* bsrc[MAXPAY];
    int bdt[MAXPAY];
    void* bdst[MAXPAY];
    const void* psrc[MAXPAY];
    int pdt[MAXPAY];
    void* pdst[MAXPAY];
};

__device__ __forceinline__ void copy_elem(const void* src, int dt, int64_t from, void* dst, int64_t to) {
    switch (dt) {
        case TQP_U8: static_cast<uint8_t*>(dst)[to] = __ldg(static_cast<const uint8_t*>(src) + from); break;
        case TQP_I32: __stcs(static_cast<int*>(dst) + to, __ldg(static_cast<const int*>(src) + from)); break;
        default: __stcs(static_cast<long long*>(dst) + to, __ldg(static_cast<const long long*>(src) + from));
    }
}

// Pass 2: order-preserving compaction at the scanned tile offsets. Each thread owns
// PIPT consecutive probe rows; ranks by warp scan of per-thread counts + block scan;
// join pairs (leftOutputIndex = build row, rightOutputIndex = probe row)
// or semi/anti rows are staged in shared memory and written coalesced.
template <bool JOIN>
__device__ __forceinline__ void emit_tile(int64_t t, const uint32_t* __restrict__ lft, const uint8_t* __restrict__ mask,
                                          int anti, int64_t np, const uint64_t* __restrict__ toff, int64_t* left_out,
                                          int64_t* right_out, const Payload& pay) {
    __shared__ uint32_t s_w[PNW];
    __shared__ uint32_t s_l[PTILE];
    __shared__ uint16_t s_r[PTILE];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t base = t * PTILE;
    const int64_t excl = (int64_t)toff[t];
    const uint32_t tot = (uint32_t)(toff[t + 1] - toff[t]);
    if (tot == 0) return;
    TQP_DCHECK(tot <= (uint32_t)PTILE && excl + (int64_t)tot <= np);
    const int64_t r0 = base + (int64_t)tid * PIPT;
    const bool full = base + PTILE <= np;
    uint32_t l[PIPT];
    bool sel[PIPT];
    if (JOIN) {
        if (full) {
            const uint4 v0 = __ldcs(reinterpret_cast<const uint4*>(lft + r0));
            const uint4 v1 = __ldcs(reinterpret_cast<const uint4*>(lft + r0) + 1);
            l[0] = v0.x; l[1] = v0.y; l[2] = v0.z; l[3] = v0.w; l[4] = v1.x; l[5] = v1.y; l[6] = v1.z; l[7] = v1.w;
        } else {
#pragma unroll
            for (int i = 0; i < PIPT; i++) l[i] = r0 + i < np ? lft[r0 + i] : NOMATCH;
        }
#pragma unroll
        for (int i = 0; i < PIPT; i++) sel[i] = l[i] != NOMATCH;
    } else {
        uint8_t mb[PIPT];
        if (full && (uintptr_t)mask % 8 == 0) {
            const uint2 v = *reinterpret_cast<const uint2*>(mask + r0);
            memcpy(mb, &v, 8);
        } else {
#pragma unroll
            for (int i = 0; i < PIPT; i++) mb[i] = r0 + i < np ? mask[r0 + i] : (uint8_t)(anti != 0);
        }
#pragma unroll
        for (int i = 0; i < PIPT; i++) sel[i] = (mb[i] != 0) != (anti != 0) && r0 + i < np;
    }
    uint32_t cnt = 0;
#pragma unroll
    for (int i = 0; i < PIPT; i++) cnt += sel[i];
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
    for (int w = 0; w < PNW; w++)
        if (w < warp) lp += s_w[w];
#pragma unroll
    for (int i = 0; i < PIPT; i++) {
        if (!sel[i]) continue;
        if (JOIN) s_l[lp] = l[i];
        s_r[lp] = (uint16_t)(tid * PIPT + i);
        lp++;
    }
    __syncthreads();
    for (uint32_t k = tid; k < tot; k += PNT) {   // streamed (evict-first) coalesced stores
        if (pay.idx32) {
            if (JOIN && left_out) __stcs((int*)left_out + excl + k, (int)s_l[k]);
            if (right_out) __stcs((int*)right_out + excl + k, (int)(base + s_r[k]));
        } else {
            if (JOIN && left_out) __stcs((long long*)left_out + excl + k, (long long)s_l[k]);
            if (right_out) __stcs((long long*)right_out + excl + k, (long long)(base + s_r[k]));
        }
        if (JOIN) {
            for (int c = 0; c < pay.nb; c++) copy_elem(pay.bsrc[c], pay.bdt[c], s_l[k], pay.bdst[c], excl + k);
            for (int c = 0; c < pay.np; c++) copy_elem(pay.psrc[c], pay.pdt[c], base + s_r[k], pay.pdst[c], excl + k);
        }
    }
}

// Persistent over the tiles (grid = resident CTAs): when the probe wrote the pairs
// directly (*direct set), every CTA exits at once instead of ~n/2048 of them.
template <bool JOIN>
__global__ void __launch_bounds__(PNT) emit_kernel(const uint32_t* __restrict__ lft, const uint8_t* __restrict__ mask,
                                                   int anti, int64_t np, const uint64_t* __restrict__ toff,
                                                   int64_t* left_out, int64_t* right_out, Payload pay,
                                                   const int* direct, const int* unsorted) {
    if (direct && *direct == 0) return;
    if (unsorted && *unsorted) return;   // speculative build side not in key order: redone by the caller
    const int64_t tiles = (np + PTILE - 1) / PTILE;
    for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
        emit_tile<JOIN>(t, lft, mask, anti, np, toff, left_out, right_out, pay);
        __syncthreads();   // the staging buffers are reused by the next tile
    }
}

struct Built {
    SortOut so;
    DevBuf<uint32_t> TR;      // bracket table T, then (packed) the records, one allocation
    DevBuf<uint32_t> slots;   // packed: per-bucket slot table (null when it would be much larger)
    uint32_t* T = nullptr;
    uint32_t* rec = nullptr;
    size_t tr_bytes = 0;
    DevBuf<int> dup;
    uint64_t base = 0, hi_bits = 0;
    int shift = 0, vbits = 0, pbits = 0;
    bool packed = false;
    int64_t nb = 0;
    DevBuf<uint32_t> rank_bm;   // presorted build side: rank bitmap (then T / records are unused)
    uint32_t rank_span = 0;     // rank bitmap: keys - base lie in [0, rank_span]
    DevBuf<int> unsorted;       // speculative rank route: set when the build side was not in key order
};

// out[0] / out[1] = the first / last key (order-preserving images); out[2] = 1 if 2,049
// evenly spaced keys (first and last included) are not in order -- a shuffled build side
// never takes the speculative route.
constexpr int SPEC_SAMPLE = 2048;
__global__ void __launch_bounds__(1024) first_last_kernel(const void* keys, int dt, int64_t n, unsigned long long* out) {
    bool bad = false;
    for (int j = threadIdx.x; j < SPEC_SAMPLE; j += blockDim.x) {
        const int64_t a = (int64_t)(((__int128)j * (n - 1)) / SPEC_SAMPLE);
        const int64_t b = (int64_t)(((__int128)(j + 1) * (n - 1)) / SPEC_SAMPLE);
        bad |= ordered_u64(load_as_i64(keys, dt, a)) > ordered_u64(load_as_i64(keys, dt, b));
    }
    bad = __syncthreads_or(bad);
    if (threadIdx.x < 2) out[threadIdx.x] = ordered_u64(load_as_i64(keys, dt, threadIdx.x == 0 ? 0 : n - 1));
    if (threadIdx.x == 0) out[2] = bad ? 1ull : 0ull;
}

// allow_rank = false: never the rank bitmap (its build row = rank + popcount of the
// distinct keys below is only right without duplicate build keys; the outer join, which
// tolerates duplicates, rebuilds without it when the duplicate flag is set).
void build_side(tqp_ctx* ctx, const tqp_col& bk, int64_t nb, Built& B, bool allow_rank = true, bool spec = true) {
    static const bool no_rank = [] {
        const char* e = std::getenv("TQP_PKFK_NO_RANK");
        return e && std::atoi(e) != 0;
    }();
    // Speculative rank route (TQP_PKFK_NO_SPEC=1 disables it): primary-key columns are
    // usually stored in key order, so read only the first and the last key (one 16-byte
    // sync instead of the sort's plan pass over the column), size the rank bitmap by them
    // and build it in one pass that also verifies the order; the probe's single readback
    // carries the verdict and an unsorted build side is redone the ordinary way.
    static const bool no_spec = [] {
        const char* e = std::getenv("TQP_PKFK_NO_SPEC");
        return e && std::atoi(e) != 0;
    }();
    if (spec && allow_rank && !no_rank && !no_spec && nb >= (1 << 16) &&
        (bk.dtype == TQP_I64 || bk.dtype == TQP_I32)) {
        DevBuf<unsigned long long> fl(ctx, 3);
        launch(ctx, "tqp_sort_andor", first_last_kernel, dim3(1), dim3(1024), 0, bk.data, (int)bk.dtype, nb, fl.get());
        uint64_t h[3];
        read_back(ctx, h, fl.get(), 24);
        const uint64_t lo = h[0], hi = h[1];
        if (!h[2] && hi > lo && (lo >> 32) == (hi >> 32)) {
            const uint64_t span = hi - lo;
            const int64_t nblk = (int64_t)((span + RB_BITS) / RB_BITS);
            if (nblk * 32 <= 8 * nb + (int64_t(1) << 20)) {
                B.nb = nb;
                B.so.k32 = true;
                B.so.identity = true;
                B.base = lo & 0xFFFFFFFFull;
                B.hi_bits = lo & 0xFFFFFFFF00000000ull;
                B.vbits = 32;   // the probe's range test is rank_span
                B.rank_span = (uint32_t)span;
                B.dup.alloc(ctx, 1);
                B.dup.zero();
                B.unsorted.alloc(ctx, 1);
                B.unsorted.zero();
                B.rank_bm.alloc(ctx, nblk * 8);
                B.rank_bm.zero();
                const int g = (int)std::min<int64_t>(ceil_div(ceil_div(nb, RBK), 256), (int64_t)ctx->num_sms * TQP_RB_GRID);
                launch(ctx, "tqp_pkfk_rank_bitmap", rank_bitmap_kernel, dim3(g), dim3(256), 0, bk.data, (int)bk.dtype,
                       nb, (uint32_t)B.base, nblk, B.rank_bm.get(), B.dup.get(), B.unsorted.get(),
                       (uint32_t)(lo >> 32), (uint32_t)span);
                ctx->add_bytes("tqp_pkfk_rank_bitmap", (double)dtype_size(bk.dtype) * (double)nb + 32.0 * (double)nblk);
                return;
            }
        }
    }
    B.so.want_internal = true;
    B.so.defer_identity = true;   // a presorted build side may take the rank bitmap straight from the keys
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
    // Build side already in key order (the sort's identity route) over a domain of at most
    // ~8 bytes of bitmap per build row: the rank bitmap replaces T + records (one sector
    // per probe, 9.6 MB at SF10 instead of 64 MB). TQP_PKFK_NO_RANK=1 disables it (A/B).
    if (B.so.identity && B.so.k32 && vbits > 0 && !no_rank && allow_rank) {
        // in key order: the keys span [first, last]; the bitmap covers exactly that range
        // (SF100 orders: 6e8 values -> 86 MB, L2-resident, where 2^vbits values took 153 MB)
        const uint64_t span = B.so.last_u - B.so.first_u;   // < 2^32 (k32)
        const int64_t nblk = (int64_t)((span + RB_BITS) / RB_BITS);
        if (nblk * 32 <= 8 * nb + (int64_t(1) << 20)) {
            B.base = B.so.first_u & 0xFFFFFFFFull;
            B.rank_span = (uint32_t)span;
            B.rank_bm.alloc(ctx, nblk * 8);
            B.rank_bm.zero();
            const int g = (int)std::min<int64_t>(ceil_div(ceil_div(nb, RBK), 256), (int64_t)ctx->num_sms * TQP_RB_GRID);
            launch(ctx, "tqp_pkfk_rank_bitmap", rank_bitmap_kernel, dim3(g), dim3(256), 0, bk.data, (int)bk.dtype, nb,
                   (uint32_t)B.base, nblk, B.rank_bm.get(), B.dup.get(), (int*)nullptr, 0u, 0u);
            ctx->add_bytes("tqp_pkfk_rank_bitmap", (double)dtype_size(bk.dtype) * (double)nb + 32.0 * (double)nblk);
            return;
        }
    }
    if (B.so.identity) sort_materialize_identity(ctx, bk.data, bk.dtype, nb, false, B.so);
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
        // slot table when the top bit is free and it is at most ~2x the records
        if (B.shift + B.pbits <= 31 && nbk * 8 <= 2 * nb + (int64_t(1) << 20) && (nbk >> 27) == 0) {
            B.slots.alloc(ctx, nbk * 8);
            const int gs = (int)std::min<int64_t>(ceil_div(nbk, 256), (int64_t)ctx->num_sms * 8);
            launch(ctx, "tqp_pkfk_records", fill_slots_kernel, dim3(gs), dim3(256), 0, (const uint32_t*)B.T,
                   (const uint32_t*)B.rec, nbk, B.slots.get());
            ctx->add_bytes("tqp_pkfk_records", 4.0 * (double)nb + 32.0 * (double)nbk);
        }
        B.so.keys32.release();
        B.so.keys64.release();
        B.so.perm32.release();
    }
}

// false: the build side taken as sorted was not (speculative rank route) -- nothing the
// probe wrote may be used; the caller rebuilds with spec = false and probes again.
bool run_probe(tqp_ctx* ctx, Built& B, const tqp_col& pk, int64_t np, int mode, int anti, int64_t* left_out,
               int64_t* right_out, uint8_t* match_out, int64_t* n_out_host, const Payload* pay = nullptr) {
    // [0] selected rows, [1] duplicate-build-key flag, [2] direct-output flag: one readback
    DevBuf<int64_t> pack(ctx, 4);   // + [3] the speculative route's unsorted flag
    pack.zero();
    const int64_t nb = B.nb;
    bool direct_capable = false;
    if (np > 0 && nb > 0) {
        const int64_t tiles = ceil_div(np, PTILE);
        DevBuf<uint32_t> tcnt(ctx, tiles);
        DevBuf<uint64_t> toff(ctx, tiles + 1);
        DevBuf<uint32_t> lft;
        DevBuf<uint8_t> tmask;
        if (mode == 0) lft.alloc(ctx, np);
        else if (mode == 1 && !match_out) tmask.alloc(ctx, np);
        ProbeArgs a{};
        a.probe = pk.data;
        a.n_probe = np;
        a.n_build = nb;
        a.unsorted = B.unsorted.get();
        a.bkeys = B.so.k32 ? (const void*)B.so.keys32.get() : (const void*)B.so.keys64.get();
        a.bperm = B.so.perm32.get();
        a.T = B.T;
        a.rec = B.rec;
        a.slots = B.slots.get();
        a.rank_bm = reinterpret_cast<const uint4*>(B.rank_bm.get());
        a.rank_span = B.rank_span;
        a.pbits = B.pbits;
        a.lowmask = B.shift >= 32 ? 0xFFFFFFFFu : ((1u << B.shift) - 1u);
        a.base = B.base;
        a.vbits = B.vbits;
        a.hi_bits = B.hi_bits;
        a.shift = B.shift;
        a.mode = mode;
        a.anti = anti;
        a.lft = lft.get();
        a.left64 = left_out;
        a.mask = match_out ? match_out : tmask.get();
        a.tcnt = tcnt.get();
        auto go = [&](auto kt, auto pk_) {
            using KT = decltype(kt);
            constexpr bool PK = decltype(pk_)::value;
            if constexpr (sizeof(KT) == 4) {
                const int route = a.rank_bm ? 0 : ((PK && a.slots) ? 1 : -1);
                if (route >= 0) {
                    auto gr = [&](auto rc) {
                        constexpr int R = decltype(rc)::value;
                        switch (pk.dtype) {
                            case TQP_I64: launch(ctx, "tqp_pkfk_probe", probe_sector_kernel<TQP_I64, R>, dim3((unsigned)tiles), dim3(PNT), 0, a); break;
                            case TQP_I32: launch(ctx, "tqp_pkfk_probe", probe_sector_kernel<TQP_I32, R>, dim3((unsigned)tiles), dim3(PNT), 0, a); break;
                            default: launch(ctx, "tqp_pkfk_probe", probe_sector_kernel<TQP_U8, R>, dim3((unsigned)tiles), dim3(PNT), 0, a); break;
                        }
                    };
                    if (route == 0) gr(std::integral_constant<int, 0>{}); else gr(std::integral_constant<int, 1>{});
                    return;
                }
            }
            switch (pk.dtype) {
                case TQP_I64: launch(ctx, "tqp_pkfk_probe", probe_kernel<KT, TQP_I64, PK>, dim3((unsigned)tiles), dim3(PNT), 0, a); break;
                case TQP_I32: launch(ctx, "tqp_pkfk_probe", probe_kernel<KT, TQP_I32, PK>, dim3((unsigned)tiles), dim3(PNT), 0, a); break;
                default: launch(ctx, "tqp_pkfk_probe", probe_kernel<KT, TQP_U8, PK>, dim3((unsigned)tiles), dim3(PNT), 0, a); break;
            }
        };
        // slices of about one L2 of T + records (TQP_PROBE_SLICE_MB overrides, for A/B)
        static const double slice_mb = [] {
            const char* e = std::getenv("TQP_PROBE_SLICE_MB");
            return e ? std::atof(e) : 128.0;
        }();
        int passes = 1;
        if (mode == 0 && B.packed && !B.slots.get() && !B.rank_bm.get() && B.vbits <= 30 && np >= nb && slice_mb > 0)
            passes = (int)std::min<double>(64.0, std::ceil((double)B.tr_bytes / (slice_mb * 1048576.0)));
        // direct output: plain index pairs (no payload columns), single-pass probe
        direct_capable = mode == 0 && passes == 1 && left_out && right_out && (!pay || (pay->nb == 0 && pay->np == 0));
        int* dflag = reinterpret_cast<int*>(pack.get() + 2);
        if (direct_capable) {
            a.direct = dflag;
            a.total = reinterpret_cast<unsigned long long*>(pack.get());
            a.out_l = left_out;
            a.out_r = right_out;
            a.idx32 = pay ? pay->idx32 : 0;
            auto gs = [&](auto kt, auto pk_) {
                using KT = decltype(kt);
                constexpr bool PK = decltype(pk_)::value;
                switch (pk.dtype) {
                    case TQP_I64: launch(ctx, "tqp_pkfk_sample", probe_sample_kernel<KT, TQP_I64, PK>, dim3(PSAMPLE / PNT), dim3(PNT), 0, a, dflag); break;
                    case TQP_I32: launch(ctx, "tqp_pkfk_sample", probe_sample_kernel<KT, TQP_I32, PK>, dim3(PSAMPLE / PNT), dim3(PNT), 0, a, dflag); break;
                    default: launch(ctx, "tqp_pkfk_sample", probe_sample_kernel<KT, TQP_U8, PK>, dim3(PSAMPLE / PNT), dim3(PNT), 0, a, dflag); break;
                }
            };
            if (B.so.k32) {
                if (B.packed) gs(uint32_t{}, std::true_type{}); else gs(uint32_t{}, std::false_type{});
            } else {
                if (B.packed) gs(uint64_t{}, std::true_type{}); else gs(uint64_t{}, std::false_type{});
            }
        }
        if (passes > 1) {
            const uint64_t nbk = uint64_t(1) << (B.vbits - B.shift);
            auto gp = [&](auto kt, auto first, auto last) {
                using KT = decltype(kt);
                constexpr bool F = decltype(first)::value, L = decltype(last)::value;
                switch (pk.dtype) {
                    case TQP_I64: launch(ctx, "tqp_pkfk_probe", probe_pass_kernel<KT, TQP_I64, F, L>, dim3((unsigned)tiles), dim3(PNT), 0, a); break;
                    case TQP_I32: launch(ctx, "tqp_pkfk_probe", probe_pass_kernel<KT, TQP_I32, F, L>, dim3((unsigned)tiles), dim3(PNT), 0, a); break;
                    default: launch(ctx, "tqp_pkfk_probe", probe_pass_kernel<KT, TQP_U8, F, L>, dim3((unsigned)tiles), dim3(PNT), 0, a); break;
                }
            };
            for (int p = 0; p < passes; p++) {
                a.blo = nbk * (uint64_t)p / (uint64_t)passes;
                a.bhi = p + 1 == passes ? nbk : nbk * (uint64_t)(p + 1) / (uint64_t)passes;
                const bool first = p == 0, last = p + 1 == passes;
                auto run = [&](auto kt) {
                    if (first) gp(kt, std::true_type{}, std::false_type{});
                    else if (last) gp(kt, std::false_type{}, std::true_type{});
                    else gp(kt, std::false_type{}, std::false_type{});
                };
                if (B.so.k32) run(uint32_t{}); else run(uint64_t{});
            }
        } else if (B.so.k32) {
            if (B.packed) go(uint32_t{}, std::true_type{}); else go(uint32_t{}, std::false_type{});
        } else {
            if (B.packed) go(uint64_t{}, std::true_type{}); else go(uint64_t{}, std::false_type{});
        }
        const int egrid = (int)std::min<int64_t>(tiles, (int64_t)ctx->num_sms * std::max(occupancy(emit_kernel<true>, PNT, 0), 1));
        if (direct_capable) {
            // one readback decides: every row matched in the direct layout -> done (no scan,
            // no compaction); else scan the tile counts and compact (after a mispredicted
            // direct layout, from the in-place pairs)
            int64_t h[4];
            if (B.dup.get()) TQP_CUDA(cudaMemcpyAsync(pack.get() + 1, B.dup.get(), 4, cudaMemcpyDeviceToDevice, ctx->stream));
            if (B.unsorted.get())
                TQP_CUDA(cudaMemcpyAsync(pack.get() + 3, B.unsorted.get(), 4, cudaMemcpyDeviceToDevice, ctx->stream));
            read_back(ctx, h, pack.get(), 32);
            if (h[3]) return false;
            if (h[1]) fail(TQP_ERR_DUPLICATE_BUILD_KEY, "pkfk: duplicate key on the build side");
            const bool direct = (int)h[2] == 0;
            const double ib = a.idx32 ? 4.0 : 8.0;
            if (!direct || h[0] < np) {
                scan_add_u32_to_u64_exclusive(ctx, tcnt.get(), toff.get(), tiles);
                if (direct) {
                    const int g = (int)std::min<int64_t>(ceil_div(np, 256), (int64_t)ctx->num_sms * 8);
                    launch(ctx, "tqp_pkfk_emit", direct_to_lft_kernel, dim3(g), dim3(256), 0, (const void*)left_out,
                           a.idx32, np, lft.get());
                    ctx->add_bytes("tqp_pkfk_emit", (ib + 4.0) * (double)np);
                }
                launch(ctx, "tqp_pkfk_emit", emit_kernel<true>, dim3((unsigned)egrid), dim3(PNT), 0,
                       (const uint32_t*)lft.get(), (const uint8_t*)nullptr, 0, np, (const uint64_t*)toff.get(), left_out,
                       right_out, pay ? *pay : Payload{}, (const int*)nullptr, (const int*)B.unsorted.get());
                ctx->add_bytes("tqp_pkfk_emit", 2.0 * ib * (double)h[0]);
            }
            if (n_out_host) *n_out_host = h[0];
            ctx->add_bytes("tqp_pkfk_probe", (double)np * dtype_size(pk.dtype) + (direct ? 2.0 * ib * (double)np : 0.0));
            return true;
        }
        scan_add_u32_to_u64_exclusive(ctx, tcnt.get(), toff.get(), tiles);
        if (mode == 0)
            launch(ctx, "tqp_pkfk_emit", emit_kernel<true>, dim3((unsigned)egrid), dim3(PNT), 0, (const uint32_t*)lft.get(),
                   (const uint8_t*)nullptr, 0, np, (const uint64_t*)toff.get(), left_out, right_out,
                   pay ? *pay : Payload{}, (const int*)nullptr, (const int*)B.unsorted.get());
        else if (mode == 1 && right_out)
            launch(ctx, "tqp_pkfk_emit", emit_kernel<false>, dim3((unsigned)egrid), dim3(PNT), 0, (const uint32_t*)nullptr,
                   (const uint8_t*)a.mask, anti, np, (const uint64_t*)toff.get(), (int64_t*)nullptr, right_out,
                   Payload{}, (const int*)nullptr, (const int*)B.unsorted.get());
        TQP_CUDA(cudaMemcpyAsync(pack.get(), toff.get() + tiles, 8, cudaMemcpyDeviceToDevice, ctx->stream));
    } else if (np > 0 && mode == 2) {
        // empty build side: no probe row matches
        TQP_CUDA(cudaMemsetAsync(left_out, 0xFF, (size_t)np * 8, ctx->stream));
        if (match_out) TQP_CUDA(cudaMemsetAsync(match_out, 0, np, ctx->stream));
    } else if (np > 0 && mode == 1) {
        // empty build side: nothing matches
        if (match_out) TQP_CUDA(cudaMemsetAsync(match_out, 0, np, ctx->stream));
        if (anti) {
            // every probe row is selected: sel = 0..np-1
            if (right_out) iota_i64(ctx, right_out, np);
            int64_t h = np;
            TQP_CUDA(cudaMemcpyAsync(pack.get(), &h, 8, cudaMemcpyHostToDevice, ctx->stream));
        }
    }
    if (B.dup.get()) TQP_CUDA(cudaMemcpyAsync(pack.get() + 1, B.dup.get(), 4, cudaMemcpyDeviceToDevice, ctx->stream));
    if (B.unsorted.get())
        TQP_CUDA(cudaMemcpyAsync(pack.get() + 3, B.unsorted.get(), 4, cudaMemcpyDeviceToDevice, ctx->stream));
    int64_t h[4];
    read_back(ctx, h, pack.get(), 32);
    if (h[3]) return false;
    if (h[1] && mode == 0) fail(TQP_ERR_DUPLICATE_BUILD_KEY, "pkfk: duplicate key on the build side");
    if (n_out_host) *n_out_host = h[0];
    if (np > 0 && nb > 0) {   // probe keys in; pairs (join) or mask + selection vector (semi) out
        ctx->add_bytes("tqp_pkfk_probe", (double)np * dtype_size(pk.dtype) + (mode != 0 && match_out ? (double)np : 0.0) +
                                             (mode == 2 ? 8.0 * (double)np : 0.0));
        double pb = 0;   // payload: read + write per output row
        for (int c = 0; pay && c < pay->nb; c++) pb += 2.0 * (double)dtype_size(pay->bdt[c]);
        for (int c = 0; pay && c < pay->np; c++) pb += 2.0 * (double)dtype_size(pay->pdt[c]);
        if (mode != 2)
            ctx->add_bytes("tqp_pkfk_emit", mode == 0 ? ((pay && pay->idx32 ? 4.0 : 8.0) * ((left_out ? 1.0 : 0.0) + (right_out ? 1.0 : 0.0)) + pb) * (double)h[0]
                                                    : (right_out ? 8.0 * (double)h[0] : 0.0));
    }
    return true;
}
// Marks the build rows that some pair references (idempotent byte stores).
__global__ void mark_rows_kernel(const int64_t* __restrict__ left, int64_t m, int64_t nb, uint8_t* __restrict__ matched) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = __ldcs((const long long*)left + i);
        TQP_DCHECK(b >= 0 && b < nb);
        matched[b] = 1;
    }
}

// ---------------------------------------------------------- hash-join ablation
// the generic hash join the paper compares against (OmniSciDB's
// hash aggregation / join beat TQP's sort-based operators on Q1 / Q9), as a
// comparison point for the sort-based PK-FK join on the same GPU. Open addressing, a
// power-of-two table of >= 2 n_build slots, linear probing; the row slot is claimed by
// CAS, then the key is written (build and probe are separate launches). The probe
// writes the same per-row u32 build row as the sort-based probe, so the scan and the
// order-preserving emit are shared and the output is identical.
__device__ __forceinline__ uint64_t hmix(uint64_t x) {
    x ^= x >> 33;
    x *= 0xff51afd7ed558ccdull;
    x ^= x >> 33;
    x *= 0xc4ceb9fe1a85ec53ull;
    x ^= x >> 33;
    return x;
}

// one 16-byte slot per entry (key and row in one sector): words {key lo, key hi, row, pad}
__global__ void hash_build_kernel(const void* keys, int dt, int64_t n, uint64_t mask, uint4* slots) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t k = load_as_i64(keys, dt, i);
        uint64_t slot = hmix((uint64_t)k) & mask;
        while (true) {
            uint32_t* row = &slots[slot].z;
            if (atomicCAS(row, NOMATCH, (uint32_t)i) == NOMATCH) {
                slots[slot].x = (uint32_t)k;
                slots[slot].y = (uint32_t)((uint64_t)k >> 32);
                break;
            }
            slot = (slot + 1) & mask;
        }
    }
}

// duplicate build keys: two slots of one probe chain holding the same key
__global__ void hash_dup_kernel(const uint4* slots, uint64_t mask, int64_t size, int* dup) {
    for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < size; s += (int64_t)gridDim.x * blockDim.x) {
        const uint4 e = slots[s];
        if (e.z == NOMATCH) continue;
        uint64_t t = hmix(((uint64_t)e.y << 32) | e.x) & mask;
        while (t != (uint64_t)s) {   // earlier slots of the key's chain
            const uint4 f = slots[t];
            if (f.z != NOMATCH && f.x == e.x && f.y == e.y) { *dup = 1; break; }
            t = (t + 1) & mask;
        }
    }
}

template <int PDT>
__global__ void __launch_bounds__(PNT) hash_probe_kernel(const void* probe, int64_t np, uint64_t mask,
                                                         const uint4* __restrict__ slots, uint32_t* lft,
                                                         uint32_t* tcnt) {
    __shared__ uint32_t s_w[PNW];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t base = (int64_t)blockIdx.x * PTILE;
    uint32_t cnt = 0;
#pragma unroll
    for (int i = 0; i < PIPT; i++) {
        const int64_t row = base + i * PNT + tid;
        if (row >= np) continue;
        int64_t k;
        if (PDT == TQP_I64) k = (int64_t)__ldcs((const long long*)probe + row);
        else if (PDT == TQP_I32) k = (int64_t)__ldcs((const int*)probe + row);
        else k = (int64_t)__ldcs((const unsigned char*)probe + row);
        uint64_t slot = hmix((uint64_t)k) & mask;
        uint32_t left = NOMATCH;
        while (true) {   // one 16-byte load per slot visited
            const uint4 e = __ldg(slots + slot);
            if (e.z == NOMATCH) break;
            if ((((uint64_t)e.y << 32) | e.x) == (uint64_t)k) { left = e.z; break; }
            slot = (slot + 1) & mask;
        }
        __stcs(lft + row, left);
        cnt += left != NOMATCH;
    }
    for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    if (lane == 0) s_w[warp] = cnt;
    __syncthreads();
    if (tid == 0) {
        uint32_t t = 0;
        for (int w = 0; w < PNW; w++) t += s_w[w];
        tcnt[blockIdx.x] = t;
    }
}
}  // namespace

void pkfk_join_hash(tqp_ctx* ctx, tqp_col bk, int64_t nb, tqp_col pk, int64_t np, int64_t* left_out,
                    int64_t* right_out, int64_t* n_out_host) {
    check_col(bk, nb, "hash build");
    check_col(pk, np, "hash probe");
    if (np > 0 && (!left_out || !right_out)) fail(TQP_ERR_INVALID_ARGUMENT, "pkfk_hash: null output");
    if (nb >= (int64_t(1) << 30) || np >= (int64_t(1) << 40)) fail(TQP_ERR_INVALID_ARGUMENT, "pkfk_hash: too large");
    int64_t size = 1;
    while (size < 2 * std::max<int64_t>(nb, 1)) size <<= 1;
    const uint64_t mask = (uint64_t)size - 1;
    DevBuf<uint4> slots(ctx, size);
    DevBuf<int64_t> pack(ctx, 2);   // [0] pairs, [1] duplicate flag
    pack.zero();
    TQP_CUDA(cudaMemsetAsync(slots.get(), 0xFF, (size_t)size * 16, ctx->stream));
    const int g = (int)std::min<int64_t>(ceil_div(std::max<int64_t>(nb, 1), 256), (int64_t)ctx->num_sms * 8);
    if (nb > 0) {
        launch(ctx, "tqp_hash_build", hash_build_kernel, dim3(g), dim3(256), 0, bk.data, bk.dtype, nb, mask, slots.get());
        const int gd = (int)std::min<int64_t>(ceil_div(size, 256), (int64_t)ctx->num_sms * 8);
        launch(ctx, "tqp_hash_build", hash_dup_kernel, dim3(gd), dim3(256), 0, (const uint4*)slots.get(), mask, size,
               (int*)(pack.get() + 1));
        ctx->add_bytes("tqp_hash_build", (double)nb * (dtype_size(bk.dtype) + 16.0) + 16.0 * (double)size);
    }
    if (np > 0) {
        const int64_t tiles = ceil_div(np, PTILE);
        DevBuf<uint32_t> lft(ctx, np), tcnt(ctx, tiles);
        DevBuf<uint64_t> toff(ctx, tiles + 1);
        switch (pk.dtype) {
            case TQP_I64: launch(ctx, "tqp_hash_probe", hash_probe_kernel<TQP_I64>, dim3((unsigned)tiles), dim3(PNT), 0, pk.data, np, mask, (const uint4*)slots.get(), lft.get(), tcnt.get()); break;
            case TQP_I32: launch(ctx, "tqp_hash_probe", hash_probe_kernel<TQP_I32>, dim3((unsigned)tiles), dim3(PNT), 0, pk.data, np, mask, (const uint4*)slots.get(), lft.get(), tcnt.get()); break;
            default: launch(ctx, "tqp_hash_probe", hash_probe_kernel<TQP_U8>, dim3((unsigned)tiles), dim3(PNT), 0, pk.data, np, mask, (const uint4*)slots.get(), lft.get(), tcnt.get()); break;
        }
        scan_add_u32_to_u64_exclusive(ctx, tcnt.get(), toff.get(), tiles);
        const int egrid = (int)std::min<int64_t>(tiles, (int64_t)ctx->num_sms * std::max(occupancy(emit_kernel<true>, PNT, 0), 1));
        launch(ctx, "tqp_pkfk_emit", emit_kernel<true>, dim3((unsigned)egrid), dim3(PNT), 0, (const uint32_t*)lft.get(),
               (const uint8_t*)nullptr, 0, np, (const uint64_t*)toff.get(), left_out, right_out, Payload{},
               (const int*)nullptr, (const int*)nullptr);
        TQP_CUDA(cudaMemcpyAsync(pack.get(), toff.get() + tiles, 8, cudaMemcpyDeviceToDevice, ctx->stream));
        ctx->add_bytes("tqp_hash_probe", (double)np * dtype_size(pk.dtype));
    }
    int64_t h[2];
    read_back(ctx, h, pack.get(), 16);
    if (h[1]) fail(TQP_ERR_DUPLICATE_BUILD_KEY, "pkfk_hash: duplicate key on the build side");
    if (n_out_host) *n_out_host = h[0];
    if (np > 0) ctx->add_bytes("tqp_pkfk_emit", 16.0 * (double)h[0]);
}

void pkfk_join(tqp_ctx* ctx, tqp_col bk, int64_t nb, tqp_col pk, int64_t np, int64_t* left_out, int64_t* right_out,
               int64_t* n_out_host) {
    check_col(bk, nb, "pkfk build");
    check_col(pk, np, "pkfk probe");
    if (np > 0 && (!left_out || !right_out)) fail(TQP_ERR_INVALID_ARGUMENT, "pkfk: null output");
    if (np >= (int64_t(1) << 40)) fail(TQP_ERR_INVALID_ARGUMENT, "pkfk: probe too large");
    Built B;
    build_side(ctx, bk, nb, B);
    if (!run_probe(ctx, B, pk, np, 0, 0, left_out, right_out, nullptr, n_out_host)) {
        B = Built();
        build_side(ctx, bk, nb, B, true, false);
        run_probe(ctx, B, pk, np, 0, 0, left_out, right_out, nullptr, n_out_host);
    }
}

// PK-FK join with payload columns gathered into the output (one row per matching probe
// row, ascending probe row): build_out[c][j] = build_payload[c][left_j],
// probe_out[c][j] = probe_payload[c][right_j]; the index pairs are optional.
void pkfk_join_payload(tqp_ctx* ctx, tqp_col bk, int64_t nb, tqp_col pk, int64_t np, const tqp_col* bp, int n_bp,
                       void* const* bp_out, const tqp_col* pp, int n_pp, void* const* pp_out, int64_t* left_out,
                       int64_t* right_out, int64_t* n_out_host) {
    check_col(bk, nb, "pkfk build");
    check_col(pk, np, "pkfk probe");
    if (n_bp < 0 || n_bp > MAXPAY || n_pp < 0 || n_pp > MAXPAY) fail(TQP_ERR_INVALID_ARGUMENT, "pkfk: at most 8 payload columns per side");
    if (np >= (int64_t(1) << 40)) fail(TQP_ERR_INVALID_ARGUMENT, "pkfk: probe too large");
    Payload pay{};
    pay.nb = n_bp;
    pay.np = n_pp;
    for (int c = 0; c < n_bp; c++) {
        check_col(bp[c], nb, "pkfk build payload");
        if (np > 0 && !bp_out[c]) fail(TQP_ERR_INVALID_ARGUMENT, "pkfk: null payload output");
        pay.bsrc[c] = bp[c].data;
        pay.bdt[c] = bp[c].dtype;
        pay.bdst[c] = bp_out[c];
    }
    for (int c = 0; c < n_pp; c++) {
        check_col(pp[c], np, "pkfk probe payload");
        if (np > 0 && !pp_out[c]) fail(TQP_ERR_INVALID_ARGUMENT, "pkfk: null payload output");
        pay.psrc[c] = pp[c].data;
        pay.pdt[c] = pp[c].dtype;
        pay.pdst[c] = pp_out[c];
    }
    Built B;
    build_side(ctx, bk, nb, B);
    if (!run_probe(ctx, B, pk, np, 0, 0, left_out, right_out, nullptr, n_out_host, &pay)) {
        B = Built();
        build_side(ctx, bk, nb, B, true, false);
        run_probe(ctx, B, pk, np, 0, 0, left_out, right_out, nullptr, n_out_host, &pay);
    }
}

// The paper's output order (reading R7): the probe side sorted
// descending first (Alg. 1 l.3 as written for the PK-FK macro), then the
// sorted keys probed in order, so the pairs come by probe key descending and, among
// equal probe keys, by ascending probe row (the sort is stable). The original probe row
// of each pair is the sort permutation gathered by the emit pass as a payload column.
void pkfk_join_paper_order(tqp_ctx* ctx, tqp_col bk, int64_t nb, tqp_col pk, int64_t np, int64_t* left_out,
                           int64_t* right_out, int64_t* n_out_host) {
    check_col(bk, nb, "pkfk build");
    check_col(pk, np, "pkfk probe");
    if (np > 0 && (!left_out || !right_out)) fail(TQP_ERR_INVALID_ARGUMENT, "pkfk: null output");
    if (np >= (int64_t(1) << 30)) fail(TQP_ERR_INVALID_ARGUMENT, "pkfk_paper_order: probe must be < 2^30 rows");
    if (np == 0 || nb == 0) {
        pkfk_join(ctx, bk, nb, pk, np, left_out, right_out, n_out_host);
        return;
    }
    DevBuf<uint8_t> sorted(ctx, (size_t)np * dtype_size(pk.dtype));
    DevBuf<int64_t> perm(ctx, np);
    SortOut so;
    so.sorted_orig = sorted.get();
    so.perm64 = perm.get();
    radix_sort(ctx, pk.data, pk.dtype, np, true, so);
    tqp_col spk = pk;
    spk.data = sorted.get();
    tqp_col pp{};
    pp.data = perm.get();
    pp.dtype = TQP_I64;
    void* pp_out[1] = {right_out};
    pkfk_join_payload(ctx, bk, nb, spk, np, nullptr, 0, nullptr, &pp, 1, pp_out, left_out, nullptr, n_out_host);
}

// PK-FK join with int32 index outputs (SURVEY §8(f) NEXT 4 variant): half the output
// bytes; both sides must have fewer than 2^31 rows.
void pkfk_join_i32(tqp_ctx* ctx, tqp_col bk, int64_t nb, tqp_col pk, int64_t np, int32_t* left_out, int32_t* right_out,
                   int64_t* n_out_host) {
    check_col(bk, nb, "pkfk build");
    check_col(pk, np, "pkfk probe");
    if (np > 0 && (!left_out || !right_out)) fail(TQP_ERR_INVALID_ARGUMENT, "pkfk: null output");
    if (nb >= (int64_t(1) << 31) || np >= (int64_t(1) << 31))
        fail(TQP_ERR_INVALID_ARGUMENT, "pkfk_i32: row counts must be < 2^31");
    Payload pay{};
    pay.idx32 = 1;
    Built B;
    build_side(ctx, bk, nb, B);
    if (!run_probe(ctx, B, pk, np, 0, 0, reinterpret_cast<int64_t*>(left_out), reinterpret_cast<int64_t*>(right_out),
                   nullptr, n_out_host, &pay)) {
        B = Built();
        build_side(ctx, bk, nb, B, true, false);
        run_probe(ctx, B, pk, np, 0, 0, reinterpret_cast<int64_t*>(left_out), reinterpret_cast<int64_t*>(right_out), nullptr,
                  n_out_host, &pay);
    }
}

void pkfk_semi(tqp_ctx* ctx, tqp_col bk, int64_t nb, tqp_col pk, int64_t np, int anti, uint8_t* match_out,
               int64_t* sel_out, int64_t* n_sel_host) {
    check_col(bk, nb, "semi build");
    check_col(pk, np, "semi probe");
    Built B;
    build_side(ctx, bk, nb, B);
    if (!run_probe(ctx, B, pk, np, 1, anti, nullptr, sel_out, match_out, n_sel_host)) {
        B = Built();
        build_side(ctx, bk, nb, B, true, false);
        run_probe(ctx, B, pk, np, 1, anti, nullptr, sel_out, match_out, n_sel_host);
    }
}

// Probe-side outer join ("outer = inner pairs + unmatched rows
// with a match-flag column"): every probe row in order, left_out[i] = its build row or
// -1; match_out (nullable) = 1 iff matched; *n_match_host (nullable) = matched rows.
void pkfk_outer(tqp_ctx* ctx, tqp_col bk, int64_t nb, tqp_col pk, int64_t np, int64_t* left_out, uint8_t* match_out,
                int64_t* n_match_host) {
    check_col(bk, nb, "outer build");
    check_col(pk, np, "outer probe");
    if (np > 0 && !left_out) fail(TQP_ERR_INVALID_ARGUMENT, "pkfk_outer: null left_out");
    if (np >= (int64_t(1) << 40)) fail(TQP_ERR_INVALID_ARGUMENT, "pkfk_outer: probe too large");
    Built B;
    build_side(ctx, bk, nb, B);
    if (B.rank_bm.get()) {   // a presorted build side with duplicate keys: rank + popcount would be wrong
        int flags[2] = {0, 0};   // duplicate, speculative route found the build side unsorted
        DevBuf<int> f(ctx, 2);
        f.zero();
        TQP_CUDA(cudaMemcpyAsync(f.get(), B.dup.get(), 4, cudaMemcpyDeviceToDevice, ctx->stream));
        if (B.unsorted.get()) TQP_CUDA(cudaMemcpyAsync(f.get() + 1, B.unsorted.get(), 4, cudaMemcpyDeviceToDevice, ctx->stream));
        read_back(ctx, flags, f.get(), 8);
        if (flags[0] || flags[1]) {
            B = Built();
            build_side(ctx, bk, nb, B, false);
        }
    }
    int64_t m = 0;
    run_probe(ctx, B, pk, np, 2, 0, left_out, nullptr, match_out, &m);
    if (n_match_host) *n_match_host = m;
}

// Outer join preserving the build (primary-key) side -- TPC-H Q13's customer LEFT OUTER
// JOIN orders shape (the left outer join TQP found slow; SURVEY.md §8(f)
// NEXT 1): the inner pairs exactly as tqp_pkfk_join returns them (ascending probe row),
// then (b, -1) for every build row b that no probe row matches, ascending b. Capacity of
// both outputs: n_probe + n_build.
void pkfk_outer_build(tqp_ctx* ctx, tqp_col bk, int64_t nb, tqp_col pk, int64_t np, int64_t* left_out,
                      int64_t* right_out, int64_t* n_out_host) {
    check_col(bk, nb, "outer build");
    check_col(pk, np, "outer probe");
    if (nb + np > 0 && (!left_out || !right_out)) fail(TQP_ERR_INVALID_ARGUMENT, "pkfk_outer_build: null output");
    if (np >= (int64_t(1) << 40) || nb >= (int64_t(1) << 32)) fail(TQP_ERR_INVALID_ARGUMENT, "pkfk_outer_build: too large");
    int64_t m = 0;
    pkfk_join(ctx, bk, nb, pk, np, left_out, right_out, &m);
    if (nb == 0) {
        *n_out_host = m;
        return;
    }
    DevBuf<uint8_t> matched(ctx, nb);
    matched.zero();
    if (m > 0) {
        const int g = (int)std::min<int64_t>(ceil_div(m, 256), (int64_t)ctx->num_sms * 8);
        launch(ctx, "tqp_pkfk_outer_mark", mark_rows_kernel, dim3(g), dim3(256), 0, (const int64_t*)left_out, m, nb,
               matched.get());
        ctx->add_bytes("tqp_pkfk_outer_mark", 9.0 * (double)m);
    }
    // unmatched build rows = the selection vector of (matched == 0), appended after the pairs
    tqp_col mc{};
    mc.data = matched.get();
    mc.dtype = TQP_U8;
    tqp_pred pr{};
    pr.col = 0;
    pr.op = TQP_EQ;
    pr.value = 0;
    int64_t u = 0;
    filter_compact(ctx, &mc, 1, nb, &pr, 1, nullptr, left_out + m, &u);
    if (u > 0) TQP_CUDA(cudaMemsetAsync(right_out + m, 0xFF, (size_t)u * 8, ctx->stream));
    *n_out_host = m + u;
}

// The sampled first / last / order check of a key column (first_last_kernel): out[0..2]
// on the device, stream-ordered (the SMJ's speculative presorted left side uses it too).
void sample_first_last(tqp_ctx* ctx, const void* keys, int dt, int64_t n, unsigned long long* out) {
    launch(ctx, "tqp_sort_andor", first_last_kernel, dim3(1), dim3(1024), 0, keys, dt, n, out);
}

}  // namespace tqp
