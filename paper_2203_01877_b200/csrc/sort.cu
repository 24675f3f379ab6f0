// sort.cu -- LSD radix sort with permutation (stable), sm_100a.
//
// Paper: the join sorts its keys (Alg. 1 l.2-3) and the
// aggregation sorts the concatenated group keys with "radix sort" (PAPER.md:256,
// prose :1148). The paper composes torch.sort; here:
//   - one AND/OR pass finds the bits that vary (fused with pass 0's histogram);
//     the digit plan covers only those bits: 8-bit digits over the bytes that
//     vary, or 9-bit digits over the varying span when that takes fewer passes;
//     when every varying bit lies in the low 32 bits the passes carry 32-bit keys
//     (half the traffic);
//   - every digit pass is reduce-then-scan, with no inter-tile waiting:
//       tile_hist   per tile of 4096 (u32) / 3072 (u64) keys: the digit counts
//       scan_tiles  per chunk of 128 tiles: exclusive prefix over tiles, per digit
//       scan_chunks prefix over chunks + global bin bases (one CTA)
//       scatter     persistent, TMA double-buffered input tiles; stable tile
//                   ranking (each key's peers by warp match, per-warp digit
//                   counters claimed with shared atomics in item order, digit slots
//                   bank-swizzled), the tile staged in shared memory in digit order
//                   and written out so consecutive threads write consecutive
//                   addresses.
//     (A decoupled look-back "onesweep" variant was measured at 0.74 ms per
//     60M-key pass on B200: its inclusive-prefix frontier serialises the tiles;
//     see DESIGN.md.)
#include "internal.h"
#include <cstdlib>

namespace tqp {

constexpr int NT = 256;   // threads per CTA in the sort kernels
constexpr int NW = NT / 32;
constexpr int CHUNK = 128;   // tiles per scan chunk (64 / 32 measured slower: 0.083 / 0.118 ms vs 0.071 for the SMJ sort)

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

// Fold one block's AND / OR / "out of order" into the three plan words. Every block of a
// 60M-key input hitting the same L2 sector with atomics serialised the pass (shuffled
// keys: one same-address atomic per warp, 240 us for 60M keys); the words settle after
// a few blocks, so each block reads them first and only issues the atomics that change
// something.
__device__ __forceinline__ void andor_fold(unsigned long long* out, uint64_t a, uint64_t o, bool uns) {
    const volatile unsigned long long* v = out;
    if ((v[0] & a) != v[0]) atomicAnd(&out[0], (unsigned long long)a);
    if ((v[1] | o) != v[1]) atomicOr(&out[1], (unsigned long long)o);
    if (uns && v[2] == 0) atomicOr(&out[2], 1ull);
}

template <int IN>
__global__ void __launch_bounds__(NT) andor_kernel(const void* keys, int64_t n, bool desc,
                                                   unsigned long long* out) {
    uint64_t a = ~0ull, o = 0;
    bool uns = false;   // some adjacent pair out of order (else the stable order is the identity)
    for (int64_t i = blockIdx.x * (int64_t)NT + threadIdx.x; i < n; i += (int64_t)gridDim.x * NT) {
        uint64_t u = load_u<IN>(keys, i, desc);
        a &= u;
        o |= u;
        if (i + 1 < n) uns |= u > load_u<IN>(keys, i + 1, desc);
    }
    uns = __syncthreads_or(uns);
    for (int s = 16; s > 0; s >>= 1) {
        a &= __shfl_xor_sync(0xffffffffu, a, s);
        o |= __shfl_xor_sync(0xffffffffu, o, s);
    }
    __shared__ uint64_t sa[NW], so[NW];
    if ((threadIdx.x & 31) == 0) { sa[threadIdx.x >> 5] = a; so[threadIdx.x >> 5] = o; }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < NW; w++) { a &= sa[w]; o |= so[w]; }
        andor_fold(out, a, o, uns);
    }
}

// AND / OR of the sort-domain keys fused with a speculative first-pass histogram: the
// low 9 bits (digit 0 of the 9-bit plan that dense integer keys take) per tile of 4096
// keys -- exactly what tile_hist_kernel<uint32_t, IN, 16, 9> would compute for pass 0
// at shift 0. The host uses it only when the plan turns out to be that one.
constexpr int H0_IPT = 16, H0_TILE = 256 * H0_IPT, H0_BINS = 512;

// Shared-memory slot of digit d in a per-warp digit array: the low 5 bits (the bank)
// are XORed with a function of the high bits, a bijection on [0, 2^RB). Keys with
// structure in their low bits (TPC-H order keys take 8 of every 32 values, keys that
// are multiples of 2^k) otherwise pile their digits onto a few banks.
__device__ __forceinline__ uint32_t dslot(uint32_t d) { return d ^ (((d >> 5) * 9u) & 31u); }

// Slot of tile rank r in the digit-ordered staging buffer: the low 4 bits XORed with
// bits 5..8, a bijection within each aligned group of 16. Consecutive ranks (the
// write-out) keep distinct banks; ranks 32 apart -- what an already ordered input
// produces, e.g. orders rows in key order, whose digits repeat every 128 rows --
// no longer land on one bank (32-way conflicts on the staging stores otherwise).
__device__ __forceinline__ uint32_t kslot(uint32_t r) { return r ^ ((r >> 5) & 15u); }
// Blocks per SM the register budget must allow: at the default 72 registers only 3 fit
// (37 % occupancy) and the one-tile blocks stalled on their loads (ncu: long scoreboard).
// Measured, 60M shuffled int64 keys: 0.147 ms at 72 registers, 0.128 ms with 4 blocks,
// 0.120 ms with 5 (16 bytes of spills), 6 spills ~250 bytes.
#ifndef TQP_H0_MINB
#define TQP_H0_MINB 5
#endif
template <int IN>
__global__ void __launch_bounds__(NT, TQP_H0_MINB) andor_hist0_kernel(const void* keys, int64_t n, bool desc,
                                                         unsigned long long* out, uint32_t* __restrict__ th0) {
    __shared__ uint32_t h[NW][H0_BINS];
    __shared__ uint64_t sa[NW], so[NW];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int d = lane; d < H0_BINS; d += 32) h[warp][d] = 0;
    __syncwarp();
    const int64_t base = (int64_t)blockIdx.x * H0_TILE;
    uint64_t a = ~0ull, o = 0;
    uint64_t u[H0_IPT];
    bool unsorted;
    if ((IN == IN_I64 || IN == IN_I32) && base + H0_TILE <= n && ((uintptr_t)keys & 15) == 0) {
        // full tile: 16-byte loads (which warp counts a key does not matter for the tile)
        constexpr int PER = IN == IN_I64 ? 2 : 4;   // keys per 16-byte load
        const uint4* p4 = reinterpret_cast<const uint4*>((const uint8_t*)keys + base * (IN == IN_I64 ? 8 : 4)) + tid;
#pragma unroll
        for (int j = 0; j < H0_IPT / PER; j++) {
            const uint4 v = __ldg(p4 + j * NT);
            if (IN == IN_I64) {
                u[2 * j] = ordered_u64((int64_t)(((uint64_t)v.y << 32) | v.x));
                u[2 * j + 1] = ordered_u64((int64_t)(((uint64_t)v.w << 32) | v.z));
            } else {
                u[4 * j] = ordered_u64((int64_t)(int32_t)v.x);
                u[4 * j + 1] = ordered_u64((int64_t)(int32_t)v.y);
                u[4 * j + 2] = ordered_u64((int64_t)(int32_t)v.z);
                u[4 * j + 3] = ordered_u64((int64_t)(int32_t)v.w);
            }
        }
        bool uns = false;
#pragma unroll
        for (int i = 0; i < H0_IPT; i++) {
            if (desc) u[i] = ~u[i];
            a &= u[i];
            o |= u[i];
            atomicAdd(&h[warp][dslot((uint32_t)u[i] & (H0_BINS - 1u))], 1u);
            if (i % PER != PER - 1) {
                uns |= u[i] > u[i + 1];
            } else {   // the key after this vector: the next lane's first (a shuffle), lane 31 loads it
                const uint64_t nxt = __shfl_down_sync(0xffffffffu, u[i + 1 - PER], 1);
                if (lane != 31) {
                    uns |= u[i] > nxt;
                } else {
                    const int64_t nx = base + ((int64_t)(i / PER) * NT + tid + 1) * PER;
                    if (nx < n) uns |= u[i] > load_u<IN>(keys, nx, desc);
                }
            }
        }
        unsorted = uns;
    } else {
#pragma unroll
        for (int i = 0; i < H0_IPT; i++) {
            const int64_t pos = base + warp * 32 * H0_IPT + i * 32 + lane;
            u[i] = pos < n ? load_u<IN>(keys, pos, desc) : 0;
            if (pos < n) { a &= u[i]; o |= u[i]; }
        }
        bool uns = false;
#pragma unroll
        for (int i = 0; i < H0_IPT; i++) {
            const int64_t pos = base + warp * 32 * H0_IPT + i * 32 + lane;
            if (pos < n) atomicAdd(&h[warp][dslot((uint32_t)u[i] & (H0_BINS - 1u))], 1u);
            if (pos + 1 < n) uns |= u[i] > load_u<IN>(keys, pos + 1, desc);
        }
        unsorted = uns;
    }
    unsorted = __syncthreads_or(unsorted);
    for (int sft = 16; sft > 0; sft >>= 1) {
        a &= __shfl_xor_sync(0xffffffffu, a, sft);
        o |= __shfl_xor_sync(0xffffffffu, o, sft);
    }
    if (lane == 0) { sa[warp] = a; so[warp] = o; }
    __syncthreads();
    if (tid == 0) {
        for (int w = 1; w < NW; w++) { a &= sa[w]; o |= so[w]; }
        andor_fold(out, a, o, unsorted);
    }
    for (int d = tid; d < H0_BINS; d += NT) {
        uint32_t c = 0;
#pragma unroll
        for (int w = 0; w < NW; w++) c += h[w][dslot(d)];
        th0[(int64_t)blockIdx.x * H0_BINS + d] = c;
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

template <typename KT, int IN>
__device__ __forceinline__ KT load_key(const void* in_keys, int64_t pos, bool desc) {
    if (IN == IN_INTERNAL) return ((const KT*)in_keys)[pos];
    return (KT)load_u<IN>(in_keys, pos, desc);
}

// (1) per-tile digit counts -> th[tile * BINS + d]
template <typename KT, int IN, int IPT, int RB, int TNT = NT>
__global__ void __launch_bounds__(TNT) tile_hist_kernel(const void* in_keys, int64_t n, int shift, bool desc,
                                                       uint32_t* __restrict__ th) {
    constexpr int TILE = TNT * IPT, BINS = 1 << RB;
    __shared__ uint32_t h[(TNT / 32)][BINS];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int d = lane; d < BINS; d += 32) h[warp][d] = 0;
    __syncwarp();
    const int64_t base = (int64_t)blockIdx.x * TILE;
    KT k[IPT];
    if (IN == IN_INTERNAL && sizeof(KT) == 4 && IPT % 4 == 0 && base + TILE <= n) {
        // full tile of internal u32 keys: 16-byte loads (which warp counts a key does
        // not matter for the tile's histogram)
        const uint4* p4 = reinterpret_cast<const uint4*>((const uint32_t*)in_keys + base) + tid;
#pragma unroll
        for (int j = 0; j < IPT / 4; j++) {
            const uint4 v = __ldg(p4 + j * TNT);
            k[4 * j] = (KT)v.x; k[4 * j + 1] = (KT)v.y; k[4 * j + 2] = (KT)v.z; k[4 * j + 3] = (KT)v.w;
        }
#pragma unroll
        for (int i = 0; i < IPT; i++) atomicAdd(&h[warp][dslot((uint32_t)(k[i] >> shift) & (BINS - 1u))], 1u);
    } else {
#pragma unroll
        for (int i = 0; i < IPT; i++) {
            const int64_t pos = base + warp * 32 * IPT + i * 32 + lane;
            k[i] = pos < n ? load_key<KT, IN>(in_keys, pos, desc) : (KT)0;
        }
#pragma unroll
        for (int i = 0; i < IPT; i++) {
            const int64_t pos = base + warp * 32 * IPT + i * 32 + lane;
            if (pos < n) atomicAdd(&h[warp][dslot((uint32_t)(k[i] >> shift) & (BINS - 1u))], 1u);
        }
    }
    __syncthreads();
    for (int d = tid; d < BINS; d += TNT) {
        uint32_t c = 0;
#pragma unroll
        for (int w = 0; w < (TNT / 32); w++) c += h[w][dslot(d)];
        th[(int64_t)blockIdx.x * BINS + d] = c;
    }
}

// (2) per chunk of CHUNK tiles: th[t][d] <- exclusive prefix within the chunk; ct[c][d] = chunk total.
// Grid (chunk, digit slice of SNT): the CTA stages its [CHUNK tiles x SNT digits] block
// into shared memory with 16-byte cp.async copies (all in flight at once), then one
// thread per digit scans its column and writes the prefixes back (coalesced rows).
constexpr int SNT = 64;
__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gmem_src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(smem_dst)), "l"(gmem_src) : "memory");
}
template <int RB>
__global__ void __launch_bounds__(SNT) scan_tiles_kernel(uint32_t* __restrict__ th, int64_t n_tiles,
                                                         uint32_t* __restrict__ ct) {
    constexpr int BINS = 1 << RB;
    constexpr int V = SNT / 4;   // 16-byte vectors per tile row of the slice
    __shared__ __align__(16) uint32_t blk[CHUNK][SNT];
    const int64_t t0 = (int64_t)blockIdx.x * CHUNK;
    const int cnt = (int)min((int64_t)CHUNK, n_tiles - t0);
    const int d0 = blockIdx.y * SNT;
    for (int q = threadIdx.x; q < cnt * V; q += SNT) {
        const int r = q / V, c = q - r * V;
        cp_async16(&blk[r][c * 4], th + (t0 + r) * BINS + d0 + c * 4);
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();
    const int d = threadIdx.x;
    uint32_t run = 0;
    for (int r = 0; r < cnt; r++) {
        const uint32_t v = blk[r][d];
        th[(t0 + r) * BINS + d0 + d] = run;
        run += v;
    }
    ct[(int64_t)blockIdx.x * BINS + d0 + d] = run;
}

// (3) one CTA of BINS threads (one digit each): ct[c][d] <- global start of digit d
// in chunk c (bin base + earlier chunks)
template <int RB>
__global__ void __launch_bounds__(1 << RB) scan_chunks_kernel(uint32_t* __restrict__ ct, int64_t n_chunks) {
    constexpr int BINS = 1 << RB, NWB = BINS / 32;
    __shared__ uint32_t s_w[NWB];
    const int d = threadIdx.x, lane = d & 31, warp = d >> 5;
    uint32_t run = 0;   // pass 1: digit total over all chunks (32 loads in flight)
    for (int64_t b = 0; b < n_chunks; b += 32) {
        uint32_t v[32];
#pragma unroll
        for (int i = 0; i < 32; i++) v[i] = (b + i < n_chunks) ? ct[(b + i) * BINS + d] : 0u;
#pragma unroll
        for (int i = 0; i < 32; i++) run += v[i];
    }
    // exclusive scan of the digit totals across the block (global bin bases)
    uint32_t x = run;
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) s_w[warp] = x;
    __syncthreads();
    uint32_t base = x - run;
    for (int w = 0; w < warp; w++) base += s_w[w];
    // pass 2: ct[c][d] <- bin base + exclusive prefix over earlier chunks
    for (int64_t b = 0; b < n_chunks; b += 32) {
        uint32_t v[32];
#pragma unroll
        for (int i = 0; i < 32; i++) v[i] = (b + i < n_chunks) ? ct[(b + i) * BINS + d] : 0u;
        asm volatile("" ::: "memory");
#pragma unroll
        for (int i = 0; i < 32; i++) {
            if (b + i < n_chunks) ct[(b + i) * BINS + d] = base;
            base += v[i];
        }
    }
}

struct ScatterArgs {
    const void* in_keys;
    const uint32_t* in_perm;      // IN_INTERNAL only
    void* out_keys;               // internal KT (nullable on the last pass)
    uint32_t* out_perm;           // nullable on the last pass
    void* out_orig;               // last pass: keys in the input dtype
    int orig_dtype;
    int64_t* out_perm64;          // last pass
    uint64_t* out_u;              // last pass: sort-domain values
    const uint32_t* th;           // per histogram tile, per digit: exclusive prefix within the chunk
    const uint32_t* ct;           // per chunk, per digit: global start
    int hr;                       // histogram tiles per scatter tile (th's tile is smaller)
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

// (4') the same stable scatter as a persistent kernel whose input tiles (keys and
// permutation) are streamed into shared memory by TMA bulk copies
// (cp.async.bulk + mbarrier), double-buffered: the stage of tile k is released as
// soon as its keys are in registers, and tile k+2's copy is issued right away, so
// HBM reads overlap ranking and write-out. Tail tile: plain loads.
template <int IN, typename KT>
struct InKey { using T = KT; };
template <typename KT> struct InKey<IN_I64, KT> { using T = long long; };
template <typename KT> struct InKey<IN_I32, KT> { using T = int; };
template <typename KT> struct InKey<IN_U8, KT> { using T = unsigned char; };
template <typename KT> struct InKey<IN_U64, KT> { using T = unsigned long long; };

template <typename KT, int IN>
__device__ __forceinline__ KT conv_key(typename InKey<IN, KT>::T v, bool desc) {
    if (IN == IN_INTERNAL) return (KT)v;
    uint64_t u = IN == IN_U64 ? (uint64_t)v : ordered_u64((int64_t)v);
    return (KT)(desc ? ~u : u);
}

template <typename KT, int IN, int IPT, int RB, int SNT = NT>
struct ScatterWork {
    static constexpr int SNW = SNT / 32;
    union {
        struct {
            uint32_t whist[SNW][1 << RB];
            uint32_t match[SNW][1 << RB];   // per-warp digit -> lane bitmask (peer detection)
        };
        struct {
            KT keys[SNT * IPT];
            uint32_t perm[SNT * IPT];
        } sorted;
    } u;
    uint32_t tstart[1 << RB], gstart[1 << RB], w[SNW];
    uint64_t mbar[2];
};

// The stage carries the keys only; a later pass's permutation is loaded from global
// memory straight into registers (issued before the stage wait, used after ranking),
// which halves the stages and leaves room for 3 CTAs per SM.
constexpr bool PERM_DIRECT = false;   // measured: 3 CTAs/SM with direct loads was slower (1.39 -> 1.50 ms, 60M keys; MIO-bound)

template <typename KT, int IN, int IPT, int SNT = NT>
constexpr int scatter_stage_bytes() {
    return SNT * IPT * (int)sizeof(typename InKey<IN, KT>::T) + (IN == IN_INTERNAL && !PERM_DIRECT ? SNT * IPT * 4 : 0);
}

// (Writing the digit-ordered tile into the tile's own input stage, which saves a barrier
// and refills the stage after the write-out, measured no faster: 1.059 -> 1.064 ms.)
// Input stages per CTA: tile k+2's copy is in flight while tile k is ranked and written.
// (One stage with 3 CTAs/SM was measured slower: 1.34 -> 1.53 ms per 60M-key sort.)
#ifndef TQP_SCATTER_STAGES
#define TQP_SCATTER_STAGES 2
#endif
constexpr int SCATTER_STAGES = TQP_SCATTER_STAGES;

// Peer detection by __match_any_sync (one MATCH.ANY per item) instead of the shared
// match words (atomicOr + read-back + clear): measured slower on B200 (60M-key sort
// scatter 1.27 -> 1.79 ms), kept off.
#ifndef TQP_PEER_MATCH_ANY
#define TQP_PEER_MATCH_ANY 0
#endif
constexpr bool PEER_MATCH_ANY = TQP_PEER_MATCH_ANY;
// Peer detection by RB ballots (one per digit bit; peers = lanes agreeing on every bit)
// and a plain read-modify-write of the warp's digit counter by the peers' leader: no
// shared atomics, no match words to clear. Measured slower (60M u32 keys, 3 passes:
// 1.108 -> 1.331 ms in the SMJ, 1.188 -> 1.415 ms int64 sort), kept off.
#ifndef TQP_PEER_BALLOT
#define TQP_PEER_BALLOT 0
#endif
constexpr bool PEER_BALLOT = TQP_PEER_BALLOT;
// (Half-warp ranking -- each 16-lane half ranks its own 256 consecutive keys with one word
// per (half, digit) holding the peer mask and the half's count, the leader's single store
// replacing the atomic add, the clear and the leader shuffle -- correct but slower:
// 1.062 -> 1.104 ms.)
// (The leader's count update as a plain load + store instead of the shared atomic add --
// it is the only writer of its digit in its warp -- measured slower: 1.065 -> 1.101 ms.)
// (A single 64-bit word per (warp, digit) -- peer mask low, warp digit count high, one
// 64-bit shared atomicOr per key, the leader's plain store replacing the atomic add and
// the clear, no leader shuffle -- measured much slower: 1.059 -> 1.502 ms.)

// L2 hints in the scatter: bit 0 = the TMA input copies evict_first (read once), bit 1 =
// the u32 key/perm output stores evict_last (run ends share sectors with the neighbouring
// tile's runs; a sector evicted half-written costs a DRAM fill and a second write-back).
// Measured off (60M-key sort, 3 passes): 1.205 ms without hints, 1.287 ms with bit 0,
// 1.212 ms with bit 1, 1.29 ms with both -- the extra middle-pass traffic is not an
// eviction-order effect the hints can steer.
#ifndef TQP_SCATTER_HINTS
#define TQP_SCATTER_HINTS 0
#endif

template <typename KT, int IN, int IPT, int RB, int SNT = NT>
constexpr size_t scatter_tma_smem() {
    return SCATTER_STAGES * (size_t)scatter_stage_bytes<KT, IN, IPT, SNT>() + sizeof(ScatterWork<KT, IN, IPT, RB, SNT>);
}

// Tile order of a persistent CTA: grid-stride (tile b + k*grid, default) or contiguous
// (TQP_SCATTER_CONTIG=1: CTA b takes tiles [b*T, (b+1)*T), so the tile after t -- whose
// digit-d run continues exactly where t's ends, sharing a half-written 32-byte sector --
// is written by the same CTA while that sector is still in L2). Measured contiguous
// slower (SMJ's 60M-key sort, 3 scatter passes: 1.15 -> 1.40 ms): with grid-stride the
// CTAs' concurrent writes of a digit land next to each other (tiles t, t+1, ... are in
// flight together), which DRAM serves better than 296 write fronts far apart.
#ifndef TQP_SCATTER_CONTIG
#define TQP_SCATTER_CONTIG 0
#endif
// Thread-block clusters of this many CTAs, held in step by a cluster barrier per tile: the
// CTAs of a cluster hold adjacent tiles (grid-stride order), whose digit runs meet in
// half-written 32-byte sectors; written at the same time, those merge in L2 instead of
// being evicted half-written (DRAM read-modify-write). Measured (3 scatter passes of 60M
// keys, ms): no clusters 1.141 (SMJ) / 1.224 (int64 sort); pairs 1.042 / 1.106; clusters
// of 4 1.605 / 1.751, of 8 1.632 / 1.763 (the barrier waits for the slowest of more CTAs).
#ifndef TQP_SCATTER_CLUSTER
#define TQP_SCATTER_CLUSTER 2
#endif

// Threads per scatter CTA for 9-bit digits on u32 keys: 512 = one CTA per SM ranking
// 8192-key tiles (16 keys per digit run instead of 8: fewer half-written sectors).
// Measured (60M keys, 3 passes; SMJ / int64 sort): 256 threads in cluster pairs 1.083 /
// 1.156 ms, 512 threads 1.058 / 1.113 ms.
#ifndef TQP_SCATTER_NT
#define TQP_SCATTER_NT 512
#endif
constexpr int SCATTER_NT = TQP_SCATTER_NT;
// cluster size of a scatter launch: the 512-thread CTA already holds the adjacent runs the
// clusters pair up (measured 1.083 -> 1.058 ms with clusters off, 1.095 with pairs)
__host__ __device__ constexpr int scatter_cluster(int snt) { return snt > NT ? 1 : TQP_SCATTER_CLUSTER; }
template <typename KT, int IN, int IPT, int RB, int SNT>
#ifndef TQP_SCATTER_MINB
#define TQP_SCATTER_MINB 2
#endif
__global__ void __launch_bounds__(SNT, (SNT > NT ? 1 : IPT <= 8 ? 4 : (PERM_DIRECT && sizeof(KT) == 4 ? 3 : TQP_SCATTER_MINB))) scatter_tma_kernel(ScatterArgs a, int64_t n_tiles, bool use_tma) {
    constexpr int TILE = SNT * IPT, BINS = 1 << RB, BPT = BINS / SNT, SNW = SNT / 32;
    static_assert(BPT >= 1, "one digit per thread at least");
    constexpr int CLS = scatter_cluster(SNT);
    constexpr uint32_t DM = BINS - 1u;
    using KIN = typename InKey<IN, KT>::T;
    constexpr bool HAS_PERM = IN == IN_INTERNAL;
    constexpr int STAGE_BYTES = scatter_stage_bytes<KT, IN, IPT, SNT>();
    extern __shared__ __align__(128) uint8_t smem[];
    constexpr int SST = SCATTER_STAGES;
    auto stage_ptr = [&](int st) { return smem + (size_t)st * STAGE_BYTES; };
    ScatterWork<KT, IN, IPT, RB, SNT>& s = *reinterpret_cast<ScatterWork<KT, IN, IPT, RB, SNT>*>(smem + SST * STAGE_BYTES);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) {
        for (int st = 0; st < SST; st++) mbar_init(&s.mbar[st], 1);
        fence_mbar_init();
    }
    __syncthreads();
    auto full = [&](int64_t t) { return use_tma && (t + 1) * TILE <= a.n; };
    auto issue = [&](int64_t t, int st) {   // thread 0
        uint8_t* dst = stage_ptr(st);
        mbar_expect_tx(&s.mbar[st], (uint32_t)STAGE_BYTES);
        if (TQP_SCATTER_HINTS & 1) {
            const uint64_t pol = policy_evict_first();
            bulk_g2s_hint(dst, (const KIN*)a.in_keys + t * TILE, TILE * (uint32_t)sizeof(KIN), &s.mbar[st], pol);
            if (HAS_PERM && !PERM_DIRECT) bulk_g2s_hint(dst + TILE * sizeof(KIN), a.in_perm + t * TILE, TILE * 4u, &s.mbar[st], pol);
        } else {
            bulk_g2s(dst, (const KIN*)a.in_keys + t * TILE, TILE * (uint32_t)sizeof(KIN), &s.mbar[st]);
            if (HAS_PERM && !PERM_DIRECT) bulk_g2s(dst + TILE * sizeof(KIN), a.in_perm + t * TILE, TILE * 4u, &s.mbar[st]);
        }
    };
    uint32_t par = 0;   // bit st: phase parity of stage st's next wait (a register, not a local array)
    // this CTA's k-th tile and the number of its tiles
    const int64_t per = (n_tiles + gridDim.x - 1) / gridDim.x;
    const int64_t t_begin = TQP_SCATTER_CONTIG ? min((int64_t)blockIdx.x * per, n_tiles) : 0;
    const int64_t t_end = TQP_SCATTER_CONTIG ? min(t_begin + per, n_tiles) : n_tiles;
    auto tile_of = [&](int64_t k) -> int64_t {
        return TQP_SCATTER_CONTIG ? t_begin + k : blockIdx.x + k * gridDim.x;
    };
    for (int st = 0; st < SST; st++) {
        const int64_t t = tile_of(st);
        if (t < t_end && full(t)) {
            if (tid == 0) issue(t, st);
        }
    }
    const unsigned lt = lanemask_lt();
    const uint64_t opol = (TQP_SCATTER_HINTS & 2) ? policy_evict_last() : 0;
    // with clusters every CTA of a cluster runs as many iterations as its first CTA (the one
    // with the most tiles), idling through its own missing ones, so the barriers match
    int64_t kmax = INT64_MAX;
    if (CLS > 1) {
        unsigned rank;
        asm("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
        const int64_t first = (int64_t)blockIdx.x - rank;
        kmax = (n_tiles - first + gridDim.x - 1) / gridDim.x;
    }
    for (int64_t k = 0; k < kmax; k++) {
        const int64_t tile = tile_of(k);
        if (tile >= t_end) {
            if (CLS > 1) {
                asm volatile("barrier.cluster.arrive.relaxed.aligned;\n\tbarrier.cluster.wait.aligned;" ::: "memory");
                continue;
            }
            break;
        }
        const int st = (int)(k % SST);
        const int64_t base = tile * TILE;
        KT key[IPT];
        uint32_t pm[IPT], rk[IPT];
        for (int d = lane * 4; d < BINS; d += 128) {   // 16-byte stores
            *reinterpret_cast<uint4*>(&s.u.whist[warp][d]) = make_uint4(0, 0, 0, 0);
            if (!PEER_BALLOT) *reinterpret_cast<uint4*>(&s.u.match[warp][d]) = make_uint4(0, 0, 0, 0);
        }
        // rows of this tile left from this thread's first slot on (32-bit compares below)
        const int rem = (int)min((int64_t)TILE + 1, a.n - base - (int64_t)(warp * 32 * IPT + lane));
        uint32_t gs[BPT];   // this tile's global digit starts: loaded now, used after ranking
#pragma unroll
        for (int j = 0; j < BPT; j++) {
            const int d = tid + j * SNT;
            gs[j] = __ldg(a.ct + (tile * a.hr / CHUNK) * BINS + d) + __ldg(a.th + tile * a.hr * BINS + d);
        }
        if (full(tile)) {
            if (HAS_PERM && PERM_DIRECT) {
#pragma unroll
                for (int i = 0; i < IPT; i++) pm[i] = __ldcs(a.in_perm + base + warp * 32 * IPT + i * 32 + lane);
            }
            mbar_wait(&s.mbar[st], (par >> st) & 1u);
            par ^= 1u << st;
            const uint8_t* sp = stage_ptr(st);
            const KIN* sk = reinterpret_cast<const KIN*>(sp);
            const uint32_t* spm = reinterpret_cast<const uint32_t*>(sp + TILE * sizeof(KIN));
#pragma unroll
            for (int i = 0; i < IPT; i++) {
                const int q = warp * 32 * IPT + i * 32 + lane;
                key[i] = conv_key<KT, IN>(sk[q], a.desc);
                if (!HAS_PERM) pm[i] = (uint32_t)(base + q);
                else if (!PERM_DIRECT) pm[i] = spm[q];
            }
        } else {
#pragma unroll
            for (int i = 0; i < IPT; i++) {
                const int64_t pos = base + warp * 32 * IPT + i * 32 + lane;
                if (pos < a.n) {
                    key[i] = conv_key<KT, IN>(((const KIN*)a.in_keys)[pos], a.desc);
                    pm[i] = HAS_PERM ? a.in_perm[pos] : (uint32_t)pos;
                } else {
                    key[i] = 0;
                    pm[i] = 0;
                }
            }
        }
        __syncthreads();   // stage st consumed by every thread; whist zeroed
        {
            const int64_t t2 = tile_of(k + SST);
            if (t2 < t_end && full(t2)) {
                if (tid == 0) {
                    fence_proxy_async();
                    issue(t2, st);
                }
            }
        }
        // ranking, specialised for full tiles (every item valid: no per-item guards)
        auto rank_items = [&](auto fullc) {
            constexpr bool FULL = decltype(fullc)::value;
#pragma unroll
            for (int i = 0; i < IPT; i++) {
                const bool valid = FULL || i * 32 < rem;
                const uint32_t d = dslot((uint32_t)(key[i] >> a.shift) & DM);
                // peers = lanes of this warp with the same digit: every lane ORs its bit into
                // the digit's match word, reads the word back, and the leader clears it
                unsigned peers;
                uint32_t* mw = &s.u.match[warp][d];
                if (PEER_BALLOT) {
                    peers = FULL ? 0xffffffffu : __ballot_sync(0xffffffffu, valid);
#pragma unroll
                    for (int b = 0; b < RB; b++) {
                        const bool bit = (d >> b) & 1u;
                        const unsigned bb = __ballot_sync(0xffffffffu, bit);
                        peers &= bit ? bb : ~bb;
                    }
                    if (!valid) peers = 0;
                } else if (PEER_MATCH_ANY) {
                    peers = __match_any_sync(0xffffffffu, valid ? d : 0xFFFFFFFFu);
                    if (!valid) peers = 0;
                } else {
                    if (valid) atomicOr(mw, 1u << lane);
                    __syncwarp();
                    peers = valid ? *reinterpret_cast<volatile uint32_t*>(mw) : 0u;
                    __syncwarp();
                }
                const uint32_t leader = 31 - __clz(peers);
                uint32_t old = 0;
                if (PEER_BALLOT) {
                    if (valid && lane == leader) {
                        old = s.u.whist[warp][d];
                        s.u.whist[warp][d] = old + (uint32_t)__popc(peers);
                    }
                    __syncwarp();
                } else if (valid && lane == leader) {
                    old = atomicAdd(&s.u.whist[warp][d], (uint32_t)__popc(peers));
                    if (!PEER_MATCH_ANY) *mw = 0;
                }
                rk[i] = old | (leader << 16) | ((uint32_t)__popc(peers & lt) << 24);
            }
        };
        if (base + TILE <= a.n) rank_items(std::true_type{});
        else rank_items(std::false_type{});
#pragma unroll
        for (int i = 0; i < IPT; i++) {
            const uint32_t b = __shfl_sync(0xffffffffu, rk[i] & 0xFFFFu, (rk[i] >> 16) & 31u);
            rk[i] = b + (rk[i] >> 24);
        }
        __syncthreads();
        {   // per digit: tile-local digit start + exclusive prefix over warps, folded into
            // whist[w][d] (thread owns BPT digits); gdelta[d] = global - tile digit start
            uint32_t c[BPT][SNW], cnt[BPT], local = 0;
#pragma unroll
            for (int j = 0; j < BPT; j++) {
                const int d = dslot(tid * BPT + j);
                uint32_t run = 0;
#pragma unroll
                for (int w = 0; w < SNW; w++) {
                    c[j][w] = s.u.whist[w][d];
                    run += c[j][w];
                }
                cnt[j] = run;
                local += run;
            }
            uint32_t ex = block_excl_scan256(local, s.w);
#pragma unroll
            for (int j = 0; j < BPT; j++) {
                const int d = tid * BPT + j;
                s.tstart[d] = ex;
                uint32_t run = ex;
#pragma unroll
                for (int w = 0; w < SNW; w++) {
                    s.u.whist[w][dslot(d)] = run;
                    run += c[j][w];
                }
                ex += cnt[j];
            }
        }
        __syncthreads();
#pragma unroll
        for (int i = 0; i < IPT; i++) {
            if (i * 32 < rem) {
                const uint32_t d = dslot((uint32_t)(key[i] >> a.shift) & DM);
                rk[i] = s.u.whist[warp][d] + rk[i];
            }
        }
        __syncthreads();
        // tile staged in digit order; u32 keys as {key, perm} pairs (one 8-byte access each way)
        uint2* kp = reinterpret_cast<uint2*>(&s.u.sorted);
#pragma unroll
        for (int i = 0; i < IPT; i++) {
            if (i * 32 < rem) {
                if (sizeof(KT) == 4) {
                    kp[kslot(rk[i])] = make_uint2((uint32_t)key[i], pm[i]);
                } else {
                    s.u.sorted.keys[kslot(rk[i])] = key[i];
                    s.u.sorted.perm[kslot(rk[i])] = pm[i];
                }
            }
        }
#pragma unroll
        for (int j = 0; j < BPT; j++) s.gstart[tid + j * SNT] = gs[j] - s.tstart[tid + j * SNT];   // global - tile start
        __syncthreads();
        const int tile_n = (int)min((int64_t)TILE, a.n - base);
        if (!a.out_perm64 && !a.out_u && !a.out_orig) {   // intermediate passes / internal outputs
            KT* ok = (KT*)a.out_keys;
            uint32_t* op = a.out_perm;
            if (sizeof(KT) == 4 && ok && op) {
                for (int j = tid; j < tile_n; j += SNT) {
                    const uint2 v = kp[kslot(j)];
                    const uint32_t dst = s.gstart[(v.x >> a.shift) & DM] + (uint32_t)j;
                    TQP_DCHECK((int64_t)dst < a.n);
                    if (TQP_SCATTER_HINTS & 2) {
                        st_hint_u32(reinterpret_cast<uint32_t*>(ok + dst), (uint32_t)v.x, opol);
                        st_hint_u32(op + dst, v.y, opol);
                    } else {
                        ok[dst] = (KT)v.x;
                        op[dst] = v.y;
                    }
                }
            } else {
                for (int j = tid; j < tile_n; j += SNT) {
                    const KT kk = sizeof(KT) == 4 ? (KT)kp[kslot(j)].x : s.u.sorted.keys[kslot(j)];
                    const uint32_t p = sizeof(KT) == 4 ? kp[kslot(j)].y : s.u.sorted.perm[kslot(j)];
                    const uint32_t dst = s.gstart[(uint32_t)(kk >> a.shift) & DM] + (uint32_t)j;
                    TQP_DCHECK((int64_t)dst < a.n);
                    if (ok) ok[dst] = kk;
                    if (op) op[dst] = p;
                }
            }
        } else
        for (int j = tid; j < tile_n; j += SNT) {
            const KT kk = sizeof(KT) == 4 ? (KT)kp[kslot(j)].x : s.u.sorted.keys[kslot(j)];
            const uint32_t p = sizeof(KT) == 4 ? kp[kslot(j)].y : s.u.sorted.perm[kslot(j)];
            const uint32_t d = (uint32_t)(kk >> a.shift) & DM;
            const int64_t dst = (int64_t)(uint32_t)(s.gstart[d] + (uint32_t)j);   // gdelta[d] + j (mod 2^32, n < 2^30)
            TQP_DCHECK(dst < a.n);
            if (a.out_keys) ((KT*)a.out_keys)[dst] = kk;
            if (a.out_perm) a.out_perm[dst] = p;
            if (a.out_perm64) a.out_perm64[dst] = (int64_t)p;
            if (a.out_u || a.out_orig) {
                const uint64_t u = to_u<KT>(kk, a.hi_bits);
                if (a.out_u) a.out_u[dst] = u;
                if (a.out_orig) {
                    const uint64_t v = a.desc ? ~u : u;
                    switch (a.orig_dtype) {
                        case TQP_U8: ((uint8_t*)a.out_orig)[dst] = (uint8_t)unordered_i64(v); break;
                        case TQP_I32: ((int32_t*)a.out_orig)[dst] = (int32_t)unordered_i64(v); break;
                        case TQP_I64: ((int64_t*)a.out_orig)[dst] = unordered_i64(v); break;
                        default: ((uint64_t*)a.out_orig)[dst] = v; break;
                    }
                }
            }
        }
        __syncthreads();   // sorted/whist/gstart reused by the next tile
        if (CLS > 1) {   // the cluster's CTAs (adjacent tiles) stay in step
            asm volatile("barrier.cluster.arrive.relaxed.aligned;\n\tbarrier.cluster.wait.aligned;" ::: "memory");
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
        case IN_INTERNAL: f(std::integral_constant<int, IN_INTERNAL>()); break;
        default: f(std::integral_constant<int, IN_U64>()); break;
    }
}

template <typename KT, int RB>
static void run_passes(tqp_ctx* ctx, const void* keys, int dtype, int64_t n, bool desc, SortOut& o,
                       const int* shifts, int P, uint32_t* th0 = nullptr) {
    constexpr int BINS = 1 << RB;
    constexpr int IPT = sizeof(KT) == 4 ? 16 : 12;   // 4096 / 3072 keys per NT-thread tile
    constexpr int TILE = NT * IPT;
    // the scatter's CTA width and tile; the tile histograms of passes after the first are
    // per scatter tile (the fused pass-0 histogram of sort_andor is per TILE keys)
    constexpr int SNTs = (RB == 9 && sizeof(KT) == 4) ? SCATTER_NT : NT;
    constexpr int HR0 = SNTs / NT;
    const int64_t tiles = ceil_div(n, TILE);
    const int64_t stiles = ceil_div(n, (int64_t)SNTs * IPT);
    const int64_t chunks_max = ceil_div(tiles, CHUNK);
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
    DevBuf<uint32_t> th(ctx, (size_t)stiles * BINS);
    DevBuf<uint32_t> ct(ctx, (size_t)chunks_max * BINS);
    const int mode0 = in_mode(dtype);
    for (int p = 0; p < P; p++) {
        const void* in = p == 0 ? keys : kb[(p - 1) % 2].get();
        const int mode = p == 0 ? mode0 : (int)IN_INTERNAL;
        const double kin = p == 0 ? (double)dtype_size(dtype) : (double)sizeof(KT);
        const bool fused = p == 0 && th0;   // pass 0: histogram fused into the AND/OR pass
        uint32_t* thp = fused ? th0 : th.get();
        const int64_t htiles = fused ? tiles : stiles;
        const int64_t chunks = ceil_div(htiles, CHUNK);
        if (!fused) {
            dispatch_in(mode, [&](auto m) {
                // one CTA of the scatter's width per scatter tile
                launch(ctx, "tqp_sort_tile_hist", tile_hist_kernel<KT, decltype(m)::value, IPT, RB, SNTs>,
                       dim3((unsigned)stiles), dim3(SNTs), 0, in, n, shifts[p], desc, thp);
            });
            ctx->add_bytes("tqp_sort_tile_hist", kin * (double)n + 4.0 * BINS * (double)stiles);
        }
        launch(ctx, "tqp_sort_scan", scan_tiles_kernel<RB>, dim3((unsigned)chunks, BINS / SNT), dim3(SNT), 0, thp,
               htiles, ct.get());
        launch(ctx, "tqp_sort_scan", scan_chunks_kernel<RB>, dim3(1), dim3(BINS), 0, ct.get(), chunks);
        ctx->add_bytes("tqp_sort_scan", 8.0 * BINS * (double)htiles + 12.0 * BINS * (double)chunks);
        ScatterArgs a{};
        a.in_keys = in;
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
        a.th = thp;
        a.ct = ct.get();
        a.hr = fused ? HR0 : 1;
        a.n = n;
        a.shift = shifts[p];
        a.desc = desc;
        a.hi_bits = o.and_bits & 0xFFFFFFFF00000000ull;
        {   // algorithmic bytes of this pass: keys + permutation in, requested outputs out
            const double rd = kin + (p == 0 ? 0.0 : 4.0);
            const double wr = (a.out_keys ? sizeof(KT) : 0) + (a.out_perm ? 4 : 0) +
                              (a.out_orig ? dtype_size(dtype) : 0) + (a.out_perm64 ? 8 : 0) + (a.out_u ? 8 : 0);
            ctx->add_bytes("tqp_sort_scatter", (rd + wr) * (double)n);
        }
        const bool aligned = ((uintptr_t)in % 16 == 0) && (p == 0 || (uintptr_t)a.in_perm % 16 == 0);
        dispatch_in(mode, [&](auto m) {
            constexpr int INM = decltype(m)::value;
            constexpr int SNTc = (RB == 9 && sizeof(KT) == 4) ? SCATTER_NT : NT;
            constexpr size_t smem = scatter_tma_smem<KT, INM, IPT, RB, SNTc>();
            auto* kfn = scatter_tma_kernel<KT, INM, IPT, RB, SNTc>;
            const int occ = occupancy(kfn, SNTc, smem);
            int64_t grid = std::min<int64_t>(stiles, (int64_t)ctx->num_sms * std::max(occ, 1));
            constexpr int CL = scatter_cluster(SNTc);
            if (CL > 1) {   // a whole number of clusters (the kernel needs them)
                grid -= grid % CL;
                if (grid < CL) grid = CL;
            }
            launch_cluster(ctx, "tqp_sort_scatter", kfn, dim3((unsigned)grid), dim3(SNTc), smem, (unsigned)CL, a,
                           stiles, aligned);
        });
    }
    const int fb = (P - 1) % 2;
    if (need_key_final) {
        if constexpr (sizeof(KT) == 4) o.keys32 = std::move(kb[fb]);
        else o.keys64 = std::move(kb[fb]);
    }
    if (need_perm_final) o.perm32 = std::move(pb[fb]);
}

// TQP_SORT_NO_PRESORTED=1 disables the presorted shortcut (A/B and tests of the radix path).
static bool force_radix() {
    static const bool f = [] {
        const char* e = std::getenv("TQP_SORT_NO_PRESORTED");
        return e && std::atoi(e) != 0;
    }();
    return f;
}

template <int IN>
__global__ void first_last_kernel(const void* keys, int64_t n, bool desc, unsigned long long* out) {
    out[threadIdx.x] = load_u<IN>(keys, threadIdx.x == 0 ? 0 : n - 1, desc);
}

void sort_andor(tqp_ctx* ctx, const void* keys, int dtype, int64_t n, bool desc, unsigned long long* ao,
                uint32_t* th0) {
    TQP_CUDA(cudaMemsetAsync(ao, 0xFF, 8, ctx->stream));
    TQP_CUDA(cudaMemsetAsync(ao + 1, 0, 32, ctx->stream));
    if (n <= 0) return;
    const int mode = in_mode(dtype);
    dispatch_in(mode, [&](auto m) {
        if constexpr (decltype(m)::value != IN_INTERNAL)
            launch(ctx, "tqp_sort_andor", first_last_kernel<decltype(m)::value>, dim3(1), dim3(2), 0, keys, n, desc, ao + 3);
    });
    const int grid = (int)std::min<int64_t>(ceil_div(n, NT * 8), (int64_t)ctx->num_sms * 4);
    dispatch_in(mode, [&](auto m) {
        if constexpr (decltype(m)::value != IN_INTERNAL) {
            if (th0)
                launch(ctx, "tqp_sort_andor", andor_hist0_kernel<decltype(m)::value>, dim3((unsigned)ceil_div(n, H0_TILE)),
                       dim3(NT), 0, keys, n, desc, ao, th0);
            else
                launch(ctx, "tqp_sort_andor", andor_kernel<decltype(m)::value>, dim3(grid), dim3(NT), 0, keys, n, desc, ao);
        }
    });
    ctx->add_bytes("tqp_sort_andor", (double)n * dtype_size(dtype) + (th0 ? 2048.0 * (double)ceil_div(n, H0_TILE) : 0.0));
}

size_t sort_hist0_words(int64_t n) { return (size_t)ceil_div(n, H0_TILE) * H0_BINS; }

void sort_materialize_identity(tqp_ctx* ctx, const void* keys, int dtype, int64_t n, bool desc, SortOut& o) {
        const int mode = in_mode(dtype);
        if (o.want_internal || o.want_perm32) o.perm32.alloc(ctx, n);
        if (o.want_internal) {
            if (o.k32) o.keys32.alloc(ctx, n); else o.keys64.alloc(ctx, n);
        }
        const int g = (int)std::min<int64_t>(ceil_div(n, NT), (int64_t)ctx->num_sms * 8);
        ctx->add_bytes("tqp_sort_trivial",
                       (double)n * (dtype_size(dtype) + (o.sorted_orig ? dtype_size(dtype) : 0) + (o.perm64 ? 8 : 0) +
                                    (o.sorted_u ? 8 : 0) + (o.perm32.n ? 4 : 0) + (o.want_internal ? (o.k32 ? 4 : 8) : 0)));
        dispatch_in(mode, [&](auto m) {
            if constexpr (decltype(m)::value != IN_INTERNAL) {
                if (o.k32)
                    launch(ctx, "tqp_sort_trivial", trivial_sort_kernel<uint32_t, decltype(m)::value>, dim3(g),
                           dim3(NT), 0, keys, n, desc, dtype, o.sorted_orig, o.perm64, o.sorted_u, o.keys32.get(),
                           o.perm32.get());
                else
                    launch(ctx, "tqp_sort_trivial", trivial_sort_kernel<uint64_t, decltype(m)::value>, dim3(g),
                           dim3(NT), 0, keys, n, desc, dtype, o.sorted_orig, o.perm64, o.sorted_u, o.keys64.get(),
                           o.perm32.get());
            }
        });
}

void radix_sort(tqp_ctx* ctx, const void* keys, int dtype, int64_t n, bool desc, SortOut& o, const uint64_t* andor,
                uint32_t* th0) {
    if (n < 0 || n >= (int64_t(1) << 30)) fail(TQP_ERR_INVALID_ARGUMENT, "sort: n must be in [0, 2^30)");
    if (n == 0) return;
    const int mode = in_mode(dtype);
    uint64_t h[SORT_PLAN_WORDS];
    DevBuf<uint32_t> th0_own;
    if (andor) {   // the caller launched sort_andor and read the plan back (one sync for several sorts)
        for (int w = 0; w < SORT_PLAN_WORDS; w++) h[w] = andor[w];
    } else {
        DevBuf<unsigned long long> ao(ctx, SORT_PLAN_WORDS);
        if (n >= (1 << 16) && mode != IN_INTERNAL) {   // large sorts: speculative pass-0 histogram
            th0_own.alloc(ctx, sort_hist0_words(n));
            th0 = th0_own.get();
        }
        sort_andor(ctx, keys, dtype, n, desc, ao.get(), th0);
        read_back(ctx, h, ao.get(), 8 * SORT_PLAN_WORDS);
    }
    o.and_bits = h[0];
    o.or_bits = h[1];
    o.first_u = h[3];
    o.last_u = h[4];
    const uint64_t diff = h[0] ^ h[1];
    o.k32 = (diff >> 32) == 0;
    // digit plan: 8-bit digits over the bytes that vary, or 9-bit digits over the
    // varying bit span when that takes fewer passes (e.g. 26-bit order keys: 3 not 4)
    int shifts[8], P = 0, rb = 8;
    for (int b = 0; b < 8; b++)
        if ((diff >> (8 * b)) & 0xFF) shifts[P++] = 8 * b;
    if (diff) {
        const int lo = __builtin_ctzll(diff), hi = 64 - __builtin_clzll(diff);
        const int p9 = (hi - lo + 8) / 9;
        if (p9 < P) {
            rb = 9;
            P = p9;
            for (int p = 0; p < P; p++) shifts[p] = lo + 9 * p;
        }
    }
    o.passes = P;
    // Already in (key, row) order -- every adjacent pair non-decreasing in the sort domain,
    // as TPC-H's orders table is by o_orderkey: the stable order is the identity, and one
    // streaming pass writes the outputs (the digit passes would reproduce the input order).
    if (P > 0 && h[2] == 0 && n >= 2 && mode != IN_INTERNAL && !force_radix()) P = 0;
    if (P == 0) {
        o.identity = true;
        if (o.defer_identity) return;
        sort_materialize_identity(ctx, keys, dtype, n, desc, o);
        return;
    }
    if (o.k32) {
        // the fused histogram is pass 0's when the plan is 9-bit digits from bit 0 on u32 keys
        uint32_t* h0 = (th0 && rb == 9 && shifts[0] == 0) ? th0 : nullptr;
        if (rb == 9) run_passes<uint32_t, 9>(ctx, keys, dtype, n, desc, o, shifts, P, h0);
        else run_passes<uint32_t, 8>(ctx, keys, dtype, n, desc, o, shifts, P);
    } else {
        if (rb == 9) run_passes<uint64_t, 9>(ctx, keys, dtype, n, desc, o, shifts, P);
        else run_passes<uint64_t, 8>(ctx, keys, dtype, n, desc, o, shifts, P);
    }
}

}  // namespace tqp
