// common.cuh -- context, errors, stream-ordered temporaries, instrumented launches,
// and the device helpers shared by every libtqp kernel (sm_100a only).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstring>
#include <map>
#include <mutex>
#include <tuple>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/tqp.h"

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ != 1000)
#error "libtqp is written for sm_100a (B200) only"
#endif

// Checked build (-DTQP_CHECKED=1; compute-sanitizer is not available on the GPU pool):
// device-side bounds checks on the global stores whose index the kernel computes (scatter
// destinations, compaction offsets, expansion positions, partial-record slots); a failed
// check prints the condition and traps, so the test that ran it fails loudly.
#ifndef TQP_CHECKED
#define TQP_CHECKED 0
#endif
#if TQP_CHECKED
#include <cstdio>
#define TQP_DCHECK(c)                                                                          \
    do {                                                                                       \
        if (!(c)) {                                                                            \
            printf("TQP_DCHECK failed %s:%d block %d thread %d: %s\n", __FILE__, __LINE__,     \
                   (int)blockIdx.x, (int)threadIdx.x, #c);                                     \
            __trap();                                                                          \
        }                                                                                      \
    } while (0)
#else
#define TQP_DCHECK(c) \
    do {              \
    } while (0)
#endif

namespace tqp {

struct Error {
    tqp_status status;
    std::string msg;
};

[[noreturn]] inline void fail(tqp_status s, const std::string& m) { throw Error{s, m}; }

#define TQP_CUDA(call)                                                                        \
    do {                                                                                      \
        cudaError_t e_ = (call);                                                              \
        if (e_ != cudaSuccess)                                                                \
            ::tqp::fail(e_ == cudaErrorMemoryAllocation ? TQP_ERR_OUT_OF_MEMORY : TQP_ERR_CUDA, \
                        std::string(#call) + ": " + cudaGetErrorString(e_));                 \
    } while (0)

}  // namespace tqp

struct tqp_ctx {
    int device = 0;
    int num_sms = 148;
    cudaStream_t stream = nullptr;
    // caching device allocator: blocks are reused stream-ordered on `stream`
    // (all libtqp work of a context is on that one stream), never returned
    // until tqp_ctx_destroy / an out-of-memory retry.
    std::multimap<size_t, void*> free_blocks;
    std::unordered_map<void*, size_t> live_blocks;
    size_t cached_bytes = 0;
    // TQP_ALLOC_EXACT=1 (sanitizer runs): every temporary is its own exact-size cudaMalloc,
    // freed (after a stream sync) when released, so memcheck sees out-of-bounds accesses
    // that a cached, rounded-up block would hide
    bool exact_alloc = false;
    // TQP_ALLOC_POISON=1 (tests): every temporary handed out is filled with 0xA5 bytes first,
    // so a kernel that reads a temporary it never wrote sees garbage, not a lucky zero
    bool poison = false;
    static constexpr size_t GUARD = 256;   // exact mode: canary bytes after every temporary
    int64_t guard_violations = 0;          // canaries found overwritten at release
    void* dalloc(size_t bytes);
    void dfree(void* p);
    void trim();
    // device memory under the cache: the caller's allocator (tqp_ctx_set_allocator) or
    // cudaMalloc / cudaFree
    void* (*alloc_fn)(void*, size_t, int, void*) = nullptr;
    void (*free_fn)(void*, void*, int, void*) = nullptr;
    void* alloc_user = nullptr;
    void* raw_alloc(size_t bytes);   // nullptr when out of memory
    void raw_free(void* p);
    std::string err;
    int64_t launches = 0;
    bool profiling = false;
    std::string prof_prefix;   // profile only kernels whose name starts with this (empty: all)
    bool profiled(const char* name) const {
        return profiling && (prof_prefix.empty() || strncmp(name, prof_prefix.c_str(), prof_prefix.size()) == 0);
    }
    struct Pending { const char* name; cudaEvent_t a, b; };
    std::vector<Pending> pending;
    std::vector<cudaEvent_t> free_events;
    struct Stat { double ms = 0; int64_t launches = 0; double bytes = 0; };
    std::map<std::string, Stat> stats;
    // algorithmic (compulsory) bytes per kernel name, accounted on the host at
    // launch time; independent of profiling
    void add_bytes(const char* name, double b) { stats[name].bytes += b; }
    void* pinned = nullptr;   // 4 KB pinned host scratch for scalar readbacks

    cudaEvent_t get_event() {
        if (!free_events.empty()) {
            cudaEvent_t e = free_events.back();
            free_events.pop_back();
            return e;
        }
        cudaEvent_t e;
        TQP_CUDA(cudaEventCreate(&e));
        return e;
    }
    void drain_profile();   // synchronises; folds pending events into stats
};

namespace tqp {

// ------------------------------------------------------------------ memory
// Device temporaries from the context's caching allocator; released back to it
// on destruction (reuse is stream-ordered), so RAII is safe on every error path.
template <typename T>
struct DevBuf {
    tqp_ctx* ctx = nullptr;
    T* p = nullptr;
    size_t n = 0;
    DevBuf() = default;
    DevBuf(tqp_ctx* c, size_t count) { alloc(c, count); }
    void alloc(tqp_ctx* c, size_t count) {
        release();
        ctx = c;
        n = count;
        if (count == 0) return;
        p = static_cast<T*>(c->dalloc(count * sizeof(T)));
    }
    void release() {
        if (p && ctx) ctx->dfree(p);
        p = nullptr;
        n = 0;
    }
    void zero() {
        if (p) TQP_CUDA(cudaMemsetAsync(p, 0, n * sizeof(T), ctx->stream));
    }
    T* get() const { return p; }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    DevBuf(DevBuf&& o) noexcept : ctx(o.ctx), p(o.p), n(o.n) { o.p = nullptr; o.n = 0; }
    DevBuf& operator=(DevBuf&& o) noexcept {
        if (this != &o) { release(); ctx = o.ctx; p = o.p; n = o.n; o.p = nullptr; o.n = 0; }
        return *this;
    }
    ~DevBuf() { release(); }
};

// Read `bytes` from device memory into host memory: one stream synchronisation.
inline void read_back(tqp_ctx* ctx, void* host, const void* dev, size_t bytes) {
    if (bytes > 4096) fail(TQP_ERR_INVALID_ARGUMENT, "read_back too large");
    TQP_CUDA(cudaMemcpyAsync(ctx->pinned, dev, bytes, cudaMemcpyDeviceToHost, ctx->stream));
    TQP_CUDA(cudaStreamSynchronize(ctx->stream));
    memcpy(host, ctx->pinned, bytes);
}

// -------------------------------------------------------------- launching
template <typename... KArgs, typename... Args>
inline void launch(tqp_ctx* ctx, const char* name, void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem,
                   Args... args) {
    if (grid.x == 0 || grid.y == 0 || grid.z == 0) return;
    cudaEvent_t a = nullptr, b = nullptr;
    const bool prof = ctx->profiled(name);
    if (prof) {
        a = ctx->get_event();
        b = ctx->get_event();
        TQP_CUDA(cudaEventRecord(a, ctx->stream));
    }
    k<<<grid, block, smem, ctx->stream>>>(args...);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) fail(TQP_ERR_CUDA, std::string("launch ") + name + ": " + cudaGetErrorString(e));
    ctx->launches++;
    if (prof) {
        TQP_CUDA(cudaEventRecord(b, ctx->stream));
        ctx->pending.push_back({name, a, b});
    }
}

// The same launch as a thread-block cluster of `cluster` CTAs along x (grid.x a multiple).
template <typename... KArgs, typename... Args>
inline void launch_cluster(tqp_ctx* ctx, const char* name, void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem,
                           unsigned cluster, Args... args) {
    if (cluster <= 1) {
        launch(ctx, name, k, grid, block, smem, args...);
        return;
    }
    if (grid.x == 0 || grid.y == 0 || grid.z == 0) return;
    cudaEvent_t a = nullptr, b = nullptr;
    const bool prof = ctx->profiled(name);
    if (prof) {
        a = ctx->get_event();
        b = ctx->get_event();
        TQP_CUDA(cudaEventRecord(a, ctx->stream));
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = ctx->stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = cluster;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, k, static_cast<KArgs>(args)...);
    if (e == cudaSuccess) e = cudaGetLastError();
    if (e != cudaSuccess) fail(TQP_ERR_CUDA, std::string("launch ") + name + ": " + cudaGetErrorString(e));
    ctx->launches++;
    if (prof) {
        TQP_CUDA(cudaEventRecord(b, ctx->stream));
        ctx->pending.push_back({name, a, b});
    }
}

// Dynamic shared-memory limit and occupancy per (kernel, block size, bytes), cached: the
// runtime queries cost host time while the GPU waits right after a readback.
inline std::mutex& kcache_mutex() {
    static std::mutex m;
    return m;
}
template <typename K>
inline void set_smem(K* k, size_t bytes) {
    static std::map<std::pair<const void*, int>, size_t> done;   // (kernel, device) -> limit set
    int dev = 0;
    TQP_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> g(kcache_mutex());
    size_t& cur = done[{(const void*)k, dev}];
    if (bytes <= cur) return;
    TQP_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
    cur = bytes;
}
template <typename K>
inline int occupancy(K* k, int nt, size_t smem) {
    static std::map<std::tuple<const void*, int, int, size_t>, int> cache;
    int dev = 0;
    TQP_CUDA(cudaGetDevice(&dev));
    {
        std::lock_guard<std::mutex> g(kcache_mutex());
        auto it = cache.find({(const void*)k, dev, nt, smem});
        if (it != cache.end()) return it->second;
    }
    set_smem(k, smem);
    int occ = 0;
    TQP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, nt, smem));
    std::lock_guard<std::mutex> g(kcache_mutex());
    cache[{(const void*)k, dev, nt, smem}] = occ;
    return occ;
}

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// ------------------------------------------------------------ key helpers
// Order-preserving map of a signed value to unsigned (sign-bit flip).
__host__ __device__ inline uint64_t ordered_u64(int64_t k) { return (uint64_t)k ^ 0x8000000000000000ull; }
__host__ __device__ inline int64_t unordered_i64(uint64_t u) { return (int64_t)(u ^ 0x8000000000000000ull); }

// Internal dtype code for unsigned 64-bit packed keys (not part of the ABI).
constexpr int DT_U64 = 100;

__device__ __forceinline__ int64_t load_as_i64(const void* p, int dtype, int64_t i) {
    switch (dtype) {
        case TQP_U8: return (int64_t)__ldg((const uint8_t*)p + i);
        case TQP_I32: return (int64_t)__ldg((const int32_t*)p + i);
        default: return (int64_t)__ldg((const long long*)p + i);
    }
}

inline size_t dtype_size(int dt) {
    switch (dt) {
        case TQP_U8: return 1;
        case TQP_I32: return 4;
        case TQP_I64: return 8;
        case DT_U64: return 8;
        case TQP_F64: return 8;
    }
    return 0;
}
inline void check_col(const tqp_col& c, int64_t n, const char* what) {
    if (n < 0) fail(TQP_ERR_INVALID_ARGUMENT, std::string(what) + ": negative length");
    if (c.dtype != TQP_U8 && c.dtype != TQP_I32 && c.dtype != TQP_I64)
        fail(TQP_ERR_INVALID_ARGUMENT, std::string(what) + ": unsupported dtype");
    if (n > 0 && c.data == nullptr) fail(TQP_ERR_INVALID_ARGUMENT, std::string(what) + ": null data");
}

// ------------------------------------------------- predicate conjunctions
// The filter of PAPER.md:829 is an AND of column-vs-constant comparisons. The host
// folds the conjunction into one closed interval per column (lo <= x <= hi, the
// intersection of the <, <=, >, >=, == bounds, clamped to the column's dtype) and
// keeps each != as a negated point interval. A row passes a term iff
// ((x - lo) mod 2^b <= (hi - lo) mod 2^b) != neg, b = 32 for u8/i32 columns and 64 for
// i64: one subtract + one unsigned compare per term and row. Same truth value as the
// predicates taken one by one; never reorders or drops a row.
struct Term {
    int col;          // column index (caller's numbering)
    int dt;           // column dtype
    int neg;          // 1: the row passes iff x is outside [lo, hi]
    uint64_t lo;      // interval start (two's complement bits; 32-bit terms use the low half)
    uint64_t width;   // hi - lo (mod 2^64)
};
struct TermSet {
    int n = 0;
    bool never = false;   // the conjunction is unsatisfiable: no row passes
    Term t[TQP_MAX_PREDS];
};

inline void dtype_domain(int dt, int64_t& lo, int64_t& hi) {
    if (dt == TQP_U8) { lo = 0; hi = 255; }
    else if (dt == TQP_I32) { lo = INT32_MIN; hi = INT32_MAX; }
    else { lo = INT64_MIN; hi = INT64_MAX; }
}

// col_dt(c) gives the dtype of column c; predicates are validated by the caller.
template <typename DtOf>
inline TermSet make_terms(const tqp_pred* preds, int n_preds, DtOf col_dt) {
    TermSet s;
    for (int q = 0; q < n_preds; q++) {   // one range term per distinct column, first-use order
        if (preds[q].op == TQP_NE) continue;
        const int c = preds[q].col;
        bool seen = false;
        for (int r = 0; r < q; r++) seen = seen || (preds[r].op != TQP_NE && preds[r].col == c);
        if (seen) continue;
        const int dt = col_dt(c);
        int64_t dlo, dhi;
        dtype_domain(dt, dlo, dhi);
        int64_t lo = dlo, hi = dhi;
        bool empty = false;
        for (int r = q; r < n_preds; r++) {
            if (preds[r].col != c || preds[r].op == TQP_NE) continue;
            const int64_t v = preds[r].value;
            switch (preds[r].op) {
                case TQP_LT: if (v == INT64_MIN) empty = true; else hi = std::min(hi, v - 1); break;
                case TQP_LE: hi = std::min(hi, v); break;
                case TQP_GT: if (v == INT64_MAX) empty = true; else lo = std::max(lo, v + 1); break;
                case TQP_GE: lo = std::max(lo, v); break;
                default: lo = std::max(lo, v); hi = std::min(hi, v); break;   // TQP_EQ
            }
        }
        if (empty || lo > hi) { s.never = true; s.n = 0; return s; }
        if (lo == dlo && hi == dhi) continue;   // the whole domain: always true
        s.t[s.n++] = Term{c, dt, 0, (uint64_t)lo, (uint64_t)hi - (uint64_t)lo};
    }
    for (int q = 0; q < n_preds; q++) {
        if (preds[q].op != TQP_NE) continue;
        const int dt = col_dt(preds[q].col);
        int64_t dlo, dhi;
        dtype_domain(dt, dlo, dhi);
        const int64_t v = preds[q].value;
        if (v < dlo || v > dhi) continue;        // no value of the column equals v: always true
        s.t[s.n++] = Term{preds[q].col, dt, 1, (uint64_t)v, 0};
    }
    return s;
}

__device__ __forceinline__ bool term32(uint32_t x, uint32_t lo, uint32_t width, bool neg) {
    return (x - lo <= width) != neg;
}
__device__ __forceinline__ bool term64(uint64_t x, uint64_t lo, uint64_t width, bool neg) {
    return (x - lo <= width) != neg;
}

// --------------------------------------------------- decoupled look-back
// Single-pass chained scan across tiles (Merrill & Garland's decoupled
// look-back). Status word: bits [63:62] flag (0 = not ready, 1 = tile aggregate,
// 2 = inclusive prefix), bits [61:0] value. Value and flag live in one aligned
// 64-bit word, so relaxed gpu-scope loads/stores are sufficient.
constexpr uint64_t LB_AGG = 1ull << 62;
constexpr uint64_t LB_PRE = 2ull << 62;
constexpr uint64_t LB_VAL = (1ull << 62) - 1;

__device__ __forceinline__ void lb_store(uint64_t* p, uint64_t v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t lb_load(const uint64_t* p) {
    uint64_t v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

// Called by ALL lanes of ONE warp. Publishes `agg` for `tile` and returns the
// exclusive prefix (sum of all earlier tiles' aggregates) in every lane.
// Dynamic tile ids (taken in launch order) guarantee forward progress.
template <typename Op>
__device__ __forceinline__ uint64_t lookback_warp(uint64_t* status, int64_t tile, uint64_t agg, Op op,
                                                  uint64_t identity) {
    const int lane = threadIdx.x & 31;
    if (tile == 0) {
        if (lane == 0) lb_store(status, LB_PRE | (agg & LB_VAL));
        return identity;
    }
    if (lane == 0) lb_store(status + tile, LB_AGG | (agg & LB_VAL));
    uint64_t excl = identity;
    int64_t win = tile - 1;   // the closest earlier tile this lane group looks at
    while (true) {
        int64_t idx = win - lane;
        uint64_t w = (idx >= 0) ? lb_load(status + idx) : (LB_PRE | (identity & LB_VAL));
        // all lanes must have a ready word before reducing; back off while waiting so
        // spinning warps do not steal issue slots and L2 bandwidth from the producers
        while (__any_sync(0xffffffffu, (w >> 62) == 0)) {
            __nanosleep(64);
            if ((w >> 62) == 0) w = lb_load(status + idx);
        }
        unsigned pre = __ballot_sync(0xffffffffu, (w >> 62) == 2);
        int stop = pre ? (__ffs(pre) - 1) : 31;   // lanes 0..stop contribute
        uint64_t v = (lane <= stop) ? (w & LB_VAL) : identity;
        for (int o = 16; o > 0; o >>= 1) v = op(v, __shfl_xor_sync(0xffffffffu, v, o));
        excl = op(excl, v);
        if (pre) break;
        win -= 32;
    }
    if (lane == 0) lb_store(status + tile, LB_PRE | (op(excl, agg) & LB_VAL));
    return excl;
}

struct OpAdd {
    __device__ __forceinline__ uint64_t operator()(uint64_t a, uint64_t b) const { return a + b; }
};
struct OpMax {
    __device__ __forceinline__ uint64_t operator()(uint64_t a, uint64_t b) const { return a > b ? a : b; }
};

// Dynamic tile id: taken by thread 0 and broadcast through shared memory.
__device__ __forceinline__ int64_t take_tile(unsigned long long* counter, int64_t* smem_slot) {
    if (threadIdx.x == 0) *smem_slot = (int64_t)atomicAdd(counter, 1ull);
    __syncthreads();
    return *smem_slot;
}

__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

}  // namespace tqp

namespace tqp {
// ------------------------------------------- TMA bulk copies + mbarriers
// 1-D bulk copies global -> shared (cp.async.bulk, the TMA engine's non-tensor
// path) completing on an mbarrier transaction count.
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
// Same copy with an L2 eviction-priority hint (a createpolicy value): the sort scatter
// streams its input once, so it can be marked evict_first.
__device__ __forceinline__ void bulk_g2s_hint(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t pol) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
                 : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ void st_hint_u32(uint32_t* p, uint32_t v, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.u32 [%0], %1, %2;" ::"l"(p), "r"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}\n" ::"r"(
            smem_u32(bar)),
        "r"(parity)
        : "memory");
}
}  // namespace tqp
