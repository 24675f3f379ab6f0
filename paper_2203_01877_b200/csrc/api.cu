// api.cu -- the extern "C" boundary of libtqp (declared in include/tqp.h).
// Every entry point converts internal exceptions into a tqp_status and a
// message; nothing C++ crosses the ABI.
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include <nvtx3/nvToolsExt.h>

#include "internal.h"
#include "jit.h"

namespace tqp {
void pkfk_join(tqp_ctx*, tqp_col, int64_t, tqp_col, int64_t, int64_t*, int64_t*, int64_t*);
void pkfk_join_i32(tqp_ctx*, tqp_col, int64_t, tqp_col, int64_t, int32_t*, int32_t*, int64_t*);
void pkfk_join_paper_order(tqp_ctx*, tqp_col, int64_t, tqp_col, int64_t, int64_t*, int64_t*, int64_t*);
void pkfk_semi(tqp_ctx*, tqp_col, int64_t, tqp_col, int64_t, int, uint8_t*, int64_t*, int64_t*);
void pkfk_outer(tqp_ctx*, tqp_col, int64_t, tqp_col, int64_t, int64_t*, uint8_t*, int64_t*);
void pkfk_join_hash(tqp_ctx*, tqp_col, int64_t, tqp_col, int64_t, int64_t*, int64_t*, int64_t*);
void pkfk_join_payload(tqp_ctx*, tqp_col, int64_t, tqp_col, int64_t, const tqp_col*, int, void* const*, const tqp_col*, int,
                       void* const*, int64_t*, int64_t*, int64_t*);
void filter_compact(tqp_ctx*, const tqp_col*, int, int64_t, const tqp_pred*, int, uint8_t*, int64_t*, int64_t*);
int pack_keys(tqp_ctx*, const tqp_col*, int64_t, const tqp_col*, int64_t, int, int64_t*, int64_t*);
tqp_smj_plan* smj_prepare(tqp_ctx*, tqp_col, int64_t, tqp_col, int64_t, int64_t*);
void smj_expand(tqp_ctx*, const tqp_smj_plan*, int64_t, int64_t, void*, void*, int);
void smj_expand_checksum(tqp_ctx*, const tqp_smj_plan*, int64_t, int64_t, uint64_t*);
void smj_release(tqp_ctx*, tqp_smj_plan*);
tqp_groupby_plan* groupby_prepare(tqp_ctx*, const tqp_col*, int, int64_t, const int32_t*, int, const tqp_pred*, int,
                                  const tqp_agg*, int, int64_t*);
void groupby_fetch(tqp_ctx*, const tqp_groupby_plan*, void* const*, void* const*);
void groupby_release(tqp_ctx*, tqp_groupby_plan*);
tqp_groupby_plan* groupby_merge(tqp_ctx*, int64_t, const tqp_col*, int, const tqp_agg*, int, const void* const*,
                                const int64_t*, int64_t*);
void smj_expand_payload(tqp_ctx*, const tqp_smj_plan*, int64_t, int64_t, const tqp_col*, int, void* const*,
                        const tqp_col*, int, void* const*, int64_t*, int64_t*);
void partition(tqp_ctx*, tqp_col, int64_t, const int64_t*, int, int64_t, void*, int64_t*, int64_t*);
void pkfk_outer_build(tqp_ctx*, tqp_col, int64_t, tqp_col, int64_t, int64_t*, int64_t*, int64_t*);
tqp_partition_plan* partition_plan(tqp_ctx*, tqp_col, int64_t, const int64_t*, int, int64_t*);
void partition_scatter(tqp_ctx*, tqp_partition_plan*, int64_t, void* const*, int64_t* const*, const int64_t*);
void partition_release(tqp_ctx*, tqp_partition_plan*);
void* ipc_alloc(size_t, void*);
void* ipc_open(const void*);
void minmax(tqp_ctx*, tqp_col, int64_t, int64_t*);
void range_splitters(tqp_ctx*, const int64_t*, int, int64_t*);
void gather(tqp_ctx*, tqp_col, const int64_t*, int64_t, void*);
}  // namespace tqp

static_assert(sizeof(tqp_col) == 16, "tqp_col layout");
static_assert(sizeof(tqp_pred) == 16, "tqp_pred layout");
static_assert(sizeof(tqp_agg) == 56, "tqp_agg layout");

static size_t round_block(size_t b) {
    if (b <= (1u << 20)) return (b + 511) & ~size_t(511);
    return (b + (2u << 20) - 1) & ~size_t((2u << 20) - 1);
}

void* tqp_ctx::raw_alloc(size_t bytes) {
    if (alloc_fn) return alloc_fn(alloc_user, bytes, device, stream);
    void* p = nullptr;
    if (cudaMalloc(&p, bytes) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    return p;
}

void tqp_ctx::raw_free(void* p) {
    if (!p) return;
    if (free_fn) free_fn(alloc_user, p, device, stream);
    else cudaFree(p);
}

void* tqp_ctx::dalloc(size_t bytes) {
    if (bytes == 0) return nullptr;
    if (exact_alloc) {   // exact size + GUARD canary bytes (0xA5), checked at release
        void* p = raw_alloc(bytes + GUARD);
        if (!p) tqp::fail(TQP_ERR_OUT_OF_MEMORY, "device allocation of a temporary failed");
        TQP_CUDA(cudaMemsetAsync(static_cast<char*>(p) + bytes, 0xA5, GUARD, stream));
        if (poison) TQP_CUDA(cudaMemsetAsync(p, 0xA5, bytes, stream));
        live_blocks[p] = bytes;
        return p;
    }
    const size_t sz = round_block(bytes);
    auto it = free_blocks.lower_bound(sz);
    if (it != free_blocks.end() && it->first <= sz + sz / 4) {   // best fit within 25 %
        void* p = it->second;
        const size_t have = it->first;
        free_blocks.erase(it);
        cached_bytes -= have;
        live_blocks[p] = have;
        if (poison) TQP_CUDA(cudaMemsetAsync(p, 0xA5, bytes, stream));
        return p;
    }
    void* p = raw_alloc(sz);
    if (!p) {   // out of memory: give the cached blocks back and retry once
        trim();
        p = raw_alloc(sz);
    }
    if (!p) tqp::fail(TQP_ERR_OUT_OF_MEMORY, "device allocation of a temporary failed (" + std::to_string(sz) + " bytes)");
    live_blocks[p] = sz;
    if (poison) TQP_CUDA(cudaMemsetAsync(p, 0xA5, bytes, stream));
    return p;
}

void tqp_ctx::dfree(void* p) {
    auto it = live_blocks.find(p);
    if (it == live_blocks.end()) return;
    if (exact_alloc) {
        unsigned char g[GUARD];
        cudaStreamSynchronize(stream);
        if (cudaMemcpy(g, static_cast<char*>(p) + it->second, GUARD, cudaMemcpyDeviceToHost) == cudaSuccess) {
            for (size_t i = 0; i < GUARD; i++)
                if (g[i] != 0xA5) {
                    guard_violations++;
                    fprintf(stderr, "libtqp: guard bytes after a %zu-byte temporary overwritten (offset %zu)\n",
                            it->second, i);
                    break;
                }
        }
        raw_free(p);
        live_blocks.erase(it);
        return;
    }
    free_blocks.emplace(it->second, p);
    cached_bytes += it->second;
    live_blocks.erase(it);
}

void tqp_ctx::trim() {
    cudaStreamSynchronize(stream);
    for (auto& kv : free_blocks) raw_free(kv.second);
    free_blocks.clear();
    cached_bytes = 0;
}

void tqp_ctx::drain_profile() {
    if (pending.empty()) return;
    TQP_CUDA(cudaStreamSynchronize(stream));
    for (auto& p : pending) {
        float ms = 0.f;
        TQP_CUDA(cudaEventElapsedTime(&ms, p.a, p.b));
        auto& st = stats[p.name];
        st.ms += ms;
        st.launches += 1;
        free_events.push_back(p.a);
        free_events.push_back(p.b);
    }
    pending.clear();
}

// Every entry point is an NVTX range named after it (nsys / ncu --nvtx timelines; nvtx3
// is header-only and costs a null check without a tool attached).
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};

#define TQP_GUARD(ctx, body)                                                   \
    do {                                                                       \
        if (!(ctx)) return TQP_ERR_INVALID_ARGUMENT;                           \
        NvtxRange nvtx_range_(__func__);                                       \
        try {                                                                  \
            int cur_ = -1;                                                     \
            cudaGetDevice(&cur_);                                              \
            if (cur_ != (ctx)->device) cudaSetDevice((ctx)->device);           \
            body;                                                              \
            (ctx)->err.clear();                                                \
            return TQP_OK;                                                     \
        } catch (const ::tqp::Error& e) {                                      \
            (ctx)->err = e.msg;                                                \
            return e.status;                                                   \
        } catch (const std::bad_alloc&) {                                      \
            (ctx)->err = "host out of memory";                                 \
            return TQP_ERR_OUT_OF_MEMORY;                                      \
        } catch (...) {                                                        \
            (ctx)->err = "unknown error";                                      \
            return TQP_ERR_CUDA;                                               \
        }                                                                      \
    } while (0)

extern "C" {

int tqp_abi_version(void) { return TQP_ABI_VERSION; }

tqp_status tqp_ctx_create(int device, void* stream, tqp_ctx** out) {
    if (!out) return TQP_ERR_INVALID_ARGUMENT;
    *out = nullptr;
    tqp_ctx* c = new (std::nothrow) tqp_ctx();
    if (!c) return TQP_ERR_OUT_OF_MEMORY;
    try {
        c->device = device;
        TQP_CUDA(cudaSetDevice(device));
        TQP_CUDA(cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device));
        c->stream = static_cast<cudaStream_t>(stream);
        const char* ex = getenv("TQP_ALLOC_EXACT");
        c->exact_alloc = ex && ex[0] == '1';
        const char* po = getenv("TQP_ALLOC_POISON");
        c->poison = po && po[0] == '1';
        TQP_CUDA(cudaMallocHost(&c->pinned, 4096));
    } catch (const tqp::Error& e) {
        delete c;
        return e.status;
    }
    *out = c;
    return TQP_OK;
}

void tqp_ctx_destroy(tqp_ctx* c) {
    if (!c) return;
    cudaSetDevice(c->device);
    cudaStreamSynchronize(c->stream);
    for (auto& p : c->pending) { cudaEventDestroy(p.a); cudaEventDestroy(p.b); }
    for (auto e : c->free_events) cudaEventDestroy(e);
    if (c->pinned) cudaFreeHost(c->pinned);
    c->trim();
    for (auto& kv : c->live_blocks) c->raw_free(kv.first);
    delete c;
}

tqp_status tqp_ctx_set_allocator(tqp_ctx* c, tqp_alloc_fn alloc, tqp_free_fn free_, void* user) {
    TQP_GUARD(c, {
        if ((alloc == nullptr) != (free_ == nullptr)) tqp::fail(TQP_ERR_INVALID_ARGUMENT, "allocator: both callbacks or neither");
        if (!c->live_blocks.empty()) tqp::fail(TQP_ERR_INVALID_ARGUMENT, "allocator: the context holds live temporaries");
        c->trim();   // cached blocks go back to the allocator they came from
        c->alloc_fn = alloc;
        c->free_fn = free_;
        c->alloc_user = user;
    });
}

tqp_status tqp_ctx_trim(tqp_ctx* c) {
    TQP_GUARD(c, { c->trim(); });
}

size_t tqp_ctx_cached_bytes(const tqp_ctx* c) { return c ? c->cached_bytes : 0; }

tqp_status tqp_ctx_set_stream(tqp_ctx* c, void* stream) {
    // cached blocks were last used on the old stream: order the switch
    TQP_GUARD(c, {
        c->drain_profile();
        TQP_CUDA(cudaStreamSynchronize(c->stream));
        c->stream = static_cast<cudaStream_t>(stream);
    });
}

const char* tqp_last_error(const tqp_ctx* c) { return c ? c->err.c_str() : "null context"; }

int64_t tqp_ctx_launch_count(const tqp_ctx* c) { return c ? c->launches : 0; }

int64_t tqp_ctx_guard_violations(const tqp_ctx* c) { return c ? c->guard_violations : 0; }

int tqp_jit_counters(int64_t* compiled, int64_t* failed, int64_t* launches) {
    const tqp::JitCounters c = tqp::jit_counters();
    if (compiled) *compiled = c.compiled;
    if (failed) *failed = c.failed;
    if (launches) *launches = c.launches;
    return tqp::jit_available() ? 1 : 0;
}

void tqp_ctx_reset_counters(tqp_ctx* c) {
    if (!c) return;
    try { c->drain_profile(); } catch (...) {}
    c->launches = 0;
    c->stats.clear();
}

tqp_status tqp_ctx_set_profiling(tqp_ctx* c, int enable) {
    TQP_GUARD(c, { c->drain_profile(); c->profiling = enable != 0; });
}

tqp_status tqp_ctx_set_profiling_filter(tqp_ctx* c, const char* name_prefix) {
    TQP_GUARD(c, { c->drain_profile(); c->prof_prefix = name_prefix ? name_prefix : ""; });
}

tqp_status tqp_ctx_kernel_stats(tqp_ctx* c, char* names, size_t names_cap, double* ms, int64_t* launches,
                                double* bytes, int max_kernels, int* n_kernels) {
    TQP_GUARD(c, {
        c->drain_profile();
        std::string all;
        int k = 0;
        for (auto& kv : c->stats) {
            if (k < max_kernels) {
                if (ms) ms[k] = kv.second.ms;
                if (launches) launches[k] = kv.second.launches;
                if (bytes) bytes[k] = kv.second.bytes;
                all += kv.first;
                all += '\n';
            }
            k++;
        }
        if (n_kernels) *n_kernels = k < max_kernels ? k : max_kernels;
        if (names && names_cap) {
            size_t m = all.size() < names_cap - 1 ? all.size() : names_cap - 1;
            memcpy(names, all.data(), m);
            names[m] = 0;
        }
    });
}

tqp_status tqp_sort(tqp_ctx* c, tqp_col keys, int64_t n, int descending, void* sorted_keys_out, int64_t* perm_out) {
    TQP_GUARD(c, {
        tqp::check_col(keys, n, "sort keys");
        if (n > 0 && !perm_out) tqp::fail(TQP_ERR_INVALID_ARGUMENT, "sort: null perm_out");
        tqp::SortOut o;
        o.sorted_orig = sorted_keys_out;
        o.perm64 = perm_out;
        tqp::radix_sort(c, keys.data, keys.dtype, n, descending != 0, o);
    });
}

tqp_status tqp_pkfk_join(tqp_ctx* c, tqp_col b, int64_t nb, tqp_col p, int64_t np, int64_t* lo, int64_t* ro,
                         int64_t* n_out_host) {
    TQP_GUARD(c, {
        if (!n_out_host) tqp::fail(TQP_ERR_INVALID_ARGUMENT, "pkfk: null n_out_host");
        tqp::pkfk_join(c, b, nb, p, np, lo, ro, n_out_host);
    });
}

tqp_status tqp_pkfk_join_i32(tqp_ctx* c, tqp_col b, int64_t nb, tqp_col p, int64_t np, int32_t* lo, int32_t* ro,
                             int64_t* n_out_host) {
    TQP_GUARD(c, {
        if (!n_out_host) tqp::fail(TQP_ERR_INVALID_ARGUMENT, "pkfk_i32: null n_out_host");
        tqp::pkfk_join_i32(c, b, nb, p, np, lo, ro, n_out_host);
    });
}

tqp_status tqp_pkfk_join_paper_order(tqp_ctx* c, tqp_col b, int64_t nb, tqp_col p, int64_t np, int64_t* lo,
                                     int64_t* ro, int64_t* n_out_host) {
    TQP_GUARD(c, {
        if (!n_out_host) tqp::fail(TQP_ERR_INVALID_ARGUMENT, "pkfk_paper_order: null n_out_host");
        tqp::pkfk_join_paper_order(c, b, nb, p, np, lo, ro, n_out_host);
    });
}

tqp_status tqp_pkfk_semi(tqp_ctx* c, tqp_col b, int64_t nb, tqp_col p, int64_t np, int anti, uint8_t* match_out,
                         int64_t* sel_out, int64_t* n_sel_host) {
    TQP_GUARD(c, { tqp::pkfk_semi(c, b, nb, p, np, anti, match_out, sel_out, n_sel_host); });
}

tqp_status tqp_pkfk_join_payload(tqp_ctx* c, tqp_col b, int64_t nb, tqp_col p, int64_t np, const tqp_col* bp, int n_bp,
                                 void* const* bp_out, const tqp_col* pp, int n_pp, void* const* pp_out, int64_t* lo,
                                 int64_t* ro, int64_t* n_out_host) {
    TQP_GUARD(c, {
        if (!n_out_host) tqp::fail(TQP_ERR_INVALID_ARGUMENT, "pkfk: null n_out_host");
        if ((n_bp > 0 && (!bp || !bp_out)) || (n_pp > 0 && (!pp || !pp_out)))
            tqp::fail(TQP_ERR_INVALID_ARGUMENT, "pkfk: null payload arrays");
        tqp::pkfk_join_payload(c, b, nb, p, np, bp, n_bp, bp_out, pp, n_pp, pp_out, lo, ro, n_out_host);
    });
}

tqp_status tqp_pkfk_join_hash(tqp_ctx* c, tqp_col b, int64_t nb, tqp_col p, int64_t np, int64_t* lo, int64_t* ro,
                              int64_t* n_out_host) {
    TQP_GUARD(c, {
        if (!n_out_host) tqp::fail(TQP_ERR_INVALID_ARGUMENT, "pkfk_hash: null n_out_host");
        tqp::pkfk_join_hash(c, b, nb, p, np, lo, ro, n_out_host);
    });
}

tqp_status tqp_pkfk_outer(tqp_ctx* c, tqp_col b, int64_t nb, tqp_col p, int64_t np, int64_t* left_out,
                          uint8_t* match_out, int64_t* n_match_host) {
    TQP_GUARD(c, { tqp::pkfk_outer(c, b, nb, p, np, left_out, match_out, n_match_host); });
}

tqp_status tqp_smj_prepare(tqp_ctx* c, tqp_col l, int64_t nl, tqp_col r, int64_t nr, tqp_smj_plan** plan,
                           int64_t* out_size_host) {
    TQP_GUARD(c, {
        if (!plan || !out_size_host) tqp::fail(TQP_ERR_INVALID_ARGUMENT, "smj_prepare: null output");
        *plan = tqp::smj_prepare(c, l, nl, r, nr, out_size_host);
    });
}

tqp_status tqp_smj_expand(tqp_ctx* c, const tqp_smj_plan* plan, int64_t begin, int64_t end, int64_t* lo,
                          int64_t* ro) {
    TQP_GUARD(c, {
        if (!plan) tqp::fail(TQP_ERR_INVALID_ARGUMENT, "smj_expand: null plan");
        tqp::smj_expand(c, plan, begin, end, lo, ro, 0);
    });
}

tqp_status tqp_smj_expand_i32(tqp_ctx* c, const tqp_smj_plan* plan, int64_t begin, int64_t end, int32_t* lo,
                              int32_t* ro) {
    TQP_GUARD(c, {
        if (!plan) tqp::fail(TQP_ERR_INVALID_ARGUMENT, "smj_expand_i32: null plan");
        tqp::smj_expand(c, plan, begin, end, lo, ro, 1);
    });
}

tqp_status tqp_smj_expand_checksum(tqp_ctx* c, const tqp_smj_plan* plan, int64_t begin, int64_t end,
                                   uint64_t* out_host) {
    TQP_GUARD(c, {
        if (!plan || !out_host) tqp::fail(TQP_ERR_INVALID_ARGUMENT, "smj_expand_checksum: null argument");
        tqp::smj_expand_checksum(c, plan, begin, end, out_host);
    });
}

void tqp_smj_release(tqp_ctx* c, tqp_smj_plan* plan) {
    if (plan) tqp::smj_release(c, plan);
}

tqp_status tqp_smj_join(tqp_ctx* c, tqp_col l, int64_t nl, tqp_col r, int64_t nr, int64_t* lo, int64_t* ro,
                        int64_t capacity, int64_t* n_out_host) {
    TQP_GUARD(c, {
        if (!n_out_host) tqp::fail(TQP_ERR_INVALID_ARGUMENT, "smj_join: null n_out_host");
        int64_t size = 0;
        tqp_smj_plan* P = tqp::smj_prepare(c, l, nl, r, nr, &size);
        *n_out_host = size;
        if (size > capacity) {
            tqp::smj_release(c, P);
            tqp::fail(TQP_ERR_CAPACITY, "smj_join: capacity smaller than the join size");
        }
        try {
            tqp::smj_expand(c, P, 0, size, lo, ro, 0);
        } catch (...) {
            tqp::smj_release(c, P);
            throw;
        }
        tqp::smj_release(c, P);
    });
}

tqp_status tqp_pack_keys(tqp_ctx* c, const tqp_col* a_cols, int64_t n_a, const tqp_col* b_cols, int64_t n_b, int n_cols,
                         int64_t* a_out, int64_t* b_out, int* bits_host) {
    TQP_GUARD(c, {
        if (!a_cols) tqp::fail(TQP_ERR_INVALID_ARGUMENT, "pack_keys: null columns");
        const int bits = tqp::pack_keys(c, a_cols, n_a, b_cols, n_b, n_cols, a_out, b_out);
        if (bits_host) *bits_host = bits;
    });
}

tqp_status tqp_filter_compact(tqp_ctx* c, const tqp_col* cols, int n_cols, int64_t n, const tqp_pred* preds,
                              int n_preds, uint8_t* mask_out, int64_t* sel_out, int64_t* n_sel_host) {
    TQP_GUARD(c, { tqp::filter_compact(c, cols, n_cols, n, preds, n_preds, mask_out, sel_out, n_sel_host); });
}

tqp_status tqp_groupby_prepare(tqp_ctx* c, const tqp_col* cols, int n_cols, int64_t n, const int32_t* key_idx,
                               int n_keys, const tqp_pred* preds, int n_preds, const tqp_agg* aggs, int n_aggs,
                               tqp_groupby_plan** plan, int64_t* n_groups_host) {
    TQP_GUARD(c, {
        if (!plan || !n_groups_host) tqp::fail(TQP_ERR_INVALID_ARGUMENT, "groupby_prepare: null output");
        if ((n_cols && !cols) || (n_keys && !key_idx) || (n_preds && !preds) || (n_aggs && !aggs))
            tqp::fail(TQP_ERR_INVALID_ARGUMENT, "groupby_prepare: null array");
        *plan = tqp::groupby_prepare(c, cols, n_cols, n, key_idx, n_keys, preds, n_preds, aggs, n_aggs, n_groups_host);
    });
}

tqp_status tqp_groupby_fetch(tqp_ctx* c, const tqp_groupby_plan* plan, void* const* keys_out,
                             void* const* results_out) {
    TQP_GUARD(c, {
        if (!plan) tqp::fail(TQP_ERR_INVALID_ARGUMENT, "groupby_fetch: null plan");
        tqp::groupby_fetch(c, plan, keys_out, results_out);
    });
}

tqp_status tqp_groupby_merge(tqp_ctx* c, int64_t m, const tqp_col* key_cols, int n_keys, const tqp_agg* aggs,
                             int n_aggs, const void* const* partial, const int64_t* counts, tqp_groupby_plan** plan,
                             int64_t* n_groups_host) {
    TQP_GUARD(c, {
        if (!plan || !n_groups_host) tqp::fail(TQP_ERR_INVALID_ARGUMENT, "groupby_merge: null output");
        if ((n_keys && !key_cols) || (n_aggs && !aggs)) tqp::fail(TQP_ERR_INVALID_ARGUMENT, "groupby_merge: null array");
        *plan = tqp::groupby_merge(c, m, key_cols, n_keys, aggs, n_aggs, partial, counts, n_groups_host);
    });
}

void tqp_groupby_release(tqp_ctx* c, tqp_groupby_plan* plan) {
    if (plan) tqp::groupby_release(c, plan);
}

tqp_status tqp_groupby_agg(tqp_ctx* c, const tqp_col* cols, int n_cols, int64_t n, const int32_t* key_idx,
                           int n_keys, const tqp_pred* preds, int n_preds, const tqp_agg* aggs, int n_aggs,
                           void* const* keys_out, void* const* results_out, int64_t capacity,
                           int64_t* n_groups_host) {
    TQP_GUARD(c, {
        if (!n_groups_host) tqp::fail(TQP_ERR_INVALID_ARGUMENT, "groupby_agg: null n_groups_host");
        if ((n_cols && !cols) || (n_keys && !key_idx) || (n_preds && !preds) || (n_aggs && !aggs))
            tqp::fail(TQP_ERR_INVALID_ARGUMENT, "groupby_agg: null array");
        tqp_groupby_plan* P =
            tqp::groupby_prepare(c, cols, n_cols, n, key_idx, n_keys, preds, n_preds, aggs, n_aggs, n_groups_host);
        if (*n_groups_host > capacity) {
            tqp::groupby_release(c, P);
            tqp::fail(TQP_ERR_CAPACITY, "groupby_agg: capacity smaller than the group count");
        }
        try {
            tqp::groupby_fetch(c, P, keys_out, results_out);
        } catch (...) {
            tqp::groupby_release(c, P);
            throw;
        }
        tqp::groupby_release(c, P);
    });
}

tqp_status tqp_smj_expand_payload(tqp_ctx* c, const tqp_smj_plan* plan, int64_t begin, int64_t end,
                                  const tqp_col* left_payload, int n_left_payload, void* const* left_payload_out,
                                  const tqp_col* right_payload, int n_right_payload, void* const* right_payload_out,
                                  int64_t* left_out_idx, int64_t* right_out_idx) {
    TQP_GUARD(c, {
        if (!plan) tqp::fail(TQP_ERR_INVALID_ARGUMENT, "smj_expand_payload: null plan");
        if ((n_left_payload && (!left_payload || !left_payload_out)) ||
            (n_right_payload && (!right_payload || !right_payload_out)))
            tqp::fail(TQP_ERR_INVALID_ARGUMENT, "smj_expand_payload: null payload array");
        tqp::smj_expand_payload(c, plan, begin, end, left_payload, n_left_payload, left_payload_out, right_payload,
                                n_right_payload, right_payload_out, left_out_idx, right_out_idx);
    });
}

tqp_status tqp_pkfk_outer_build(tqp_ctx* c, tqp_col b, int64_t nb, tqp_col p, int64_t np, int64_t* left_out,
                                int64_t* right_out, int64_t* n_out_host) {
    TQP_GUARD(c, {
        if (!n_out_host) tqp::fail(TQP_ERR_INVALID_ARGUMENT, "pkfk_outer_build: null n_out_host");
        tqp::pkfk_outer_build(c, b, nb, p, np, left_out, right_out, n_out_host);
    });
}

tqp_status tqp_partition(tqp_ctx* c, tqp_col keys, int64_t n, const int64_t* splitters, int n_parts, int64_t row_base,
                         void* keys_out, int64_t* rows_out, int64_t* counts_out) {
    TQP_GUARD(c, { tqp::partition(c, keys, n, splitters, n_parts, row_base, keys_out, rows_out, counts_out); });
}

tqp_status tqp_partition_plan_create(tqp_ctx* c, tqp_col keys, int64_t n, const int64_t* splitters, int n_parts,
                                     int64_t* counts_out, tqp_partition_plan** plan) {
    TQP_GUARD(c, {
        if (!plan) tqp::fail(TQP_ERR_INVALID_ARGUMENT, "partition_plan: null plan");
        *plan = tqp::partition_plan(c, keys, n, splitters, n_parts, counts_out);
    });
}

tqp_status tqp_partition_scatter(tqp_ctx* c, tqp_partition_plan* plan, int64_t row_base, void* const* dst_keys_host,
                                 int64_t* const* dst_rows_host, const int64_t* dst_base_host) {
    TQP_GUARD(c, {
        if (!plan) tqp::fail(TQP_ERR_INVALID_ARGUMENT, "partition_scatter: null plan");
        tqp::partition_scatter(c, plan, row_base, dst_keys_host, dst_rows_host, dst_base_host);
    });
}

void tqp_partition_release(tqp_ctx* c, tqp_partition_plan* plan) {
    if (c && plan) tqp::partition_release(c, plan);
}

tqp_status tqp_ipc_alloc(tqp_ctx* c, size_t bytes, void** dev_ptr_out, void* handle_out) {
    TQP_GUARD(c, {
        if (!dev_ptr_out || !handle_out) tqp::fail(TQP_ERR_INVALID_ARGUMENT, "ipc_alloc: null output");
        *dev_ptr_out = tqp::ipc_alloc(bytes, handle_out);
    });
}

tqp_status tqp_ipc_free(tqp_ctx* c, void* dev_ptr) {
    TQP_GUARD(c, { TQP_CUDA(cudaFree(dev_ptr)); });
}

tqp_status tqp_ipc_open(tqp_ctx* c, const void* handle, void** dev_ptr_out) {
    TQP_GUARD(c, {
        if (!handle || !dev_ptr_out) tqp::fail(TQP_ERR_INVALID_ARGUMENT, "ipc_open: null argument");
        *dev_ptr_out = tqp::ipc_open(handle);
    });
}

tqp_status tqp_ipc_close(tqp_ctx* c, void* dev_ptr) {
    TQP_GUARD(c, { TQP_CUDA(cudaIpcCloseMemHandle(dev_ptr)); });
}

tqp_status tqp_minmax(tqp_ctx* c, tqp_col keys, int64_t n, int64_t* lohi_out) {
    TQP_GUARD(c, { tqp::minmax(c, keys, n, lohi_out); });
}

tqp_status tqp_range_splitters(tqp_ctx* c, const int64_t* lohi, int n_parts, int64_t* splitters_out) {
    TQP_GUARD(c, { tqp::range_splitters(c, lohi, n_parts, splitters_out); });
}

tqp_status tqp_gather(tqp_ctx* c, tqp_col src, const int64_t* idx, int64_t n, void* out) {
    TQP_GUARD(c, { tqp::gather(c, src, idx, n, out); });
}

}  // extern "C"
