// internal.h -- interfaces shared between libtqp translation units (not part of the ABI).
#pragma once

#include "common.cuh"

namespace tqp {

// Radix sort of one key column (stable; "radix sort" :256/:1148).
// Sort domain value u = ordered_u64(key) (DT_U64: the key itself); descending: u = ~u.
// Requested outputs (all nullable / optional):
struct SortOut {
    void* sorted_orig = nullptr;       // n elements of the input dtype = keys[perm]
    int64_t* perm64 = nullptr;         // n x int64 permutation
    uint64_t* sorted_u = nullptr;      // n x sort-domain values u (ascending)
    bool want_internal = false;        // keep internal sorted keys + u32 permutation below
    bool want_perm32 = false;          // keep the u32 permutation only
    bool defer_identity = false;       // presorted input: return with identity = true and nothing
                                       // written (the caller reads the input keys themselves or
                                       // calls sort_materialize_identity)
    // results
    bool k32 = false;                  // internal keys are the low 32 bits of u
    uint64_t and_bits = 0, or_bits = 0;   // AND / OR of all u (varying-bit mask = and ^ or)
    uint64_t first_u = 0, last_u = 0;     // u of keys[0] and keys[n - 1] (= min / max when identity)
    int passes = 0;
    bool identity = false;             // the input was already in (key, row) order: perm = 0..n-1
    DevBuf<uint32_t> keys32;           // internal sorted keys (k32)
    DevBuf<uint64_t> keys64;           // internal sorted keys (!k32)
    DevBuf<uint32_t> perm32;           // internal permutation
};

// andor (nullable, SORT_PLAN_WORDS words): the AND / OR of the sort-domain keys, an "out
// of order" flag (0 = already sorted) and the sort-domain values of the first and last
// key, read back by the caller from sort_andor (so several sorts share one host sync);
// null = computed here.
// th0 (nullable, sort_hist0_words(n) u32): the first-pass histogram sort_andor fused in.
constexpr int SORT_PLAN_WORDS = 5;
void radix_sort(tqp_ctx* ctx, const void* keys, int dtype, int64_t n, bool desc, SortOut& out,
                const uint64_t* andor = nullptr, uint32_t* th0 = nullptr);
// AND / OR of the sort-domain keys into ao[0..1], the unsorted flag into ao[2], the first /
// last key's sort-domain value into ao[3..4] (device, stream-ordered; no sync); with
// th0, also the speculative pass-0 tile histogram (9-bit digits at bit 0, 4096-key tiles)
void sort_andor(tqp_ctx* ctx, const void* keys, int dtype, int64_t n, bool desc, unsigned long long* ao,
                uint32_t* th0 = nullptr);
size_t sort_hist0_words(int64_t n);
// The identity route's outputs (the trivial pass) for a sort that returned with
// defer_identity and identity set.
void sort_materialize_identity(tqp_ctx* ctx, const void* keys, int dtype, int64_t n, bool desc, SortOut& o);

// First / last key (order-preserving images) and an order check of 2,049 evenly spaced
// keys (pkfk.cu): out[0] = first, out[1] = last, out[2] = 1 if the sample is not in order.
void sample_first_last(tqp_ctx* ctx, const void* keys, int dt, int64_t n, unsigned long long* out);

// Filter + compaction (filter.cu), used by the group-by sort path for its selection.
void filter_compact(tqp_ctx* ctx, const tqp_col* cols, int n_cols, int64_t n, const tqp_pred* preds, int n_preds,
                    uint8_t* mask_out, int64_t* sel_out, int64_t* n_sel_host);

// Exclusive / inclusive scans over device arrays (decoupled look-back).
void iota_i64(tqp_ctx* ctx, int64_t* p, int64_t n);
void scan_max_u32_exclusive(tqp_ctx* ctx, const uint32_t* in, uint32_t* out, int64_t n);
// out[i] = sum(in[0..i-1]), out[n] = total (out has n + 1 entries; sums must fit 32 bits)
void scan_add_u32_exclusive(tqp_ctx* ctx, const uint32_t* in, uint32_t* out, int64_t n);
void scan_add_u32_to_u64_exclusive(tqp_ctx* ctx, const uint32_t* in, uint64_t* out, int64_t n);
void scan_add_u64_exclusive(tqp_ctx* ctx, const uint64_t* in, uint64_t* out, int64_t n);

}  // namespace tqp
