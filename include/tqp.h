/*
 * tqp.h -- C ABI of libtqp: the data-parallel hot path of TQP
 * ("Query Processing on Tensor Computation Runtimes", He et al., PVLDB 2022,
 * arXiv 2203.01877; PAPER.md = the paper's LaTeX source) on NVIDIA B200 (sm_100a).
 *
 * The paper states each operator as forward(self, x) over "input columns passed
 * as an array of tensors" returning "an array of tensors representing the join
 * output". Here the arguments are key / payload
 * columns and the results are index pairs and aggregate columns.
 *
 * Conventions (apply to every entry point)
 *  - Pointers are CUDA DEVICE pointers (HBM) unless the parameter name ends in
 *    `_host`. Lengths are int64_t. Index outputs are int64 row numbers into the
 *    caller's input columns.
 *  - Ownership: inputs are borrowed and never modified. Outputs are
 *    caller-allocated (the bound is stated per function). Temporaries come from a
 *    caching device allocator owned by the context (blocks are reused
 *    stream-ordered on the context stream and returned on tqp_ctx_destroy).
 *    Plans (tqp_smj_plan, tqp_groupby_plan) must be released before their context.
 *  - Ordering: all work is enqueued on the context's stream. A `*_host` output
 *    costs one stream synchronisation; functions that need a data-dependent size
 *    (sort pass plan, join sizes, group count) synchronise internally and say so.
 *  - Errors: a status code; the message is available from tqp_last_error().
 *    No C++ exception crosses the ABI. Outputs are unspecified on error. After
 *    TQP_ERR_CUDA the context should be destroyed.
 *  - Determinism: identical inputs give bit-identical outputs (every scan and
 *    compaction is order-preserving; integer sums are associative).
 *  - Threading: one context per host thread / stream.
 */
#ifndef TQP_H_
#define TQP_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TQP_ABI_VERSION 1

typedef enum {
    TQP_OK = 0,
    TQP_ERR_INVALID_ARGUMENT = 1,
    TQP_ERR_DUPLICATE_BUILD_KEY = 2,   /* PK-FK build side has a repeated key (reading R10) */
    TQP_ERR_OUT_OF_MEMORY = 3,
    TQP_ERR_CUDA = 4,
    TQP_ERR_OVERFLOW = 5,              /* int64 aggregate value / join size >= 2^62 */
    TQP_ERR_CAPACITY = 6               /* output buffer too small; required size reported */
} tqp_status;

/* Column element types ("§4.1 Data Representation": numeric
 * n x 1 tensors; 1-character strings as uint8 (reading R19); dates as int32 days
 * or int64 microseconds (reading R18)). Comparisons: u8 unsigned, ints signed. */
/* TQP_F64: IEEE double value columns, accepted only as factor columns of group-by
 * aggregates; every other use -> TQP_ERR_INVALID_ARGUMENT. */
typedef enum { TQP_U8 = 1, TQP_I32 = 2, TQP_I64 = 3, TQP_F64 = 4 } tqp_dtype;

/* A column: `data` points to n elements of `dtype`, contiguous. */
typedef struct {
    const void* data;
    int32_t dtype;      /* tqp_dtype */
    int32_t reserved;   /* must be 0 */
} tqp_col;

typedef struct tqp_ctx tqp_ctx;

/* Create a context on CUDA device `device` issuing work on `stream`
 * (a cudaStream_t; NULL = legacy default stream). */
tqp_status tqp_ctx_create(int device, void* stream, tqp_ctx** out);
void tqp_ctx_destroy(tqp_ctx* ctx);
tqp_status tqp_ctx_set_stream(tqp_ctx* ctx, void* stream);

/* Device memory for the context's temporaries (SURVEY.md §8(b) tqp_alloc_fn /
 * tqp_free_fn): by default cudaMalloc / cudaFree; with tqp_ctx_set_allocator, the
 * caller's allocator (e.g. the framework's caching allocator, so both draw on one pool
 * of HBM). `stream` is the context stream (a cudaStream_t), `device` its device.
 * alloc returns NULL when out of memory; it must not call back into libtqp.
 * libtqp keeps the blocks it releases in a per-context cache in front of the allocator
 * (reused stream-ordered on the context stream), so the callbacks run on a cache miss,
 * at tqp_ctx_trim and at tqp_ctx_destroy only; on an allocation failure the cache is
 * returned to the allocator and the allocation retried once.
 * tqp_ctx_set_allocator: both callbacks or neither (NULL, NULL = cudaMalloc / cudaFree);
 * call it before the context's first operator -- with live temporaries it returns
 * TQP_ERR_INVALID_ARGUMENT; cached blocks of the previous allocator are returned to it
 * first. `user` is passed through to the callbacks (not owned). */
typedef void* (*tqp_alloc_fn)(void* user, size_t bytes, int device, void* stream);
typedef void (*tqp_free_fn)(void* user, void* ptr, int device, void* stream);
tqp_status tqp_ctx_set_allocator(tqp_ctx* ctx, tqp_alloc_fn alloc, tqp_free_fn free_fn, void* user);
/* Return every cached temporary block to the allocator (synchronises the context stream). */
tqp_status tqp_ctx_trim(tqp_ctx* ctx);
/* Bytes held in the context's cache of released temporaries. */
size_t tqp_ctx_cached_bytes(const tqp_ctx* ctx);
const char* tqp_last_error(const tqp_ctx* ctx);
int tqp_abi_version(void);

/* Instrumentation. Every kernel launch is counted; with profiling enabled each
 * launch is bracketed by CUDA events on the context stream and the device time
 * is accumulated per kernel name. Each kernel's ALGORITHMIC bytes (the
 * compulsory HBM traffic of the work it did) are
 * accounted on the host per launch. tqp_ctx_kernel_stats synchronises the
 * stream; per kernel k: ms_host[k] (profiled device time), launches_host[k]
 * (profiled launches), bytes_host[k] (algorithmic bytes, all launches).
 * names_host: '\n'-separated kernel names written into a caller buffer. */
int64_t tqp_ctx_launch_count(const tqp_ctx* ctx);
/* Poisoned temporaries (environment TQP_ALLOC_POISON=1 at context creation; tests): every
 * libtqp temporary is filled with 0xA5 bytes when handed out, so reads of never-written
 * temporary memory give garbage deterministically instead of a fresh allocation's zeros.
 * Checked mode (environment TQP_ALLOC_EXACT=1 at context creation; test builds):
 * every temporary is its own cudaMalloc followed by 256 canary bytes, verified when
 * the temporary is released; returns the number of overwritten canaries seen. */
int64_t tqp_ctx_guard_violations(const tqp_ctx* ctx);
void tqp_ctx_reset_counters(tqp_ctx* ctx);
/* Plan-compiled kernels (process-wide, all contexts): the dense group-by kernel of
 * tqp_groupby_agg is compiled at run time for each distinct aggregation plan (NVRTC,
 * sm_100a; environment TQP_JIT=0 disables it, TQP_JIT_MIN_ROWS (default 2^20) is the
 * smallest input that uses it; at most 256 plans are compiled per process, later ones run
 * on the generic kernel). Writes the number of plans compiled successfully, the
 * compilations that failed (the generic kernel ran instead) and the launches of compiled
 * kernels; any pointer may be NULL. Returns 1 if the runtime compiler was found, else 0. */
int tqp_jit_counters(int64_t* compiled_host, int64_t* failed_host, int64_t* launches_host);
tqp_status tqp_ctx_set_profiling(tqp_ctx* ctx, int enable);
/* Restrict profiling to kernels whose name starts with name_prefix (NULL or ""
 * = every kernel). Two event records per profiled launch cost host time that the
 * GPU waits for after each readback; the bench profiles only its dominant kernel. */
tqp_status tqp_ctx_set_profiling_filter(tqp_ctx* ctx, const char* name_prefix);
tqp_status tqp_ctx_kernel_stats(tqp_ctx* ctx, char* names_host, size_t names_cap, double* ms_host,
                                int64_t* launches_host, double* bytes_host, int max_kernels, int* n_kernels_host);

/* ------------------------------------------------------------------ sort */
/* (1) Stable sort with permutation -- Alg. 1 l.2-3, Alg. 2
 * l.3 "radix sort" (prose :1148); reading R1 (stable).
 * keys: n elements (I32 or I64; U8 also accepted).
 * perm_out[i] = input row of the i-th element of the stable (key, row) order
 * (n x int64, caller-allocated). descending != 0 orders keys descending with
 * ties still in ascending row order (descending is NOT the reverse).
 * sorted_keys_out: nullable; if given, n elements of the input dtype = keys[perm].
 * Implementation: reduce-then-scan LSD radix sort (per-tile digit histograms,
 * prefix scans, stable tile scatter); digits that are constant across all keys
 * are skipped. Synchronises once (pass plan). Requires n < 2^30, else
 * TQP_ERR_INVALID_ARGUMENT. */
tqp_status tqp_sort(tqp_ctx* ctx, tqp_col keys, int64_t n, int descending,
                    void* sorted_keys_out, int64_t* perm_out);

/* ------------------------------------------------------------ PK-FK join */
/* (2) Primary-key / foreign-key join -- PAPER.md:55-100 ("Find matches using
 * binary search"). build = unique-key side (the paper's `left`), probe = FK side
 * (`right`). Output: one pair per matching probe row, in ascending probe-row
 * order (reading R7): left_out_idx[j] = build row, right_out_idx[j] = probe row.
 * Buffers: capacity n_probe each (caller-allocated). *n_out_host = pairs.
 * The build side is radix-sorted; each probe key is located by a radix bracket
 * table plus a branch-free lower_bound (reading R8: the answer equals
 * lower_bound on the unpadded sorted build keys), matched by equality and
 * compacted order-preservingly. Duplicate build keys -> TQP_ERR_DUPLICATE_BUILD_KEY.
 * Key dtypes may differ (compared as int64). Synchronises twice. */
tqp_status tqp_pkfk_join(tqp_ctx* ctx, tqp_col build_keys, int64_t n_build, tqp_col probe_keys, int64_t n_probe,
                         int64_t* left_out_idx, int64_t* right_out_idx, int64_t* n_out_host);

/* tqp_pkfk_join with int32 index outputs (output-width
 * variant): identical pairs and order, written as int32 (half the output bytes of
 * the emit pass). Requires n_build < 2^31 and n_probe < 2^31, else
 * TQP_ERR_INVALID_ARGUMENT. Synchronises twice. */
tqp_status tqp_pkfk_join_i32(tqp_ctx* ctx, tqp_col build_keys, int64_t n_build, tqp_col probe_keys, int64_t n_probe,
                             int32_t* left_out_idx, int32_t* right_out_idx, int64_t* n_out_host);

/* tqp_pkfk_join in the paper's output order (reading R7):
 * the probe side is sorted descending first (stable radix sort) and
 * the sorted keys are probed in order, so the same pairs come ordered by probe key
 * descending, then by ascending probe row. Outputs as tqp_pkfk_join (capacity
 * n_probe x int64 each). Requires n_probe < 2^30. Synchronises three times. */
tqp_status tqp_pkfk_join_paper_order(tqp_ctx* ctx, tqp_col build_keys, int64_t n_build, tqp_col probe_keys,
                                     int64_t n_probe, int64_t* left_out_idx, int64_t* right_out_idx,
                                     int64_t* n_out_host);

/* Left-semi / left-anti variant ("left-semi, and left-anti
 * joins"): match_out (nullable, n_probe x u8) = 1 iff the probe row has a build
 * match; sel_out (nullable, capacity n_probe x int64) = ascending probe rows
 * with a match (anti != 0: without a match); *n_sel_host = their count. */
tqp_status tqp_pkfk_semi(tqp_ctx* ctx, tqp_col build_keys, int64_t n_build, tqp_col probe_keys, int64_t n_probe,
                         int anti, uint8_t* match_out, int64_t* sel_out, int64_t* n_sel_host);

/* PK-FK join with payload materialisation fused into the output (SURVEY.md
 * §8(f) NEXT 2: the paper's GenerateOutput / createOutput, PAPER.md:89, :333,
 * gathering payload columns by the index pairs). Same rows and order as
 * tqp_pkfk_join; for each j < *n_out_host:
 *   build_payload_out[c][j] = build_payload[c][left_j]   (n_build rows each)
 *   probe_payload_out[c][j] = probe_payload[c][right_j]  (n_probe rows each)
 * Outputs have the payload column's dtype and capacity n_probe (caller-allocated
 * device buffers; host arrays of pointers). At most 8 payload columns per side.
 * left_out_idx / right_out_idx are nullable here. Synchronises twice. */
tqp_status tqp_pkfk_join_payload(tqp_ctx* ctx, tqp_col build_keys, int64_t n_build, tqp_col probe_keys,
                                 int64_t n_probe, const tqp_col* build_payload_host, int n_build_payload,
                                 void* const* build_payload_out_host, const tqp_col* probe_payload_host,
                                 int n_probe_payload, void* const* probe_payload_out_host, int64_t* left_out_idx,
                                 int64_t* right_out_idx, int64_t* n_out_host);

/* Hash-join ablation (the comparison point of PAPER.md:1299,
 * not the paper's method): the same PK-FK join contract and output (pairs in
 * ascending probe row, TQP_ERR_DUPLICATE_BUILD_KEY on a repeated build key) from
 * an open-addressing hash table (>= 2 n_build slots, linear probing) instead of
 * the sorted build side. Requires n_build < 2^30. Synchronises once. */
tqp_status tqp_pkfk_join_hash(tqp_ctx* ctx, tqp_col build_keys, int64_t n_build, tqp_col probe_keys,
                              int64_t n_probe, int64_t* left_out_idx, int64_t* right_out_idx, int64_t* n_out_host);

/* Probe-side outer join (the PK-FK match mask of
 * PAPER.md:81 kept for every row): every probe row i in order gets
 * left_out[i] = its build row, or -1 without a match (n_probe x int64,
 * caller-allocated, required); the right index of row i is i itself.
 * match_out (nullable, n_probe x u8) = 1 iff matched; *n_match_host (nullable)
 * = matched rows. Duplicate build keys are not an error: each probe row takes
 * one of the equal build rows. Synchronises twice (three times when the build
 * side is already in key order: its duplicate flag is read before the probe). */
tqp_status tqp_pkfk_outer(tqp_ctx* ctx, tqp_col build_keys, int64_t n_build, tqp_col probe_keys, int64_t n_probe,
                          int64_t* left_out, uint8_t* match_out, int64_t* n_match_host);

/* Outer join preserving the BUILD (primary-key) side -- TPC-H Q13's customer
 * LEFT OUTER JOIN orders shape, where every customer appears with each of its
 * orders or once with a NULL (PAPER.md:1218 names TQP's left outer join as slow;
 * SURVEY.md §8(f) NEXT 1). Output: the inner pairs exactly as tqp_pkfk_join
 * returns them (ascending probe row), followed by (b, -1) for every build row b
 * that no probe row matches, ascending b; right_out = -1 is the match flag.
 * left_out / right_out: device int64, capacity n_probe + n_build (caller-
 * allocated); *n_out_host = pairs + unmatched build rows. Duplicate build keys ->
 * TQP_ERR_DUPLICATE_BUILD_KEY. n_build < 2^32. Synchronises three times. */
tqp_status tqp_pkfk_outer_build(tqp_ctx* ctx, tqp_col build_keys, int64_t n_build, tqp_col probe_keys,
                                int64_t n_probe, int64_t* left_out, int64_t* right_out, int64_t* n_out_host);

/* ------------------------------------------------ m:n sort-merge join */
/* (3) Generic sort-merge join -- Alg. 1 (prose :1114-1137)
 * with readings R2 (ascending sort), R3 (bucketize right=True),
 * R4 (div and remainder by rightHist), R5 (histograms over the
 * keys present on both sides). Output order: key ascending, then left row
 * ascending, then right row ascending (reading R6).
 * prepare: sorts both sides, run-length encodes them (the "bincount"), forms
 * histMul = L*R and cumHistMul over the common keys; *out_size_host = outSize
 * (synchronises; TQP_ERR_OVERFLOW if >= 2^62). The plan lives on the device.
 * expand: writes pairs for output offsets [begin, end) into left_out_idx /
 * right_out_idx ((end - begin) elements each); asynchronous, may be called on
 * any windows of [0, outSize). */
typedef struct tqp_smj_plan tqp_smj_plan;
tqp_status tqp_smj_prepare(tqp_ctx* ctx, tqp_col left, int64_t n_left, tqp_col right, int64_t n_right,
                           tqp_smj_plan** plan, int64_t* out_size_host);
tqp_status tqp_smj_expand(tqp_ctx* ctx, const tqp_smj_plan* plan, int64_t begin, int64_t end,
                          int64_t* left_out_idx, int64_t* right_out_idx);
/* tqp_smj_expand writing int32 indices (same pairs, half the bytes). Requires
 * n_left < 2^31 and n_right < 2^31, else TQP_ERR_INVALID_ARGUMENT. */
tqp_status tqp_smj_expand_i32(tqp_ctx* ctx, const tqp_smj_plan* plan, int64_t begin, int64_t end,
                              int32_t* left_out_idx, int32_t* right_out_idx);
/* Fused consumer of the expansion (for joins whose
 * outSize cannot be materialised, e.g. both-Zipf config 4 with ~4.6e13 pairs):
 * the pairs (l_j, r_j) at output positions j in [begin, end) -- exactly those
 * tqp_smj_expand would write -- are consumed in registers, and
 *   out_host[0] = sum_j mix64(mix64((l_j << 32) | r_j) ^ j)
 *   out_host[1] = sum_j l_j,   out_host[2] = sum_j r_j        (all mod 2^64)
 * with mix64(x): x ^= x >> 30; x *= 0xbf58476d1ce4e5b9; x ^= x >> 27;
 * x *= 0x94d049bb133111eb; x ^= x >> 31 (the splitmix64 finaliser). out_host:
 * 3 x uint64 host array. Synchronises once. */
tqp_status tqp_smj_expand_checksum(tqp_ctx* ctx, const tqp_smj_plan* plan, int64_t begin, int64_t end,
                                   uint64_t* out_host);
/* createOutput fused into the expansion (Alg. 1's return, PAPER.md:333;
 * SURVEY.md §8(f) NEXT 2): for the pairs (l_j, r_j) of output positions j in
 * [begin, end), left_payload_out[c][j - begin] = left_payload[c][l_j] and
 * right_payload_out[c][j - begin] = right_payload[c][r_j]. Payload columns are
 * device columns of the left (n_left rows) / right (n_right rows) relation, any
 * dtype (u8 / i32 / i64 / f64), at most 8 per side (host arrays of columns and of
 * device output pointers, each output end - begin elements of its column's dtype).
 * left_out_idx / right_out_idx (nullable) also receive the index pairs. Asynchronous. */
tqp_status tqp_smj_expand_payload(tqp_ctx* ctx, const tqp_smj_plan* plan, int64_t begin, int64_t end,
                                  const tqp_col* left_payload_host, int n_left_payload, void* const* left_payload_out_host,
                                  const tqp_col* right_payload_host, int n_right_payload,
                                  void* const* right_payload_out_host, int64_t* left_out_idx, int64_t* right_out_idx);
void tqp_smj_release(tqp_ctx* ctx, tqp_smj_plan* plan);
/* prepare + expand of everything into caller buffers of `capacity` pairs.
 * If capacity < outSize: TQP_ERR_CAPACITY and *n_out_host = outSize. */
tqp_status tqp_smj_join(tqp_ctx* ctx, tqp_col left, int64_t n_left, tqp_col right, int64_t n_right,
                        int64_t* left_out_idx, int64_t* right_out_idx, int64_t capacity, int64_t* n_out_host);

/* Multi-column join keys (the key packing of PAPER.md:350,
 * column 0 most significant): the n_cols key columns of two relations a and b are
 * packed into one int64 key per row with a layout shared by both sides:
 *   out[row] = sum_c (u_c(row) - min_c) << shift_c,
 * u_c = the order-preserving unsigned image of column c (value XOR 2^63 of the
 * sign-extended int64), min_c / max_c over both sides, width_c = bits(max_c -
 * min_c), shift_c = sum of the widths of columns c+1 .. n_cols-1. Equal tuples
 * pack equal, different tuples differently, and packed order = lexicographic tuple
 * order, so tqp_pkfk_join / tqp_smj_* on the packed columns join on the tuples.
 * a_cols_host / b_cols_host: host arrays of n_cols columns (n_a / n_b rows; b may be
 * NULL with n_b = 0); a_out / b_out: device int64 (n_a / n_b). *bits_host (nullable):
 * total width. More than 63 bits, or n_cols outside 1..8: TQP_ERR_INVALID_ARGUMENT.
 * Synchronises once. */
tqp_status tqp_pack_keys(tqp_ctx* ctx, const tqp_col* a_cols_host, int64_t n_a, const tqp_col* b_cols_host,
                         int64_t n_b, int n_cols, int64_t* a_out, int64_t* b_out, int* bits_host);

/* ---------------------------------------------------- filter/compaction */
/* (4) Filter -- Listing 1 (bitmap) and Listing 2 (selection
 * vector, reading R20). A row passes iff every predicate
 * `cols[col] <op> value` holds (conjunction, "intersecting the
 * masks using logical_and"). mask_out (nullable): n x u8 in {0,1}; sel_out
 * (nullable): ascending passing rows (capacity n x int64); at least one given.
 * n_sel_host (nullable): number of passing rows (synchronises if given).
 * n < 2^32, else TQP_ERR_INVALID_ARGUMENT. */
typedef enum { TQP_LT = 0, TQP_LE = 1, TQP_GT = 2, TQP_GE = 3, TQP_EQ = 4, TQP_NE = 5 } tqp_cmp;
typedef struct {
    int32_t col;     /* index into cols */
    int32_t op;      /* tqp_cmp */
    int64_t value;   /* compared as int64 with the column value */
} tqp_pred;
#define TQP_MAX_PREDS 16
tqp_status tqp_filter_compact(tqp_ctx* ctx, const tqp_col* cols_host, int n_cols, int64_t n,
                              const tqp_pred* preds_host, int n_preds,
                              uint8_t* mask_out, int64_t* sel_out, int64_t* n_sel_host);

/* -------------------------------------------------------------- group-by */
/* (5) Sort-based group-by aggregation -- Alg. 2 (prose
 * :1146-1152) with an optional fused pre-filter (same predicate form as (4)).
 * Group keys: up to 8 columns, concatenated column 0 most significant
 * (reading R12) into at most 64 bits (u8: 8, i32: 32, i64: 64 bits).
 * Aggregate value per row = prod_{f < n_factors} (add[f] + sign[f] * cols[col[f]])
 * in int64 fixed point (reading R16; the expression form of PAPER.md:1103-1110
 * "sum(l_extendedprice * (1 - l_discount))"); overflow -> TQP_ERR_OVERFLOW.
 * Results: SUM -> int128 (16 bytes, little-endian two's complement, exact);
 * COUNT -> int64 rows of the group (COUNT(*), n_factors ignored);
 * MIN / MAX -> int64; AVG -> double = rn((double)sum / (double)count) (R15/R17).
 * fp64 aggregates: an aggregate with a TQP_F64 factor
 * column is evaluated in fp64, prod_f (add_f + sign_f * x_f) left to right, and
 * SUM / MIN / MAX / AVG return double (8 bytes): SUM in an unspecified order
 * (|error| <= (m - 1) * 2^-53 * sum|v| for a group of m rows), MIN / MAX exact
 * (no NaN inputs), AVG = SUM / COUNT; with no row: SUM 0, MIN +inf, MAX -inf.
 * TQP_F64 columns may not be keys or predicate columns.
 * Groups come out in ascending key order. n_keys == 0 -> exactly one group even
 * if no row passes (SUM 0, COUNT 0, MIN INT64_MAX, MAX INT64_MIN, AVG NaN).
 * Method: each tile of rows is radix-sorted by key in shared memory and reduced
 * per run (segment boundaries + segmented sums); the per-tile partials are
 * radix-sorted globally and reduced again (two-level sort-based aggregation).
 * When at most 16 packed keys occur (packed width <= 16 bits), the keys get dense
 * ids in key order from a presence pass instead and rows are reduced per id without
 * a sort; without group keys the partials are reduced per block. Same results.
 * prepare synchronises and reports *n_groups_host = G; fetch writes:
 *   keys_out[k]   : G elements of key column k's dtype (nullable each)
 *   results_out[a]: G elements of the aggregate's result type (nullable each). */
typedef enum { TQP_SUM = 0, TQP_COUNT = 1, TQP_MIN = 2, TQP_MAX = 3, TQP_AVG = 4 } tqp_aggop;
typedef struct {
    int32_t op;          /* tqp_aggop */
    int32_t n_factors;   /* 0..3 */
    int32_t col[3];
    int32_t sign[3];     /* +1 or -1 */
    int64_t add[3];
} tqp_agg;
#define TQP_MAX_KEYS 8
#define TQP_MAX_AGGS 16
typedef struct tqp_groupby_plan tqp_groupby_plan;
tqp_status tqp_groupby_prepare(tqp_ctx* ctx, const tqp_col* cols_host, int n_cols, int64_t n,
                               const int32_t* key_idx_host, int n_keys,
                               const tqp_pred* preds_host, int n_preds,
                               const tqp_agg* aggs_host, int n_aggs,
                               tqp_groupby_plan** plan, int64_t* n_groups_host);
tqp_status tqp_groupby_fetch(tqp_ctx* ctx, const tqp_groupby_plan* plan, void* const* keys_out_host,
                             void* const* results_out_host);
void tqp_groupby_release(tqp_ctx* ctx, tqp_groupby_plan* plan);
/* Merge partial group-by results -- the "gather and final reduce" of
 * multi-GPU aggregation (the paper's data-parallel future work,
 * PAPER.md:1076). Inputs: m partial rows (e.g. the tqp_groupby_fetch outputs of
 * R ranks, concatenated): key_cols_host[k] = device column of key k (dtype of
 * the original key column); counts = COUNT(*) of each partial row (device,
 * m x int64); partial_host[a] = device array per aggregate a: SUM and AVG ->
 * the exact int128 SUM of aggregate a's expression (m x 16 bytes, fetch
 * layout), MIN / MAX -> m x int64, COUNT -> ignored (may be NULL). The merged
 * groups are fetched with tqp_groupby_fetch; AVG = rn(merged SUM / merged
 * COUNT) -- averages are never averaged. Synchronises once. */
tqp_status tqp_groupby_merge(tqp_ctx* ctx, int64_t m, const tqp_col* key_cols_host, int n_keys,
                             const tqp_agg* aggs_host, int n_aggs, const void* const* partial_host,
                             const int64_t* counts, tqp_groupby_plan** plan, int64_t* n_groups_host);
/* prepare + fetch into caller buffers of `capacity` groups; if capacity < G:
 * TQP_ERR_CAPACITY and *n_groups_host = G. */
tqp_status tqp_groupby_agg(tqp_ctx* ctx, const tqp_col* cols_host, int n_cols, int64_t n,
                           const int32_t* key_idx_host, int n_keys, const tqp_pred* preds_host, int n_preds,
                           const tqp_agg* aggs_host, int n_aggs, void* const* keys_out_host,
                           void* const* results_out_host, int64_t capacity, int64_t* n_groups_host);

/* ------------------------------------------- data-parallel exchange steps */
/* Multi-GPU execution (the paper names data-parallel execution as
 * future work): one process per GPU exchanges (key, global row)
 * pairs with NCCL all_to_all. These calls are the on-GPU steps around that
 * collective; none synchronises with the host.
 *
 * Stable partition by key range. dest(k) = the number of splitters <= k
 * (splitters: device, n_parts - 1 sorted int64; keys compare as signed int64).
 * keys_out (device, n elements of the key dtype) receives the keys grouped by
 * destination 0..n_parts-1, in input order within a destination; rows_out
 * (device int64, nullable) the matching row_base + input row; counts_out (device
 * int64, n_parts) the rows per destination -- the send buffer and split sizes
 * of one all_to_all_single. 1 <= n_parts <= 256; keys u8 / i32 / i64. */
tqp_status tqp_partition(tqp_ctx* ctx, tqp_col keys, int64_t n, const int64_t* splitters, int n_parts,
                         int64_t row_base, void* keys_out, int64_t* rows_out, int64_t* counts_out);
/* The same partition as a fused exchange: no local send buffer, each destination's
 * block written straight into that destination's receive buffer (a peer GPU's memory
 * mapped with tqp_ipc_open -- NVLink P2P stores -- or local memory), so the partition's
 * stores are the all-to-all. Two steps around the count exchange:
 *   tqp_partition_plan_create: the destination histogram + scan; counts_out (device
 *     int64, n_parts) = rows per destination; keys and splitters must stay valid until
 *     the plan is released;
 *   tqp_partition_scatter: destination d's rows (input order kept) go to
 *     dst_keys_host[d] + dst_base_host[d] (elements of the key dtype) and, if
 *     dst_rows_host is not NULL, dst_rows_host[d] + dst_base_host[d] (int64 row_base +
 *     input row). The pointers (host arrays of n_parts device pointers) may be peers'.
 * The caller orders the exchange (all destinations' buffers ready before the scatter,
 * the scatter finished -- device sync + barrier -- before a destination reads). */
typedef struct tqp_partition_plan tqp_partition_plan;
tqp_status tqp_partition_plan_create(tqp_ctx* ctx, tqp_col keys, int64_t n, const int64_t* splitters, int n_parts,
                                     int64_t* counts_out, tqp_partition_plan** plan);
tqp_status tqp_partition_scatter(tqp_ctx* ctx, tqp_partition_plan* plan, int64_t row_base,
                                 void* const* dst_keys_host, int64_t* const* dst_rows_host,
                                 const int64_t* dst_base_host);
void tqp_partition_release(tqp_ctx* ctx, tqp_partition_plan* plan);
/* Receive buffers shared between processes (CUDA IPC): tqp_ipc_alloc = an exact
 * cudaMalloc of `bytes` and its 64-byte IPC handle (handle_out: host, 64 bytes);
 * tqp_ipc_open maps a peer process's handle (peer access enabled lazily: NVLink P2P
 * between GPUs, or the same GPU); tqp_ipc_close unmaps; tqp_ipc_free frees. */
tqp_status tqp_ipc_alloc(tqp_ctx* ctx, size_t bytes, void** dev_ptr_out, void* handle_out);
tqp_status tqp_ipc_free(tqp_ctx* ctx, void* dev_ptr);
tqp_status tqp_ipc_open(tqp_ctx* ctx, const void* handle, void** dev_ptr_out);
tqp_status tqp_ipc_close(tqp_ctx* ctx, void* dev_ptr);
/* lohi_out (device, 2 x int64) = [min, max] of the key column; an empty column
 * gives [INT64_MAX, INT64_MIN] (so MIN / MAX all-reduces across ranks ignore it). */
tqp_status tqp_minmax(tqp_ctx* ctx, tqp_col keys, int64_t n, int64_t* lohi_out);
/* Equal-width key ranges from a device [lo, hi] (e.g. all-reduced tqp_minmax):
 * width = (hi - lo) / n_parts + 1, splitters_out[j] = lo + (j + 1) * width
 * (saturating at INT64_MAX), j < n_parts - 1: key k goes to (k - lo) / width. */
tqp_status tqp_range_splitters(tqp_ctx* ctx, const int64_t* lohi, int n_parts, int64_t* splitters_out);
/* out[i] = src[idx[i]] for i < n (device; src any column dtype, out the same
 * dtype; idx device int64 in [0, len(src))). The row mapping of createOutput
 * (PAPER.md:333): join indices into received blocks -> global row numbers. */
tqp_status tqp_gather(tqp_ctx* ctx, tqp_col src, const int64_t* idx, int64_t n, void* out);

#ifdef __cplusplus
}
#endif
#endif /* TQP_H_ */
