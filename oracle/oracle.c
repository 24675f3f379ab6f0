/*
 * oracle.c -- TEST INFRASTRUCTURE ONLY. NOT PART OF THE PRODUCT PATH.
 *
 * A plain, slow, obviously-correct, single-threaded CPU implementation of what
 * the TQP hot path computes (He et al., "Query Processing on Tensor Computation
 * Runtimes", arXiv 2203.01877; PAPER.md = /root/reference/PAPER.md).
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * `--impl reference` legs may load this library. It shares no code, header or
 * table with the CUDA path (paper_2203_01877_b200/csrc); the only numbers both
 * contain are public hash constants (murmur3's fmix64 here for the hash map, also
 * in the CUDA hash-join ablation), which never influence a result.
 *
 * The method reaches exactly (integers are exact) the plain relational result,
 * so every entry point below is the PLAIN DEFINITION written out, not a
 * transcription of the paper's tensor program:
 *
 *   oracle_sort          stable (key, row) order          PAPER.md:296-297 (Alg.1 l.2-3), :352 (Alg.2 l.3)
 *   oracle_pkfk_join     {(b,p): build[b]==probe[p]}       PAPER.md:55-100 (PK-FK join macro)
 *   oracle_nested_join   brute force O(n*m) pairs          SPEC.md:548 (oracle design)
 *   oracle_smj_join      {(l,r): left[l]==right[r]} in (key, l, r) order
 *                                                          PAPER.md:286-338 (Alg. 1), readings R2-R6
 *   oracle_smj_window    the same pairs at output offsets [begin,end), by an
 *                        independent per-offset route (exact cumulative table
 *                        + upper_bound)                    PAPER.md:310-330 (Alg.1 l.9-14)
 *   oracle_filter        rows where every predicate holds  PAPER.md:825-851 (Listings 1-2)
 *   oracle_groupby       per distinct key tuple (lexicographic): sum (int128),
 *                        count, min, max, avg              PAPER.md:340-367 (Alg. 2), :1088 (aggregates)
 *
 * Integer-only except AVG = (double)sum / (double)count (gcc's __int128 -> double
 * conversion is correctly rounded; reading R15/R17 in DESIGN.md).
 * Every function returns a status: 0 ok, 1 invalid argument, 2 duplicate
 * build key, 3 out of memory, 5 overflow, 6 capacity too small.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>

#define OR_OK 0
#define OR_ERR_ARG 1
#define OR_ERR_DUP 2
#define OR_ERR_OOM 3
#define OR_ERR_OVERFLOW 5
#define OR_ERR_CAPACITY 6

typedef __int128 i128;

/* ------------------------------------------------------------------ sort */

typedef struct { int64_t key; int64_t row; } kr_t;

static int cmp_kr_asc(const void* a, const void* b) {
    const kr_t* x = (const kr_t*)a; const kr_t* y = (const kr_t*)b;
    if (x->key != y->key) return x->key < y->key ? -1 : 1;
    return x->row < y->row ? -1 : (x->row > y->row);
}
static int cmp_kr_desc(const void* a, const void* b) {
    const kr_t* x = (const kr_t*)a; const kr_t* y = (const kr_t*)b;
    if (x->key != y->key) return x->key > y->key ? -1 : 1;   /* key descending  */
    return x->row < y->row ? -1 : (x->row > y->row);         /* ties: row ascending (stable) */
}

/* Stable sort (reading R1): perm_out[i] = input row of the i-th element of the
 * (key, row) order; descending orders keys descending with ties still by
 * ascending row. sorted_out (nullable) = keys[perm]. */
int oracle_sort(const int64_t* keys, int64_t n, int descending, int64_t* perm_out, int64_t* sorted_out) {
    if (n < 0) return OR_ERR_ARG;
    if (n == 0) return OR_OK;
    kr_t* a = (kr_t*)malloc(sizeof(kr_t) * (size_t)n);
    if (!a) return OR_ERR_OOM;
    for (int64_t i = 0; i < n; i++) { a[i].key = keys[i]; a[i].row = i; }
    qsort(a, (size_t)n, sizeof(kr_t), descending ? cmp_kr_desc : cmp_kr_asc);
    for (int64_t i = 0; i < n; i++) {
        perm_out[i] = a[i].row;
        if (sorted_out) sorted_out[i] = a[i].key;
    }
    free(a);
    return OR_OK;
}

/* ------------------------------------------------------------ hash map  */
/* open addressing, int64 key -> int64 value; used only by the oracle. */
typedef struct { int64_t* keys; int64_t* vals; uint8_t* used; uint64_t cap; } hmap_t;

static uint64_t hmix(uint64_t x) {
    x ^= x >> 33; x *= 0xff51afd7ed558ccdULL; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ULL; x ^= x >> 33;
    return x;
}
static int hmap_init(hmap_t* h, int64_t n) {
    uint64_t cap = 16;
    while (cap < (uint64_t)n * 2) cap <<= 1;
    h->cap = cap;
    h->keys = (int64_t*)malloc(cap * sizeof(int64_t));
    h->vals = (int64_t*)malloc(cap * sizeof(int64_t));
    h->used = (uint8_t*)calloc(cap, 1);
    return (h->keys && h->vals && h->used) ? OR_OK : OR_ERR_OOM;
}
static void hmap_free(hmap_t* h) { free(h->keys); free(h->vals); free(h->used); }
/* returns slot of key; *found tells whether it existed */
static uint64_t hmap_find(const hmap_t* h, int64_t key, int* found) {
    uint64_t m = h->cap - 1, s = hmix((uint64_t)key) & m;
    while (h->used[s]) {
        if (h->keys[s] == key) { *found = 1; return s; }
        s = (s + 1) & m;
    }
    *found = 0;
    return s;
}

/* --------------------------------------------------------- PK-FK join  */
/* Plain definition: all pairs (b, p) with build[b] == probe[p]; build keys
 * unique (reading R10: duplicate -> status 2); output ordered by probe row p
 * ascending (reading R7). left_out/right_out have capacity n_probe. */
int oracle_pkfk_join(const int64_t* build, int64_t n_build, const int64_t* probe, int64_t n_probe,
                     int64_t* left_out, int64_t* right_out, int64_t* n_out) {
    if (n_build < 0 || n_probe < 0) return OR_ERR_ARG;
    *n_out = 0;
    hmap_t h;
    int st = hmap_init(&h, n_build);
    if (st) { hmap_free(&h); return st; }
    for (int64_t b = 0; b < n_build; b++) {
        int found;
        uint64_t s = hmap_find(&h, build[b], &found);
        if (found) { hmap_free(&h); return OR_ERR_DUP; }
        h.used[s] = 1; h.keys[s] = build[b]; h.vals[s] = b;
    }
    int64_t m = 0;
    for (int64_t p = 0; p < n_probe; p++) {
        int found;
        uint64_t s = hmap_find(&h, probe[p], &found);
        if (found) { left_out[m] = h.vals[s]; right_out[m] = p; m++; }
    }
    *n_out = m;
    hmap_free(&h);
    return OR_OK;
}

/* ------------------------------------------------- nested-loop (brute)  */
/* O(n_left * n_right): every pair (l, r) with left[l] == right[r], emitted in
 * (l, r) loop order. If cap is too small, counts only and returns status 6. */
int oracle_nested_join(const int64_t* left, int64_t n_left, const int64_t* right, int64_t n_right,
                       int64_t* left_out, int64_t* right_out, int64_t cap, int64_t* n_out) {
    int64_t m = 0;
    for (int64_t l = 0; l < n_left; l++)
        for (int64_t r = 0; r < n_right; r++)
            if (left[l] == right[r]) {
                if (m < cap) { left_out[m] = l; right_out[m] = r; }
                m++;
            }
    *n_out = m;
    return m > cap ? OR_ERR_CAPACITY : OR_OK;
}

/* ------------------------------------------------------ m:n join (SMJ)  */
/* Plain definition: all pairs (l, r) with left[l] == right[r], in the order
 * (key ascending, l ascending, r ascending) -- readings R2/R3/R4/R6. Algorithm:
 * sort (key,row) pairs of each side, then for every key present on both sides
 * emit the nested loop over its rows. *out_size = total pairs (status 5 if it
 * exceeds INT64_MAX); if cap < total only counts (status 6). */
int oracle_smj_join(const int64_t* left, int64_t n_left, const int64_t* right, int64_t n_right,
                    int64_t* left_out, int64_t* right_out, int64_t cap, int64_t* out_size) {
    *out_size = 0;
    kr_t* a = (kr_t*)malloc(sizeof(kr_t) * (size_t)(n_left > 0 ? n_left : 1));
    kr_t* b = (kr_t*)malloc(sizeof(kr_t) * (size_t)(n_right > 0 ? n_right : 1));
    if (!a || !b) { free(a); free(b); return OR_ERR_OOM; }
    for (int64_t i = 0; i < n_left; i++) { a[i].key = left[i]; a[i].row = i; }
    for (int64_t i = 0; i < n_right; i++) { b[i].key = right[i]; b[i].row = i; }
    qsort(a, (size_t)n_left, sizeof(kr_t), cmp_kr_asc);
    qsort(b, (size_t)n_right, sizeof(kr_t), cmp_kr_asc);
    i128 total = 0;
    int64_t i = 0, j = 0;
    while (i < n_left && j < n_right) {
        if (a[i].key < b[j].key) { i++; continue; }
        if (a[i].key > b[j].key) { j++; continue; }
        int64_t key = a[i].key, i1 = i, j1 = j;
        while (i1 < n_left && a[i1].key == key) i1++;
        while (j1 < n_right && b[j1].key == key) j1++;
        for (int64_t x = i; x < i1; x++)
            for (int64_t y = j; y < j1; y++) {
                if (total < (i128)cap) { left_out[(int64_t)total] = a[x].row; right_out[(int64_t)total] = b[y].row; }
                total++;
            }
        i = i1; j = j1;
    }
    free(a); free(b);
    if (total > (i128)INT64_MAX) return OR_ERR_OVERFLOW;
    *out_size = (int64_t)total;
    return total > (i128)cap ? OR_ERR_CAPACITY : OR_OK;
}

/* Count-only variant (no pair emission, no nested loops): exact
 * sum over common keys of countL(k) * countR(k). */
int oracle_smj_count(const int64_t* left, int64_t n_left, const int64_t* right, int64_t n_right,
                     int64_t* out_size) {
    *out_size = 0;
    int64_t* a = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n_left > 0 ? n_left : 1));
    int64_t* b = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n_right > 0 ? n_right : 1));
    if (!a || !b) { free(a); free(b); return OR_ERR_OOM; }
    int64_t* pa = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n_left > 0 ? n_left : 1));
    int64_t* pb = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n_right > 0 ? n_right : 1));
    if (!pa || !pb) { free(a); free(b); free(pa); free(pb); return OR_ERR_OOM; }
    oracle_sort(left, n_left, 0, pa, a);
    oracle_sort(right, n_right, 0, pb, b);
    free(pa); free(pb);
    i128 total = 0;
    int64_t i = 0, j = 0;
    while (i < n_left && j < n_right) {
        if (a[i] < b[j]) { i++; continue; }
        if (a[i] > b[j]) { j++; continue; }
        int64_t key = a[i], i1 = i, j1 = j;
        while (i1 < n_left && a[i1] == key) i1++;
        while (j1 < n_right && b[j1] == key) j1++;
        total += (i128)(i1 - i) * (i128)(j1 - j);
        i = i1; j = j1;
    }
    free(a); free(b);
    if (total > (i128)INT64_MAX) return OR_ERR_OVERFLOW;
    *out_size = (int64_t)total;
    return OR_OK;
}

/* Windowed route, independent of oracle_smj_join's emission loop: for each
 * output offset o in [begin, end): find the common key k whose cumulative pair
 * count first exceeds o (upper_bound over an exact cumulative table), then
 * o' = o - pairs before k; left = o' / R_k -th left row of k (ascending),
 * right = o' % R_k -th right row of k (Alg.1 l.12-14, with
 * reading R4: both div and remainder by rightHist). */
int oracle_smj_window(const int64_t* left, int64_t n_left, const int64_t* right, int64_t n_right,
                      int64_t begin, int64_t end, int64_t* left_out, int64_t* right_out) {
    if (begin < 0 || end < begin) return OR_ERR_ARG;
    kr_t* a = (kr_t*)malloc(sizeof(kr_t) * (size_t)(n_left > 0 ? n_left : 1));
    kr_t* b = (kr_t*)malloc(sizeof(kr_t) * (size_t)(n_right > 0 ? n_right : 1));
    /* per common key: start in a, start in b, L, R, cumulative pairs (inclusive) */
    int64_t nk_cap = (n_left < n_right ? n_left : n_right) + 1;
    int64_t* sa = (int64_t*)malloc(sizeof(int64_t) * (size_t)nk_cap);
    int64_t* sb = (int64_t*)malloc(sizeof(int64_t) * (size_t)nk_cap);
    int64_t* cl = (int64_t*)malloc(sizeof(int64_t) * (size_t)nk_cap);
    int64_t* cr = (int64_t*)malloc(sizeof(int64_t) * (size_t)nk_cap);
    i128* cum = (i128*)malloc(sizeof(i128) * (size_t)nk_cap);
    if (!a || !b || !sa || !sb || !cl || !cr || !cum) {
        free(a); free(b); free(sa); free(sb); free(cl); free(cr); free(cum); return OR_ERR_OOM;
    }
    for (int64_t i = 0; i < n_left; i++) { a[i].key = left[i]; a[i].row = i; }
    for (int64_t i = 0; i < n_right; i++) { b[i].key = right[i]; b[i].row = i; }
    qsort(a, (size_t)n_left, sizeof(kr_t), cmp_kr_asc);
    qsort(b, (size_t)n_right, sizeof(kr_t), cmp_kr_asc);
    int64_t nk = 0, i = 0, j = 0;
    i128 run = 0;
    while (i < n_left && j < n_right) {
        if (a[i].key < b[j].key) { i++; continue; }
        if (a[i].key > b[j].key) { j++; continue; }
        int64_t key = a[i].key, i1 = i, j1 = j;
        while (i1 < n_left && a[i1].key == key) i1++;
        while (j1 < n_right && b[j1].key == key) j1++;
        sa[nk] = i; sb[nk] = j; cl[nk] = i1 - i; cr[nk] = j1 - j;
        run += (i128)cl[nk] * (i128)cr[nk];
        cum[nk] = run;
        nk++;
        i = i1; j = j1;
    }
    int st = OR_OK;
    if ((i128)end > run) st = OR_ERR_ARG;
    for (int64_t o = begin; st == OR_OK && o < end; o++) {
        /* upper_bound: smallest k with o < cum[k] */
        int64_t lo = 0, hi = nk;
        while (lo < hi) {
            int64_t mid = lo + (hi - lo) / 2;
            if ((i128)o < cum[mid]) hi = mid; else lo = mid + 1;
        }
        int64_t k = lo;
        i128 before = cum[k] - (i128)cl[k] * (i128)cr[k];
        int64_t off = (int64_t)((i128)o - before);
        int64_t q = off / cr[k], r = off % cr[k];
        left_out[o - begin] = a[sa[k] + q].row;
        right_out[o - begin] = b[sb[k] + r].row;
    }
    free(a); free(b); free(sa); free(sb); free(cl); free(cr); free(cum);
    return st;
}

/* ------------------------------------------------------------- filter  */
/* predicate: cols[col][row] <op> value, all columns widened to int64 by the
 * caller (u8 unsigned, i32/i64 signed -- values compare identically). */
typedef struct { int32_t col; int32_t op; int64_t value; } or_pred;
enum { OR_LT = 0, OR_LE = 1, OR_GT = 2, OR_GE = 3, OR_EQ = 4, OR_NE = 5 };

static int pred_holds(const int64_t* const* cols, const or_pred* p, int64_t row) {
    int64_t x = cols[p->col][row], v = p->value;
    switch (p->op) {
        case OR_LT: return x < v;
        case OR_LE: return x <= v;
        case OR_GT: return x > v;
        case OR_GE: return x >= v;
        case OR_EQ: return x == v;
        case OR_NE: return x != v;
    }
    return 0;
}
static int row_passes(const int64_t* const* cols, const or_pred* preds, int n_preds, int64_t row) {
    for (int q = 0; q < n_preds; q++)
        if (!pred_holds(cols, &preds[q], row)) return 0;
    return 1;
}

/* Listing 1 (bitmap) and Listing 2 (selection vector), PAPER.md:832-850:
 * mask[row] = AND of predicates; sel = ascending rows with mask == 1. */
int oracle_filter(const int64_t* const* cols, int n_cols, int64_t n, const or_pred* preds, int n_preds,
                  uint8_t* mask_out, int64_t* sel_out, int64_t* n_sel) {
    for (int q = 0; q < n_preds; q++)
        if (preds[q].col < 0 || preds[q].col >= n_cols || preds[q].op < 0 || preds[q].op > 5) return OR_ERR_ARG;
    int64_t m = 0;
    for (int64_t row = 0; row < n; row++) {
        int pass = row_passes(cols, preds, n_preds, row);
        if (mask_out) mask_out[row] = (uint8_t)pass;
        if (pass) { if (sel_out) sel_out[m] = row; m++; }
    }
    *n_sel = m;
    return OR_OK;
}

/* ------------------------------------------------------------ group-by */
/* aggregate: op over the per-row value v = prod_{f < n_factors}(add[f] + sign[f]*cols[col[f]][row])
 * computed in int64 (overflow -> status 5). COUNT = number of rows (COUNT(*)). */
typedef struct { int32_t op; int32_t n_factors; int32_t col[3]; int32_t sign[3]; int64_t add[3]; } or_agg;
enum { OR_SUM = 0, OR_COUNT = 1, OR_MIN = 2, OR_MAX = 3, OR_AVG = 4 };

typedef struct {
    i128* sum;      /* per aggregate */
    int64_t* mn;
    int64_t* mx;
    int64_t count;
    int64_t first_row; /* a row of this group, to read back its key tuple */
} grp_t;

static int agg_value(const int64_t* const* cols, const or_agg* a, int64_t row, int64_t* out) {
    int64_t v = 1;
    for (int f = 0; f < a->n_factors; f++) {
        int64_t x = cols[a->col[f]][row], t, term;
        if (__builtin_mul_overflow((int64_t)a->sign[f], x, &t)) return OR_ERR_OVERFLOW;
        if (__builtin_add_overflow(a->add[f], t, &term)) return OR_ERR_OVERFLOW;
        if (__builtin_mul_overflow(v, term, &v)) return OR_ERR_OVERFLOW;
    }
    *out = v;
    return OR_OK;
}

/* key tuples are compared lexicographically, column 0 most significant
 * (reading R12); the hash map below is keyed by the tuple. */
static const int64_t* const* g_cols;
static const int* g_key_idx;
static int g_n_keys;
static int cmp_group_rows(const void* a, const void* b) {
    int64_t ra = *(const int64_t*)a, rb = *(const int64_t*)b;
    for (int k = 0; k < g_n_keys; k++) {
        int64_t x = g_cols[g_key_idx[k]][ra], y = g_cols[g_key_idx[k]][rb];
        if (x != y) return x < y ? -1 : 1;
    }
    return 0;
}
static uint64_t tuple_hash(const int64_t* const* cols, const int* key_idx, int n_keys, int64_t row) {
    uint64_t h = 0x9E3779B97F4A7C15ULL;
    for (int k = 0; k < n_keys; k++) h = hmix(h ^ (uint64_t)cols[key_idx[k]][row]) + (uint64_t)k;
    return h;
}
static int tuple_eq(const int64_t* const* cols, const int* key_idx, int n_keys, int64_t r1, int64_t r2) {
    for (int k = 0; k < n_keys; k++)
        if (cols[key_idx[k]][r1] != cols[key_idx[k]][r2]) return 0;
    return 1;
}

/*
 * Output: *n_groups = G; keys_out[g*n_keys + k] = key column k of group g;
 * results[(g*n_aggs + a)*2 + {0,1}]:
 *   SUM   -> (low 64 bits, high 64 bits) of the int128 sum
 *   COUNT -> (count, 0);  MIN/MAX -> (value, 0);  AVG -> (bits of the double, 0)
 * Groups are in lexicographic key order. n_keys == 0 -> exactly one group even
 * when no row passes (SUM 0, COUNT 0, MIN INT64_MAX, MAX INT64_MIN, AVG NaN).
 * If cap < G: *n_groups = G and status 6 (nothing written).
 */
int oracle_groupby(const int64_t* const* cols, int n_cols, int64_t n, const int* key_idx, int n_keys,
                   const or_pred* preds, int n_preds, const or_agg* aggs, int n_aggs,
                   int64_t cap, int64_t* n_groups, int64_t* keys_out, int64_t* results) {
    if (n < 0 || n_keys < 0 || n_aggs < 0) return OR_ERR_ARG;
    for (int k = 0; k < n_keys; k++) if (key_idx[k] < 0 || key_idx[k] >= n_cols) return OR_ERR_ARG;
    for (int q = 0; q < n_preds; q++)
        if (preds[q].col < 0 || preds[q].col >= n_cols || preds[q].op < 0 || preds[q].op > 5) return OR_ERR_ARG;
    for (int a = 0; a < n_aggs; a++) {
        if (aggs[a].op < 0 || aggs[a].op > 4 || aggs[a].n_factors < 0 || aggs[a].n_factors > 3) return OR_ERR_ARG;
        for (int f = 0; f < aggs[a].n_factors; f++)
            if (aggs[a].col[f] < 0 || aggs[a].col[f] >= n_cols) return OR_ERR_ARG;
    }
    /* hash map: tuple -> group index (grown by doubling) */
    uint64_t hcap = 1024;
    int64_t* slot_row = (int64_t*)malloc(hcap * sizeof(int64_t));
    int64_t* slot_grp = (int64_t*)malloc(hcap * sizeof(int64_t));
    if (!slot_row || !slot_grp) { free(slot_row); free(slot_grp); return OR_ERR_OOM; }
    for (uint64_t s = 0; s < hcap; s++) slot_row[s] = -1;
    int64_t gcap = 64, G = 0;
    grp_t* g = (grp_t*)malloc(sizeof(grp_t) * (size_t)gcap);
    int st = OR_OK;
    if (n_keys == 0) { /* the single global group always exists */
        g[0].sum = (i128*)calloc((size_t)(n_aggs + 1), sizeof(i128));
        g[0].mn = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n_aggs + 1));
        g[0].mx = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n_aggs + 1));
        for (int a = 0; a < n_aggs; a++) { g[0].mn[a] = INT64_MAX; g[0].mx[a] = INT64_MIN; }
        g[0].count = 0; g[0].first_row = -1; G = 1;
    }
    for (int64_t row = 0; row < n && st == OR_OK; row++) {
        if (!row_passes(cols, preds, n_preds, row)) continue;
        int64_t gi = 0;
        if (n_keys > 0) {
            uint64_t m = hcap - 1, s = tuple_hash(cols, key_idx, n_keys, row) & m;
            while (slot_row[s] >= 0 && !tuple_eq(cols, key_idx, n_keys, slot_row[s], row)) s = (s + 1) & m;
            if (slot_row[s] >= 0) gi = slot_grp[s];
            else {
                if (G == gcap) { gcap *= 2; g = (grp_t*)realloc(g, sizeof(grp_t) * (size_t)gcap); }
                gi = G++;
                g[gi].sum = (i128*)calloc((size_t)(n_aggs + 1), sizeof(i128));
                g[gi].mn = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n_aggs + 1));
                g[gi].mx = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n_aggs + 1));
                for (int a = 0; a < n_aggs; a++) { g[gi].mn[a] = INT64_MAX; g[gi].mx[a] = INT64_MIN; }
                g[gi].count = 0; g[gi].first_row = row;
                slot_row[s] = row; slot_grp[s] = gi;
                if ((uint64_t)G * 2 > hcap) { /* rehash */
                    uint64_t ncap = hcap * 2;
                    int64_t* nr = (int64_t*)malloc(ncap * sizeof(int64_t));
                    int64_t* ng = (int64_t*)malloc(ncap * sizeof(int64_t));
                    for (uint64_t t = 0; t < ncap; t++) nr[t] = -1;
                    for (uint64_t t = 0; t < hcap; t++) if (slot_row[t] >= 0) {
                        uint64_t u = tuple_hash(cols, key_idx, n_keys, slot_row[t]) & (ncap - 1);
                        while (nr[u] >= 0) u = (u + 1) & (ncap - 1);
                        nr[u] = slot_row[t]; ng[u] = slot_grp[t];
                    }
                    free(slot_row); free(slot_grp); slot_row = nr; slot_grp = ng; hcap = ncap;
                }
            }
        }
        g[gi].count++;
        for (int a = 0; a < n_aggs; a++) {
            if (aggs[a].op == OR_COUNT) continue;
            int64_t v;
            st = agg_value(cols, &aggs[a], row, &v);
            if (st) break;
            g[gi].sum[a] += (i128)v;
            if (v < g[gi].mn[a]) g[gi].mn[a] = v;
            if (v > g[gi].mx[a]) g[gi].mx[a] = v;
        }
    }
    if (st == OR_OK) {
        *n_groups = G;
        if (G > cap) st = OR_ERR_CAPACITY;
    }
    if (st == OR_OK) {
        /* order groups lexicographically by key tuple (via a representative row) */
        int64_t* rows = (int64_t*)malloc(sizeof(int64_t) * (size_t)(G ? G : 1));
        int64_t* idx_of_row_order = (int64_t*)malloc(sizeof(int64_t) * (size_t)(G ? G : 1));
        for (int64_t i = 0; i < G; i++) rows[i] = g[i].first_row;
        g_cols = cols; g_key_idx = key_idx; g_n_keys = n_keys;
        if (n_keys > 0) qsort(rows, (size_t)G, sizeof(int64_t), cmp_group_rows);
        /* map sorted representative rows back to group slots via the hash map */
        for (int64_t i = 0; i < G; i++) {
            if (n_keys == 0) { idx_of_row_order[i] = 0; continue; }
            uint64_t m = hcap - 1, s = tuple_hash(cols, key_idx, n_keys, rows[i]) & m;
            while (!tuple_eq(cols, key_idx, n_keys, slot_row[s], rows[i])) s = (s + 1) & m;
            idx_of_row_order[i] = slot_grp[s];
        }
        for (int64_t i = 0; i < G; i++) {
            grp_t* gg = &g[idx_of_row_order[i]];
            for (int k = 0; k < n_keys; k++) keys_out[i * n_keys + k] = cols[key_idx[k]][gg->first_row];
            for (int a = 0; a < n_aggs; a++) {
                int64_t* r = &results[(i * n_aggs + a) * 2];
                switch (aggs[a].op) {
                    case OR_SUM: { unsigned __int128 u = (unsigned __int128)gg->sum[a];
                                   r[0] = (int64_t)(uint64_t)u; r[1] = (int64_t)(uint64_t)(u >> 64); break; }
                    case OR_COUNT: r[0] = gg->count; r[1] = 0; break;
                    case OR_MIN: r[0] = gg->mn[a]; r[1] = 0; break;
                    case OR_MAX: r[0] = gg->mx[a]; r[1] = 0; break;
                    case OR_AVG: { double d = gg->count ? (double)gg->sum[a] / (double)gg->count : NAN;
                                   memcpy(&r[0], &d, sizeof(double)); r[1] = 0; break; }
                }
            }
        }
        free(rows); free(idx_of_row_order);
    }
    for (int64_t i = 0; i < G; i++) { free(g[i].sum); free(g[i].mn); free(g[i].mx); }
    free(g); free(slot_row); free(slot_grp);
    return st;
}
