/*
 * ahs_oracle.c — plain, slow, single-threaded CPU oracle for the Adaptive
 * Hybrid Sort hot path (arXiv 2506.20677).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * It shares no code, header, table or constant generator with the CUDA path
 * (paper_2506_20677_b200/csrc); neither includes or links the other.
 *
 * Everything follows the paper's definitions / listings in the paper's order;
 * citations are PAPER.md line numbers ("P:n") with section / listing, and the
 * readings taken where the paper is garbled are the ones listed in DESIGN.md
 * §3.
 *
 *   oracle_features   P:96 (§III.A state vector v = (n, k, H)),
 *                     P:292 (§III.H H = -sum p_i log2 p_i), reading A1/A16
 *                     (equal power-of-two-width buckets, at most 2^bits),
 *                     descents per BASELINE.json north_star / reading A14.
 *   oracle_h_exact    P:96 per-value entropy (reading "P"), context only.
 *   oracle_select     P:96-98 (§III.A FSM), Table II P:140-145 thresholds,
 *                     P:411 (§III.K empty / constant shortcuts), A2..A8.
 *   oracle_insertion  Listing 1, P:157-180 (§III.E).
 *   oracle_counting   Listing 2, P:182-216 (§III.F): histogram, inclusive
 *                     prefix, reverse traversal (stable).
 *   oracle_radix      §III.G P:218-251 base 256 for k > 10^6, digit count
 *                     d = ceil(log_256 k) (Eq. 4), each digit a
 *                     stable counting pass as in Listing 2; offset key - min
 *                     (reading A9/A10 instead of Listing 7's unstable reverse).
 *   oracle_quicksort  Listing 4, P:253-288 (§III.G.1): median-of-three pivot;
 *                     3-way partition, insertion leaf and heapsort depth guard
 *                     (reading A13).  Records compare (key, original index),
 *                     so the result is the unique stable order.
 *
 * Key types: int32, uint32, int64, uint64 (SPEC's SortKey is i64, S:20;
 * NEXT-3 in SURVEY §8(f)).  Every function works on the ORDER-PRESERVING
 * UNSIGNED IMAGE u of a key (signed types: the sign bit flipped), so unsigned
 * comparison of images is the keys' order and u - u_min = key - min exactly.
 * k = max - min + 1 can be 2^64 for 64-bit keys: it is computed in 128-bit
 * arithmetic and reported saturated at 2^64 - 1 with ORF_K_SATURATED.
 *
 * Parity pins: tests/test_oracle.py (brute force over all permutations for
 * n <= 8 against Python's sorted(), entropy closed forms, SPEC worked examples,
 * golden fixtures in tests/golden/).  H_exact is context only ("parity
 * unpinned" for the A1/A2 reading choice itself).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ---- independent type definitions (NOT shared with include/ahs.h) ---- */
typedef struct {
    uint64_t n;
    int64_t min, max;
    uint64_t k;
    uint32_t bits, shift, nb, dtype;
    double entropy;
    uint64_t descents;
    uint32_t flags;
    uint32_t pad;
} oracle_features_t;

enum { OR_I32 = 0, OR_U32 = 1, OR_I64 = 2, OR_U64 = 3 };
enum { ORF_EMPTY = 1, ORF_CONSTANT = 2, ORF_BUCKETED = 4, ORF_SORTED = 8,
       ORF_STRICT_DESC = 16, ORF_SIGNED = 32, ORF_K_SATURATED = 64 };
/* the paper's four algorithms, §III.A */
enum { OR_INSERTION = 0, OR_COUNTING = 1, OR_RADIX = 2, OR_QUICK = 3 };
enum { ORR_EMPTY = 0, ORR_CONSTANT = 1, ORR_SMALL_N = 2, ORR_SMALL_RANGE = 3,
       ORR_LOW_ENTROPY = 4, ORR_DEFAULT = 5 };

static int dtype_ok(int dtype) { return dtype >= OR_I32 && dtype <= OR_U64; }
static int dtype_signed(int dtype) { return dtype == OR_I32 || dtype == OR_I64; }
static size_t key_bytes(int dtype) { return dtype >= OR_I64 ? 8 : 4; }

/* order-preserving unsigned image of key i (sign bit flipped for signed types) */
static uint64_t key_at(const void *keys, int dtype, uint64_t i)
{
    switch (dtype) {
    case OR_I32: return (uint64_t)(((const uint32_t *)keys)[i] ^ 0x80000000u);
    case OR_U32: return (uint64_t)((const uint32_t *)keys)[i];
    case OR_I64: return ((const uint64_t *)keys)[i] ^ 0x8000000000000000ull;
    default: return ((const uint64_t *)keys)[i];
    }
}

/* inverse of key_at: store the key whose image is u */
static void key_put(void *keys, int dtype, uint64_t i, uint64_t u)
{
    switch (dtype) {
    case OR_I32: ((uint32_t *)keys)[i] = (uint32_t)u ^ 0x80000000u; break;
    case OR_U32: ((uint32_t *)keys)[i] = (uint32_t)u; break;
    case OR_I64: ((uint64_t *)keys)[i] = u ^ 0x8000000000000000ull; break;
    default: ((uint64_t *)keys)[i] = u; break;
    }
}

/* the key with image u as a 64-bit integer: its value for the signed types
 * and uint32, its bit pattern for uint64 */
static int64_t key_value(int dtype, uint64_t u)
{
    switch (dtype) {
    case OR_I32: return (int64_t)(int32_t)((uint32_t)u ^ 0x80000000u);
    case OR_U32: return (int64_t)u;
    case OR_I64: return (int64_t)(u ^ 0x8000000000000000ull);
    default: return (int64_t)u;
    }
}

/* number of bits needed to write x in binary; bitlen(0) = 0 */
static uint32_t bitlen(uint64_t x)
{
    uint32_t b = 0;
    while (x) { b++; x >>= 1; }
    return b;
}

/* -------------------------------------------------------------------------
 * Features: v = (n, k, H), plus min, max and the descent count.
 * hist_out (nullable) receives the nb bucket counts.
 * Returns 0, or -1 on bad arguments.
 * ------------------------------------------------------------------------- */
int oracle_features(const void *keys, uint64_t n, int dtype, uint32_t entropy_bits,
                    oracle_features_t *out, uint64_t *hist_out)
{
    if (!out || !dtype_ok(dtype) || entropy_bits == 0 || entropy_bits > 32)
        return -1;
    memset(out, 0, sizeof(*out));
    out->n = n;
    out->dtype = (uint32_t)dtype;
    if (dtype_signed(dtype)) out->flags |= ORF_SIGNED;
    if (n == 0) {                      /* empty array, O(1) exit */
        out->flags |= ORF_EMPTY;
        return 0;
    }
    if (!keys) return -1;

    /* pass 1: min, max (P:397 Math.min/max), descents (reading A14) */
    uint64_t mn = key_at(keys, dtype, 0), mx = mn;
    uint64_t desc = 0;
    for (uint64_t i = 0; i < n; i++) {
        uint64_t v = key_at(keys, dtype, i);
        if (v < mn) mn = v;
        if (v > mx) mx = v;
        if (i + 1 < n && v > key_at(keys, dtype, i + 1)) desc++;
    }
    out->min = key_value(dtype, mn);
    out->max = key_value(dtype, mx);
    out->descents = desc;
    /* k = max(arr) - min(arr) + 1, in 128-bit arithmetic: up to
     * 2^64 for 64-bit keys, reported saturated at 2^64 - 1 */
    unsigned __int128 k = (unsigned __int128)(mx - mn) + 1u;
    out->k = k > (unsigned __int128)UINT64_MAX ? UINT64_MAX : (uint64_t)k;
    if (k > (unsigned __int128)UINT64_MAX) out->flags |= ORF_K_SATURATED;
    out->bits = bitlen(mx - mn); /* = bitlen(k - 1) */
    out->shift = out->bits > entropy_bits ? out->bits - entropy_bits : 0;
    out->nb = (uint32_t)(((mx - mn) >> out->shift) + 1);
    if (out->shift > 0) out->flags |= ORF_BUCKETED;
    if (k == 1) out->flags |= ORF_CONSTANT;
    if (desc == 0) out->flags |= ORF_SORTED;
    if (n >= 2 && desc == n - 1) out->flags |= ORF_STRICT_DESC;

    /* pass 2: bucket counts c_b = #{i : (key_i - min) >> s == b} (reading A1/A16) */
    uint64_t *c = (uint64_t *)calloc(out->nb, sizeof(uint64_t));
    if (!c) return -2;
    for (uint64_t i = 0; i < n; i++) {
        uint64_t off = key_at(keys, dtype, i) - mn;
        c[off >> out->shift]++;
    }

    /* H = -sum_b p_b log2 p_b, p_b = c_b / n, ascending b,
     * Kahan-compensated (reading A15); then clamp to [0, log2 nb]. */
    double sum = 0.0, comp = 0.0;
    for (uint32_t b = 0; b < out->nb; b++) {
        if (c[b] == 0) continue;
        double p = (double)c[b] / (double)n;
        double term = -p * log2(p);
        double y = term - comp;
        double t = sum + y;
        comp = (t - sum) - y;
        sum = t;
    }
    double hmax = log2((double)out->nb);
    if (sum < 0.0) sum = 0.0;
    if (sum > hmax) sum = hmax;
    out->entropy = sum;
    if (hist_out) memcpy(hist_out, c, sizeof(uint64_t) * out->nb);
    free(c);
    return 0;
}

/* Exact per-value entropy (reading "P") from the run lengths of an
 * already sorted key array.  Context only, not a parity field. */
double oracle_h_exact(const void *sorted_keys, uint64_t n, int dtype)
{
    if (n == 0) return 0.0;
    double sum = 0.0, comp = 0.0;
    uint64_t run = 1;
    for (uint64_t i = 1; i <= n; i++) {
        if (i < n && key_at(sorted_keys, dtype, i) == key_at(sorted_keys, dtype, i - 1)) {
            run++;
            continue;
        }
        double p = (double)run / (double)n;
        double term = -p * log2(p);
        double y = term - comp;
        double t = sum + y;
        comp = (t - sum) - y;
        sum = t;
        run = 1;
    }
    return sum < 0.0 ? 0.0 : sum;
}

/* -------------------------------------------------------------------------
 * FSM (§III.A, Fig. 2; shortcuts P:411 §III.K; reading A2..A8).
 * norm: 0 = BUCKETS (H < c*log2 nb, reading A2), 1 = RANGE (H < c*log2 k).
 * strategy4 receives the paper's algorithm (OR_INSERTION .. OR_QUICK),
 * rule which rule fired.  Returns 0 or -1 for invalid thresholds.
 * ------------------------------------------------------------------------- */
int oracle_select(const oracle_features_t *f, uint64_t n_insertion, uint64_t k_counting,
                  uint64_t k_radix, double entropy_coeff, int norm,
                  int *strategy4, int *rule)
{
    if (!f || !strategy4 || !rule) return -1;
    if (n_insertion == 0 || k_counting == 0 || k_radix == 0 || !(k_counting < k_radix) ||
        !(entropy_coeff > 0.0 && entropy_coeff <= 1.0) || (norm != 0 && norm != 1))
        return -1;
    if (f->n == 0) { *strategy4 = OR_COUNTING; *rule = ORR_EMPTY; return 0; }
    if (f->k == 1) { *strategy4 = OR_COUNTING; *rule = ORR_CONSTANT; return 0; }
    if (f->n <= n_insertion) { *strategy4 = OR_INSERTION; *rule = ORR_SMALL_N; return 0; }
    if (f->k <= k_counting) { *strategy4 = OR_COUNTING; *rule = ORR_SMALL_RANGE; return 0; }
    double base = norm == 0 ? (double)f->nb : (double)f->k;
    if (f->k > k_radix && f->entropy < entropy_coeff * log2(base)) {
        *strategy4 = OR_RADIX; *rule = ORR_LOW_ENTROPY; return 0;
    }
    *strategy4 = OR_QUICK; *rule = ORR_DEFAULT;
    return 0;
}

/* -------------------------------------------------------------------------
 * Insertion sort, Listing 1.  Values move with their keys.
 * ------------------------------------------------------------------------- */
void oracle_insertion(void *keys, uint32_t *vals, uint64_t n, int dtype)
{
    for (uint64_t i = 1; i < n; i++) {
        uint64_t key = key_at(keys, dtype, i);
        uint32_t val = vals ? vals[i] : 0;
        int64_t j = (int64_t)i - 1;
        while (j >= 0 && key_at(keys, dtype, (uint64_t)j) > key) {
            key_put(keys, dtype, (uint64_t)j + 1, key_at(keys, dtype, (uint64_t)j));
            if (vals) vals[j + 1] = vals[j];
            j--;
        }
        key_put(keys, dtype, (uint64_t)(j + 1), key);
        if (vals) vals[j + 1] = val;
    }
}

/* -------------------------------------------------------------------------
 * Counting sort, Listing 2.  range = max - min + 1 counters,
 * inclusive prefix, reverse traversal output[--count[x - min]] = x.
 * Returns 0, or -3 if the range is too large for a dense count array.
 * ------------------------------------------------------------------------- */
#define ORACLE_COUNTING_MAX_RANGE (1ull << 28)
int oracle_counting(const void *keys, const uint32_t *vals, uint64_t n, int dtype,
                    void *out_keys, uint32_t *out_vals)
{
    if (n == 0) return 0;
    uint64_t mn = key_at(keys, dtype, 0), mx = mn;
    for (uint64_t i = 0; i < n; i++) {
        uint64_t v = key_at(keys, dtype, i);
        if (v < mn) mn = v;
        if (v > mx) mx = v;
    }
    if (mx - mn >= ORACLE_COUNTING_MAX_RANGE) return -3;
    uint64_t range = mx - mn + 1;
    uint64_t *count = (uint64_t *)calloc(range, sizeof(uint64_t));
    if (!count) return -2;
    for (uint64_t i = 0; i < n; i++) count[key_at(keys, dtype, i) - mn]++;      /* count */
    for (uint64_t i = 1; i < range; i++) count[i] += count[i - 1];             /* prefix */
    for (uint64_t i = n; i-- > 0;) {                                           /* output */
        uint64_t x = key_at(keys, dtype, i);
        uint64_t pos = --count[x - mn];
        key_put(out_keys, dtype, pos, x);
        if (out_vals) out_vals[pos] = vals[i];
    }
    free(count);
    return 0;
}

/* -------------------------------------------------------------------------
 * Radix sort (§III.G): base b = 256, on u = key - min (reading A9),
 * d = ceil(log_b k) digits (Eq. 4), each digit sorted by a stable
 * counting pass exactly as Listing 2 (count, inclusive prefix, reverse
 * traversal).  Output key = u + min.
 * ------------------------------------------------------------------------- */
int oracle_radix(const void *keys, const uint32_t *vals, uint64_t n, int dtype,
                 void *out_keys, uint32_t *out_vals)
{
    if (n == 0) return 0;
    uint64_t mn = key_at(keys, dtype, 0), mx = mn;
    for (uint64_t i = 0; i < n; i++) {
        uint64_t v = key_at(keys, dtype, i);
        if (v < mn) mn = v;
        if (v > mx) mx = v;
    }
    unsigned __int128 k = (unsigned __int128)(mx - mn) + 1u; /* up to 2^64 */
    /* Eq. 4: d = ceil(log_256 k) = least d with 256^d >= k */
    uint32_t d = 0;
    for (unsigned __int128 p = 1; p < k; p *= 256) d++;

    uint64_t *a = (uint64_t *)malloc(n * sizeof(uint64_t));
    uint64_t *b = (uint64_t *)malloc(n * sizeof(uint64_t));
    uint32_t *va = vals ? (uint32_t *)malloc(n * sizeof(uint32_t)) : NULL;
    uint32_t *vb = vals ? (uint32_t *)malloc(n * sizeof(uint32_t)) : NULL;
    if (!a || !b || (vals && (!va || !vb))) { free(a); free(b); free(va); free(vb); return -2; }
    for (uint64_t i = 0; i < n; i++) {
        a[i] = key_at(keys, dtype, i) - mn;
        if (vals) va[i] = vals[i];
    }
    for (uint32_t digit = 0; digit < d; digit++) {
        uint64_t count[256];
        memset(count, 0, sizeof(count));
        uint32_t sh = 8 * digit;
        for (uint64_t i = 0; i < n; i++) count[(a[i] >> sh) & 255]++;
        for (int i = 1; i < 256; i++) count[i] += count[i - 1];
        for (uint64_t i = n; i-- > 0;) {
            uint64_t pos = --count[(a[i] >> sh) & 255];
            b[pos] = a[i];
            if (vals) vb[pos] = va[i];
        }
        uint64_t *t = a; a = b; b = t;
        if (vals) { uint32_t *tv = va; va = vb; vb = tv; }
    }
    for (uint64_t i = 0; i < n; i++) {
        key_put(out_keys, dtype, i, a[i] + mn);
        if (vals) out_vals[i] = va[i];
    }
    free(a); free(b); free(va); free(vb);
    return 0;
}

/* -------------------------------------------------------------------------
 * QuickSort (Listing 4) over records (key, original index).
 * Pivot = median of a[lo], a[lo + len/2], a[hi].  3-way
 * partition, insertion sort for len <= 20 (Listing 1 as the leaf), recurse
 * on the smaller side / loop on the larger, heapsort past depth
 * 2*log2(n) + 64 (reading A13).
 * ------------------------------------------------------------------------- */
typedef struct { uint64_t key; uint64_t idx; } rec_t; /* key: the ordered image */

static int rec_lt(const rec_t *x, const rec_t *y)
{
    return x->key < y->key || (x->key == y->key && x->idx < y->idx);
}

static void rec_insertion(rec_t *a, int64_t lo, int64_t hi)
{
    for (int64_t i = lo + 1; i <= hi; i++) {
        rec_t key = a[i];
        int64_t j = i - 1;
        while (j >= lo && rec_lt(&key, &a[j])) { a[j + 1] = a[j]; j--; }
        a[j + 1] = key;
    }
}

static void rec_sift(rec_t *a, int64_t lo, int64_t start, int64_t len)
{
    int64_t root = start;
    for (;;) {
        int64_t child = 2 * root + 1;
        if (child >= len) break;
        if (child + 1 < len && rec_lt(&a[lo + child], &a[lo + child + 1])) child++;
        if (!rec_lt(&a[lo + root], &a[lo + child])) break;
        rec_t t = a[lo + root]; a[lo + root] = a[lo + child]; a[lo + child] = t;
        root = child;
    }
}

static void rec_heapsort(rec_t *a, int64_t lo, int64_t hi)
{
    int64_t len = hi - lo + 1;
    for (int64_t s = len / 2 - 1; s >= 0; s--) rec_sift(a, lo, s, len);
    for (int64_t end = len - 1; end > 0; end--) {
        rec_t t = a[lo]; a[lo] = a[lo + end]; a[lo + end] = t;
        rec_sift(a, lo, 0, end);
    }
}

static rec_t median_of_three(const rec_t *a, int64_t lo, int64_t hi)
{
    rec_t x = a[lo], y = a[lo + (hi - lo + 1) / 2], z = a[hi];
    /* sort three and take the middle */
    if (rec_lt(&y, &x)) { rec_t t = x; x = y; y = t; }
    if (rec_lt(&z, &y)) { rec_t t = y; y = z; z = t; }
    if (rec_lt(&y, &x)) { rec_t t = x; x = y; y = t; }
    return y;
}

static void rec_quicksort(rec_t *a, int64_t lo, int64_t hi, int depth_left)
{
    while (hi - lo + 1 > 20) {
        if (depth_left-- <= 0) { rec_heapsort(a, lo, hi); return; }
        rec_t pivot = median_of_three(a, lo, hi);
        /* 3-way partition: [lo, lt) < pivot, [lt, gt] == pivot, (gt, hi] > pivot */
        int64_t lt = lo, i = lo, gt = hi;
        while (i <= gt) {
            if (rec_lt(&a[i], &pivot)) { rec_t t = a[lt]; a[lt] = a[i]; a[i] = t; lt++; i++; }
            else if (rec_lt(&pivot, &a[i])) { rec_t t = a[gt]; a[gt] = a[i]; a[i] = t; gt--; }
            else i++;
        }
        if (lt - lo < hi - gt) { rec_quicksort(a, lo, lt - 1, depth_left); lo = gt + 1; }
        else { rec_quicksort(a, gt + 1, hi, depth_left); hi = lt - 1; }
    }
    if (hi > lo) rec_insertion(a, lo, hi);
}

int oracle_quicksort(const void *keys, const uint32_t *vals, uint64_t n, int dtype,
                     void *out_keys, uint32_t *out_vals)
{
    if (n == 0) return 0;
    rec_t *a = (rec_t *)malloc(n * sizeof(rec_t));
    if (!a) return -2;
    for (uint64_t i = 0; i < n; i++) { a[i].key = key_at(keys, dtype, i); a[i].idx = i; }
    int depth = 2 * (int)bitlen(n) + 64;
    rec_quicksort(a, 0, (int64_t)n - 1, depth);
    for (uint64_t i = 0; i < n; i++) {
        key_put(out_keys, dtype, i, a[i].key);
        if (out_vals) out_vals[i] = vals[a[i].idx];
    }
    free(a);
    return 0;
}

/* Dispatch one of the paper's four algorithms (strategy4).  out may not alias in. */
int oracle_sort(const void *keys, const uint32_t *vals, uint64_t n, int dtype, int strategy4,
                void *out_keys, uint32_t *out_vals)
{
    if (n == 0) return 0;
    if (!dtype_ok(dtype)) return -1;
    size_t kb = key_bytes(dtype);
    switch (strategy4) {
    case OR_INSERTION:
        memcpy(out_keys, keys, n * kb);
        if (vals) memcpy(out_vals, vals, n * sizeof(uint32_t));
        oracle_insertion(out_keys, vals ? out_vals : NULL, n, dtype);
        return 0;
    case OR_COUNTING: return oracle_counting(keys, vals, n, dtype, out_keys, out_vals);
    case OR_RADIX: return oracle_radix(keys, vals, n, dtype, out_keys, out_vals);
    case OR_QUICK: return oracle_quicksort(keys, vals, n, dtype, out_keys, out_vals);
    default: return -1;
    }
}

/* The whole pipeline of Listing 6 with §III.A's entropy rule:
 * features -> FSM -> chosen algorithm.  EMPTY / CONSTANT are no-op copies
 * (P:411). */
int oracle_ahs(const void *keys, const uint32_t *vals, uint64_t n, int dtype,
               uint64_t n_insertion, uint64_t k_counting, uint64_t k_radix,
               double entropy_coeff, int norm, uint32_t entropy_bits,
               void *out_keys, uint32_t *out_vals,
               oracle_features_t *feat, int *strategy4, int *rule)
{
    int rc = oracle_features(keys, n, dtype, entropy_bits, feat, NULL);
    if (rc) return rc;
    rc = oracle_select(feat, n_insertion, k_counting, k_radix, entropy_coeff, norm, strategy4, rule);
    if (rc) return rc;
    if (n == 0) return 0;
    if (*rule == ORR_CONSTANT) {
        size_t kb = key_bytes(dtype);
        memcpy(out_keys, keys, n * kb);
        if (vals) memcpy(out_vals, vals, n * sizeof(uint32_t));
        return 0;
    }
    return oracle_sort(keys, vals, n, dtype, *strategy4, out_keys, out_vals);
}
