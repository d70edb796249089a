/*
 * ahs.h — C ABI of libahs.so, the B200-native (sm_100a) hot path of
 * Adaptive Hybrid Sort (arXiv 2506.20677).
 *
 * Three calls make the method (BASELINE.json north_star):
 *
 *   ahs_features  feature extraction, §III.A line 96: the state vector
 *                 v = (n, k, H) with k = max - min + 1 and
 *                 H = -sum_i p_i log2 p_i, plus min/max and the descent count
 *                 (presortedness, §I line 25 / north_star).
 *   ahs_select    the decision FSM, §III.A lines 96-98 (Fig. 2), with
 *                 Table II thresholds (lines 140-145) and the §III.K shortcuts
 *                 (line 411), applied on the host to the feature struct.
 *   ahs_sort      the chosen strategy on the device:
 *                   COUNTING  Listing 2 (§III.F), reusing the
 *                             feature histogram (run fill for keys only, stable
 *                             scatter for key-value pairs);
 *                   RADIX     §III.G (lines 218-251) base 256 on key - min with
 *                             d = ceil(log_256 k) passes (Eq. 4);
 *                   GENERAL   the paper's QuickSort branch (§III.G.1, lines
 *                             253-288) served by a full-width 4-pass radix sort
 *                             (identical, stable output).
 *
 * All pointers named d_* are DEVICE pointers owned by the caller (the library
 * never allocates device memory).  `stream` is a cudaStream_t passed as void*
 * (NULL = legacy default stream).  Keys are 32-bit integers (§III.K
 * line 409: integer-only input) stored contiguously, 4-byte aligned; values
 * are uint32 payloads that travel with their keys.  Every call returns an
 * ahs_status (0 = OK, < 0 = error; no exception crosses the ABI).  Calls are
 * thread-safe when concurrent calls use distinct ws/tmp buffers; the
 * profiling switch (ahs_profile_*) is process-global.
 */
#ifndef AHS_H
#define AHS_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define AHS_API __attribute__((visibility("default")))
#else
#define AHS_API
#endif

/* ------------------------------------------------------------------ enums */
typedef enum {
    AHS_OK = 0,
    AHS_EINVAL = -1,   /* NULL pointer with n > 0, bad dtype / strategy / thresholds,
                          misaligned key pointer, vals_out missing when vals_in given */
    AHS_ENOSPACE = -2, /* ws or tmp smaller than ahs_workspace_bytes / ahs_sort_tmp_bytes */
    AHS_ERANGE = -3,   /* n > AHS_MAX_N */
    AHS_EFEAT = -4,    /* feat does not describe these keys (n or dtype mismatch) */
    AHS_ECUDA = -5,    /* CUDA launch / runtime error (cudaGetLastError) */
    AHS_ENODEV = -6,   /* no CUDA device or not an sm_100 device */
    AHS_EMODEL = -7,   /* ahs_model_load: malformed JSON or a schema violation (err names the tree / node) */
    AHS_EMODELVER = -8 /* ahs_model_load: version other than "ahs-model/1" */
} ahs_status;

/* Key types: 32-bit keys (PAPER.md P:409 integers) and, NEXT-3, 64-bit keys
 * (SPEC.md S:20 SortKey is i64).  Values are always uint32. */
typedef enum { AHS_I32 = 0, AHS_U32 = 1, AHS_I64 = 2, AHS_U64 = 3 } ahs_dtype;

/* The GPU's three strategies.  The paper's Insertion (n <= 20) and QuickSort
 * branches both run as AHS_GENERAL; ahs_rule keeps which rule fired. */
typedef enum { AHS_COUNTING = 0, AHS_RADIX = 1, AHS_GENERAL = 2 } ahs_strategy;

typedef enum {
    AHS_RULE_EMPTY = 0,       /* n = 0  -> COUNTING, no-op  */
    AHS_RULE_CONSTANT = 1,    /* k = 1  -> COUNTING, no-op  */
    AHS_RULE_SMALL_N = 2,     /* n <= n_insertion   -> GENERAL (Insertion) */
    AHS_RULE_SMALL_RANGE = 3, /* k <= k_counting   -> COUNTING         */
    AHS_RULE_LOW_ENTROPY = 4, /* k > k_radix and H < c*log2(norm) -> RADIX */
    AHS_RULE_DEFAULT = 5,     /* otherwise   -> GENERAL (QuickSort) */
    AHS_RULE_MODEL = 6        /* the classifier chose (ahs_select_model) */
} ahs_rule;

/* Entropy normalisation of the RADIX rule (reading R2):
 * BUCKETS compares H against c*log2(nbins), RANGE against c*log2(k)
 * (paper-literal; identical whenever shift = 0). */
typedef enum { AHS_NORM_BUCKETS = 0, AHS_NORM_RANGE = 1 } ahs_entropy_norm;

/* feature flags (informational; only EMPTY / CONSTANT change ahs_select) */
#define AHS_FLAG_EMPTY 1u        /* n = 0 */
#define AHS_FLAG_CONSTANT 2u     /* k = 1 */
#define AHS_FLAG_BUCKETED 4u     /* shift > 0: H is a 2^16-bucket entropy */
#define AHS_FLAG_SORTED 8u       /* descents = 0 */
#define AHS_FLAG_STRICT_DESC 16u /* descents = n - 1 (n >= 2) */
#define AHS_FLAG_SIGNED 32u      /* dtype = AHS_I32 or AHS_I64 */
#define AHS_FLAG_K_SATURATED 64u /* 64-bit keys spanning the whole range: k = 2^64, reported
                                    as 2^64 - 1 */

#define AHS_ENTROPY_BITS 16u     /* at most 2^16 histogram bins (reading R1) */
#define AHS_MAX_N ((1ull << 30) - 1) /* look-back counts are 30-bit */

/* ------------------------------------------------------------------ types */
/* The state vector v = (n, k, H) of PAPER.md §III.A (line 96) and friends.
 *   min, max   in the key's own signedness (sign-extended for AHS_I32); for
 *              AHS_U64 the key's bit pattern (reinterpret as uint64)
 *   k          max - min + 1 (up to 2^32 for 32-bit keys; for 64-bit keys up
 *              to 2^64, saturated at 2^64 - 1 with AHS_FLAG_K_SATURATED)
 *   bits       bitlen(k - 1); shift = max(0, bits - 16);
 *   nbins      ((k - 1) >> shift) + 1  — histogram bins of (key - min) >> shift
 *   entropy    H = -sum_b p_b log2 p_b over those bins, fp64, clamped to
 *              [0, log2 nbins]  (equals the per-value entropy when shift = 0)
 *   descents   #{ i < n-1 : key[i] > key[i+1] } */
typedef struct {
    uint64_t n;
    int64_t min, max;
    uint64_t k;
    uint32_t bits, shift, nbins, dtype;
    double entropy;
    uint64_t descents;
    uint32_t flags;
    uint32_t entropy_bits;
} ahs_features_t;

/* Decision thresholds (Table II; R3-R5).
 * Valid iff all > 0, k_counting < k_radix, 0 < entropy_coeff <= 1
 * and entropy_norm is an ahs_entropy_norm. */
typedef struct {
    uint64_t n_insertion;   /* 20        : n <= n_insertion -> Insertion (GENERAL) */
    uint64_t k_counting;    /* 1024      : k <= k_counting  -> COUNTING            */
    uint64_t k_radix;       /* 1000000   : k >  k_radix and H < coeff*log2(norm)    */
    double entropy_coeff;   /* 0.7                                                   */
    uint32_t entropy_norm;  /* AHS_NORM_BUCKETS                                      */
    uint32_t reserved;      /* must be 0                                             */
} ahs_thresholds_t;

/* ------------------------------------------------------------ utilities */
AHS_API const char *ahs_version(void);
AHS_API const char *ahs_status_string(int status);
AHS_API void ahs_thresholds_default(ahs_thresholds_t *th);
/* Table II's defaults (ahs_thresholds_default) with environment overrides named
 * after SPEC's CLI flags: AHS_N_INSERTION, AHS_K_COUNTING, AHS_K_RADIX
 * (unsigned decimal), AHS_ENTROPY_COEFF (decimal), AHS_ENTROPY_NORM ("buckets" /
 * "range" or 0 / 1).  Unset or empty variables keep the default.  Returns AHS_OK,
 * or AHS_EINVAL when a variable is malformed or the result fails ahs_select's
 * threshold check (th then holds the defaults).  ahs_select(f, NULL, ...) does
 * NOT read the environment; the Python binding's sort() does, through this. */
AHS_API int ahs_thresholds_from_env(ahs_thresholds_t *th);

/* Device workspace for ahs_features (histogram, scan, reduction partials).
 * Independent of n in this version (~600 KiB); pass n anyway. */
AHS_API size_t ahs_workspace_bytes(uint64_t n);

/* Device scratch for ahs_sort: a second key buffer (and value buffer when
 * has_vals) plus per-tile look-back status.  Sufficient for every strategy.
 * ahs_sort_tmp_bytes assumes 32-bit keys; ahs_sort_tmp_bytes_dtype takes the
 * key type (0 for an invalid dtype). */
AHS_API size_t ahs_sort_tmp_bytes(uint64_t n, int has_vals);
AHS_API size_t ahs_sort_tmp_bytes_dtype(uint64_t n, int has_vals, int32_t dtype);
/* value_bytes: 0 (keys only), 4 or 8 (64-bit payloads, NEXT-3); 0 for invalid arguments. */
AHS_API size_t ahs_sort_tmp_bytes_ex(uint64_t n, uint32_t value_bytes, int32_t dtype);

/* Number of 8-bit digit passes ahs_sort will run for this strategy
 * (RADIX: ceil(bits/8) per Eq. 4; GENERAL: 4; COUNTING: 0 keys-only or 1 KV). */
AHS_API int ahs_sort_passes(const ahs_features_t *feat, int32_t strategy, int has_vals);

/* ---------------------------------------------------------- the hot path */

/* Feature extraction.  Reads d_keys[0..n) twice (min/max/descents, then the
 * histogram of (key - min) >> shift), computes H in fp64 on the device, and
 * WAITS for the result on the host (the one host sync of the pipeline: the FSM
 * runs on the host): the last kernel writes the 64-byte record into a mapped
 * pinned per-thread buffer that the call polls (spinning for ~100 us, then
 * yielding the core between polls; falling back to a copy + stream sync when
 * mapped memory is unavailable).  On return every read of d_keys is
 * complete; later work on `stream` is ordered after the kernels as usual.
 * d_ws (>= ahs_workspace_bytes) keeps the histogram and the digit rows for a
 * following ahs_sort on the same keys.
 * n = 0 returns AHS_OK with feat->flags = EMPTY and launches nothing. */
AHS_API int ahs_features(const void *d_keys, uint64_t n, int32_t dtype, void *d_ws, size_t ws_bytes,
                 ahs_features_t *feat, void *stream);

/* The FSM, host only, O(1).  th = NULL uses ahs_thresholds_default.  Rules in
 * order: EMPTY, CONSTANT, SMALL_N, SMALL_RANGE, LOW_ENTROPY, DEFAULT (see
 * ahs_rule).  rule may be NULL.  AHS_EINVAL for invalid thresholds. */
AHS_API int ahs_select(const ahs_features_t *feat, const ahs_thresholds_t *th, int32_t *strategy,
               int32_t *rule);

/* Sort n keys (and their values) with `strategy`, asynchronously on `stream`.
 *   d_keys_in / d_vals_in     input (d_vals_in NULL = keys only)
 *   d_keys_out / d_vals_out   output, ascending, stable (ties keep input order);
 *                             may alias the inputs (in place: odd pass counts
 *                             then cost one extra device copy)
 *   feat                      from ahs_features on the same keys (n, dtype, min,
 *                             bits, shift must match; AHS_EFEAT otherwise)
 *   d_ws                      the ahs_features workspace (COUNTING reads its
 *                             histogram and writes the exclusive scan of it
 *                             there; RADIX / GENERAL read its digit rows)
 *   d_tmp                     >= ahs_sort_tmp_bytes(n, d_vals_in != NULL)
 * COUNTING with shift > 0 (only reachable with k_counting > 65536) runs as
 * radix passes on key - min; the output is identical.  Empty and constant
 * inputs are copies.  The keys must not change between the two calls. */
AHS_API int ahs_sort(const void *d_keys_in, const uint32_t *d_vals_in, void *d_keys_out,
             uint32_t *d_vals_out, uint64_t n, int32_t strategy, const ahs_features_t *feat,
             void *d_ws, size_t ws_bytes, void *d_tmp, size_t tmp_bytes, void *stream);
/* ahs_sort with 4- or 8-byte values (value_bytes; ignored when d_vals_in is
 * NULL): 64-bit payloads (NEXT-3).  The values are moved bit-exactly; d_tmp >=
 * ahs_sort_tmp_bytes_ex(n, value_bytes, dtype).  EINVAL for another value_bytes
 * or value pointers not aligned to it. */
AHS_API int ahs_sort_ex(const void *d_keys_in, const void *d_vals_in, void *d_keys_out, void *d_vals_out,
                        uint64_t n, uint32_t value_bytes, int32_t strategy, const ahs_features_t *feat,
                        void *d_ws, size_t ws_bytes, void *d_tmp, size_t tmp_bytes, void *stream);

/* End to end from HOST buffers: H2D copy, ahs_features, ahs_select, ahs_sort,
 * D2H copy, stream sync.  h_* are host pointers (pinned for full speed);
 * d_scratch (>= ahs_host_scratch_bytes) is carved into the device buffers.
 * feat / strategy / rule may be NULL. */
AHS_API size_t ahs_host_scratch_bytes(uint64_t n, int has_vals);                 /* 32-bit keys */
AHS_API size_t ahs_host_scratch_bytes_dtype(uint64_t n, int has_vals, int32_t dtype); /* any key type */
AHS_API int ahs_sort_host(const void *h_keys_in, const uint32_t *h_vals_in, void *h_keys_out,
                  uint32_t *h_vals_out, uint64_t n, int32_t dtype, const ahs_thresholds_t *th,
                  void *d_scratch, size_t scratch_bytes, ahs_features_t *feat,
                  int32_t *strategy, int32_t *rule, void *stream);
/* The same without the final stream sync: returns once the sort and the D2H
 * copies are enqueued on `stream` (the features round trip inside is the only
 * wait).  h_keys_out / h_vals_out are valid, and the host inputs and d_scratch
 * reusable, after `stream` completes.  Two streams with two scratch buffers
 * overlap one sort's D2H with the next one's H2D and compute (PCIe is full
 * duplex). */
AHS_API int ahs_sort_host_async(const void *h_keys_in, const uint32_t *h_vals_in, void *h_keys_out,
                                uint32_t *h_vals_out, uint64_t n, int32_t dtype, const ahs_thresholds_t *th,
                                void *d_scratch, size_t scratch_bytes, ahs_features_t *feat, int32_t *strategy,
                                int32_t *rule, void *stream);

/* ------------------------------------------ paper-literal entropy (NEXT-2) */
/* H over the DISTINCT key values (§III.A line 96, H = -sum_v p_v
 * log2 p_v; reading "P" of SURVEY Appendix A, where ahs_features computes the
 * bucketed H16 of reading "B"), from a device key array in which equal keys
 * are contiguous, e.g. the keys_out of ahs_sort:
 *   H = log2 n - (1/n) sum over runs of c log2 c,  clamped to >= 0.
 * Key equality only (int32 and uint32 alike).  d_ws: an ahs_features workspace
 * (this call uses its own scratch area in it).  Synchronizes `stream`; *H on
 * return.  n = 0 gives H = 0.  Errors: EINVAL (NULL / misaligned pointer),
 * ENOSPACE, ERANGE (n > AHS_MAX_N), ENODEV, ECUDA. */
AHS_API int ahs_entropy_sorted(const void *d_keys, uint64_t n, void *d_ws, size_t ws_bytes, double *H,
                               void *stream);
/* The same for any key type (64-bit keys: NEXT-3); ahs_entropy_sorted = AHS_U32. */
AHS_API int ahs_entropy_sorted_dtype(const void *d_keys, uint64_t n, int32_t dtype, void *d_ws, size_t ws_bytes,
                                     double *H, void *stream);

/* ------------------------------------------- batched segment sort (NEXT-4) */
/* Many small independent sorts in one call: the GPU form of the paper's small-n
 * path (Insertion Sort for n <= 20, §III.E Listing 1).
 * Segment s = keys[d_offsets[s] .. d_offsets[s+1]) (device uint32 array of
 * num_segments + 1 non-decreasing offsets <= n; segments need not start at 0),
 * each sorted ascending and stably, values travelling with their keys; keys
 * outside every segment are not touched.  max_segment: an upper bound on the
 * segment lengths, <= 8192 (ERANGE above); <= 32 runs one thread per segment
 * with Listing 1's insertion sort in shared memory, otherwise 32 .. 512
 * threads per segment (a stable LSD radix sort in shared memory, 8-bit digits,
 * digits all keys of the segment share skipped).  Out may alias in.
 * d_bad (device uint32, required) receives the number of segments found longer
 * than max_segment or reaching past n: those are left unsorted (never an
 * out-of-bounds access).  Asynchronous.  Errors: EINVAL, ERANGE, ENODEV, ECUDA. */
AHS_API int ahs_sort_segments(const void *d_keys_in, const uint32_t *d_vals_in, void *d_keys_out,
                              uint32_t *d_vals_out, uint64_t n, const uint32_t *d_offsets, uint32_t num_segments,
                              uint32_t max_segment, int32_t dtype, uint32_t *d_bad, void *stream);

/* --------------------------------------- strategy classifier (NEXT-4, host) */
/* PAPER.md §III.H (lines 290-332, Listing 5 loadModel / predictStrategy): a
 * gradient-boosted tree ensemble over the raw features (n, k, H), used for
 * n >= 1000 beside the static rules (Table IV).  Model format: SPEC.md's
 * "ahs-model/1" JSON (classifier.hpp states it); validated eagerly on load.
 * The library ships no trained model (none exists offline); the tests use an
 * FSM-consistent fixture.  Host only, no device work, thread-safe after load. */
typedef struct ahs_model ahs_model_t;

/* Parse + validate json[0..len).  *model receives a handle to free with
 * ahs_model_free.  err (nullable) receives a NUL-terminated message naming the
 * offending tree / node.  Errors: EINVAL (NULL json / model), EMODEL,
 * EMODELVER. */
AHS_API int ahs_model_load(const char *json, size_t len, ahs_model_t **model, char *err, size_t err_len);
AHS_API void ahs_model_free(ahs_model_t *model);

/* score_c = base_c + sum over trees of the reached leaf's score (left iff
 * feature < threshold); *algo4 = argmax (ties: earlier class) as the paper's
 * algorithm: 0 insertion, 1 counting, 2 radix, 3 quick.  scores4 (nullable)
 * receives the 4 scores in the model's class order. */
AHS_API int ahs_model_predict(const ahs_model_t *model, double n, double k, double H, int32_t *algo4,
                              double *scores4);

/* Strategy selection with the classifier: the P:411 shortcuts (EMPTY,
 * CONSTANT) first; then, when model != NULL and n >= ml_min_n (Table IV: 1000),
 * the classifier (rule AHS_RULE_MODEL; insertion and quick map to GENERAL);
 * otherwise ahs_select.  *source (nullable): 0 = rules, 1 = classifier. */
AHS_API int ahs_select_model(const ahs_features_t *feat, const ahs_thresholds_t *th, const ahs_model_t *model,
                             uint64_t ml_min_n, int32_t *strategy, int32_t *rule, int32_t *source);

/* ------------------------------------------------------- ranking mode (K6) */
/* The onesweep pass ranks keys stably in one of two ways (onesweep.cuh):
 *   AHS_RANK_MASKED   {lane mask, slot} words: atomic add, read-back, clear;
 *                     valid on any CUDA device;
 *   AHS_RANK_ORDERED  one atomic add with return per key; valid only where the
 *                     same-address lanes of one shared-memory atomic instruction
 *                     are served in ascending lane order (unspecified by the
 *                     CUDA model; B200 does).  Selected by default only when a
 *                     self-test of that property passes on the device at first
 *                     use; environment AHS_RANK=masked forces the masked mode.
 * ahs_rank_mode(-1) returns the current mode of the current device; 0 / 1 set
 * it (AHS_EINVAL for ORDERED when the self-test failed).  Both modes give
 * identical output.  ahs_lane_order_ok() returns 1 if the self-test passed. */
#define AHS_RANK_MASKED 0
#define AHS_RANK_ORDERED 1
AHS_API int ahs_rank_mode(int mode);
AHS_API int ahs_lane_order_ok(void);

/* ------------------------------------------- trivial-pass skipping (NEXT-1) */
/* A radix pass whose digit is the same for every key is an identity
 * permutation.  With skipping on (default; environment AHS_SKIP_TRIVIAL=0
 * turns it off), K5 writes a device-side pass plan into d_tmp and such passes
 * return at once; the remaining passes keep the buffer parity so the result
 * still lands in keys_out.  With skipping on, when every key shares its bits
 * below a bit lo that is not a multiple of 8 and the feature bins resolve the
 * bits from lo up, the digits are placed at lo, lo + 8, ... instead of 0, 8, ...
 * (Eq. 4, fixes the digit count, not the digit positions;
 * DESIGN.md R20): the same or fewer passes over denser digits.  Not used in place
 * (keys_out == keys_in), where the parity must be known on the host.  Output is
 * identical either way.
 * ahs_set_skip_trivial(0/1) sets it (any other value queries); returns the
 * setting.  ahs_sort_executed_passes() reads the plan of the last ahs_sort on
 * that d_tmp (synchronizes `stream`): the number of executed digit passes, or
 * -1 if that sort wrote no plan (COUNTING paths), or AHS_ECUDA if one of its
 * digit passes gave up waiting for a predecessor tile's look-back status (more
 * than 2^28 empty polls, > 17 s: a stalled or preempted CTA; the output is then
 * invalid, and the pass finished instead of trapping the context).
 * ahs_sort_host() performs the same check after its final synchronisation. */
AHS_API int ahs_set_skip_trivial(int on);

/* Key-value COUNTING with 256 < k <= 1024 (§III.F Listing 2, lines
 * 187-214; k_counting = 1024, Table II): one stable scatter by the
 * 10-bit digit key - min (16 n bytes moved: read and write of keys and values)
 * instead of two 8-bit radix passes over key - min (32 n bytes).  Output is
 * identical.  Default off (environment AHS_COUNT_KV_SINGLE=1 turns it on):
 * on B200 the single pass measured slower, because 1024 digit runs per
 * 4096-key tile fragment its write-out (profiles/r02_summary.md).  32-bit keys
 * with 4-byte values and the ordered ranking only; otherwise the two passes
 * run.  ahs_set_count_kv_single(0/1) sets it (any other value queries);
 * returns the setting.  ahs_sort_passes() reports 1 for such inputs when on. */
AHS_API int ahs_set_count_kv_single(int on);

/* Bucket-local GENERAL plan (the paper's GENERAL branch, QuickSort in
 * Listing 4, served by radix passes, R14).  For 32-bit keys whose
 * feature bins (key - min) >> s are coarser than single values (s > 0), with
 * 4-byte or no values and out of place: two stable LSD passes over the two bytes
 * of the bin make every bin a contiguous bucket (its boundaries are the exclusive
 * scan of the feature histogram), then K10 sorts each bucket in shared memory by
 * its low s bits (K10, bucket.cuh: one CTA per bucket, digits a bucket shares
 * skipped; it sorts key - min, and for pairs whose bucket keys differ only in
 * their low 16 bits it sorts 32-bit (key bits, index) slots and gathers the
 * values once) -- three reads and writes of the keys instead of four.  Used where
 * it pays on B200: bins of >= 1536 keys on average (environment AHS_BL_MIN_KEYS
 * changes the bound; 2^28 pairs, keys over 20..32 bits: sort 3.72-4.96 ms ->
 * 3.57-3.90 ms; with smaller bins the bucket pass is slower than the passes it
 * replaces, profiles/r02_summary.md).  The library picks K10's capacity from the
 * mean bin size (up to 8192 keys); K5 falls back to the four full-width passes on
 * the device when a bin is larger.  Default on (environment AHS_BUCKET_LOCAL=0
 * turns it off).  Output identical.
 * ahs_set_bucket_local(0/1) sets it (any other value queries); returns the setting.
 * ahs_sort_plan() reads the plan of the last ahs_sort on d_tmp (synchronizes):
 * executed digit passes and whether the bucket-local pass ran.
 * ahs_sort_executed_passes() counts the bucket-local pass as one pass. */
AHS_API int ahs_set_bucket_local(int on);
AHS_API int ahs_sort_plan(const void *d_tmp, size_t tmp_bytes, int *digit_passes, int *bucket_local,
                          void *stream);
AHS_API int ahs_sort_executed_passes(const void *d_tmp, size_t tmp_bytes, uint64_t n, int has_vals,
                                     void *stream);

/* -------------------------------------------------------- instrumentation */
/* Kernels launched by this library since load (all streams, all threads). */
AHS_API uint64_t ahs_launch_count(void);

/* Per-kernel timing: while enabled, every launch is bracketed by CUDA events
 * on its own stream.  ahs_profile_read synchronizes those events and returns,
 * per kernel id (0 .. ahs_kernel_count()-1), the summed milliseconds and the
 * launch count since ahs_profile_begin. */
AHS_API int ahs_kernel_count(void);
AHS_API const char *ahs_kernel_name(int id);
AHS_API int ahs_profile_begin(void);
AHS_API int ahs_profile_end(void);
AHS_API int ahs_profile_read(double *ms, uint64_t *launches, int n_ids);

#ifdef __cplusplus
}
#endif
#endif /* AHS_H */
