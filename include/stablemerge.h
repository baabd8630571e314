/*
 * stablemerge.h -- C ABI of the B200 (sm_100a) stable parallel merge and
 * stable merge sort of arXiv 1202.6575 (J. L. Traff, "A simple, stable
 * parallel two-way merge").  Citations are PAPER.md line numbers
 * and SURVEY.md §8 rows.
 *
 * Library: paper_1202_6575_b200/lib/libstablemerge.so (CUDA runtime linked
 * statically).  No torch types appear here: keys and payloads are plain
 * pointers, sizes are int64_t, the stream is a cudaStream_t passed as void*.
 *
 * ------------------------------------------------------------------------
 * Problem (§2): A (n elements) and B (m elements) are
 * non-decreasing under the key order; repeated keys are allowed.  C (n+m
 * elements) receives the STABLE merge: keys non-decreasing, each input's
 * order preserved, and every element of A placed before every equal-keyed
 * element of B (L158-166, L354-357).  Equivalently A[i] lands at
 * C[i + rank_low(A[i], B)] and B[j] at C[j + rank_high(B[j], A)].  The
 * paper's "m <= n without loss of generality" (L66) is NOT required: any n, m
 * (swapping would flip the tie rule).  Sentinels A[-1] = -inf, A[n] = +inf are
 * virtual and never stored (L69-71).
 *
 * Key order ("<=" of PAPER.md L63): _u32 / _u64 compare unsigned, _i32 /
 * _i64 signed (two's complement), _f32 / _f64 by IEEE 754 totalOrder
 * (-NaN < -inf < ... < -0.0 < +0.0 < ... < +inf < +NaN; SURVEY.md §8(f)
 * row 2) -- a total order, so the stable merge is unique.  Inputs must be
 * non-decreasing in that order (e.g. sorted by mergesort_stable_f32).
 * Payloads are uint32 and travel with their key.
 *
 * Memory: every pointer may be DEVICE memory (cudaMalloc / torch CUDA
 * tensors / managed) or HOST memory (pinned or pageable).  With device
 * pointers the call is fully asynchronous on `stream`.  If any key/payload
 * pointer of a call is host memory, the library stages all of that call's
 * buffers through device memory (cudaMemcpyAsync host->device, the kernels,
 * device->host) ordered after `stream`; host outputs are valid once `stream`
 * has been synchronised (for pageable outputs the final copy is
 * synchronous).  merge_stable with host inputs of 64 MB or more is cut on the
 * host into 2 p_h independent sub-merges (Steps 1-4 at p_h <= 16 blocks per
 * array) pipelined over three internal streams (uploads || merges || downloads),
 * joined back into `stream`; the library reads the host keys for that
 * partition (2 p_h binary searches).  mergesort_stable with host keys (and
 * payloads) of 64 MB or more uploads in chunks sorted as they arrive and
 * downloads the last merge round in sub-merges as they finish (one host
 * synchronisation for that round's coarse partition).
 * Device: a call runs on the device of `stream`, whatever the calling
 * thread's current device (restored on return); with the NULL, legacy or
 * per-thread default stream, or a stream under graph capture, it runs on the
 * current device.  Device buffers must be accessible from that device.
 * Device-pointer calls can be captured into a CUDA graph (the scratch
 * allocations become graph memory nodes); host-pointer calls cannot.
 * Ownership: the caller owns every buffer; the library never frees or
 * retains them past the stream point of the call.  Scratch (the two
 * cross-rank arrays of p+1 entries, L373-375; the merge sort's auxiliary
 * array of N keys + N payloads, §3) comes from
 * cudaMallocAsync on `stream` and is freed stream-ordered.
 *
 * Errors (return value; no host synchronisation is done to detect them):
 *   SM_OK       success (n = m = 0 / N <= 1: nothing launched)
 *   SM_EINVAL   negative size; NULL key pointer with a nonzero size; payload
 *               pointers not all set or all NULL; invalid options; n + m > 2^31 - 1
 *               for the batched, wide-payload, plan and merge-path calls
 *               (32-bit in-kernel indices)
 *   SM_EALIAS   output overlaps an input (the merge is not in place)
 *   SM_ENOMEM   scratch allocation failed
 *   SM_ECUDA    a CUDA launch or copy failed (see sm_last_error())
 * Unsorted inputs violate the precondition: the output is then unspecified
 * (but every write stays inside C).
 * Sizes of 2^31 elements or more (merge_stable, mergesort_stable): the kernels
 * index 32-bit, so the library applies the paper's Steps 1-4 once more at
 * coarse granularity (p blocks of <= 2^29 elements per array, their
 * block-start keys ranked by the rank kernel, the cases on the host) and runs
 * 2p sub-merges below 2^31; a sort sorts chunks of 2^30 and merges them
 * pairwise.  One host synchronisation per coarse partition.
 */
#ifndef STABLEMERGE_H
#define STABLEMERGE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* An unsigned 128-bit key (the _u128 entry points): value = hi * 2^64 + lo,
 * i.e. (hi, lo) tuples in lexicographic order -- "(key, tie)" pairs.  Same
 * bytes as a little-endian unsigned __int128.  Arrays of sm_u128 keys must be
 * 16-byte aligned (SM_EINVAL otherwise). */
typedef struct {
    uint64_t lo;
    uint64_t hi;
} sm_u128;

typedef enum {
    SM_OK = 0,
    SM_EINVAL = 1,
    SM_EALIAS = 2,
    SM_ENOMEM = 3,
    SM_ECUDA = 4
} sm_status;

/* ---------------------------------------------------------------------
 * merge_stable_<K>  -- SURVEY.md §8 rows a0-a7 (§2 Steps 1-4).
 *
 *   keys_A[n], vals_A[n]   A, non-decreasing keys (+ uint32 payload)
 *   keys_B[m], vals_B[m]   B, non-decreasing keys (+ uint32 payload)
 *   out_keys[n+m], out_vals[n+m]   C
 *   vals_A, vals_B, out_vals: all three set, or all three NULL (keys only)
 *   stream: cudaStream_t (NULL = legacy default stream)
 *
 * Device path: a cross-rank kernel computes xbar_i = rank_low(A[x_i], B) and
 * ybar_j = rank_high(B[y_j], A) for the block starts x_i, y_j (L304-309);
 * stream order is the paper's single synchronisation (L373-375); a task
 * kernel then classifies each block start into cases (a)-(e) (L310-340) and
 * copies or stably merges each disjoint subproblem into C[x_i + xbar_i ..]
 * or C[y_j + ybar_j ..].  Block counts: p_A = ceil(n / T), p_B = ceil(m / T)
 * with the tile-derived block size T (reading R7 of DESIGN.md).
 * ------------------------------------------------------------------- */
sm_status merge_stable_u32(const uint32_t *keys_A, const uint32_t *vals_A, int64_t n,
                           const uint32_t *keys_B, const uint32_t *vals_B, int64_t m,
                           uint32_t *out_keys, uint32_t *out_vals, void *stream);
sm_status merge_stable_i32(const int32_t *keys_A, const uint32_t *vals_A, int64_t n,
                           const int32_t *keys_B, const uint32_t *vals_B, int64_t m,
                           int32_t *out_keys, uint32_t *out_vals, void *stream);
sm_status merge_stable_i64(const int64_t *keys_A, const uint32_t *vals_A, int64_t n,
                           const int64_t *keys_B, const uint32_t *vals_B, int64_t m,
                           int64_t *out_keys, uint32_t *out_vals, void *stream);
sm_status merge_stable_u64(const uint64_t *keys_A, const uint32_t *vals_A, int64_t n,
                           const uint64_t *keys_B, const uint32_t *vals_B, int64_t m,
                           uint64_t *out_keys, uint32_t *out_vals, void *stream);
sm_status merge_stable_f32(const float *keys_A, const uint32_t *vals_A, int64_t n,
                           const float *keys_B, const uint32_t *vals_B, int64_t m,
                           float *out_keys, uint32_t *out_vals, void *stream);
sm_status merge_stable_f64(const double *keys_A, const uint32_t *vals_A, int64_t n,
                           const double *keys_B, const uint32_t *vals_B, int64_t m,
                           double *out_keys, uint32_t *out_vals, void *stream);

/* ---------------------------------------------------------------------
 * merge_stable_batched_<K>  -- SURVEY.md §8(f) row 1: S independent stable
 * merges in one call (variable lengths), through the segmented machinery of
 * the merge-sort rounds (§3, "modifying the merge
 * algorithm to work in parallel on the pairs").
 *
 *   keys_A[n], vals_A[n]     the A segments, concatenated
 *   a_offsets[S+1]  int64    segment s of A is keys_A[a_offsets[s], a_offsets[s+1])
 *   keys_B[m], vals_B[m], b_offsets[S+1]   likewise for B
 *   out_keys[n+m], out_vals[n+m]   segment s of C starts at
 *                            a_offsets[s] + b_offsets[s] and holds the stable
 *                            merge (ties: A first) of the two segments
 *   vals_*: all three set or all NULL; stream as above.
 *
 * DEVICE pointers only (keys, payloads and both offset arrays; a host
 * pointer gives SM_EINVAL).  Precondition: a_offsets[0] = 0,
 * a_offsets[S] = n, non-decreasing (same for b_offsets with m), and every
 * segment sorted.  The offsets are read on the device only; a violated
 * precondition gives unspecified output but no write outside C (offsets
 * are clamped into [0, n] / [0, m] and each segment to a non-negative
 * length).  Errors and scratch as merge_stable_<K>.
 * ------------------------------------------------------------------- */
sm_status merge_stable_batched_u32(const uint32_t *keys_A, const uint32_t *vals_A, int64_t n,
                                   const int64_t *a_offsets, const uint32_t *keys_B, const uint32_t *vals_B,
                                   int64_t m, const int64_t *b_offsets, int64_t S, uint32_t *out_keys,
                                   uint32_t *out_vals, void *stream);
sm_status merge_stable_batched_i32(const int32_t *keys_A, const uint32_t *vals_A, int64_t n,
                                   const int64_t *a_offsets, const int32_t *keys_B, const uint32_t *vals_B,
                                   int64_t m, const int64_t *b_offsets, int64_t S, int32_t *out_keys,
                                   uint32_t *out_vals, void *stream);
sm_status merge_stable_batched_i64(const int64_t *keys_A, const uint32_t *vals_A, int64_t n,
                                   const int64_t *a_offsets, const int64_t *keys_B, const uint32_t *vals_B,
                                   int64_t m, const int64_t *b_offsets, int64_t S, int64_t *out_keys,
                                   uint32_t *out_vals, void *stream);
sm_status merge_stable_batched_u64(const uint64_t *keys_A, const uint32_t *vals_A, int64_t n,
                                   const int64_t *a_offsets, const uint64_t *keys_B, const uint32_t *vals_B,
                                   int64_t m, const int64_t *b_offsets, int64_t S, uint64_t *out_keys,
                                   uint32_t *out_vals, void *stream);
sm_status merge_stable_batched_f32(const float *keys_A, const uint32_t *vals_A, int64_t n,
                                   const int64_t *a_offsets, const float *keys_B, const uint32_t *vals_B,
                                   int64_t m, const int64_t *b_offsets, int64_t S, float *out_keys,
                                   uint32_t *out_vals, void *stream);
sm_status merge_stable_batched_f64(const double *keys_A, const uint32_t *vals_A, int64_t n,
                                   const int64_t *a_offsets, const double *keys_B, const uint32_t *vals_B,
                                   int64_t m, const int64_t *b_offsets, int64_t S, double *out_keys,
                                   uint32_t *out_vals, void *stream);

/* ---------------------------------------------------------------------
 * ranks_stable_<K>  -- rank queries, the primitive of rows a1/a2 on its own
 * (PAPER.md L119-128): out[i] = rank_low(keys[i], X) = #{X[t] < keys[i]}
 * when high = 0, rank_high(keys[i], X) = #{X[t] <= keys[i]} when high != 0,
 * for X[len] non-decreasing in the key order.  One binary search per key.
 * DEVICE pointers only; out is int64[nkeys].  Used by the sharded
 * multi-GPU merge (paper_1202_6575_b200.distributed): the
 * global cross rank of a block start is the sum of its ranks in the shards.
 * ------------------------------------------------------------------- */
sm_status ranks_stable_u32(const uint32_t *X, int64_t len, const uint32_t *keys, int64_t nkeys, int32_t high,
                             int64_t *out, void *stream);
sm_status ranks_stable_i32(const int32_t *X, int64_t len, const int32_t *keys, int64_t nkeys, int32_t high,
                             int64_t *out, void *stream);
sm_status ranks_stable_i64(const int64_t *X, int64_t len, const int64_t *keys, int64_t nkeys, int32_t high,
                             int64_t *out, void *stream);
sm_status ranks_stable_u64(const uint64_t *X, int64_t len, const uint64_t *keys, int64_t nkeys, int32_t high,
                             int64_t *out, void *stream);
sm_status ranks_stable_f32(const float *X, int64_t len, const float *keys, int64_t nkeys, int32_t high,
                             int64_t *out, void *stream);
sm_status ranks_stable_f64(const double *X, int64_t len, const double *keys, int64_t nkeys, int32_t high,
                             int64_t *out, void *stream);

/* ---------------------------------------------------------------------
 * mergesort_stable_<K>  -- SURVEY.md §8 rows a8-a9 (§3).
 *
 *   keys[N], vals[N] (vals may be NULL: keys only), sorted IN PLACE from the
 *   caller's view; stable: equal keys keep their input order.
 *
 * Device path, phase 1 ("sorting sequentially in parallel p consecutive
 * blocks", L406-407): p blocks of R consecutive elements, each sorted
 * stably by one CTA.  Keys of <= 8 bytes with 16-byte-aligned buffers and
 * N / (SM count) >= 2^15: p = the SM count (the paper's p processing
 * elements), each block radix-sorted through global memory (8-bit digits,
 * one pass per byte on which the block's keys differ); otherwise runs of
 * sm_sort_run() elements sorted in shared memory.  Either sort is stable
 * by construction (sm_sort_run_n() gives R for a given N).
 * Then ceil(log2(N/R)) rounds merge run pairs (2k, 2k+1) with the left run
 * playing A, every pair of a round in one segmented launch of the merge
 * above ("modifying the merge algorithm to work in parallel on the
 * ceil(p/2^i) pairs", L413-414); an odd trailing run is copied (L409-410).
 * One auxiliary array (N keys + N payloads) is ping-ponged.
 * ------------------------------------------------------------------- */
sm_status mergesort_stable_u32(uint32_t *keys, uint32_t *vals, int64_t N, void *stream);
sm_status mergesort_stable_i32(int32_t *keys, uint32_t *vals, int64_t N, void *stream);
sm_status mergesort_stable_i64(int64_t *keys, uint32_t *vals, int64_t N, void *stream);
sm_status mergesort_stable_u64(uint64_t *keys, uint32_t *vals, int64_t N, void *stream);
sm_status mergesort_stable_f32(float *keys, uint32_t *vals, int64_t N, void *stream);
sm_status mergesort_stable_f64(double *keys, uint32_t *vals, int64_t N, void *stream);

/* ---------------------------------------------------------------------
 * Test / tuning variants (not the contract).
 *
 * sm_options: zero fields mean "default".
 *   p_A, p_B   explicit block counts (PAPER.md's single p: p_A = p_B = p).
 *              Every task must then fit one tile:
 *              ceil(n/p_A) + ceil(m/p_B) <= sm_tile_capacity(key bytes,
 *              has_vals), else SM_EINVAL.
 *   block      block size T (elements) when p_A/p_B are 0:
 *              p_A = ceil(n/T), p_B = ceil(m/T); 2T <= tile capacity.
 *   sort_run   merge sort initial run length R (0 = default): the
 *              shared-memory block-sort tile sm_sort_run(), or any multiple
 *              of 16 for one-CTA-per-block phase 1 (keys <= 8 bytes,
 *              16-byte-aligned buffers); anything else: SM_EINVAL
 *   flags      bit 0 (SM_FLAG_NO_PDL): disable programmatic dependent launch
 *              between the cross-rank and task kernels; bit 1
 *              (SM_FLAG_MERGE_PATH): the merge-path comparison below.
 * ------------------------------------------------------------------- */
typedef struct {
    int64_t p_A;
    int64_t p_B;
    int64_t block;
    int64_t sort_run;
    int64_t flags;
} sm_options;

#define SM_FLAG_NO_PDL 1
/* merge_stable_ex only, device pointers only: the merge-path COMPARISON
 * ([AklSantoro87]) -- C cut into
 * tiles of exactly tile-capacity outputs by one binary search per diagonal,
 * instead of the paper's cross ranks and cases.  Same output; exists to
 * measure what the paper's factor-two task imbalance costs.  Not the method. */
#define SM_FLAG_MERGE_PATH 2

sm_status merge_stable_ex_u32(const uint32_t *keys_A, const uint32_t *vals_A, int64_t n,
                              const uint32_t *keys_B, const uint32_t *vals_B, int64_t m,
                              uint32_t *out_keys, uint32_t *out_vals, void *stream,
                              const sm_options *opt);
sm_status merge_stable_ex_i32(const int32_t *keys_A, const uint32_t *vals_A, int64_t n,
                              const int32_t *keys_B, const uint32_t *vals_B, int64_t m,
                              int32_t *out_keys, uint32_t *out_vals, void *stream,
                              const sm_options *opt);
sm_status merge_stable_ex_i64(const int64_t *keys_A, const uint32_t *vals_A, int64_t n,
                              const int64_t *keys_B, const uint32_t *vals_B, int64_t m,
                              int64_t *out_keys, uint32_t *out_vals, void *stream,
                              const sm_options *opt);
sm_status merge_stable_ex_u64(const uint64_t *keys_A, const uint32_t *vals_A, int64_t n,
                              const uint64_t *keys_B, const uint32_t *vals_B, int64_t m,
                              uint64_t *out_keys, uint32_t *out_vals, void *stream,
                              const sm_options *opt);
sm_status merge_stable_ex_f32(const float *keys_A, const uint32_t *vals_A, int64_t n,
                              const float *keys_B, const uint32_t *vals_B, int64_t m,
                              float *out_keys, uint32_t *out_vals, void *stream,
                              const sm_options *opt);
sm_status merge_stable_ex_f64(const double *keys_A, const uint32_t *vals_A, int64_t n,
                              const double *keys_B, const uint32_t *vals_B, int64_t m,
                              double *out_keys, uint32_t *out_vals, void *stream,
                              const sm_options *opt);

/* merge_plan_ex_<K>: Steps 1-4 only, dumped for parity with the oracle's plan
 * (Fig. 1, L73-117).  DEVICE pointers only (host -> SM_EINVAL).
 *   p_A >= 1, p_B >= 1 (block counts; no tile limit here)
 *   xbar[p_A+1]  int64: x̄_i = rank_low(A[x_i], B), x̄_{p_A} = m   (L304-306)
 *   ybar[p_B+1]  int64: ȳ_j = rank_high(B[y_j], A), ȳ_{p_B} = n  (L307-309)
 *   tasks[(p_A+p_B)*6] int64 rows (side 0=A/1=B, case 0..4 = (a)..(e),
 *                a0, a1, b0, b1): A-side tasks 0..p_A-1, then B-side.
 *                The output offset of a task is a0 + b0.                  */
sm_status merge_plan_ex_u32(const uint32_t *keys_A, int64_t n, const uint32_t *keys_B, int64_t m,
                            int64_t p_A, int64_t p_B, int64_t *xbar, int64_t *ybar, int64_t *tasks,
                            void *stream);
sm_status merge_plan_ex_i32(const int32_t *keys_A, int64_t n, const int32_t *keys_B, int64_t m,
                            int64_t p_A, int64_t p_B, int64_t *xbar, int64_t *ybar, int64_t *tasks,
                            void *stream);
sm_status merge_plan_ex_i64(const int64_t *keys_A, int64_t n, const int64_t *keys_B, int64_t m,
                            int64_t p_A, int64_t p_B, int64_t *xbar, int64_t *ybar, int64_t *tasks,
                            void *stream);
sm_status merge_plan_ex_u64(const uint64_t *keys_A, int64_t n, const uint64_t *keys_B, int64_t m,
                            int64_t p_A, int64_t p_B, int64_t *xbar, int64_t *ybar, int64_t *tasks,
                            void *stream);
sm_status merge_plan_ex_f32(const float *keys_A, int64_t n, const float *keys_B, int64_t m,
                            int64_t p_A, int64_t p_B, int64_t *xbar, int64_t *ybar, int64_t *tasks,
                            void *stream);
sm_status merge_plan_ex_f64(const double *keys_A, int64_t n, const double *keys_B, int64_t m,
                            int64_t p_A, int64_t p_B, int64_t *xbar, int64_t *ybar, int64_t *tasks,
                            void *stream);

sm_status mergesort_stable_ex_u32(uint32_t *keys, uint32_t *vals, int64_t N, void *stream,
                                  const sm_options *opt);
sm_status mergesort_stable_ex_i32(int32_t *keys, uint32_t *vals, int64_t N, void *stream,
                                  const sm_options *opt);
sm_status mergesort_stable_ex_i64(int64_t *keys, uint32_t *vals, int64_t N, void *stream,
                                  const sm_options *opt);
sm_status mergesort_stable_ex_u64(uint64_t *keys, uint32_t *vals, int64_t N, void *stream,
                                  const sm_options *opt);
sm_status mergesort_stable_ex_f32(float *keys, uint32_t *vals, int64_t N, void *stream,
                                  const sm_options *opt);
sm_status mergesort_stable_ex_f64(double *keys, uint32_t *vals, int64_t N, void *stream,
                                  const sm_options *opt);

/* Largest task (elements) one CTA tile holds for this key width / payload
 * mode: the default block size is T = capacity / 2 (the task bound
 * ceil(n/p_A) + ceil(m/p_B) <= 2T). */
int64_t sm_tile_capacity(int32_t key_bytes, int32_t has_vals);

/* Run length of the shared-memory block sort (the merge sort's initial run
 * length R for small N and 128-bit keys) for this key width / payload mode. */
int64_t sm_sort_run(int32_t key_bytes, int32_t has_vals);

/* The merge sort's initial run length R for N elements on the current
 * device (16-byte-aligned buffers): ceil(N / SM count) rounded up to 16
 * when that is >= 2^15 and keys have <= 8 bytes, else sm_sort_run(). */
int64_t sm_sort_run_n(int32_t key_bytes, int32_t has_vals, int64_t n);

/* Test hooks (not the contract).
 *
 * sm_set_k1_variant: which cross-rank kernel (rows a1/a2) later calls on
 *   this process launch -- 0 automatic (the default: a warp per search below
 *   10240 searches, else the shared-memory-sample kernel for a plain merge and
 *   one thread per search for the segmented modes), 1 a warp per search,
 *   2 the sample kernel (plain merges), 3 one thread per search.  Lets the
 *   tests compare every variant's x̄ / ȳ with the oracle (merge_plan_ex).
 *   A variant other than 0 also turns the one-launch small merges off.
 *
 * sm_set_small_fuse: 1 -- a plain merge on device buffers with at most 8
 *   tasks per resident K2 CTA (C1's size) is ONE launch: each CTA computes
 *   the cross ranks its own tasks read (Steps 1-2, L304-309; a warp per
 *   search) before classifying them, so every rank a task reads is final
 *   first (L373-375, per CTA); 0 (the default) -- K1 then K2 as for larger
 *   merges (measured faster when the inputs are not in L2: K2's launch then
 *   overlaps K1 under PDL).  Both give the same output.
 *
 * sm_set_sort_ways: how the merge sort's phase 2 (§3,
 *   row a9) runs its ceil(log2 p) rounds on later calls of this process --
 *   4: two rounds per HBM pass (keys of <= 8 bytes): the four runs R0..R3
 *   of two consecutive rounds are partitioned at once (every block start of
 *   a run ranked in the three others: Steps 1-2 of L304-309 for four
 *   arrays, reading R20 in DESIGN.md) and each subproblem is merged twice in
 *   shared memory (R0 with R1, R2 with R3, then the two results), an odd
 *   round first as a plain round; 2: one round per pass (the paper's rounds
 *   as they stand); 0 (the default, also any other value): 4 where it
 *   measured faster -- N >= 3 * 2^19 (~1.5 M) elements, except 4-byte
 *   keys without a payload from N = 2^28 on -- else 2.  Same output, bit for bit; 128-bit keys always take one round
 *   per pass.
 *
 * sm_sort_merge_passes: the number of phase-2 HBM passes (k_tasks / k_tasks4
 *   launches) a sort of n elements takes on the current device under the
 *   current sm_set_sort_ways setting (16-byte-aligned buffers).
 *
 * sm_plan_from_ranks: the host's own Steps 3-4 (readings
 *   R1, R8) on given cross ranks xbar[0..p], ybar[0..p] with p blocks per
 *   array: the coarse partition the host-buffer pipeline and the >= 2^31
 *   merges use.  Writes the 2p tasks as rows (a0, a1, b0, b1) into
 *   tasks[2p * 4], ordered by output offset a0 + b0.  Host memory, no GPU;
 *   SM_EINVAL on bad arguments. */
void sm_set_k1_variant(int32_t variant);
void sm_set_small_fuse(int32_t on);
void sm_set_sort_ways(int32_t ways);
int32_t sm_sort_merge_passes(int32_t key_bytes, int32_t has_vals, int64_t n);

/* SM_DEBUG builds (build_native.build_debug(): lib/libstablemerge_debug.so)
 * check the paper's disjoint-write invariant on the device (PAPER.md
 * L343-361): every K2 store lies inside its task's output range and inside
 * C, every K3 / K3H store inside its run, else the kernel traps (printf +
 * __trap).  sm_debug_cover(cover, len): later K2 launches add 1 to
 * cover[i] for every output element i they store (cover: device memory the
 * caller zeroed, len >= the output length; NULL stops counting) -- a merge
 * must leave exactly 1 everywhere.  Release builds: SM_EINVAL.
 * sm_is_debug_build: 1 in SM_DEBUG builds, else 0. */
sm_status sm_debug_cover(uint32_t *cover, int64_t len);
int32_t sm_is_debug_build(void);
sm_status sm_plan_from_ranks(int64_t n, int64_t m, int64_t p, const int64_t *xbar, const int64_t *ybar,
                             int64_t *tasks);

/* Steps 3-4 on the host (readings R1, R7, R8) for cross
 * ranks computed elsewhere -- the sharded merge ranks block
 * starts across GPUs and classifies the p_A + p_B tasks here.
 *   xbar[0..pA], ybar[0..pB]: x̄ (rank_low of A's block starts in B, the
 *   sentinel x̄_pA = m, m for empty block starts) and ȳ likewise (n).
 *   tasks[(pA + pB) * 4]: rows (a0, a1, b0, b1) in task order -- A-side task
 *   i = 0..pA-1, then B-side task j = 0..pB-1 -- the ranges A[a0, a1) and
 *   B[b0, b1) merged into C[a0 + b0, a1 + b1).
 * The same classification code as the device's K2 (64-bit indices).  Host
 * memory, no GPU; caller-owned arrays; SM_EINVAL on bad arguments. */
sm_status sm_plan_tasks(int64_t n, int64_t m, int64_t pA, int64_t pB, const int64_t *xbar, const int64_t *ybar,
                        int64_t *tasks);

/* Human-readable text for a status, and the last CUDA error message seen by
 * this library in the calling thread ("" if none). */
const char *sm_status_string(sm_status s);
const char *sm_last_error(void);

/* Number of kernel launches the last call on this host thread issued. */
int64_t sm_last_launch_count(void);

/* Profiling (bench.py only).  While enabled, every kernel the library
 * launches is bracketed by two CUDA events recorded on its launch stream
 * (this also turns programmatic dependent launch off).  Enabling resets the
 * record.  sm_profile_read synchronises the recorded events and returns the
 * summed duration (ms) and launch count of one kernel kind:
 * 0 = cross ranks (K1), 1 = tasks (K2: classify + copy/merge), 2 = block
 * sort (K3).  Not thread-safe; process-wide. */
void sm_profile_enable(int on);
sm_status sm_profile_read(int kind, double *total_ms, int64_t *launches);


/* ---------------------------------------------------------------------
 * Descending order -- SURVEY.md §8(f) row 2: the method for an arbitrary
 * total order "<=", instantiated with the REVERSED key order
 * (u32/u64 unsigned, i32/i64 signed, f32/f64 IEEE totalOrder, each
 * reversed).  <op>_desc_<K> has exactly the signature and contract of
 * <op>_<K> above, with "non-decreasing" read as "non-increasing":
 *   inputs sorted non-increasingly; C non-increasing; stability unchanged --
 *   every element of A precedes every equal-keyed element of B, and
 *   mergesort_stable_desc keeps equal keys in input order;
 *   ranks_stable_desc: rank_low(x, X) = #{X[t] > x}, rank_high = #{X[t] >= x}.
 * Same kernels (one template instantiation per key type), same bytes moved.
 * ------------------------------------------------------------------- */
sm_status merge_stable_desc_u32(const uint32_t *keys_A, const uint32_t *vals_A, int64_t n,
                                const uint32_t *keys_B, const uint32_t *vals_B, int64_t m,
                                uint32_t *out_keys, uint32_t *out_vals, void *stream);
sm_status merge_stable_desc_i32(const int32_t *keys_A, const uint32_t *vals_A, int64_t n,
                                const int32_t *keys_B, const uint32_t *vals_B, int64_t m,
                                int32_t *out_keys, uint32_t *out_vals, void *stream);
sm_status merge_stable_desc_i64(const int64_t *keys_A, const uint32_t *vals_A, int64_t n,
                                const int64_t *keys_B, const uint32_t *vals_B, int64_t m,
                                int64_t *out_keys, uint32_t *out_vals, void *stream);
sm_status merge_stable_desc_u64(const uint64_t *keys_A, const uint32_t *vals_A, int64_t n,
                                const uint64_t *keys_B, const uint32_t *vals_B, int64_t m,
                                uint64_t *out_keys, uint32_t *out_vals, void *stream);
sm_status merge_stable_desc_f32(const float *keys_A, const uint32_t *vals_A, int64_t n,
                                const float *keys_B, const uint32_t *vals_B, int64_t m,
                                float *out_keys, uint32_t *out_vals, void *stream);
sm_status merge_stable_desc_f64(const double *keys_A, const uint32_t *vals_A, int64_t n,
                                const double *keys_B, const uint32_t *vals_B, int64_t m,
                                double *out_keys, uint32_t *out_vals, void *stream);
sm_status merge_stable_ex_desc_u32(const uint32_t *keys_A, const uint32_t *vals_A, int64_t n,
                                   const uint32_t *keys_B, const uint32_t *vals_B, int64_t m,
                                   uint32_t *out_keys, uint32_t *out_vals, void *stream,
                                   const sm_options *opt);
sm_status merge_stable_ex_desc_i32(const int32_t *keys_A, const uint32_t *vals_A, int64_t n,
                                   const int32_t *keys_B, const uint32_t *vals_B, int64_t m,
                                   int32_t *out_keys, uint32_t *out_vals, void *stream,
                                   const sm_options *opt);
sm_status merge_stable_ex_desc_i64(const int64_t *keys_A, const uint32_t *vals_A, int64_t n,
                                   const int64_t *keys_B, const uint32_t *vals_B, int64_t m,
                                   int64_t *out_keys, uint32_t *out_vals, void *stream,
                                   const sm_options *opt);
sm_status merge_stable_ex_desc_u64(const uint64_t *keys_A, const uint32_t *vals_A, int64_t n,
                                   const uint64_t *keys_B, const uint32_t *vals_B, int64_t m,
                                   uint64_t *out_keys, uint32_t *out_vals, void *stream,
                                   const sm_options *opt);
sm_status merge_stable_ex_desc_f32(const float *keys_A, const uint32_t *vals_A, int64_t n,
                                   const float *keys_B, const uint32_t *vals_B, int64_t m,
                                   float *out_keys, uint32_t *out_vals, void *stream,
                                   const sm_options *opt);
sm_status merge_stable_ex_desc_f64(const double *keys_A, const uint32_t *vals_A, int64_t n,
                                   const double *keys_B, const uint32_t *vals_B, int64_t m,
                                   double *out_keys, uint32_t *out_vals, void *stream,
                                   const sm_options *opt);
sm_status merge_plan_ex_desc_u32(const uint32_t *keys_A, int64_t n, const uint32_t *keys_B, int64_t m,
                                 int64_t p_A, int64_t p_B, int64_t *xbar, int64_t *ybar, int64_t *tasks,
                                 void *stream);
sm_status merge_plan_ex_desc_i32(const int32_t *keys_A, int64_t n, const int32_t *keys_B, int64_t m,
                                 int64_t p_A, int64_t p_B, int64_t *xbar, int64_t *ybar, int64_t *tasks,
                                 void *stream);
sm_status merge_plan_ex_desc_i64(const int64_t *keys_A, int64_t n, const int64_t *keys_B, int64_t m,
                                 int64_t p_A, int64_t p_B, int64_t *xbar, int64_t *ybar, int64_t *tasks,
                                 void *stream);
sm_status merge_plan_ex_desc_u64(const uint64_t *keys_A, int64_t n, const uint64_t *keys_B, int64_t m,
                                 int64_t p_A, int64_t p_B, int64_t *xbar, int64_t *ybar, int64_t *tasks,
                                 void *stream);
sm_status merge_plan_ex_desc_f32(const float *keys_A, int64_t n, const float *keys_B, int64_t m,
                                 int64_t p_A, int64_t p_B, int64_t *xbar, int64_t *ybar, int64_t *tasks,
                                 void *stream);
sm_status merge_plan_ex_desc_f64(const double *keys_A, int64_t n, const double *keys_B, int64_t m,
                                 int64_t p_A, int64_t p_B, int64_t *xbar, int64_t *ybar, int64_t *tasks,
                                 void *stream);
sm_status merge_stable_batched_desc_u32(const uint32_t *keys_A, const uint32_t *vals_A, int64_t n,
                                        const int64_t *a_offsets, const uint32_t *keys_B, const uint32_t *vals_B,
                                        int64_t m, const int64_t *b_offsets, int64_t S, uint32_t *out_keys,
                                        uint32_t *out_vals, void *stream);
sm_status merge_stable_batched_desc_i32(const int32_t *keys_A, const uint32_t *vals_A, int64_t n,
                                        const int64_t *a_offsets, const int32_t *keys_B, const uint32_t *vals_B,
                                        int64_t m, const int64_t *b_offsets, int64_t S, int32_t *out_keys,
                                        uint32_t *out_vals, void *stream);
sm_status merge_stable_batched_desc_i64(const int64_t *keys_A, const uint32_t *vals_A, int64_t n,
                                        const int64_t *a_offsets, const int64_t *keys_B, const uint32_t *vals_B,
                                        int64_t m, const int64_t *b_offsets, int64_t S, int64_t *out_keys,
                                        uint32_t *out_vals, void *stream);
sm_status merge_stable_batched_desc_u64(const uint64_t *keys_A, const uint32_t *vals_A, int64_t n,
                                        const int64_t *a_offsets, const uint64_t *keys_B, const uint32_t *vals_B,
                                        int64_t m, const int64_t *b_offsets, int64_t S, uint64_t *out_keys,
                                        uint32_t *out_vals, void *stream);
sm_status merge_stable_batched_desc_f32(const float *keys_A, const uint32_t *vals_A, int64_t n,
                                        const int64_t *a_offsets, const float *keys_B, const uint32_t *vals_B,
                                        int64_t m, const int64_t *b_offsets, int64_t S, float *out_keys,
                                        uint32_t *out_vals, void *stream);
sm_status merge_stable_batched_desc_f64(const double *keys_A, const uint32_t *vals_A, int64_t n,
                                        const int64_t *a_offsets, const double *keys_B, const uint32_t *vals_B,
                                        int64_t m, const int64_t *b_offsets, int64_t S, double *out_keys,
                                        uint32_t *out_vals, void *stream);
sm_status ranks_stable_desc_u32(const uint32_t *X, int64_t len, const uint32_t *keys, int64_t nkeys, int32_t high,
                                  int64_t *out, void *stream);
sm_status ranks_stable_desc_i32(const int32_t *X, int64_t len, const int32_t *keys, int64_t nkeys, int32_t high,
                                  int64_t *out, void *stream);
sm_status ranks_stable_desc_i64(const int64_t *X, int64_t len, const int64_t *keys, int64_t nkeys, int32_t high,
                                  int64_t *out, void *stream);
sm_status ranks_stable_desc_u64(const uint64_t *X, int64_t len, const uint64_t *keys, int64_t nkeys, int32_t high,
                                  int64_t *out, void *stream);
sm_status ranks_stable_desc_f32(const float *X, int64_t len, const float *keys, int64_t nkeys, int32_t high,
                                  int64_t *out, void *stream);
sm_status ranks_stable_desc_f64(const double *X, int64_t len, const double *keys, int64_t nkeys, int32_t high,
                                  int64_t *out, void *stream);
sm_status mergesort_stable_desc_u32(uint32_t *keys, uint32_t *vals, int64_t N, void *stream);
sm_status mergesort_stable_desc_i32(int32_t *keys, uint32_t *vals, int64_t N, void *stream);
sm_status mergesort_stable_desc_i64(int64_t *keys, uint32_t *vals, int64_t N, void *stream);
sm_status mergesort_stable_desc_u64(uint64_t *keys, uint32_t *vals, int64_t N, void *stream);
sm_status mergesort_stable_desc_f32(float *keys, uint32_t *vals, int64_t N, void *stream);
sm_status mergesort_stable_desc_f64(double *keys, uint32_t *vals, int64_t N, void *stream);
sm_status mergesort_stable_ex_desc_u32(uint32_t *keys, uint32_t *vals, int64_t N, void *stream,
                                       const sm_options *opt);
sm_status mergesort_stable_ex_desc_i32(int32_t *keys, uint32_t *vals, int64_t N, void *stream,
                                       const sm_options *opt);
sm_status mergesort_stable_ex_desc_i64(int64_t *keys, uint32_t *vals, int64_t N, void *stream,
                                       const sm_options *opt);
sm_status mergesort_stable_ex_desc_u64(uint64_t *keys, uint32_t *vals, int64_t N, void *stream,
                                       const sm_options *opt);
sm_status mergesort_stable_ex_desc_f32(float *keys, uint32_t *vals, int64_t N, void *stream,
                                       const sm_options *opt);
sm_status mergesort_stable_ex_desc_f64(double *keys, uint32_t *vals, int64_t N, void *stream,
                                       const sm_options *opt);


/* ---------------------------------------------------------------------
 * Wide / struct payloads -- SURVEY.md §8(f) row 2.  Each element carries a
 * payload ROW of val_bytes bytes (1 <= val_bytes <= 4096: 64-bit values,
 * structs, fixed-size records), moved with its key:
 *   merge_stable_wide_<K>          as merge_stable_<K>, vals_* = rows
 *   merge_stable_batched_wide_<K>  as merge_stable_batched_<K>
 *   mergesort_stable_wide_<K>      as mergesort_stable_<K> (rows sorted in
 *                                  place with their keys, stable)
 * and the same for the descending order (_wide_desc_<K>).  Payload
 * pointers are required (use the uint32 / keys-only calls otherwise).
 * DEVICE pointers only (host -> SM_EINVAL).  Rows are copied in the widest
 * word (16/8/4/2/1 bytes) that divides val_bytes and the three payload
 * pointers' alignment.
 * Device path: the method runs unchanged with a uint32 INDEX payload (the
 * position of each element in A||B, or in the sort input), then one gather
 * kernel moves row idx[k] to output row k.  merge_stable_wide and
 * merge_stable_batched_wide with 8-byte rows and 8-byte-aligned payload
 * pointers move the rows directly as the merge kernel's 64-bit payload (no
 * index, no gather).  Scratch: 2 (n+m) uint32 (merge), N uint32 + N rows
 * (sort), stream-ordered as above.
 * ------------------------------------------------------------------- */
sm_status merge_stable_wide_u32(const uint32_t *keys_A, const void *vals_A, int64_t n,
                                const uint32_t *keys_B, const void *vals_B, int64_t m,
                                uint32_t *out_keys, void *out_vals, int64_t val_bytes, void *stream);
sm_status merge_stable_wide_i32(const int32_t *keys_A, const void *vals_A, int64_t n,
                                const int32_t *keys_B, const void *vals_B, int64_t m,
                                int32_t *out_keys, void *out_vals, int64_t val_bytes, void *stream);
sm_status merge_stable_wide_i64(const int64_t *keys_A, const void *vals_A, int64_t n,
                                const int64_t *keys_B, const void *vals_B, int64_t m,
                                int64_t *out_keys, void *out_vals, int64_t val_bytes, void *stream);
sm_status merge_stable_wide_u64(const uint64_t *keys_A, const void *vals_A, int64_t n,
                                const uint64_t *keys_B, const void *vals_B, int64_t m,
                                uint64_t *out_keys, void *out_vals, int64_t val_bytes, void *stream);
sm_status merge_stable_wide_f32(const float *keys_A, const void *vals_A, int64_t n,
                                const float *keys_B, const void *vals_B, int64_t m,
                                float *out_keys, void *out_vals, int64_t val_bytes, void *stream);
sm_status merge_stable_wide_f64(const double *keys_A, const void *vals_A, int64_t n,
                                const double *keys_B, const void *vals_B, int64_t m,
                                double *out_keys, void *out_vals, int64_t val_bytes, void *stream);
sm_status merge_stable_wide_desc_u32(const uint32_t *keys_A, const void *vals_A, int64_t n,
                                     const uint32_t *keys_B, const void *vals_B, int64_t m,
                                     uint32_t *out_keys, void *out_vals, int64_t val_bytes, void *stream);
sm_status merge_stable_wide_desc_i32(const int32_t *keys_A, const void *vals_A, int64_t n,
                                     const int32_t *keys_B, const void *vals_B, int64_t m,
                                     int32_t *out_keys, void *out_vals, int64_t val_bytes, void *stream);
sm_status merge_stable_wide_desc_i64(const int64_t *keys_A, const void *vals_A, int64_t n,
                                     const int64_t *keys_B, const void *vals_B, int64_t m,
                                     int64_t *out_keys, void *out_vals, int64_t val_bytes, void *stream);
sm_status merge_stable_wide_desc_u64(const uint64_t *keys_A, const void *vals_A, int64_t n,
                                     const uint64_t *keys_B, const void *vals_B, int64_t m,
                                     uint64_t *out_keys, void *out_vals, int64_t val_bytes, void *stream);
sm_status merge_stable_wide_desc_f32(const float *keys_A, const void *vals_A, int64_t n,
                                     const float *keys_B, const void *vals_B, int64_t m,
                                     float *out_keys, void *out_vals, int64_t val_bytes, void *stream);
sm_status merge_stable_wide_desc_f64(const double *keys_A, const void *vals_A, int64_t n,
                                     const double *keys_B, const void *vals_B, int64_t m,
                                     double *out_keys, void *out_vals, int64_t val_bytes, void *stream);
sm_status merge_stable_batched_wide_u32(const uint32_t *keys_A, const void *vals_A, int64_t n,
                                        const int64_t *a_offsets, const uint32_t *keys_B, const void *vals_B,
                                        int64_t m, const int64_t *b_offsets, int64_t S, uint32_t *out_keys,
                                        void *out_vals, int64_t val_bytes, void *stream);
sm_status merge_stable_batched_wide_i32(const int32_t *keys_A, const void *vals_A, int64_t n,
                                        const int64_t *a_offsets, const int32_t *keys_B, const void *vals_B,
                                        int64_t m, const int64_t *b_offsets, int64_t S, int32_t *out_keys,
                                        void *out_vals, int64_t val_bytes, void *stream);
sm_status merge_stable_batched_wide_i64(const int64_t *keys_A, const void *vals_A, int64_t n,
                                        const int64_t *a_offsets, const int64_t *keys_B, const void *vals_B,
                                        int64_t m, const int64_t *b_offsets, int64_t S, int64_t *out_keys,
                                        void *out_vals, int64_t val_bytes, void *stream);
sm_status merge_stable_batched_wide_u64(const uint64_t *keys_A, const void *vals_A, int64_t n,
                                        const int64_t *a_offsets, const uint64_t *keys_B, const void *vals_B,
                                        int64_t m, const int64_t *b_offsets, int64_t S, uint64_t *out_keys,
                                        void *out_vals, int64_t val_bytes, void *stream);
sm_status merge_stable_batched_wide_f32(const float *keys_A, const void *vals_A, int64_t n,
                                        const int64_t *a_offsets, const float *keys_B, const void *vals_B,
                                        int64_t m, const int64_t *b_offsets, int64_t S, float *out_keys,
                                        void *out_vals, int64_t val_bytes, void *stream);
sm_status merge_stable_batched_wide_f64(const double *keys_A, const void *vals_A, int64_t n,
                                        const int64_t *a_offsets, const double *keys_B, const void *vals_B,
                                        int64_t m, const int64_t *b_offsets, int64_t S, double *out_keys,
                                        void *out_vals, int64_t val_bytes, void *stream);
sm_status merge_stable_batched_wide_desc_u32(const uint32_t *keys_A, const void *vals_A, int64_t n,
                                             const int64_t *a_offsets, const uint32_t *keys_B, const void *vals_B,
                                             int64_t m, const int64_t *b_offsets, int64_t S, uint32_t *out_keys,
                                             void *out_vals, int64_t val_bytes, void *stream);
sm_status merge_stable_batched_wide_desc_i32(const int32_t *keys_A, const void *vals_A, int64_t n,
                                             const int64_t *a_offsets, const int32_t *keys_B, const void *vals_B,
                                             int64_t m, const int64_t *b_offsets, int64_t S, int32_t *out_keys,
                                             void *out_vals, int64_t val_bytes, void *stream);
sm_status merge_stable_batched_wide_desc_i64(const int64_t *keys_A, const void *vals_A, int64_t n,
                                             const int64_t *a_offsets, const int64_t *keys_B, const void *vals_B,
                                             int64_t m, const int64_t *b_offsets, int64_t S, int64_t *out_keys,
                                             void *out_vals, int64_t val_bytes, void *stream);
sm_status merge_stable_batched_wide_desc_u64(const uint64_t *keys_A, const void *vals_A, int64_t n,
                                             const int64_t *a_offsets, const uint64_t *keys_B, const void *vals_B,
                                             int64_t m, const int64_t *b_offsets, int64_t S, uint64_t *out_keys,
                                             void *out_vals, int64_t val_bytes, void *stream);
sm_status merge_stable_batched_wide_desc_f32(const float *keys_A, const void *vals_A, int64_t n,
                                             const int64_t *a_offsets, const float *keys_B, const void *vals_B,
                                             int64_t m, const int64_t *b_offsets, int64_t S, float *out_keys,
                                             void *out_vals, int64_t val_bytes, void *stream);
sm_status merge_stable_batched_wide_desc_f64(const double *keys_A, const void *vals_A, int64_t n,
                                             const int64_t *a_offsets, const double *keys_B, const void *vals_B,
                                             int64_t m, const int64_t *b_offsets, int64_t S, double *out_keys,
                                             void *out_vals, int64_t val_bytes, void *stream);
sm_status mergesort_stable_wide_u32(uint32_t *keys, void *vals, int64_t N, int64_t val_bytes, void *stream);
sm_status mergesort_stable_wide_i32(int32_t *keys, void *vals, int64_t N, int64_t val_bytes, void *stream);
sm_status mergesort_stable_wide_i64(int64_t *keys, void *vals, int64_t N, int64_t val_bytes, void *stream);
sm_status mergesort_stable_wide_u64(uint64_t *keys, void *vals, int64_t N, int64_t val_bytes, void *stream);
sm_status mergesort_stable_wide_f32(float *keys, void *vals, int64_t N, int64_t val_bytes, void *stream);
sm_status mergesort_stable_wide_f64(double *keys, void *vals, int64_t N, int64_t val_bytes, void *stream);
sm_status mergesort_stable_wide_desc_u32(uint32_t *keys, void *vals, int64_t N, int64_t val_bytes, void *stream);
sm_status mergesort_stable_wide_desc_i32(int32_t *keys, void *vals, int64_t N, int64_t val_bytes, void *stream);
sm_status mergesort_stable_wide_desc_i64(int64_t *keys, void *vals, int64_t N, int64_t val_bytes, void *stream);
sm_status mergesort_stable_wide_desc_u64(uint64_t *keys, void *vals, int64_t N, int64_t val_bytes, void *stream);
sm_status mergesort_stable_wide_desc_f32(float *keys, void *vals, int64_t N, int64_t val_bytes, void *stream);
sm_status mergesort_stable_wide_desc_f64(double *keys, void *vals, int64_t N, int64_t val_bytes, void *stream);


/* ---------------------------------------------------------------------
 * 128-bit keys -- SURVEY.md §8(f) row 2 (128-bit keys, (key, tie) tuples):
 * every call above for sm_u128 keys (unsigned, = lexicographic (hi, lo)),
 * ascending and descending, uint32 / wide payloads.  Same contracts; the
 * key arrays must be 16-byte aligned.  Device path: the same kernels with
 * 16-byte keys (the C++ merge over the order view; 32 radix digits in the
 * block sort).
 * ------------------------------------------------------------------- */
sm_status merge_stable_u128(const sm_u128 *keys_A, const uint32_t *vals_A, int64_t n,
                            const sm_u128 *keys_B, const uint32_t *vals_B, int64_t m,
                            sm_u128 *out_keys, uint32_t *out_vals, void *stream);
sm_status merge_stable_batched_u128(const sm_u128 *keys_A, const uint32_t *vals_A, int64_t n,
                                    const int64_t *a_offsets, const sm_u128 *keys_B, const uint32_t *vals_B,
                                    int64_t m, const int64_t *b_offsets, int64_t S, sm_u128 *out_keys,
                                    uint32_t *out_vals, void *stream);
sm_status ranks_stable_u128(const sm_u128 *X, int64_t len, const sm_u128 *keys, int64_t nkeys, int32_t high,
                              int64_t *out, void *stream);
sm_status mergesort_stable_u128(sm_u128 *keys, uint32_t *vals, int64_t N, void *stream);
sm_status merge_stable_ex_u128(const sm_u128 *keys_A, const uint32_t *vals_A, int64_t n,
                               const sm_u128 *keys_B, const uint32_t *vals_B, int64_t m,
                               sm_u128 *out_keys, uint32_t *out_vals, void *stream,
                               const sm_options *opt);
sm_status merge_plan_ex_u128(const sm_u128 *keys_A, int64_t n, const sm_u128 *keys_B, int64_t m,
                             int64_t p_A, int64_t p_B, int64_t *xbar, int64_t *ybar, int64_t *tasks,
                             void *stream);
sm_status mergesort_stable_ex_u128(sm_u128 *keys, uint32_t *vals, int64_t N, void *stream,
                                   const sm_options *opt);
sm_status merge_stable_desc_u128(const sm_u128 *keys_A, const uint32_t *vals_A, int64_t n,
                                 const sm_u128 *keys_B, const uint32_t *vals_B, int64_t m,
                                 sm_u128 *out_keys, uint32_t *out_vals, void *stream);
sm_status merge_stable_ex_desc_u128(const sm_u128 *keys_A, const uint32_t *vals_A, int64_t n,
                                    const sm_u128 *keys_B, const uint32_t *vals_B, int64_t m,
                                    sm_u128 *out_keys, uint32_t *out_vals, void *stream,
                                    const sm_options *opt);
sm_status merge_plan_ex_desc_u128(const sm_u128 *keys_A, int64_t n, const sm_u128 *keys_B, int64_t m,
                                  int64_t p_A, int64_t p_B, int64_t *xbar, int64_t *ybar, int64_t *tasks,
                                  void *stream);
sm_status merge_stable_batched_desc_u128(const sm_u128 *keys_A, const uint32_t *vals_A, int64_t n,
                                         const int64_t *a_offsets, const sm_u128 *keys_B, const uint32_t *vals_B,
                                         int64_t m, const int64_t *b_offsets, int64_t S, sm_u128 *out_keys,
                                         uint32_t *out_vals, void *stream);
sm_status ranks_stable_desc_u128(const sm_u128 *X, int64_t len, const sm_u128 *keys, int64_t nkeys, int32_t high,
                                   int64_t *out, void *stream);
sm_status mergesort_stable_desc_u128(sm_u128 *keys, uint32_t *vals, int64_t N, void *stream);
sm_status mergesort_stable_ex_desc_u128(sm_u128 *keys, uint32_t *vals, int64_t N, void *stream,
                                        const sm_options *opt);
sm_status merge_stable_wide_u128(const sm_u128 *keys_A, const void *vals_A, int64_t n,
                                 const sm_u128 *keys_B, const void *vals_B, int64_t m,
                                 sm_u128 *out_keys, void *out_vals, int64_t val_bytes, void *stream);
sm_status merge_stable_wide_desc_u128(const sm_u128 *keys_A, const void *vals_A, int64_t n,
                                      const sm_u128 *keys_B, const void *vals_B, int64_t m,
                                      sm_u128 *out_keys, void *out_vals, int64_t val_bytes, void *stream);
sm_status merge_stable_batched_wide_u128(const sm_u128 *keys_A, const void *vals_A, int64_t n,
                                         const int64_t *a_offsets, const sm_u128 *keys_B, const void *vals_B,
                                         int64_t m, const int64_t *b_offsets, int64_t S, sm_u128 *out_keys,
                                         void *out_vals, int64_t val_bytes, void *stream);
sm_status merge_stable_batched_wide_desc_u128(const sm_u128 *keys_A, const void *vals_A, int64_t n,
                                              const int64_t *a_offsets, const sm_u128 *keys_B, const void *vals_B,
                                              int64_t m, const int64_t *b_offsets, int64_t S, sm_u128 *out_keys,
                                              void *out_vals, int64_t val_bytes, void *stream);
sm_status mergesort_stable_wide_u128(sm_u128 *keys, void *vals, int64_t N, int64_t val_bytes, void *stream);
sm_status mergesort_stable_wide_desc_u128(sm_u128 *keys, void *vals, int64_t N, int64_t val_bytes, void *stream);

#ifdef __cplusplus
}
#endif

#endif /* STABLEMERGE_H */
