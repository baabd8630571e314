// sm_kernels.cuh -- the kernels of the B200 stable merge / merge sort.
//
//   K1  k_cross_ranks   rows a1/a2: one search per block start, rank_low of
//                       A[x_i] in B / rank_high of B[y_j] in A  (L304-309)
//   --  stream order (or PDL griddepcontrol.wait) = the single
//       synchronisation of L373-375 (row a3)
//   K2  k_tasks         rows a4-a7: persistent, warp-specialised; O(1)
//                       classification of every block start's task, then
//                       copy (a, e) or stable merge (b, c, d) through a TMA
//                       shared-memory ring, several tasks packed per stage
//   K3  k_block_sort    row a8: stable LSD radix sort of one run per CTA
//   --  k_cross_ranks_smp  K1 for one plain merge, top levels from a shared-
//                       memory sample of the searched array
//   --  k_classify      Steps 3-4 ahead of K2 for the segmented modes
//   --  k_batch_*       batched merges: segment table
//   --  k_iota, k_gather_rows   wide / struct payloads (§8(f) row 2)
//   --  k_block_start_keys, k_rank_keys   coarse partition (>= 2^31), ranks
//   --  k_plan_dump     Steps 1-4 only: the task table for parity tests
//
// All in-kernel indices are 32-bit (larger calls are cut into sub-problems
// below 2^31 on the host side: stablemerge.cu, merge_large_device).
#pragma once
#include "sm_device.cuh"

namespace sm {
namespace {   // internal linkage: every translation unit keeps its own kernels

// ----------------------------------------------------------------- K1
#ifndef K1_WAYS_SORT
#define K1_WAYS_SORT 2   // fan-out of the one-thread-per-search kernel in the sort rounds (binary: C5 K1 -10%)
#endif
#ifndef K1_WAYS_SEG
#define K1_WAYS_SEG 4    // ... for the batched merges (4-ary: binary measured +18%)
#endif
#ifndef K1_WAYS
#define K1_WAYS 4
#endif
// Rows a1/a2.  A group of G lanes performs one rank search cooperatively:
// each round the G lanes probe G evenly spaced keys of the remaining
// interval and a group ballot picks the sub-interval holding the rank:
// ~log_{G+1}(len) dependent rounds.  Used (G = 32) when there are few
// searches, so latency, not probe traffic, is what counts.
//   high = false: rank_low(x, X)  = #{X[t] <  x}   (L119-123)
//   high = true:  rank_high(x, X) = #{X[t] <= x}   (L124-128)
template <int GG>
__device__ __forceinline__ int probe_pos(int lo, int n, int s) {
    return lo + (int)(((long long)(s + 1) * n) / (GG + 1));
}

template <typename K, int G>
__device__ __forceinline__ int group_rank(const K* __restrict__ X, int len, K x, bool high, bool active) {
    const int lane = threadIdx.x & 31;
    const int sub = lane % G;
    const int shift = lane - sub;
    int lo = 0, hi = active ? len : 0;     // rank in [lo, hi]; X[lo, hi) undecided
    while (__any_sync(0xffffffffu, hi > lo)) {
        const int n = hi - lo;
        const int pos = n > G ? probe_pos<G>(lo, n, sub) : lo + sub;   // n <= G: probe every key left
        bool pred = false;
        if (hi > lo && sub < min(G, n)) {
            const K v = ldg_key(X + pos);
            pred = high ? key_le(v, x) : key_lt(v, x);
        }
        const unsigned bal = (__ballot_sync(0xffffffffu, pred) >> shift) & (G == 32 ? 0xffffffffu : ((1u << (G & 31)) - 1u));
        const int t = __popc(bal);          // probes passed: a prefix of the probing lanes
        if (hi > lo) {
            if (n <= G) {
                lo = lo + t;
                hi = lo;
            } else {
                const int plast = t > 0 ? probe_pos<G>(lo, n, t - 1) : lo - 1;
                const int pnext = t < G ? probe_pos<G>(lo, n, t) : hi;
                lo = plast + 1;
                hi = pnext;
            }
        }
    }
    return lo;
}

// One-thread rank search with WAYS-1 independent probes per round (the
// quantile points of the remaining interval): log_WAYS(len) dependent
// memory rounds instead of log_2(len), (WAYS-1)/log2(WAYS) loads per level.
//   high = false: rank_low(x, X) = #{X[t] < x};  high = true: rank_high = #{X[t] <= x}
// FINAL > 0: once at most FINAL keys are undecided they are all loaded at once
// (independent loads of one or two lines) and counted, instead of
// log_WAYS(FINAL) more dependent rounds on those same lines.
#ifndef K1_FINAL
#define K1_FINAL 0       // measured on C2 (K1 per call): off 23.2 us, 16 keys 23.5, 32 keys 26.5, 64 keys 28.2
#endif
template <typename K, int WAYS, int FINAL = 0>
__device__ __forceinline__ int rank_kary(const K* __restrict__ X, int len, K x, bool high) {
    int lo = 0, n = len;                     // rank in [lo, lo + n]; X[lo, lo+n) undecided
    while (n >= WAYS && n > FINAL) {
        const int q = n / WAYS;
        K v[WAYS - 1];
#pragma unroll
        for (int k = 0; k < WAYS - 1; ++k) v[k] = ldg_key(X + lo + (k + 1) * q - 1);   // independent loads
        int t = 0;                           // probes passed: a prefix
#pragma unroll
        for (int k = 0; k < WAYS - 1; ++k) t += (high ? key_le(v[k], x) : key_lt(v[k], x)) ? 1 : 0;
        // probes at lo + (k+1)q - 1: passing t of them leaves [lo + t*q, lo + (t+1)q - 1)
        // (the last sub-interval runs to the end of the interval)
        lo += t * q;
        n = (t == WAYS - 1) ? n - t * q : q - 1;
    }
    if constexpr (FINAL > 0) {
        // X sorted: the keys passing are a prefix of the n left
        int t = 0;
#pragma unroll
        for (int k = 0; k < FINAL; ++k) {
            if (k < n) {
                const K v = ldg_key(X + lo + k);
                t += (high ? key_le(v, x) : key_lt(v, x)) ? 1 : 0;
            }
        }
        return lo + t;
    }
    while (n > 0) {                          // binary tail
        const int half = n >> 1;
        const bool right = high ? key_le(ldg_key(X + lo + half), x) : key_lt(ldg_key(X + lo + half), x);
        lo = right ? lo + half + 1 : lo;
        n = right ? n - half - 1 : half;
    }
    return lo;
}

// K1 (rows a1/a2): one group of G lanes per cross rank, searching the whole
// other array (G = 1: a plain binary search per thread, measured fastest on
// B200 for every config: the top levels are shared by all searches and hit
// L1/L2, the bottom levels are private DRAM probes, one sector each).
//   Step 1: xbar_i = rank_low(A[x_i], B) (L304-306), xbar_pA = m, empty block start -> m (R4)
//   Step 2: ybar_j = rank_high(B[y_j], A) (L307-309), ybar_pB = n
template <typename K, int G>
__global__ void __launch_bounds__(256) k_cross_ranks(const K* __restrict__ A, const K* __restrict__ B, Geom g,
                                                     int* __restrict__ xbar, int* __restrict__ ybar) {
    pdl_wait();   // a batch's segment table (no-op for plain launches)
    zero_task_counter(g.ctr);
    const long long item = ((long long)blockIdx.x * blockDim.x + threadIdx.x) / G;
    const bool valid = item < (long long)total_rank_items(g);
    int s = 0, t = 0;
    if (valid) s = locate(g, (int)item, true, t);
    const Seg sg = segment(g, s, xbar, ybar);
    const bool sideA = t <= sg.pA;
    const int idx = sideA ? t : t - sg.pA - 1;
    const int plen = sideA ? sg.pA : sg.pB;          // own blocks
    const int own_len = sideA ? sg.n : sg.m;
    const int oth_len = sideA ? sg.m : sg.n;         // searched array
    const bool search = valid && idx < plen && idx < own_len;   // x_idx < own_len  <=>  idx < own_len
    K x = K(0);
    if (search) x = ldg_key((sideA ? A + sg.aoff : B + sg.boff) + Blocks(own_len, plen).start(idx));
    int r;
    if constexpr (G == 1) {
        const K* X = sideA ? B + sg.boff : A + sg.aoff;
        r = !search ? 0
            : g.sort == 1 ? rank_kary<K, K1_WAYS_SORT>(X, oth_len, x, !sideA) : rank_kary<K, K1_WAYS_SEG>(X, oth_len, x, !sideA);
    } else {
        r = group_rank<K, G>(sideA ? B + sg.boff : A + sg.aoff, oth_len, x, !sideA, search);
    }
    if (valid && (threadIdx.x % G) == 0) {
        const int v = search ? r : oth_len;
        if (sideA) sg.xs[idx] = v;
        else sg.ys[idx] = v;
    }
    pdl_launch_dependents();
}

// K1 for one plain merge (mode 0) with the top levels of every search in
// shared memory (BASELINE.json north_star): each CTA first loads a sample
// of the searched array(s) -- the last key of each of SMP equal chunks --
// with all its threads at once (one round of independent loads, mostly L2
// hits after the first CTA), binary-searches it in shared memory, and only
// the chunk found (len / SMP keys) is searched in global memory.
//   rank_low(x):  c = #{chunks whose last key < x}: every key of chunks < c
//                 is < x, chunk c's last is >= x, so the rank lies in chunk c
//   rank_high:    the same with <=
template <typename K, int SMP>
__global__ void __launch_bounds__(256) k_cross_ranks_smp(const K* __restrict__ A, const K* __restrict__ B, Geom g,
                                                         int* __restrict__ xbar, int* __restrict__ ybar) {
    extern __shared__ __align__(16) char k1_smem[];
    K (*smp)[SMP] = reinterpret_cast<K (*)[SMP]>(k1_smem);   // [0]: sample of B (A-side searches), [1]: of A
    pdl_wait();
    zero_task_counter(g.ctr);
    const int n = g.n, m = g.m, pA = g.pA, pB = g.pB;
    const int items = pA + 1 + pB + 1;
    const int i0 = blockIdx.x * blockDim.x;
    const int i1 = min(items, i0 + (int)blockDim.x);
    const bool need[2] = {i0 <= pA && m > 0, i1 > pA + 1 && n > 0};
    const K* X[2] = {B, A};
    const int len[2] = {m, n};
    // this thread's own block-start key first: its load is in flight while
    // the sample is gathered (one dependent memory round less)
    const int item = i0 + threadIdx.x;
    const bool sideA = item <= pA;
    const int idx = sideA ? item : item - pA - 1;
    const int plen = sideA ? pA : pB;
    const int own_len = sideA ? n : m;
    const int q = sideA ? 0 : 1;
    const int oth = len[q];
    const bool search = item < items && idx < plen && idx < own_len && oth > 0;
    K x = K(0);
    if (search) x = ldg_key((sideA ? A : B) + Blocks(own_len, plen).start(idx));
#pragma unroll
    for (int q2 = 0; q2 < 2; ++q2) {
        if (!need[q2]) continue;
        const int stride = (len[q2] + SMP - 1) / SMP;
        for (int k = threadIdx.x; k < SMP; k += blockDim.x) {
            const long long at = min((long long)(k + 1) * stride, (long long)len[q2]) - 1;
            smp[q2][k] = ldg_key(X[q2] + at);
        }
    }
    __syncthreads();
    if (item >= items) return;
    int r = oth;                                       // empty block start / sentinel: the other length (R4)
    if (search) {
        const bool high = !sideA;
        const int stride = (oth + SMP - 1) / SMP;
        const int chunks = (oth + stride - 1) / stride;
        int lo = 0, hi = chunks;                       // chunks whose last key passes
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            const bool pass = high ? key_le(smp[q][mid], x) : key_lt(smp[q][mid], x);
            lo = pass ? mid + 1 : lo;
            hi = pass ? hi : mid;
        }
        const int c0 = lo * stride;
        r = c0 >= oth ? oth : c0 + rank_kary<K, K1_WAYS, K1_FINAL>(X[q] + c0, min(stride, oth - c0), x, high);
    }
    const int v = (idx < plen && idx < own_len) ? r : oth;
    if (sideA) xbar[idx] = v;
    else ybar[idx] = v;
    pdl_launch_dependents();
}

#ifndef SM_REFILL_TDESC
#define SM_REFILL_TDESC 8     // window refill threshold when tasks come pre-classified (k_classify)
#endif
#ifndef SM_K2_CHUNK
#define SM_K2_CHUNK 8         // tasks per reservation of the dynamic assignment, at most (<= 8-byte elements;
#endif                        //   measured: 4 and 16 within 1% on C2 / C5)
#ifndef SM_K2_CHUNK_WIDE
#define SM_K2_CHUNK_WIDE 4    // ... wider elements (C3 / C4: 4 measured 0.5% faster than 8)
#endif
#ifndef SM_K2_TAILWIN
#define SM_K2_TAILWIN 16      // the shortest refill threshold near the end of the dynamic part (4 / 8 / 32
                              //   measured within 0.5%; a fixed static share first: no gain)
#endif
#ifndef SM_K2_DYN_MIN
#define SM_K2_DYN_MIN 8       // dynamic assignment only above this many tasks per CTA
#endif
#ifndef SM_K2_DYN
#define SM_K2_DYN 1           // 0: static round-robin task assignment (experiment)
#endif
#ifndef SM_K2_INTERLEAVE
#define SM_K2_INTERLEAVE 1    // balanced segments: K2 takes A-side and B-side tasks alternately
#endif
// The order in which K2 takes a segment's tasks.  When the segment's block
// counts are balanced (p_A, p_B within a factor 2), A-side task i and
// B-side task i alternate: their ranges lie at nearby places of A, B and C,
// so the CTAs' reads of A and B and their writes of C advance as one front
// each (measured: C2 K2 -2%); unbalanced segments (C3, C4) keep index order,
// where whole runs of A-side tasks are contiguous in C (alternating there
// was 5% slower on C4).  Position k -> local task index, and its inverse.
__device__ __forceinline__ bool interleaved(int pA, int pB) {
    return SM_K2_INTERLEAVE && pA > 0 && pB > 0 && 2 * min(pA, pB) >= max(pA, pB);
}
__device__ __forceinline__ int task_at(int k, int pA, int pB) {
    if (!interleaved(pA, pB)) return k;
    const int mn = min(pA, pB);
    if (k < 2 * mn) return (k & 1) ? pA + (k >> 1) : (k >> 1);
    return pA >= pB ? k - mn : pA + k - mn;        // the rest of the larger side, in order
}
__device__ __forceinline__ int task_pos(int t, int pA, int pB) {
    if (!interleaved(pA, pB)) return t;
    const int mn = min(pA, pB);
    const int side_i = t < pA ? t : t - pA;
    if (side_i < mn) return 2 * side_i + (t < pA ? 0 : 1);
    return 2 * mn + (side_i - mn);
}
// Decode a task (rows a4/a5).  Mode 3 (the merge-path comparison, not the
// paper's method): task k is output tile [kT, (k+1)T) with the diagonal
// splits of K1mp in xbar.
__device__ __forceinline__ Task decode_task(const Geom& g, int task, const int* xbar, const int* ybar, Seg& sg) {
    if (g.sort == 3) {
        sg = segment(g, 0, (int*)xbar, (int*)ybar);
        const int d0 = task * g.T, d1 = min(g.n + g.m, d0 + g.T);
        Task t;
        t.side = 0; t.kase = CASE_B;
        t.a0 = xbar[task]; t.a1 = xbar[task + 1];
        t.b0 = d0 - t.a0; t.b1 = d1 - t.a1;
        return t;
    }
    int t;
    const int s = locate(g, task, false, t);
    sg = segment(g, s, (int*)xbar, (int*)ybar);
    if (sg.pA == 0) {                                  // batched segment within one tile (R19)
        Task w;
        w.side = 0;
        w.kase = (sg.n > 0 && sg.m > 0) ? CASE_B : CASE_A;
        w.a0 = 0; w.a1 = sg.n; w.b0 = 0; w.b1 = sg.m;
        return w;
    }
    const Blocks xa(sg.n, sg.pA), yb(sg.m, sg.pB);
    return t < sg.pA ? classify_a_side(t, xa, yb, sg.xs, sg.ys) : classify_b_side(t - sg.pA, xa, yb, sg.xs, sg.ys);
}

// ---- small plain merges in one launch (g.fuse) ----------------------------
// When every CTA has at most K2L_MAXP tasks (C1: 2^20 + 2^20 elements,
// 1094 tasks on 296 CTAs), K1 is a latency-bound launch of its own (~10 of
// the call's 23 µs).  Then no K1 runs: CTA b takes the consecutive positions
// [bP, (b+1)P) of K2's order and its warps compute the cross ranks its
// tasks read (Steps 1-2: x̄ over the A-side tasks' block
// starts and the next one, ȳ likewise, plus a margin), a warp per search;
// then each task is classified (Steps 3-4); the one rank of the other side
// a case (c) or (e) task may still need (ȳ_j / x̄_i)
// comes from a second round of searches.  Every rank a task reads is final
// before the task is classified -- the single synchronisation of L373-375,
// per CTA -- and no CTA depends on another.
constexpr int K2L_MAXP = 8;                 // tasks per CTA at most in this mode
#ifndef SM_SMALL_PREFETCH
#define SM_SMALL_PREFETCH 1                 // own blocks prefetched to L2 while the ranks are searched
#endif
constexpr int K2L_MAXR = K2L_MAXP + 4;      // local x̄ / ȳ entries
struct K2Local {
    int k0, k1;                             // the CTA's positions
    int ia0, nx, jb0, ny;                   // x̄ over [ia0, ia0 + nx), ȳ over [jb0, jb0 + ny)
    int xl[K2L_MAXR], yl[K2L_MAXR];
    int miss_side[K2L_MAXP], miss_idx[K2L_MAXP], miss_val[K2L_MAXP];
    int4 desc[K2L_MAXP];                    // the tasks, classified: A start, B start, C start, la << 16 | lb
};
// A rank array as classification reads it: the local entries, the sentinel
// and empty block starts (the other length, R4), the second round's extras;
// an entry not there is recorded in *miss (first one only) and reads as 0.
struct LocalView {
    const K2Local* L;
    int side;                               // 0: x̄ (A's block starts in B), 1: ȳ
    int p, own_len, oth_len;
    int* miss;
    __device__ __forceinline__ int operator[](int i) const {
        if (i >= p || i >= own_len) return oth_len;
        const int lo = side ? L->jb0 : L->ia0, cnt = side ? L->ny : L->nx;
        if (i >= lo && i < lo + cnt) return side ? L->yl[i - lo] : L->xl[i - lo];
        for (int k = 0; k < L->k1 - L->k0; ++k)
            if (L->miss_side[k] == side && L->miss_idx[k] == i) return L->miss_val[k];
        if (miss && *miss < 0) *miss = i;
        return 0;
    }
};
template <typename K>
__device__ __forceinline__ int warp_rank(const K* A, const K* B, const Geom& g, const Blocks& xa, const Blocks& yb,
                                         int side, int i) {
    // x̄_i = rank_low(A[x_i], B) (side 0) or ȳ_i = rank_high(B[y_i], A) (side 1), a whole warp per search
    const int p = side ? g.pB : g.pA, own_len = side ? g.m : g.n, oth_len = side ? g.n : g.m;
    const bool search = i < p && i < own_len;
    K x = K(0);
    if (search) x = ldg_key(side ? B + yb.start(i) : A + xa.start(i));
    const int r = group_rank<K, 32>(side ? A : B, oth_len, x, side == 1, search);
    return search ? r : oth_len;
}
template <typename K, int NV>
__device__ void k2_local_prologue(const K* A, const K* B, const Geom& g, K2Local* L) {
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5, NW = (int)(blockDim.x >> 5);
    const int ntasks = g.pA + g.pB;
    const int P = (ntasks + (int)gridDim.x - 1) / (int)gridDim.x;
    const Blocks xa(g.n, g.pA), yb(g.m, g.pB);
    if (tid == 0) {
        const int k0 = min(ntasks, (int)blockIdx.x * P), k1 = min(ntasks, k0 + P);
        int a_lo = INT_MAX, a_hi = -1, b_lo = INT_MAX, b_hi = -1;
        for (int k = k0; k < k1; ++k) {
            const int t = task_at(k, g.pA, g.pB);
            if (t < g.pA) { a_lo = min(a_lo, t); a_hi = max(a_hi, t); }
            else { b_lo = min(b_lo, t - g.pA); b_hi = max(b_hi, t - g.pA); }
        }
        // own tasks' entries i, i + 1 and a margin of one before, two after
        // (balanced inputs: the other side's entries case (c) / (e) reads)
        if (a_hi < 0) { a_lo = b_lo; a_hi = b_hi; }
        if (b_hi < 0) { b_lo = a_lo; b_hi = a_hi; }
        L->k0 = k0;
        L->k1 = k1;
        L->ia0 = max(0, a_lo - 1);
        L->nx = min(g.pA - 1, a_hi + 2) - L->ia0 + 1;
        L->jb0 = max(0, b_lo - 1);
        L->ny = min(g.pB - 1, b_hi + 2) - L->jb0 + 1;
        if (k0 >= k1) L->nx = L->ny = 0;
    }
    __syncthreads();
    const int nx = max(0, L->nx), ny = max(0, L->ny), np = L->k1 - L->k0;
    for (int e = w; e < nx + ny; e += NW) {                 // round 1: a warp per entry
        const int side = e < nx ? 0 : 1;
        const int i = side ? L->jb0 + e - nx : L->ia0 + e;
        const int r = warp_rank<K>(A, B, g, xa, yb, side, i);
        if (lane == 0) (side ? L->yl : L->xl)[i - (side ? L->jb0 : L->ia0)] = r;
    }
    if (tid < K2L_MAXP) L->miss_side[tid] = -1;
    __syncthreads();
    int miss = -1, side = 0;
    if (tid < np) {                                          // classify; note the entry it lacks, if any
        const int t0 = task_at(L->k0 + tid, g.pA, g.pB);
        side = t0 < g.pA ? 1 : 0;                            // an A-side task reads ȳ, a B-side task x̄
        const LocalView xv{L, 0, g.pA, g.n, g.m, side == 0 ? &miss : nullptr};
        const LocalView yv{L, 1, g.pB, g.m, g.n, side == 1 ? &miss : nullptr};
        if (t0 < g.pA) classify_a_side(t0, xa, yb, xv, yv);
        else classify_b_side(t0 - g.pA, xa, yb, xv, yv);
        if (miss >= 0) {
            L->miss_side[tid] = side;
            L->miss_idx[tid] = miss;
        }
    }
    __syncthreads();
    for (int k = w; k < np; k += NW) {                      // round 2: the missing entries
        if (L->miss_side[k] < 0) continue;
        const int r = warp_rank<K>(A, B, g, xa, yb, L->miss_side[k], L->miss_idx[k]);
        if (lane == 0) L->miss_val[k] = r;
    }
    __syncthreads();
    if (tid < np) {
        const int t0 = task_at(L->k0 + tid, g.pA, g.pB);
        const LocalView xv{L, 0, g.pA, g.n, g.m, nullptr};
        const LocalView yv{L, 1, g.pB, g.m, g.n, nullptr};
        const Task t = t0 < g.pA ? classify_a_side(t0, xa, yb, xv, yv) : classify_b_side(t0 - g.pA, xa, yb, xv, yv);
        // clamped as in the producer (unsorted inputs, a precondition violation)
        const int la = max(0, min(t.a1 - t.a0, NV));
        const int lb = max(0, min(t.b1 - t.b0, NV - la));
        L->desc[tid] = make_int4(t.a0, t.b0, t.a0 + t.b0, (la << 16) | lb);
    }
    __syncthreads();
}

// ----------------------------------------------------------------- K2
// SM_K2_TSTAMP builds (experiments, scripts/k2_timeline.py): K2 records
// per-CTA event times (%globaltimer, ns) in g.ts[8 * CTA + slot]: 0 entry,
// 1 first stage issued, 2 producer done, 3 storer done.
#ifdef SM_K2_TSTAMP
#define K2_TS(slot)                                                                    \
    do {                                                                               \
        if (g.ts) {                                                                    \
            unsigned long long t_;                                                     \
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                   \
            g.ts[8 * blockIdx.x + (slot)] = t_;                                        \
        }                                                                              \
    } while (0)
#else
#define K2_TS(slot) do {} while (0)
#endif
// A ring stage holds the input ranges of up to MAXT tasks ("packing"): the
// paper's subproblems range from O(1) to ~2T elements (L388-393), so one task
// per tile would leave half the consumer threads idle on average.  The
// producer packs consecutive tasks of this CTA while their sizes, each
// rounded up to VT, sum to at most NV = NC * VT; consumer thread c then owns
// padded diagonal c * VT of the stage and finds its task by binary search.
struct TaskDesc {
    int la, lb;        // lengths of the A and B ranges
    int a_s, b_s;      // stage key index of A[a0] / B[b0]
    int va_s, vb_s;    // stage payload index of vA[a0] / vB[b0]
    int ob, obv;       // (in-place store) stage index of output key / payload 0 of the task
    int off;           // global output element index (segment base + a0 + b0)
    int pst;           // first padded diagonal of the task in the stage
};

// Outputs are written back in place into the stage (phase-aligned to the
// destination) and a storer warp bulk-stores them; the stage is held until
// its bulk reads complete.  (A variant with per-warp output buffers, freeing
// the stage as soon as it was read, measured 2-4% slower on C2: fewer stages
// fit in shared memory.)
template <typename K, bool HAS_V, int NC, int VT, int STAGES, int MAXT, typename PV = uint32_t>
struct K2Layout {
    static constexpr int NV = NC * VT;                     // padded diagonals per stage
    static constexpr int KB = (int)sizeof(K);
    static constexpr int EPV = 16 / KB;                    // keys per 16 bytes
    // Task k's key region: its A span and B span (16-byte aligned supersets,
    // <= L*KB + 2*30 bytes) plus 16 bytes: room for the in-place output
    // phase-aligned to the destination, and for the merge's look-ahead reads
    // past the end of a range.
    static constexpr int KREG = NV * KB + MAXT * 80;
    static constexpr int VREG = HAS_V ? NV * (int)sizeof(PV) + MAXT * 80 : 0;   // payloads (PV: 4 or 8 bytes)
    static constexpr int STAGE_BYTES = KREG + VREG;
    static constexpr int OFF_DESC = STAGES * STAGE_BYTES;
    static constexpr int OFF_PST = OFF_DESC + STAGES * MAXT * (int)sizeof(TaskDesc);
    static constexpr int OFF_BAR = ((OFF_PST + STAGES * (MAXT + 2) * 4) + 15) & ~15;
    static constexpr int OFF_LOC = (OFF_BAR + 3 * STAGES * 8 + 15) & ~15;   // full, empty, written; then
    static constexpr int SMEM = OFF_LOC + (int)sizeof(K2Local);              //   the small-merge ranks (g.fuse)
    static constexpr int THREADS = NC + 64;                 // producer + storer + consumers
};

#ifndef SM_BULK_CHUNK
#define SM_BULK_CHUNK 0       // > 0: bulk loads cut into chunks of this many bytes (experiment)
#endif
#ifndef SM_BULK_CHUNK_ST
#define SM_BULK_CHUNK_ST 0    // > 0: bulk stores cut likewise
#endif
// Bytes of the 16-byte-aligned superset of p[0, len).
template <typename T>
__device__ __forceinline__ int span_bytes(const T* p, int len) {
    if (len <= 0) return 0;
    const uintptr_t g = (uintptr_t)p;
    return (int)(((g + (uintptr_t)len * sizeof(T) + 15) & ~(uintptr_t)15) - (g & ~(uintptr_t)15));
}

// Bulk-load the aligned superset of p[0, len) to smem byte `at` of `base`;
// returns the stage element index of p[0].
template <typename T>
__device__ __forceinline__ int issue_span(char* base, int at, const T* p, int len, uint64_t* bar) {
    const uintptr_t g = (uintptr_t)p;
    const uintptr_t g0 = g & ~(uintptr_t)15;
#if SM_BULK_CHUNK > 0
    // experiment: cut each span into bulk copies of <= SM_BULK_CHUNK bytes
    const int nb = len > 0 ? span_bytes(p, len) : 0;
    for (int o = 0; o < nb; o += SM_BULK_CHUNK)
        bulk_g2s(base + at + o, (const void*)(g0 + o), (uint32_t)min(SM_BULK_CHUNK, nb - o), bar);
#else
    if (len > 0) bulk_g2s(base + at, (const void*)g0, (uint32_t)span_bytes(p, len), bar);
#endif
    return (at + (int)(g - g0)) / (int)sizeof(T);
}

template <typename T>
__device__ __forceinline__ int phase_of(const T* p) {
    return (int)(((uintptr_t)p & 15) / sizeof(T));
}

// Store smem elements sbuf[o, o+L) to dst[0, L): the 16-byte-aligned middle
// with one bulk copy (issued by the calling thread).
template <typename T>
__device__ __forceinline__ void store_middle(T* dst, const T* sbuf, int o, int L) {
    const uintptr_t g = (uintptr_t)dst;
    const uintptr_t gl = (g + 15) & ~(uintptr_t)15;
    const uintptr_t gh = (g + (uintptr_t)L * sizeof(T)) & ~(uintptr_t)15;
    SM_DCHECK(gh <= gl || (gl >= g && gh <= g + (uintptr_t)L * sizeof(T)), "K2 bulk store outside its task range");
#if SM_BULK_CHUNK_ST > 0
    for (uintptr_t c = gl; c < gh; c += SM_BULK_CHUNK_ST)
        bulk_s2g((void*)c, (const char*)(sbuf + o + (int)((gl - g) / sizeof(T))) + (c - gl),
                 (uint32_t)min((uintptr_t)SM_BULK_CHUNK_ST, gh - c));
#else
    if (gh > gl) bulk_s2g((void*)gl, sbuf + o + (int)((gl - g) / sizeof(T)), (uint32_t)(gh - gl));
#endif
}

// Edge element r (0 <= r < 2*(16/sizeof(T)-1)) of the store above: the
// elements before the first and after the last 16-byte boundary.
template <typename T>
__device__ __forceinline__ void store_edge(T* dst, const T* sbuf, int o, int L, int r) {
    const uintptr_t g = (uintptr_t)dst;
    const uintptr_t gl = (g + 15) & ~(uintptr_t)15;
    const uintptr_t gh = (g + (uintptr_t)L * sizeof(T)) & ~(uintptr_t)15;
    int head = (int)((gl - g) / sizeof(T));
    if (head > L) head = L;
    const int tail0 = gh > gl ? (int)((gh - g) / sizeof(T)) : head;
    const int e = r < head ? r : tail0 + (r - head);
    if (e < L && (r < head || e >= tail0)) {
        SM_DCHECK(e >= 0 && e < L, "K2 edge store outside its task range");
        dst[e] = sbuf[o + e];
    }
}

// ---- producer (warp 0): classify, pack, bulk-load (rows a4/a5) ----------
// Its lanes classify a window of up to 32 tasks of this CTA in parallel
// (O(1) each, L310-340); a prefix of the window whose padded sizes fit NV
// goes into the next ring stage; every packed task's lane issues the TMA bulk
// loads of its A and B ranges (keys, payloads).  A stage with task count -1
// terminates the consumers.
// Tasks are handed out dynamically: the producer takes chunks of consecutive
// positions of K2's order from the launch's task counter, so the CTAs
// advance as one front and finish together -- a static round-robin left the
// CTAs' finishing times 50 us apart on C2 (per-CTA timelines,
// scripts/k2_timeline.py).  Each refill uses the chunk reserved at the
// previous one and reserves the next (one atomicAdd, whose latency overlaps
// the stages in between).  The window is refilled (classified in parallel,
// one task per lane) whenever fewer than `refill` tasks are left: after every
// stage for plain merges of wide elements (mode 0, > 8 bytes), else when it
// runs low (8); chunks shrink to half a fair share of what is left
// (remaining / (2 x grid)) and, near the end, windows to ~4 tasks, so no CTA
// is left holding a long queue.
template <typename K, bool HAS_V, int VT, int STAGES, int MAXT, bool FIRSTFIT, typename Lay, typename PV>
__device__ __forceinline__ void k2_producer(const K* __restrict__ A, const PV* __restrict__ vA,
                                            const K* __restrict__ B, const PV* __restrict__ vB,
                                            const K* C, const PV* vC, const Geom& g,
                                            const int* xbar, const int* ybar, char* smem,
                                            TaskDesc* desc, int* pst, uint64_t* full, uint64_t* empty) {
    constexpr int NV = Lay::NV;
    constexpr int KB = Lay::KB;
    constexpr int EPV = Lay::EPV;
    const int ntasks = total_tasks(g);
    const int lane = threadIdx.x;
    const int G = (int)gridDim.x;
    int la = 0, lb = 0, off = 0, ag = 0, bg = 0;   // window slot `lane`
    int cnt = 0;                                    // slots [0, cnt) hold tasks
    int seen = 0;                                   // end of this CTA's last reservation (progress estimate)
    bool more = ntasks > 0;
    // few tasks per CTA (C1): static round-robin -- one refill takes them all
    int* const ctr = (SM_K2_DYN && !g.fuse && ntasks > SM_K2_DYN_MIN * G) ? g.ctr : nullptr;
    const int refill =
        g.tdesc ? SM_REFILL_TDESC : (g.sort == 0 && KB + (HAS_V ? (int)sizeof(PV) : 0) > 8) ? 32 : 8;
    constexpr int CH = KB + (HAS_V ? (int)sizeof(PV) : 0) > 8 ? SM_K2_CHUNK_WIDE : SM_K2_CHUNK;
    int resv = 0, resv_n = 0;                       // (lane 0) positions reserved for the next refill
    int next = blockIdx.x;                          // (no counter: static round-robin, CTA b takes b, b+G, ...)
    const K2Local* loc = (const K2Local*)(smem + Lay::OFF_LOC);
    if (g.fuse) {                                   // small merge: this CTA's positions, classified (prologue)
        next = loc->k0;
        more = loc->k0 < loc->k1;
    }
    for (int it = 0;; ++it) {
        // dynamic: refill while the window has room for a chunk; near the end
        // (fewer than SM_K2_TAILWIN tasks per CTA left) keep the window short
        const bool dyn = ctr != nullptr;
        const int thr = dyn ? min(min(refill, 33 - CH), max(SM_K2_TAILWIN, (ntasks - seen) / G)) : refill;
        if (cnt < thr && more) {
            int base, stride, take = 32;
            if (dyn) {
                if (resv_n == 0) {                  // first refill: reserve now
                    resv_n = max(1, min(CH, ntasks / (2 * G)));
                    if (lane == 0) resv = atomicAdd(ctr, resv_n);
                }
                base = __shfl_sync(0xffffffffu, resv, 0);   // (waits for the reservation)
                take = resv_n;
                seen = base + take;
                more = seen < ntasks;
                if (more) {
                    // reserve the next chunk now: the atomic's latency overlaps
                    // the stages until the next refill.  Chunks shrink to half
                    // a fair share of what is left, down to single tasks.
                    resv_n = max(1, min(CH, (ntasks - seen) / (2 * G)));
                    if (lane == 0) resv = atomicAdd(ctr, resv_n);
                }
                stride = 1;
                base -= cnt;                        // lane l in [cnt, cnt + take) takes position base + l
            } else if (g.fuse) {
                base = next;
                stride = 1;
                take = loc->k1 - loc->k0;                   // <= K2L_MAXP: one refill
                more = false;
            } else {
                base = next;
                stride = G;
                next += (32 - cnt) * G;
                more = next < ntasks;
            }
            const int my = base + (lane - (dyn ? 0 : cnt)) * stride;
            const bool fill = lane >= cnt && lane < cnt + take && my < ntasks;
            if (fill) {
                if (g.tdesc || g.fuse) {            // classified ahead (k_classify / the prologue): one load
                    const int4 q = g.fuse ? loc->desc[my - loc->k0] : __ldg(g.tdesc + my);
                    ag = q.x;
                    bg = q.y;
                    off = q.z;
                    la = q.w >> 16;
                    lb = q.w & 0xFFFF;
                } else {
                    Seg sg;
                    const Task t = decode_task(g, g.sort == 0 ? task_at(my, g.pA, g.pB) : my, xbar, ybar, sg);
                    // sorted inputs give 0 <= la + lb <= NV (the task bound of
                    // L388-393); unsorted ones (a precondition violation) may
                    // not: clamp so the kernel still terminates in its buffers
                    la = max(0, min(t.a1 - t.a0, NV));
                    lb = max(0, min(t.b1 - t.b0, NV - la));
                    off = sg.coff + t.a0 + t.b0;
                    ag = sg.aoff + t.a0;
                    bg = sg.boff + t.b0;
                }
            }
            cnt += __popc(__ballot_sync(0xffffffffu, fill));
        }
        const int st = it % STAGES;
        if (it >= STAGES) mbar_wait_sleep(&empty[st], ((it / STAGES) - 1) & 1);
        int* ps = pst + st * (MAXT + 2);
        if (cnt == 0) {                             // no task left: terminate the consumers
            if (lane == 0) {
                ps[MAXT + 1] = -1;
                mbar_arrive(&full[st]);
                K2_TS(2);
            }
            return;
        }
        // pack the window: the longest prefix that fits, or (FIRSTFIT)
        // first-fit in lane order -- the paper's tasks range from 0 to 2T
        // elements (L388-393), so after the first task that does not fit,
        // later (smaller) ones may still fill the stage; a skipped task leads
        // the next stage's window, so none starves.  Measured: first-fit
        // +2% on 4-byte keys-only merges, -1..3% on wider elements.
        const int L = la + lb;
        const int P = ((L + VT - 1) / VT) * VT;
        unsigned taken = 0u;
        if constexpr (FIRSTFIT) {
            int used = 0;
            for (int k = 0; k < MAXT; ++k) {
                const unsigned cand =
                    __ballot_sync(0xffffffffu, lane < cnt && !((taken >> lane) & 1u) && P <= NV - used);
                if (!cand) break;
                const int l = __ffs(cand) - 1;
                taken |= 1u << l;
                used += __shfl_sync(0xffffffffu, P, l);
            }
        } else {
            int pre = lane < cnt ? P : NV + 1;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int t = __shfl_up_sync(0xffffffffu, pre, o);
                if (lane >= o) pre += t;
            }
            taken = __ballot_sync(0xffffffffu, lane < cnt && lane < MAXT && pre <= NV);
        }
        const bool take_me = (taken >> lane) & 1u;
        const int take = __popc(taken);
        const int slot = __popc(taken & ((1u << lane) - 1u));   // position among the packed tasks
        // stage offsets of each packed task: padded diagonals, key / payload regions
        const int pme = take_me ? P : 0;
        const int kreg = take_me ? span_bytes(A + ag, la) + span_bytes(B + bg, lb) + 16 : 0;
        const int vreg = (HAS_V && take_me) ? span_bytes(vA + ag, la) + span_bytes(vB + bg, lb) + 16 : 0;
        int incl = pme, kat = kreg, vat = vreg;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int t0 = __shfl_up_sync(0xffffffffu, incl, o);
            const int t1 = __shfl_up_sync(0xffffffffu, kat, o);
            const int t2 = __shfl_up_sync(0xffffffffu, vat, o);
            if (lane >= o) { incl += t0; kat += t1; vat += t2; }
        }
        kat -= kreg;                                 // exclusive
        vat -= vreg;
        const int last = 31 - __clz(taken);
        const int ktot = __shfl_sync(0xffffffffu, kat + kreg, last);
        const int vtot = __shfl_sync(0xffffffffu, vat + vreg, last);
        char* stage = smem + st * Lay::STAGE_BYTES;
        char* vstage = stage + Lay::KREG;
        if (take_me) {
            TaskDesc d;
            d.la = la;
            d.lb = lb;
            d.off = off;
            d.pst = incl - pme;
            d.a_s = issue_span(stage, kat, A + ag, la, &full[st]);
            d.b_s = issue_span(stage, kat + span_bytes(A + ag, la), B + bg, lb, &full[st]);
            // in-place output position: where a copy's source already has the
            // destination's 16-byte phase, else phase-aligned at the region start
            const int phC = phase_of(C + off);
            if (lb == 0 && (d.a_s & (EPV - 1)) == phC) d.ob = d.a_s;
            else if (la == 0 && (d.b_s & (EPV - 1)) == phC) d.ob = d.b_s;
            else d.ob = kat / KB + phC;
            d.va_s = d.vb_s = d.obv = 0;
            if (HAS_V) {
                d.va_s = issue_span(vstage, vat, vA + ag, la, &full[st]);
                d.vb_s = issue_span(vstage, vat + span_bytes(vA + ag, la), vB + bg, lb, &full[st]);
                const int phV = phase_of(vC + off);
                constexpr int VM = 16 / (int)sizeof(PV) - 1;   // payload phase mask
                if (lb == 0 && (d.va_s & VM) == phV) d.obv = d.va_s;
                else if (la == 0 && (d.vb_s & VM) == phV) d.obv = d.vb_s;
                else d.obv = vat / (int)sizeof(PV) + phV;
            }
            desc[st * MAXT + slot] = d;
            if (lane == last) {
                ps[take] = incl;
                ps[MAXT + 1] = take;
            }
            ps[slot] = incl - pme;
        }
        // the descriptors are released by the arrive; the bulk loads may
        // complete_tx before the expect_tx (the phase needs both)
        __syncwarp();
        if (lane == 0) {
            mbar_arrive_expect_tx(&full[st], (uint32_t)(ktot - 16 * take + (HAS_V ? vtot - 16 * take : 0)));
            if (it == 0) K2_TS(1);
        }
        // drop the packed tasks from the window, keeping the order of the rest
        int sl = lane + take;                            // prefix packed: shift down
        if constexpr (FIRSTFIT) {
            const unsigned keep = ~taken & (cnt >= 32 ? 0xffffffffu : ((1u << cnt) - 1u));
            const unsigned src = __fns(keep, 0, lane + 1);   // (lane+1)-th kept lane, or ~0u
            sl = src < 32u ? (int)src : lane;
        } else if (sl > 31) {
            sl = lane;
        }
        la = __shfl_sync(0xffffffffu, la, sl);
        lb = __shfl_sync(0xffffffffu, lb, sl);
        off = __shfl_sync(0xffffffffu, off, sl);
        ag = __shfl_sync(0xffffffffu, ag, sl);
        bg = __shfl_sync(0xffffffffu, bg, sl);
        cnt -= take;
    }
}

// ---- k_classify: Steps 3-4 of every task ahead of K2 (modes 1, 2) --------
// The segmented classifications take three dependent loads (segment table,
// then ranks); done here once per task, in parallel, so K2's producer reads
// one 16-byte descriptor per task: (A start, B start, C start, la<<16 | lb),
// global element indices, lengths clamped as in the producer.
template <int NV>
__global__ void __launch_bounds__(256) k_classify(Geom g, const int* __restrict__ xbar, const int* __restrict__ ybar,
                                                  int4* __restrict__ tdesc) {
    pdl_wait();
    zero_task_counter(g.ctr);
    const int task = blockIdx.x * blockDim.x + threadIdx.x;
    if (task < total_tasks(g)) {
        Seg sg;
        const Task t = decode_task(g, task, xbar, ybar, sg);
        const int la = max(0, min(t.a1 - t.a0, NV));
        const int lb = max(0, min(t.b1 - t.b0, NV - la));
        int lt;
        locate(g, task, false, lt);                  // its place in K2's order within the segment
        const int at = task - lt + (sg.pA > 0 ? task_pos(lt, sg.pA, sg.pB) : lt);
        tdesc[at] = make_int4(sg.aoff + t.a0, sg.boff + t.b0, sg.coff + t.a0 + t.b0, (la << 16) | lb);
    }
    pdl_launch_dependents();
}

// ---- consumer compute (rows a6/a7) ----------------------------------------
// Thread with padded diagonal D of stage s: its task (binary search over the
// packed tasks' first diagonals), its diagonal d inside the task, and its
// cnt <= VT outputs in registers.  Returns false when D lies in no task.
//   copy = the task is a copy (cases a, e) and out/v were not filled because
//          the in-place store needs no movement (INPLACE only).
template <typename K, bool HAS_V, int VT, int MAXT, int LOG2NV, bool INPLACE, typename PV>
__device__ __forceinline__ bool k2_compute(const K* sk, const PV* sv, const TaskDesc* desc_s, const int* ps,
                                           int nt, int D, TaskDesc& td, int& d, int& cnt, bool& write, K (&out)[VT],
                                           PV (&v)[HAS_V ? VT : 1]) {
    constexpr int KB = (int)sizeof(K);
    write = false;
    cnt = 0;
    if (D >= ps[nt]) return false;
    int lo = 0, hi = nt - 1;                       // task k: last with pst[k] <= D
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (ps[mid] <= D) lo = mid;
        else hi = mid - 1;
    }
    td = desc_s[lo];
    d = D - td.pst;
    cnt = min(VT, td.la + td.lb - d);
    if (cnt <= 0) return true;
#ifdef SM_K2_NOCOMPUTE
    // experiment only (wrong output): the same data movement without the merge
    if (td.la > 0 && td.lb > 0) return true;
#endif
    if (td.la > 0 && td.lb > 0) {
        // cases (b), (c), (d): stable merge (row a7), ties to A (R17)
        if constexpr (!KeyOrd<K>::PTX && !KeyOrd<K>::FLOAT) {
            // 128-bit keys: the same merge on the order view (C++ path)
            using U = typename KeyOrd<K>::U;
            const K* a = sk + td.a_s;
            const K* b = sk + td.b_s;
            int lo = max(0, d - td.lb), hi = min(d, td.la);
            while (lo < hi) {
                const int mid = (lo + hi) >> 1;
                if (KeyOrd<K>::to(a[mid]) <= KeyOrd<K>::to(b[d - 1 - mid])) lo = mid + 1;
                else hi = mid;
            }
            int ai = lo, bi = d - lo;
            U ka = KeyOrd<K>::to(a[min(ai, td.la - 1)]), kb = KeyOrd<K>::to(b[min(bi, td.lb - 1)]);
#pragma unroll
            for (int k = 0; k < VT; ++k) {
                const bool t = bi >= td.lb || (ai < td.la && ka <= kb);
                out[k] = t ? a[min(ai, td.la - 1)] : b[min(bi, td.lb - 1)];
                if (HAS_V) v[k] = t ? sv[td.va_s + min(ai, td.la - 1)] : sv[td.vb_s + min(bi, td.lb - 1)];
                if (t) {
                    ++ai;
                    ka = KeyOrd<K>::to(a[min(ai, td.la - 1)]);
                } else {
                    ++bi;
                    kb = KeyOrd<K>::to(b[min(bi, td.lb - 1)]);
                }
            }
        } else {
            // PTX path: integer keys as they are, floating-point keys as
            // their totalOrder integer view (V), mapped back at the end
            using V = typename FViewOf<K>::type;
            const uint32_t sa0 = smem_addr(sk + td.a_s);
            const uint32_t sb0 = smem_addr(sk + td.b_s);
            const int ai = split_smem<V, LOG2NV>(sa0, td.la, sb0, td.lb, d);
            const int bi = d - ai;
            uint32_t pa = sa0 + ai * KB, pb = sb0 + bi * KB;
            const uint32_t pae = sa0 + td.la * KB, pbe = sb0 + td.lb * KB;
            V ka = lds<V>(pa), kb = lds<V>(pb), na = lds<V>(pa + KB), nb = lds<V>(pb + KB);
            V ov[VT];
            int src[VT];
            int ia = td.va_s + ai, ib = td.vb_s + bi;
            // warp-uniform choice: no exhaustion checks when no lane can run
            // out of A or B within its VT outputs (all but the last warps of
            // a task)
            if (__all_sync(__activemask(), ai + VT <= td.la && bi + VT <= td.lb)) {
#pragma unroll
                for (int k = 0; k < VT; ++k) {
                    if (HAS_V) merge_step_idx_fast<V>(pa, pb, ka, kb, na, nb, ov[k], ia, ib, src[k]);
                    else merge_step_fast<V>(pa, pb, ka, kb, na, nb, ov[k]);
                }
            } else {
#pragma unroll
                for (int k = 0; k < VT; ++k) {
                    if (HAS_V) merge_step_idx<V>(pa, pb, ka, kb, na, nb, pae, pbe, ov[k], ia, ib, src[k]);
                    else merge_step<V>(pa, pb, ka, kb, na, nb, pae, pbe, ov[k]);
                }
            }
#pragma unroll
            for (int k = 0; k < VT; ++k) out[k] = from_reg<K>(ov[k]);
            if (HAS_V) {
#pragma unroll
                for (int k = 0; k < VT; ++k)
                    if (k < cnt) v[k] = sv[src[k]];
            }
        }
        write = true;
    } else {
        // cases (a), (e): copy (row a6); in place: no movement when the source
        // already has the destination's phase
        const int ks = td.la ? td.a_s : td.b_s;
        const int vs = td.la ? td.va_s : td.vb_s;
        if (!INPLACE || ks != td.ob || (HAS_V && vs != td.obv)) {
#pragma unroll
            for (int k = 0; k < VT; ++k) {
                if (k < cnt) {
                    out[k] = sk[ks + d + k];
                    if (HAS_V) v[k] = sv[vs + d + k];
                }
            }
            write = true;
        }
    }
    return true;
}

// K2 (rows a4-a7): persistent, warp-specialised.
//   warp 0 (producer): k2_producer above (full[s]).
//   warps 2.. (NC consumers): k2_compute, then write back in place,
//     phase-aligned to the destination, and hand the stage to the storer
//     (written[s]).
//   warp 1 (storer): bulk-stores each task's 16-byte-aligned middle,
//     plain-stores the edge elements, and frees the stage once the bulk reads
//     complete (empty[s]), so the consumers never wait on the stores.
template <typename K, bool HAS_V, int NC, int VT, int STAGES, int MAXT, int MINB, typename PV = uint32_t>
__global__ void __launch_bounds__(K2Layout<K, HAS_V, NC, VT, STAGES, MAXT, PV>::THREADS, MINB)
    k_tasks(const K* __restrict__ A, const PV* __restrict__ vA, const K* __restrict__ B,
            const PV* __restrict__ vB, K* __restrict__ C, PV* __restrict__ vC, Geom g,
            const int* xbar, const int* ybar) {
    using Lay = K2Layout<K, HAS_V, NC, VT, STAGES, MAXT, PV>;
    static_assert(NC % 32 == 0 && MAXT <= 32 && STAGES >= 2, "warp-granular roles; one producer lane per task");
    constexpr int NV = Lay::NV;
    constexpr int LOG2NV = 31 - __builtin_clz(NV);   // 2^(LOG2NV+1) - 1 >= NV probes cover any range
    constexpr int EPV = Lay::EPV;
    constexpr int EK = 2 * (EPV - 1);                // key edge elements per store
    constexpr int EV = HAS_V ? 2 * (16 / (int)sizeof(PV) - 1) : 0;   // payload edge elements per store
    extern __shared__ __align__(128) char smem[];
    TaskDesc* desc = (TaskDesc*)(smem + Lay::OFF_DESC);
    int* pst = (int*)(smem + Lay::OFF_PST);          // [STAGES][MAXT + 2]: pst[0..nt], nt at MAXT+1
    uint64_t* full = (uint64_t*)(smem + Lay::OFF_BAR);
    uint64_t* empty = full + STAGES;
    uint64_t* written = empty + STAGES;

    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
            mbar_init(&written[s], NC / 32);
        }
        fence_barrier_init();
        fence_proxy_async();
    }
    __syncthreads();
    pdl_wait();   // the single synchronisation (L373-375): all ranks visible
    if (threadIdx.x == 0) K2_TS(0);

    if (g.fuse) {                                    // small plain merge
#if SM_SMALL_PREFETCH
        // each task's own block (its A range starts at x_i, a B-side task's
        // B range at y_j) to L2 while the ranks are searched
        const int ntasks = g.pA + g.pB, P = (ntasks + (int)gridDim.x - 1) / (int)gridDim.x;
        const int k = (int)blockIdx.x * P + (int)threadIdx.x;
        if ((int)threadIdx.x < P && k < ntasks) {
            const int t = task_at(k, g.pA, g.pB);
            const bool sa = t < g.pA;
            const Blocks bl = sa ? Blocks(g.n, g.pA) : Blocks(g.m, g.pB);
            const int i = sa ? t : t - g.pA;
            const int s0 = min(bl.start(i), bl.len), s1 = i + 1 < bl.p ? bl.start(i + 1) : bl.len;
            prefetch_l2((sa ? A : B) + s0, s1 - s0);
            if (HAS_V) prefetch_l2((sa ? vA : vB) + s0, s1 - s0);
        }
#endif
        k2_local_prologue<K, NV>(A, B, g, (K2Local*)(smem + Lay::OFF_LOC));
    }
    if (threadIdx.x < 32) {
        k2_producer<K, HAS_V, VT, STAGES, MAXT, (sizeof(K) == 4 && !HAS_V), Lay, PV>(A, vA, B, vB, C, vC, g, xbar, ybar,
                                                                               smem, desc, pst, full, empty);
        return;
    }

    if (threadIdx.x < 64) {
        // -------------------------------------------------------- storer
        const int lane = threadIdx.x - 32;
        for (int it = 0;; ++it) {
            const int s = it % STAGES;
            mbar_wait_sleep(&written[s], (it / STAGES) & 1);
            const int nt = pst[s * (MAXT + 2) + MAXT + 1];
            if (nt < 0) {
#ifdef SM_K2_TSTAMP
                bulk_wait_all();
                if (lane == 0) K2_TS(3);
#endif
                break;
            }
            const K* sk = (const K*)(smem + s * Lay::STAGE_BYTES);
            const PV* sv = (const PV*)(smem + s * Lay::STAGE_BYTES + Lay::KREG);
#ifdef SM_DEBUG
            {   // every task's output range inside C; every element counted once
                const long long lim = g.sort == 1 ? g.N : (g.sort == 2 ? -1 : (long long)g.n + g.m);
                for (int k = 0; k < nt; ++k) {
                    const TaskDesc& t = desc[s * MAXT + k];
                    const int L = t.la + t.lb;
                    SM_DCHECK(t.off >= 0 && L >= 0 && (lim < 0 || (long long)t.off + L <= lim),
                              "K2 task range outside C");
                    if (g.cover)
                        for (int e = lane; e < L; e += 32) atomicAdd(&g.cover[t.off + e], 1u);
                }
            }
#endif
            if (lane < nt) {
                const TaskDesc& t = desc[s * MAXT + lane];
                const int L = t.la + t.lb;
                if (L > 0) {
                    store_middle<K>(C + t.off, sk, t.ob, L);
                    if (HAS_V) store_middle<PV>(vC + t.off, sv, t.obv, L);
                }
                bulk_commit();
            }
            if constexpr (EK + EV > 0) {                 // (16-byte keys alone have no edges)
                for (int e = lane; e < nt * (EK + EV); e += 32) {
                    const int k = e / (EK + EV), r = e % (EK + EV);
                    const TaskDesc& t = desc[s * MAXT + k];
                    const int L = t.la + t.lb;
                    if (r < EK) store_edge<K>(C + t.off, sk, t.ob, L, r);
                    else if (HAS_V) store_edge<PV>(vC + t.off, sv, t.obv, L, r - EK);
                }
            }
            bulk_wait_read<0>();                       // this lane's bulk stores have read the stage
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[s]);
        }
        return;
    }

    // ---------------------------------------------------------- consumers
    const int c = threadIdx.x - 64;
    const int lane = threadIdx.x & 31;
    for (int it = 0;; ++it) {
        const int s = it % STAGES;
        mbar_wait(&full[s], (it / STAGES) & 1);
        const int* ps = pst + s * (MAXT + 2);
        const int nt = ps[MAXT + 1];
        if (nt < 0) {
            if (lane == 0) mbar_arrive(&written[s]);   // pass the termination on to the storer
            break;
        }
        K* sk = (K*)(smem + s * Lay::STAGE_BYTES);
        PV* sv = (PV*)(smem + s * Lay::STAGE_BYTES + Lay::KREG);
        TaskDesc td;
        int d = 0, cnt = 0;
        bool write = false;
        K out[VT];
        PV v[HAS_V ? VT : 1];
        k2_compute<K, HAS_V, VT, MAXT, LOG2NV, true, PV>(sk, sv, desc + s * MAXT, ps, nt, c * VT, td, d, cnt, write, out,
                                                    v);
        named_sync(1, NC);                             // every input of the stage has been read
        if (write) {
#pragma unroll
            for (int k = 0; k < VT; ++k) {
                if (k < cnt) {
                    sk[td.ob + d + k] = out[k];
                    if (HAS_V) sv[td.obv + d + k] = v[k];
                }
            }
        }
        fence_proxy_async();                           // generic writes -> the storer's bulk reads
        __syncwarp();
        if (lane == 0) mbar_arrive(&written[s]);
    }
}

// ------------------------------------------------------- wide payloads
// SURVEY.md §8(f) row 2 (wide and struct payloads): the merge / sort runs
// with a uint32 INDEX payload (each element's position in A||B, or in the
// sort input), then k_gather_rows moves payload row idx[k] to output row k
// in W-byte words (consecutive outputs mostly come from consecutive rows of
// one input, so both sides stay coalesced).
__global__ void __launch_bounds__(256) k_iota(uint32_t* __restrict__ out, int64_t count) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = (uint32_t)i;
}

template <typename W>
__global__ void __launch_bounds__(256) k_gather_rows(const uint32_t* __restrict__ idx, const W* __restrict__ PA,
                                                     int64_t n, const W* __restrict__ PB, W* __restrict__ out,
                                                     int64_t rows, int wpr) {
    const uint64_t total = (uint64_t)rows * (uint64_t)wpr;
    const bool small = total < (1ull << 32);
    for (uint64_t w = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; w < total;
         w += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t r = small ? (uint64_t)((uint32_t)w / (uint32_t)wpr) : w / (uint64_t)wpr;
        const int c = (int)(w - r * (uint64_t)wpr);
        const int64_t src = (int64_t)__ldg(idx + r);
        const W* row = src < n ? PA + src * wpr : PB + (src - n) * wpr;
        st_stream(out + w, __ldg(row + c));
    }
}

// ------------------------------------------------ coarse partition (>= 2^31)
// The keys at the block starts of the paper's partition of X[0, len) into p
// blocks, 64-bit indices; empty blocks are skipped.
template <typename K>
__global__ void __launch_bounds__(256) k_block_start_keys(const K* __restrict__ X, int64_t len, int64_t p,
                                                          K* __restrict__ out) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= p) return;
    const int64_t q = len / p, r = len % p;
    const int64_t xi = i < r ? i * (q + 1) : i * q + r;
    if (xi < len) out[i] = ldg_key(X + xi);
}

// ------------------------------------------------------- rank queries
// rank_low (high = 0) or rank_high (high = 1) of a batch of keys in one
// sorted array: the primitive of rows a1/a2 on its own,
// used by the sharded multi-GPU merge (each rank ranks every block-start key
// in its local shard; the sums over ranks are the global cross ranks).
template <typename K>
__global__ void __launch_bounds__(256) k_rank_keys(const K* __restrict__ X, int64_t len, const K* __restrict__ keys,
                                                   int64_t nkeys, int high, int64_t* __restrict__ out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nkeys) return;
    const K x = keys[i];
    int64_t lo = 0, hi = len;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        const K v = ldg_key(X + mid);
        if (high ? key_le(v, x) : key_lt(v, x)) lo = mid + 1;
        else hi = mid;
    }
    out[i] = lo;
}

// ------------------------------------------------ merge-path comparison
// SURVEY.md §8(f) row 4, an A/B comparison only (the equal-output
// partitioning of [AklSantoro87], the class the paper contrasts itself with,
// P:L49-59): split C into tiles of exactly T outputs; the split of diagonal
// D is the smallest i in [max(0, D-m), min(D, n)] with A[i] > B[D-1-i]
// (ties to A, reading R17), one binary search per diagonal over global
// memory.  Same output bytes as the method; no factor-two imbalance.
template <typename K>
__global__ void __launch_bounds__(256) k_diag_splits(const K* __restrict__ A, const K* __restrict__ B, int n, int m,
                                                     int T, int* __restrict__ split, int* ctr) {
    zero_task_counter(ctr);
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    const int tiles = (n + m + T - 1) / T;
    if (k <= tiles) {
        const int D = min(n + m, k * T);
        int lo = max(0, D - m), hi = min(D, n);
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (key_le(ldg_key(A + mid), ldg_key(B + (D - 1 - mid)))) lo = mid + 1;
            else hi = mid;
        }
        split[k] = lo;
    }
    pdl_launch_dependents();
}

// ------------------------------------------------------- batch setup
// Batched merges (mode 2): segment s merges A[a_off[s], a_off[s+1]) with
// B[b_off[s], b_off[s+1]) into C[a_off[s] + b_off[s], ...).  Offsets are
// clamped into [0, n] / [0, m] and made non-decreasing per segment, so a
// malformed table can give a wrong result but never a write outside C.
// Block counts per segment: p_A = max(1, ceil(n_s / T)) (same for B), the
// single-merge rule (reading R7).  Three passes: per-block counts and local
// exclusive scans (tasks p_A + p_B, rank entries p_A + p_B + 2), a scan of the
// block sums, and the block offsets added.
constexpr int BATCH_NT = 256;

__global__ void __launch_bounds__(BATCH_NT) k_batch_count(const int64_t* __restrict__ a_off,
                                                          const int64_t* __restrict__ b_off, int S, int64_t n,
                                                          int64_t m, int T, int NV, SegInfo* __restrict__ segs,
                                                          int2* __restrict__ blk) {
    __shared__ int2 wsum[BATCH_NT / 32];
    const int s = blockIdx.x * BATCH_NT + threadIdx.x;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    int tasks = 0, ranks = 0;
    SegInfo e;
    if (s < S) {
        const int64_t a0 = min(max(a_off[s], (int64_t)0), n), a1 = min(max(a_off[s + 1], a0), n);
        const int64_t b0 = min(max(b_off[s], (int64_t)0), m), b1 = min(max(b_off[s + 1], b0), m);
        e.aoff = (int)a0; e.n = (int)(a1 - a0); e.boff = (int)b0; e.m = (int)(b1 - b0); e.coff = (int)(a0 + b0);
        if (e.n + e.m <= NV) {
            // the whole segment fits one tile: one task, no cross ranks (the
            // two tasks of p_A = p_B = 1 concatenated: reading R19)
            e.pA = e.pB = 0;
            tasks = 1;
            ranks = 0;
        } else {
            e.pA = max(1, (e.n + T - 1) / T);
            e.pB = max(1, (e.m + T - 1) / T);
            tasks = e.pA + e.pB;
            ranks = tasks + 2;
        }
    }
    int ti = tasks, ri = ranks;                         // block-inclusive scan
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int t1 = __shfl_up_sync(0xffffffffu, ti, o), t2 = __shfl_up_sync(0xffffffffu, ri, o);
        if (lane >= o) { ti += t1; ri += t2; }
    }
    if (lane == 31) wsum[w] = make_int2(ti, ri);
    __syncthreads();
    int bt = 0, br = 0;
    for (int i = 0; i < w; ++i) { bt += wsum[i].x; br += wsum[i].y; }
    if (s < S) {
        e.tbase = bt + ti - tasks;
        e.rbase = br + ri - ranks;
        segs[s] = e;
    }
    if (threadIdx.x == BATCH_NT - 1) blk[blockIdx.x] = make_int2(bt + ti, br + ri);
}

// One CTA: exclusive scan of the nblk block sums in place; totals[0..1].
__global__ void __launch_bounds__(BATCH_NT) k_batch_scan(int2* __restrict__ blk, int nblk, int* __restrict__ totals) {
    __shared__ int2 wsum[BATCH_NT / 32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    int ct = 0, cr = 0;                                 // carry across chunks
    for (int c0 = 0; c0 < nblk; c0 += BATCH_NT) {
        const int i = c0 + threadIdx.x;
        const int2 v = i < nblk ? blk[i] : make_int2(0, 0);
        int ti = v.x, ri = v.y;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int t1 = __shfl_up_sync(0xffffffffu, ti, o), t2 = __shfl_up_sync(0xffffffffu, ri, o);
            if (lane >= o) { ti += t1; ri += t2; }
        }
        if (lane == 31) wsum[w] = make_int2(ti, ri);
        __syncthreads();
        int bt = 0, br = 0, at = 0, ar = 0;
        for (int k = 0; k < BATCH_NT / 32; ++k) {
            if (k < w) { bt += wsum[k].x; br += wsum[k].y; }
            at += wsum[k].x; ar += wsum[k].y;
        }
        if (i < nblk) blk[i] = make_int2(ct + bt + ti - v.x, cr + br + ri - v.y);
        ct += at;
        cr += ar;
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        totals[0] = ct;
        totals[1] = cr;
    }
}

__global__ void __launch_bounds__(BATCH_NT) k_batch_apply(const int2* __restrict__ blk, int S,
                                                          SegInfo* __restrict__ segs, int* __restrict__ task_seg,
                                                          int* __restrict__ rank_seg) {
    const int s = blockIdx.x * BATCH_NT + threadIdx.x;
    if (s < S) {
        const int2 b = blk[blockIdx.x];
        SegInfo e = segs[s];
        e.tbase += b.x;
        e.rbase += b.y;
        segs[s] = e;
        // task -> segment and rank entry -> segment maps (K1/K2 locate in O(1))
        const bool whole = e.pA == 0;
        for (int t = 0; t < (whole ? 1 : e.pA + e.pB); ++t) task_seg[e.tbase + t] = s;
        for (int t = 0; t < (whole ? 0 : e.pA + e.pB + 2); ++t) rank_seg[e.rbase + t] = s;
    }
    pdl_launch_dependents();
}

// ----------------------------------------------------------- plan dump
template <typename K>
__global__ void k_plan_dump(Geom g, const int* __restrict__ xbar, const int* __restrict__ ybar,
                            int64_t* __restrict__ tasks) {
    const int task = blockIdx.x * blockDim.x + threadIdx.x;
    if (task >= total_tasks(g)) return;
    Seg sg;
    const Task t = decode_task(g, task, xbar, ybar, sg);
    int64_t* row = tasks + (size_t)task * 6;
    row[0] = t.side; row[1] = t.kase; row[2] = t.a0; row[3] = t.a1; row[4] = t.b0; row[5] = t.b1;
}

// ----------------------------------------------------------------- K3
// Row a8 (§3: "sorting sequentially in parallel p
// consecutive blocks"): a stable sort of each run of R = NT * IPT consecutive
// elements, one CTA per run, in shared memory.  The paper leaves the block
// sort open; a least-significant-digit radix sort is stable by construction
// and costs a fixed number of passes whatever R, so the runs can be long
// (fewer merge rounds, row a9).
//   - keys are ranked through their unsigned order view (KeyOrd: sign bit
//     flipped for signed keys, IEEE totalOrder for floats); 4-bit digits;
//   - digits on which every key of the run agrees are skipped (the pass
//     would be the identity);
//   - blocked arrangement: thread t owns run positions [t*IPT, t*IPT+IPT)
//     (IPT odd: conflict-free strided shared loads), counts its digits in two
//     registers of packed 8-bit counters (its in-thread ranks), and one
//     block-wide exclusive scan in (digit, thread) order gives every
//     thread's base offset per digit -- equal digits keep sequence order;
//   - a partial last run is padded with the maximum unsigned view AFTER the
//     real elements: stability keeps the padding last, and it is never stored.
#ifndef SM_K3_NBUF
#define SM_K3_NBUF 1
#endif
template <typename K, bool HAS_V, int NT, int IPT>
struct K3Layout {
    using U = typename KeyOrd<K>::U;
    static constexpr int R = NT * IPT;
    static constexpr int NW = NT / 32;
    static constexpr int ND = 16;                        // 4-bit digits
    static constexpr int ROW = ND + 1;                   // padded per-thread base row
    static constexpr int NBUF = SM_K3_NBUF;              // 1: passes scatter in place
    static constexpr int OFF_V = NBUF * R * (int)sizeof(U);
    static constexpr int OFF_ROW = OFF_V + (HAS_V ? NBUF * R * 4 : 0);
    static constexpr int OFF_W = OFF_ROW + NT * ROW * 4; // warp totals [NW][ND]
    static constexpr int OFF_RED = OFF_W + NW * ND * 4;
    static constexpr int SMEM = OFF_RED + NW * (int)sizeof(U) + 16;
};

// 16 packed 8-bit counters in two 64-bit words: field d of (lo, hi).
__device__ __forceinline__ uint32_t cnt_get(uint64_t lo, uint64_t hi, int d) {
    const uint64_t w = d < 8 ? lo : hi;
    return (uint32_t)(w >> ((d & 7) * 8)) & 0xFFu;
}

#ifndef SM_K3_MINB
#define SM_K3_MINB 2
#endif
template <typename K, bool HAS_V, int NT, int IPT>
// (in and out may be the same array -- phase 1 in place -- so they are not
// __restrict__: every load of the run completes before the first barrier)
__global__ void __launch_bounds__(NT, sizeof(K) <= 8 ? SM_K3_MINB : 1) k_block_sort(const K* in, const uint32_t* vin,
                                                                                  K* out, uint32_t* vout, int N) {
    using Lay = K3Layout<K, HAS_V, NT, IPT>;
    using U = typename Lay::U;
    constexpr int R = Lay::R, NW = Lay::NW, ND = Lay::ND, ROW = Lay::ROW;
    constexpr int NDIG = (int)sizeof(U) * 2;             // 4-bit digits per key
    static_assert(IPT % 2 == 1 && IPT < 256 && NT % 32 == 0 && NT >= 32 && R < 65536,
                  "odd IPT; 8-bit counters; 16-bit scan fields");
    extern __shared__ __align__(128) char smem[];
    U* ku0 = (U*)smem;
    uint32_t* vv0 = (uint32_t*)(smem + Lay::OFF_V);
    uint32_t* rowb = (uint32_t*)(smem + Lay::OFF_ROW);  // [NT][ROW] per-thread digit bases
    uint32_t* wtot = (uint32_t*)(smem + Lay::OFF_W);    // [NW][ND] warp digit totals
    U* red = (U*)(smem + Lay::OFF_RED);                  // [NW]
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int base = blockIdx.x * R;
    const int len = min(R, N - base);

    {   // coalesced load, all loads in flight before the shared stores
        U u[IPT];
        uint32_t vl[HAS_V ? IPT : 1];
#pragma unroll
        for (int k = 0; k < IPT; ++k) {
            const int e = k * NT + tid;
            u[k] = e < len ? KeyOrd<K>::to(ld_stream(in + base + e)) : ~(U)0;
            if (HAS_V) vl[k] = e < len ? ld_stream(vin + base + e) : 0u;
        }
#pragma unroll
        for (int k = 0; k < IPT; ++k) {
            ku0[k * NT + tid] = u[k];
            if (HAS_V) vv0[k * NT + tid] = vl[k];
        }
    }
    __syncthreads();
    // digits on which the run's keys differ
    U diff = 0;
    {
        const U first = ku0[0];
        for (int e = tid; e < len; e += NT) diff |= ku0[e] ^ first;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            if constexpr (sizeof(U) == 16) {
                const uint64_t lo = __shfl_xor_sync(0xffffffffu, (uint64_t)diff, o);
                const uint64_t hi = __shfl_xor_sync(0xffffffffu, (uint64_t)(diff >> 64), o);
                diff |= ((U)hi << 64) | (U)lo;
            } else {
                diff |= __shfl_xor_sync(0xffffffffu, diff, o);
            }
        }
        if (lane == 0) red[w] = diff;
        __syncthreads();
        diff = 0;
#pragma unroll
        for (int i = 0; i < NW; ++i) diff |= red[i];
    }

    int cur = 0;
    for (int dg = 0; dg < NDIG; ++dg) {
        const int sh = dg * 4;
        if (((diff >> sh) & 0xF) == 0) continue;       // every key of the run has this digit
        // in place (NBUF = 1): every thread has read its items (step 1)
        // before the first barrier of the pass, the scatter follows the second
        const U* ks = ku0 + cur * R;
        U* kd = ku0 + ((cur ^ 1) % Lay::NBUF) * R;
        const uint32_t* vs = vv0 + cur * R;
        uint32_t* vd = vv0 + ((cur ^ 1) % Lay::NBUF) * R;
        // 1. this thread's items (blocked) and in-thread ranks
        // long runs (IPT > 17): ranks packed two 16-bit fields per register
        // (every rank < R < 2^16), so the pass fits two CTAs per SM
        constexpr bool PACK = IPT > 17;
        U key[IPT];
        uint32_t val[HAS_V ? IPT : 1];
        uint32_t rank[PACK ? (IPT + 1) / 2 : IPT];
        uint64_t clo = 0, chi = 0;
#pragma unroll
        for (int k = 0; k < IPT; ++k) {
            key[k] = ks[tid * IPT + k];
            if (HAS_V) val[k] = vs[tid * IPT + k];
            const int d = (int)(key[k] >> sh) & 0xF;
            const uint32_t r0 = cnt_get(clo, chi, d);
            if (!PACK) rank[k] = r0;
            else if (k & 1) rank[k >> 1] |= r0 << 16;
            else rank[k >> 1] = r0;
            const uint64_t inc = 1ull << ((d & 7) * 8);
            if (d < 8) clo += inc;
            else chi += inc;
        }
        // 2. warp-inclusive scan of the 16 counts, packed two 16-bit fields per word
        uint32_t c[ND / 2], x[ND / 2];
#pragma unroll
        for (int i = 0; i < ND / 2; ++i) {
            const uint32_t a0 = cnt_get(clo, chi, 2 * i), a1 = cnt_get(clo, chi, 2 * i + 1);
            c[i] = a0 | (a1 << 16);
            x[i] = c[i];
        }
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
#pragma unroll
            for (int i = 0; i < ND / 2; ++i) {
                const uint32_t t = __shfl_up_sync(0xffffffffu, x[i], o);
                if (lane >= o) x[i] += t;
            }
        }
        if (lane == 31) {
#pragma unroll
            for (int i = 0; i < ND / 2; ++i) {
                wtot[w * ND + 2 * i] = x[i] & 0xFFFFu;
                wtot[w * ND + 2 * i + 1] = x[i] >> 16;
            }
        }
        __syncthreads();
        // 3. digit-major, warp-minor bases: lanes d < ND of warp 0
        if (tid < ND) {
            uint32_t tot = 0;
            for (int i = 0; i < NW; ++i) tot += wtot[i * ND + tid];
            uint32_t ex = tot;                           // exclusive scan over the 16 digits
#pragma unroll
            for (int o = 1; o < ND; o <<= 1) {
                const uint32_t t = __shfl_up_sync(0xFFFFu, ex, o);
                if (tid >= o) ex += t;
            }
            uint32_t b = ex - tot;
            for (int i = 0; i < NW; ++i) {
                const uint32_t t = wtot[i * ND + tid];
                wtot[i * ND + tid] = b;
                b += t;
            }
        }
        __syncthreads();
        // 4. this thread's base per digit: warp base + exclusive lane prefix
#pragma unroll
        for (int i = 0; i < ND / 2; ++i) {
            const uint32_t ex = x[i] - c[i];
            rowb[tid * ROW + 2 * i] = wtot[w * ND + 2 * i] + (ex & 0xFFFFu);
            rowb[tid * ROW + 2 * i + 1] = wtot[w * ND + 2 * i + 1] + (ex >> 16);
        }
        __syncwarp();
        // 5. scatter: every destination first (the shared loads of the bases
        //    cannot be ordered behind the stores: the compiler does not know
        //    rowb and kd never alias), then the stores
#pragma unroll
        for (int k = 0; k < IPT; ++k) {
            const int d = (int)(key[k] >> sh) & 0xF;
            if (PACK) rank[k >> 1] += rowb[tid * ROW + d] << (16 * (k & 1));
            else rank[k] += rowb[tid * ROW + d];
        }
#pragma unroll
        for (int k = 0; k < IPT; ++k) {
            const uint32_t at = PACK ? (rank[k >> 1] >> (16 * (k & 1))) & 0xFFFFu : rank[k];
            kd[at] = key[k];
            if (HAS_V) vd[at] = val[k];
        }
        __syncthreads();
        cur = (cur ^ 1) % Lay::NBUF;
    }
    const U* kf = ku0 + cur * R;
    const uint32_t* vf = vv0 + cur * R;
#pragma unroll
    for (int k = 0; k < IPT; ++k) {
        const int e = k * NT + tid;
        if (e < len) {
            SM_DCHECK(base + e < N, "K3 store outside the input");
            st_stream(out + base + e, KeyOrd<K>::from(kf[e]));
            if (HAS_V) st_stream(vout + base + e, vf[e]);
        }
    }
}

// ---------------------------------------------------------------- K3H
// Row a8 with the paper's own block count (§3: "sorting
// sequentially in parallel p consecutive blocks", p = the processing
// elements): one CTA per SM sorts one block of ~N/p elements, so phase 2
// needs only ceil(log2 p) merge rounds (p = 148: 8 rounds for any N, against
// 15 with the shared-memory runs of K3 for N = 2^28).  The CTA's sort is a
// stable least-significant-digit radix sort of its block through global
// memory (8-bit digits of the key's unsigned order view, KeyOrd), ping-
// ponging between the caller's buffer (buf0) and the auxiliary one (buf1):
//   pre-pass  one read of the block's keys: the 256-bucket histogram of every
//             byte of the order view that varies, and the bytes on which keys
//             differ (bytes every key of the block shares are skipped);
//   pass      tiles of TILE elements in order, bulk-loaded (TMA) two tiles
//             ahead: each warp ranks its items by digit (peers with the same
//             digit from one ballot per digit bit, ranks in (item, lane)
//             order = input order, warp counters in shared memory), a block
//             scan over (digit, warp) places every item in the tile sorted by
//             digit (stable), and the sorted tile is written to the other
//             buffer at run[d] + (position - tile start of d), run[d] the
//             block's running offset of digit d.
// The result lands in the buffer the merge rounds start from (a third
// buffer, so no pass is spent on the parity of the pass count).
constexpr int K3H_NB = 256;          // buckets of an 8-bit digit
#ifndef SM_K3H_VREG
#define SM_K3H_VREG 0         // 1: payloads held in registers from the load to the scatter (128 regs: spills)
#endif
#ifndef SM_K3H_GROUPS
#define SM_K3H_GROUPS 2      // 2: two warp groups take alternate tiles (one ranks while the other writes)
#endif
#ifndef SM_K3H_REGKEYS
#define SM_K3H_REGKEYS 1     // items stay in registers from the ranking to the scatter (0: re-read from smem)
#endif

template <typename K, bool HAS_V, int NT, int TILE>
struct K3HLayout {
    using U = typename KeyOrd<K>::U;
    static constexpr int KB = (int)sizeof(K);
    static constexpr int NW = NT / 32;
    static constexpr int IPT = TILE / NT;
    static constexpr int NPOS = (int)sizeof(U);
    static constexpr int TILE_BYTES = TILE * (KB + (HAS_V ? 4 : 0));
    static constexpr int GROUPS = SM_K3H_GROUPS;                 // warp groups working on alternate tiles
    static constexpr int GT = NT / GROUPS;                       // threads per group
    static constexpr int GIPT = TILE / GT;                       // items per thread of a group's tile
    static constexpr int OFF_IN = 0;                            // 2 TMA targets: keys[TILE], vals[TILE]
    static constexpr int OFF_SORT = OFF_IN + 2 * TILE_BYTES;    // per group: the tile sorted by digit
    static constexpr int OFF_W = OFF_SORT + GROUPS * TILE_BYTES;  // warp counters [NW][256]
    static constexpr int OFF_HIST = OFF_W + NW * K3H_NB * 4;    // [NPOS][256]
    static constexpr int OFF_RUN = OFF_HIST + NPOS * 256 * 4;   // running offsets [256]
    static constexpr int OFF_TOT = OFF_RUN + K3H_NB * 4;        // tile totals [256]
    static constexpr int OFF_OFS = OFF_TOT + K3H_NB * 4;        // per group: run[d] - tile start[d] [256]
    static constexpr int OFF_TST = OFF_OFS + GROUPS * K3H_NB * 4;  // tile starts [256]
    static constexpr int OFF_RED = OFF_TST + K3H_NB * 4;        // [NW] diff (U), [8] scan sums
    static constexpr int OFF_BAR = (OFF_RED + NW * 16 + 64 + 15) & ~15;
    static constexpr int SMEM = OFF_BAR + 4 * 8;                // 4 mbarriers (the pre-pass's 4 TMA targets)
    // the pre-pass reads keys only, four TMA targets deep: the two input
    // targets and the two sorted-tile buffers, PT keys each
    static constexpr int PT = TILE_BYTES / KB;
    static constexpr int PIPT = PT / NT;
    static_assert(TILE % NT == 0 && NT % 32 == 0 && NT >= K3H_NB && (TILE * KB) % 16 == 0, "tile shape");
    static_assert(PT % NT == 0, "the pre-pass reads whole TMA targets: PT keys over NT threads");
    static_assert(GROUPS == 1 || (GROUPS == 2 && GT == K3H_NB), "two groups of 256 threads");
};

// L2-coherent load of any 4/8/16-byte element (bypasses L1: the block's
// other buffer is rewritten between passes)
template <typename T>
__device__ __forceinline__ T ld_cg(const T* p) {
    T v;
    if constexpr (sizeof(T) == 4) { const unsigned x = __ldcg((const unsigned*)p); memcpy(&v, &x, 4); }
    else if constexpr (sizeof(T) == 8) { const unsigned long long x = __ldcg((const unsigned long long*)p); memcpy(&v, &x, 8); }
    else { const ulonglong2 x = __ldcg((const ulonglong2*)p); memcpy(&v, &x, 16); }
    return v;
}

// Bulk-load X[0, cnt) (16-byte-aligned start) into smem; the < 16-byte tail
// with plain loads by the calling thread.  Returns the bytes for expect_tx.
template <typename T>
__device__ __forceinline__ uint32_t k3h_load(T* sdst, const T* X, int cnt, uint64_t* bar) {
    const uint32_t bytes = (uint32_t)cnt * (uint32_t)sizeof(T);
    const uint32_t body = bytes & ~15u;
    if (body) bulk_g2s(sdst, X, body, bar);
    for (uint32_t b = body / sizeof(T); b < (uint32_t)cnt; ++b) sdst[b] = ld_cg(X + b);
    return body;
}

// Block exclusive scan of v over threads 0..255 (8 warps); `sums` holds 8
// words; one barrier inside.  Returns the exclusive prefix of thread t < 256.
__device__ __forceinline__ uint32_t k3h_scan256(uint32_t v, uint32_t* sums) {
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (tid < K3H_NB && lane == 31) sums[w] = x;
    __syncthreads();
    uint32_t pre = 0;
    if (tid < K3H_NB)
        for (int i = 0; i < w; ++i) pre += sums[i];
    return pre + x - v;
}

// The lanes whose BITS-bit digit equals this lane's (within `act`): one
// ballot per digit bit, each folded in with one predicated AND / AND-NOT.
template <int BITS>
__device__ __forceinline__ uint32_t k3h_peers(uint32_t d, uint32_t act) {
    uint32_t peers = act;
#pragma unroll
    for (int b = 0; b < BITS; ++b) {
        asm("{\n\t.reg .pred q;\n\t.reg .b32 bl, t;\n\t"
            "and.b32 t, %1, %2;\n\t"
            "setp.ne.u32 q, t, 0;\n\t"
            "vote.sync.ballot.b32 bl, q, 0xffffffff;\n\t"
            "@!q not.b32 bl, bl;\n\t"
            "and.b32 %0, %0, bl;\n\t}"
            : "+r"(peers)
            : "r"(d), "r"(1u << b));
    }
    return peers;
}

// The stable rank of this lane's item in its warp's running count: the
// group of lanes with the same digit (`peers`) advances the warp counter of
// the digit once -- its highest lane adds the group size with one shared
// atomic, and every lane gets the count before it by a shuffle -- and the
// item's place is that count plus its peers in lower lanes.  A warp barrier
// orders the next item's atomic after this one's.
__device__ __forceinline__ uint32_t k3h_rank(uint32_t wc_s, uint32_t d, uint32_t peers, int lane, bool valid) {
    uint32_t r;
    asm volatile(
        "{\n\t.reg .pred lead, v;\n\t.reg .b32 hi, cnt, addr, old, src, lt, below;\n\t"
        "setp.ne.u32 v, %5, 0;\n\t"
        "shr.b32 hi, %2, %3;\n\t"
        "setp.eq.and.u32 lead, hi, 1, v;\n\t"
        "popc.b32 cnt, %2;\n\t"
        "mad.lo.u32 addr, %1, 4, %4;\n\t"
        "mov.u32 old, 0;\n\t"
        "@lead atom.shared.add.u32 old, [addr], cnt;\n\t"
        "bfind.u32 src, %2;\n\t"
        "shfl.sync.idx.b32 old, old, src, 0x1f, 0xffffffff;\n\t"
        "mov.u32 lt, %%lanemask_lt;\n\t"
        "and.b32 below, %2, lt;\n\t"
        "popc.b32 below, below;\n\t"
        "add.u32 %0, old, below;\n\t"
        "bar.warp.sync 0xffffffff;\n\t}"
        : "=r"(r)
        : "r"(d), "r"(peers), "r"(lane), "r"(wc_s), "r"((uint32_t)valid)
        : "memory");
    return r;
}

// L2-only store of any 4/8-byte element (K3H's sorted-tile write-out: the
// runs of a digit are short, L2 merges them into full lines)
template <typename T>
__device__ __forceinline__ void st_cg(T* p, T v) {
    if constexpr (sizeof(T) == 4) { unsigned x; memcpy(&x, &v, 4); __stcg((unsigned*)p, x); }
    else { unsigned long long x; memcpy(&x, &v, 8); __stcg((unsigned long long*)p, x); }
}

// One tile of a K3H pass (FULL: TILE elements, no padding items): rank the
// warps' items, scan over (digit, warp), scatter into the tile sorted by
// digit, write the sorted tile to dkb at run[d] + (position - tile start).
// Registers hold one word per item -- (rank << 9) | digit -- and the keys
// and payloads are re-read from the TMA target for the scatter, so the
// target is released (`release`: the next-but-one tile's load is issued
// there) only after the scatter.
template <typename K, bool HAS_V, int NT, int TILE, int BITS, bool FULL, typename F>
__device__ __forceinline__ void k3h_tile(const K* ik, const uint32_t* iv, int cnt, int shift, char* smem, K* dkb,
                                         uint32_t* dvb, int len, F release) {
    using Lay = K3HLayout<K, HAS_V, NT, TILE>;
    constexpr int NW = Lay::NW, IPT = Lay::IPT;
    constexpr uint32_t DMASK = (1u << BITS) - 1u;
    constexpr uint32_t PAD = 256u;                         // digit of a padding item (ranked nowhere)
    static_assert(TILE <= (1 << 22), "rank field");
    K* so_k = (K*)(smem + Lay::OFF_SORT);
    uint32_t* so_v = (uint32_t*)(smem + Lay::OFF_SORT + TILE * Lay::KB);
    uint32_t* wcnt = (uint32_t*)(smem + Lay::OFF_W);
    uint32_t* run = (uint32_t*)(smem + Lay::OFF_RUN);
    uint32_t* ofs = (uint32_t*)(smem + Lay::OFF_OFS);
    uint32_t* sums = (uint32_t*)(smem + Lay::OFF_RED + NW * 16);
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    uint32_t* wc = wcnt + w * K3H_NB;
    const uint32_t wc_s = smem_addr(wc);
    uint32_t dr[IPT];                                      // (rank in the warp << 9) | digit
#if SM_K3H_REGKEYS
    K key[IPT];
    uint32_t val[HAS_V ? IPT : 1];
#endif
#pragma unroll
    for (int k = 0; k < IPT; ++k) {                        // warp w: elements [w*32*IPT, ...), item k = k*32 + lane
        const int e = (w * IPT + k) * 32 + lane;
        const bool valid = FULL || e < cnt;
#if SM_K3H_REGKEYS
        if (valid) {
            key[k] = ik[e];
            if (HAS_V) val[k] = iv[e];
        }
        const uint32_t d = valid ? (BITS ? (uint32_t)(KeyOrd<K>::to(key[k]) >> shift) & DMASK : 0u) : PAD;
#else
        const uint32_t d = valid ? (BITS ? (uint32_t)(KeyOrd<K>::to(ik[e]) >> shift) & DMASK : 0u) : PAD;
#endif
        const uint32_t peers = k3h_peers<BITS>(d, FULL ? 0xffffffffu : __ballot_sync(0xffffffffu, valid));
        dr[k] = (k3h_rank(wc_s, d, peers, lane, valid) << 9) | d;
    }
    __syncthreads();                                       // every warp's counts are in wcnt
#if SM_K3H_REGKEYS
    release();                                             // (the items are in registers)
#endif
    // per digit: the tile total, its exclusive scan (tile start), then every
    // warp's first place of that digit in the sorted tile (start + earlier warps)
    uint32_t tc = 0;
    if (tid < K3H_NB) {
#pragma unroll
        for (int i = 0; i < NW; ++i) tc += wcnt[i * K3H_NB + tid];
    }
    const uint32_t ts = k3h_scan256(tc, sums);
    if (tid < K3H_NB) {
        uint32_t at = ts;
#pragma unroll
        for (int i = 0; i < NW; ++i) {
            const uint32_t x = wcnt[i * K3H_NB + tid];
            wcnt[i * K3H_NB + tid] = at;
            at += x;
        }
        ofs[tid] = run[tid] - ts;
        run[tid] += tc;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < IPT; ++k) {
        const uint32_t d = dr[k] & 511u;
        if (FULL || d != PAD) {
            const int e = (w * IPT + k) * 32 + lane;
            const uint32_t at = wc[d] + (dr[k] >> 9);
#if SM_K3H_REGKEYS
            (void)e;
            so_k[at] = key[k];
            if (HAS_V) so_v[at] = val[k];
#else
            so_k[at] = ik[e];
            if (HAS_V) so_v[at] = iv[e];
#endif
        }
    }
    __syncwarp();
    for (int i = lane; i < K3H_NB; i += 32) wc[i] = 0;     // this warp's counters, for the next tile
    __syncthreads();                                       // sorted tile complete; the TMA target is free
#if !SM_K3H_REGKEYS
    release();
#endif
#pragma unroll
    for (int k = 0; k < IPT; ++k) {
        const int j = k * NT + tid;
        if (FULL || j < cnt) {
            const K x = so_k[j];
            const uint32_t d = BITS ? (uint32_t)(KeyOrd<K>::to(x) >> shift) & DMASK : 0u;
            const uint32_t g = ofs[d] + (uint32_t)j;
            SM_DCHECK(g < (uint32_t)len, "K3H store outside its block");
            st_cg(dkb + g, x);
            if (HAS_V) st_cg(dvb + g, so_v[j]);
        }
    }
}

// One pass of K3H over the block: tiles of TILE elements in order, stable
// by the BITS-bit digit at `shift` (BITS = 0: a copy).  Per tile: each
// warp ranks its items (warp w: elements [w*32*IPT, (w+1)*32*IPT), item k
// of lane l = element (w*IPT + k)*32 + l, i.e. (item, lane) order = input
// order): lanes with the same digit from one ballot per digit bit, the
// warp's running count of each digit in shared memory, advanced by the
// lowest lane of each group (atomicAdd returns the count before it; warp
// barriers keep the items in order); then a scan over (digit, warp) places
// every item in the tile sorted by digit, and the sorted tile is written at
// run[d] + (position - tile start of d).
template <typename K, bool HAS_V, int NT, int TILE, int BITS>
__device__ __forceinline__ void k3h_pass(const K* sk, const uint32_t* sv, K* dk, uint32_t* dv, int64_t base, int len,
                                         int shift, char* smem, uint64_t* bar, uint32_t& ph) {
    using Lay = K3HLayout<K, HAS_V, NT, TILE>;
    const int tid = threadIdx.x;
    const int ntiles = (len + TILE - 1) / TILE;
    auto in_k = [&](int b) { return (K*)(smem + Lay::OFF_IN + b * Lay::TILE_BYTES); };
    auto in_v = [&](int b) { return (uint32_t*)(smem + Lay::OFF_IN + b * Lay::TILE_BYTES + TILE * Lay::KB); };
    auto issue = [&](int t) {
        if (tid == 0 && t < ntiles) {
            const int e0 = t * TILE, cnt = min(TILE, len - e0), b = t & 1;
            uint32_t tx = k3h_load<K>(in_k(b), sk + base + e0, cnt, &bar[b]);
            if (HAS_V) tx += k3h_load<uint32_t>(in_v(b), sv + base + e0, cnt, &bar[b]);
            mbar_arrive_expect_tx(&bar[b], tx);
        }
    };
    issue(0);
    issue(1);
    K* dkb = dk + base;
    uint32_t* dvb = HAS_V ? dv + base : nullptr;
    for (int t = 0; t < ntiles; ++t) {
        const int cnt = min(TILE, len - t * TILE);
        mbar_wait(&bar[t & 1], (ph >> (t & 1)) & 1u);
        ph ^= 1u << (t & 1);
        if (cnt == TILE)
            k3h_tile<K, HAS_V, NT, TILE, BITS, true>(in_k(t & 1), in_v(t & 1), TILE, shift, smem, dkb, dvb, len,
                                                     [&] { issue(t + 2); });
        else
            k3h_tile<K, HAS_V, NT, TILE, BITS, false>(in_k(t & 1), in_v(t & 1), cnt, shift, smem, dkb, dvb, len,
                                                      [&] { issue(t + 2); });
    }
}

// ---- K3H with two warp groups (SM_K3H_GROUPS = 2): group g (threads
// 256g .. 256g+255) takes tiles t = g, g+2, ... of a pass, so one group ranks
// its tile while the other scatters and writes its own (their barriers are
// named barriers of 256 threads).  The block's running digit offsets run[]
// advance in tile order: the group of tile t waits (bar.sync, 512 threads)
// for the group of tile t-1 to have added that tile's counts (bar.arrive).
__device__ __forceinline__ void k3h_gbar(int g) { named_sync(1 + g, 256); }
__device__ __forceinline__ void k3h_hand_arrive(int id) {
    asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(512) : "memory");
}

// Exclusive scan of v over the 256 threads of group g (one group barrier).
__device__ __forceinline__ uint32_t k3h_scan_group(uint32_t v, uint32_t* sums, int g) {
    const int tg = threadIdx.x & 255, lane = tg & 31, wg = tg >> 5;
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) sums[wg] = x;
    k3h_gbar(g);
    uint32_t pre = 0;
    for (int i = 0; i < wg; ++i) pre += sums[i];
    return pre + x - v;
}

// hnext (or null): the histogram of the next pass's byte at nshift, counted
// here as the sorted tile is written out (the pre-pass counts the first
// pass's byte only)
template <typename K, bool HAS_V, int NT, int TILE, int BITS, bool FULL, typename F>
__device__ __forceinline__ void k3h_tile_group(const K* ik, const uint32_t* iv, int cnt, int shift, char* smem, K* dkb,
                                               uint32_t* dvb, int len, int g, int t, int ntiles, F release,
                                               uint32_t* hnext, int nshift) {
    using Lay = K3HLayout<K, HAS_V, NT, TILE>;
    constexpr int IPT = Lay::GIPT;
    constexpr uint32_t DMASK = (1u << BITS) - 1u;
    constexpr uint32_t PAD = 256u;
    K* so_k = (K*)(smem + Lay::OFF_SORT + g * Lay::TILE_BYTES);
    uint32_t* so_v = (uint32_t*)(smem + Lay::OFF_SORT + g * Lay::TILE_BYTES + TILE * Lay::KB);
    uint32_t* wcnt = (uint32_t*)(smem + Lay::OFF_W);
    uint32_t* run = (uint32_t*)(smem + Lay::OFF_RUN);
    uint32_t* ofs = (uint32_t*)(smem + Lay::OFF_OFS) + g * K3H_NB;
    uint32_t* sums = (uint32_t*)(smem + Lay::OFF_RED + Lay::NW * 16) + 8 * g;
    const int tid = threadIdx.x, tg = tid & 255, lane = tid & 31, w = tid >> 5, wg = tg >> 5;
    uint32_t* wc = wcnt + w * K3H_NB;
    const uint32_t wc_s = smem_addr(wc);
    constexpr bool VREG = HAS_V && SM_K3H_VREG;            // payloads held in registers (else re-read)
    uint32_t dr[IPT];
    K key[IPT];
    uint32_t val[VREG ? IPT : 1];
#pragma unroll
    for (int k = 0; k < IPT; ++k) {                        // group warp wg: elements [wg*32*IPT, ...)
        const int e = (wg * IPT + k) * 32 + lane;
        const bool valid = FULL || e < cnt;
        if (valid) {
            key[k] = ik[e];
            if (VREG) val[k] = iv[e];
        }
        const uint32_t d = valid ? (BITS ? (uint32_t)(KeyOrd<K>::to(key[k]) >> shift) & DMASK : 0u) : PAD;
        const uint32_t peers = k3h_peers<BITS>(d, FULL ? 0xffffffffu : __ballot_sync(0xffffffffu, valid));
        dr[k] = (k3h_rank(wc_s, d, peers, lane, valid) << 9) | d;
    }
    k3h_gbar(g);                                           // the group's counts are in wcnt
    if (!HAS_V || VREG) release();                         // (the items are in registers)
    uint32_t tc = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) tc += wcnt[(8 * g + i) * K3H_NB + tg];
    const uint32_t ts = k3h_scan_group(tc, sums, g);
    {
        uint32_t at = ts;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const uint32_t x = wcnt[(8 * g + i) * K3H_NB + tg];
            wcnt[(8 * g + i) * K3H_NB + tg] = at;
            at += x;
        }
    }
    if (t > 0) named_sync(3 + ((t - 1) & 1), 512);        // run[] holds tiles < t
    ofs[tg] = run[tg] - ts;
    run[tg] += tc;
    if (t + 1 < ntiles) k3h_hand_arrive(3 + (t & 1));     // ... and now tile t too
    k3h_gbar(g);
#pragma unroll
    for (int k = 0; k < IPT; ++k) {
        const uint32_t d = dr[k] & 511u;
        if (FULL || d != PAD) {
            const uint32_t at = wc[d] + (dr[k] >> 9);
            so_k[at] = key[k];
            if (VREG) so_v[at] = val[k];
            else if (HAS_V) so_v[at] = iv[(wg * IPT + k) * 32 + lane];
        }
    }
    __syncwarp();
    for (int i = lane; i < K3H_NB; i += 32) wc[i] = 0;
    k3h_gbar(g);
    if (HAS_V && !VREG) release();                         // the payloads were read from the TMA target
#pragma unroll
    for (int k = 0; k < IPT; ++k) {
        const int j = k * 256 + tg;
        if (FULL || j < cnt) {
            const K x = so_k[j];
            const uint32_t d = BITS ? (uint32_t)(KeyOrd<K>::to(x) >> shift) & DMASK : 0u;
            const uint32_t gi = ofs[d] + (uint32_t)j;
            SM_DCHECK(gi < (uint32_t)len, "K3H store outside its block");
            st_cg(dkb + gi, x);
            if (HAS_V) st_cg(dvb + gi, so_v[j]);
            if (hnext) atomicAdd(&hnext[(uint32_t)(KeyOrd<K>::to(x) >> nshift) & 0xFFu], 1u);
        }
    }
}

template <typename K, bool HAS_V, int NT, int TILE, int BITS>
__device__ __forceinline__ void k3h_pass_group(const K* sk, const uint32_t* sv, K* dk, uint32_t* dv, int64_t base,
                                               int len, int shift, char* smem, uint64_t* bar, uint32_t& ph,
                                               uint32_t* hnext = nullptr, int nshift = 0) {
    using Lay = K3HLayout<K, HAS_V, NT, TILE>;
    const int g = threadIdx.x >> 8, tg = threadIdx.x & 255;
    const int ntiles = (len + TILE - 1) / TILE;
    auto issue = [&](int t) {
        if (tg == 0 && t < ntiles) {
            const int e0 = t * TILE, cnt = min(TILE, len - e0), b = t & 1;
            K* ik = (K*)(smem + Lay::OFF_IN + b * Lay::TILE_BYTES);
            uint32_t* iv = (uint32_t*)(smem + Lay::OFF_IN + b * Lay::TILE_BYTES + TILE * Lay::KB);
            uint32_t tx = k3h_load<K>(ik, sk + base + e0, cnt, &bar[b]);
            if (HAS_V) tx += k3h_load<uint32_t>(iv, sv + base + e0, cnt, &bar[b]);
            mbar_arrive_expect_tx(&bar[b], tx);
        }
    };
    issue(g);
    K* dkb = dk + base;
    uint32_t* dvb = HAS_V ? dv + base : nullptr;
    for (int t = g; t < ntiles; t += 2) {
        const int cnt = min(TILE, len - t * TILE);
        mbar_wait(&bar[g], (ph >> g) & 1u);
        ph ^= 1u << g;
        const K* ik = (const K*)(smem + Lay::OFF_IN + g * Lay::TILE_BYTES);
        const uint32_t* iv = (const uint32_t*)(smem + Lay::OFF_IN + g * Lay::TILE_BYTES + TILE * Lay::KB);
        if (cnt == TILE)
            k3h_tile_group<K, HAS_V, NT, TILE, BITS, true>(ik, iv, TILE, shift, smem, dkb, dvb, len, g, t, ntiles,
                                                           [&] { issue(t + 2); }, hnext, nshift);
        else
            k3h_tile_group<K, HAS_V, NT, TILE, BITS, false>(ik, iv, cnt, shift, smem, dkb, dvb, len, g, t, ntiles,
                                                            [&] { issue(t + 2); }, hnext, nshift);
    }
}

template <typename K, bool HAS_V, int NT, int TILE>
#ifndef SM_K3H_MINB
#define SM_K3H_MINB 1
#endif
#ifndef SM_K3H_DEFER
#define SM_K3H_DEFER 1        // the pre-pass counts the first pass's byte only; each pass counts the next one's
#endif
__global__ void __launch_bounds__(NT, SM_K3H_MINB) k_block_sort_hbm(K* buf0, uint32_t* vbuf0, K* buf1, uint32_t* vbuf1,
                                                           K* buf2, uint32_t* vbuf2, int64_t N, int64_t L0,
                                                           int final_buf, unsigned long long* ts) {
    using Lay = K3HLayout<K, HAS_V, NT, TILE>;
    using U = typename Lay::U;
    constexpr int NW = Lay::NW, NPOS = Lay::NPOS;
    extern __shared__ __align__(128) char smem[];
    uint32_t* wcnt = (uint32_t*)(smem + Lay::OFF_W);
    uint32_t* hist = (uint32_t*)(smem + Lay::OFF_HIST);
    uint32_t* run = (uint32_t*)(smem + Lay::OFF_RUN);
    U* red = (U*)(smem + Lay::OFF_RED);
    uint32_t* sums = (uint32_t*)(smem + Lay::OFF_RED + NW * 16);
    uint64_t* bar = (uint64_t*)(smem + Lay::OFF_BAR);      // [4]: one per TMA target (passes: 0, 1)
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int64_t base = (int64_t)blockIdx.x * L0;
    if (base >= N) return;
    const int len = (int)min(L0, N - base);              // < 2^31 (host check)
    uint32_t ph = 0u;                                   // bit b: the phase of TMA target b

    if (tid == 0) {
        for (int b = 0; b < 4; ++b) mbar_init(&bar[b], 1);
        fence_barrier_init();
    }
    for (int i = tid; i < NPOS * 256; i += NT) hist[i] = 0;
    for (int i = tid; i < NW * K3H_NB; i += NT) wcnt[i] = 0;
    __syncthreads();

    // pre-pass tile t (PT keys of the block) -> TMA target t % 4
    constexpr int PT = Lay::PT, PIPT = Lay::PIPT;
    const int ntp = (len + PT - 1) / PT;
    auto pissue = [&](int t) {
        if (tid == 0 && t < ntp) {
            const int e0 = t * PT, cnt = min(PT, len - e0), b = t & 3;
            K* dst = (K*)(smem + Lay::OFF_IN + b * Lay::TILE_BYTES);
            mbar_arrive_expect_tx(&bar[b], k3h_load<K>(dst, buf0 + base + e0, cnt, &bar[b]));
        }
    };
    auto pwait = [&](int t) {
        mbar_wait(&bar[t & 3], (ph >> (t & 3)) & 1u);
        ph ^= 1u << (t & 3);
    };

    // SM_K2_TSTAMP builds: per-CTA event times at ts[8 * (4096 + CTA) + slot]:
    // 0 entry, 1 pre-pass done, 2 + i pass i done
#ifdef SM_K2_TSTAMP
    auto k3_ts = [&](int slot) {
        if (ts && tid == 0) {
            unsigned long long t_;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));
            ts[8 * (4096 + blockIdx.x) + slot] = t_;
        }
    };
#else
    auto k3_ts = [](int) {};
    (void)ts;
#endif
    k3_ts(0);
    // ---- pre-pass: the bytes on which the block's keys differ, and the
    // histograms of the bytes in `posmask` (keys only, four targets of PT keys
    // in flight).  With two warp groups (SM_K3H_DEFER) it counts the first
    // pass's byte only -- byte 0, or after a second read the lowest varying
    // byte when byte 0 is shared -- and each pass counts the next pass's byte
    // as it writes its tiles out.
    const U first = KeyOrd<K>::to(ld_cg(buf0 + base));
    auto prepass = [&](uint32_t posmask) -> U {
        U diff = 0;
        for (int t = 0; t < 4; ++t) pissue(t);
        for (int t = 0; t < ntp; ++t) {
            pwait(t);
            const int cnt = min(PT, len - t * PT);
            const K* ik = (const K*)(smem + Lay::OFF_IN + (t & 3) * Lay::TILE_BYTES);
            U u[PIPT];
#pragma unroll
            for (int k = 0; k < PIPT; ++k) {
                const int e = k * NT + tid;
                u[k] = e < cnt ? KeyOrd<K>::to(ik[e]) : first;
            }
            __syncthreads();                             // TMA target t & 3 is free
            pissue(t + 4);
#pragma unroll
            for (int k = 0; k < PIPT; ++k) {
                const bool valid = k * NT + tid < cnt;
                const U x = u[k] ^ first;                 // the bits where this key differs from the block's first
                U m = x;                                  // ... OR-ed over the warp's valid lanes
                if constexpr (sizeof(U) == 4) {
                    m = __reduce_or_sync(0xffffffffu, valid ? (uint32_t)x : 0u);
                } else {
                    const uint32_t lo = __reduce_or_sync(0xffffffffu, valid ? (uint32_t)x : 0u);
                    const uint32_t hi = __reduce_or_sync(0xffffffffu, valid ? (uint32_t)(x >> 32) : 0u);
                    m = ((U)hi << 32) | lo;
                }
                diff |= m;
                const uint32_t nv = __popc(__ballot_sync(0xffffffffu, valid));
#pragma unroll
                for (int pos = 0; pos < NPOS; ++pos) {
                    if (!((posmask >> pos) & 1u)) continue;
                    const uint32_t b = (uint32_t)(u[k] >> (8 * pos)) & 0xFFu;
                    if (((m >> (8 * pos)) & 0xFF) == 0) { // warp-uniform: every valid lane has the first key's byte
                        if (lane == 0 && nv) atomicAdd(&hist[pos * 256 + ((uint32_t)(first >> (8 * pos)) & 0xFFu)], nv);
                    } else if (valid) {
                        atomicAdd(&hist[pos * 256 + b], 1u);
                    }
                }
            }
        }
        if (lane == 0) red[w] = diff;
        __syncthreads();
        diff = 0;
#pragma unroll
        for (int i = 0; i < NW; ++i) diff |= red[i];
        __syncthreads();                                 // (red[] reused by a second read)
        return diff;
    };
    // (keys-only sorts count every byte in the pre-pass: with the deferred counts
    // ptxas fails to allocate their kernel, C7600, around the R2P multisplit)
    constexpr bool DEFER = SM_K3H_DEFER && Lay::GROUPS == 2 && HAS_V;
    U diff = 0;
    uint32_t posmask = DEFER ? 1u : 0xFFu;
#pragma unroll 1
    for (int rd = 0; rd < 2; ++rd) {                     // (one call site: one inlined copy)
        const U d = prepass(posmask);
        if (rd == 0) diff = d;
        if (!DEFER || (diff & 0xFF) != 0 || diff == 0) break;
        int p0 = 1;                                      // byte 0 shared: count the lowest varying byte
        while (((diff >> (8 * p0)) & 0xFF) == 0) ++p0;
        posmask = 1u << p0;
    }
    k3_ts(1);

    // ---- the pass plan: one pass per varying byte, low to high.  Three
    // buffers: pass i writes the buffer that is neither its source nor the
    // final one (final_buf: 2 = buf2, the merge rounds' start; 0 = buf0,
    // a sort that is one block), the last pass writes the final buffer; a
    // block whose keys are all equal is copied (a pass on a 0-bit digit)
    int np = 0, hpos = 0;
#pragma unroll
    for (int pos = NPOS - 1; pos >= 0; --pos)
        if ((diff >> (8 * pos)) & 0xFF) { ++np; hpos = pos; }
    int npass = max(np, 1);
    if (final_buf == 0) npass = np == 0 ? 0 : max(np, 2);   // (one block: in place, or one more copying pass)
    auto bk = [&](int b) { return b == 0 ? buf0 : (b == 1 ? buf1 : buf2); };
    auto bv = [&](int b) { return b == 0 ? vbuf0 : (b == 1 ? vbuf1 : vbuf2); };
    int src = 0;
    for (int ps = 0; ps < npass; ++ps) {
        const int dst = ps == npass - 1 ? final_buf : (src != 1 && final_buf != 1 ? 1 : (src != 2 && final_buf != 2 ? 2 : 0));
        const bool digit_pass = ps < np;               // else: a copying pass
        if (digit_pass && ps > 0)
            do { ++hpos; } while (((diff >> (8 * hpos)) & 0xFF) == 0);
        const int bits = digit_pass ? 8 : 0;
        const int shift = 8 * hpos;
        // block exclusive prefix of this digit's histogram -> run[]
        uint32_t c = 0;
        if (tid < K3H_NB) c = bits ? hist[hpos * 256 + tid] : (tid == 0 ? (uint32_t)len : 0u);
        const uint32_t r0 = k3h_scan256(c, sums);
        if (tid < K3H_NB) run[tid] = r0;
        if constexpr (Lay::GROUPS == 2) {
            __syncthreads();                               // run[] of every digit before either group reads it
            // the next pass's byte, counted during this one (DEFER)
            int npos = -1;
            if (DEFER && digit_pass && ps + 1 < np) {
                npos = hpos + 1;
                while (((diff >> (8 * npos)) & 0xFF) == 0) ++npos;
            }
            uint32_t* hn = npos >= 0 ? hist + npos * 256 : nullptr;
            if (bits) k3h_pass_group<K, HAS_V, NT, TILE, 8>(bk(src), bv(src), bk(dst), bv(dst), base, len, shift, smem, bar, ph,
                                                            hn, 8 * max(npos, 0));
            else k3h_pass_group<K, HAS_V, NT, TILE, 0>(bk(src), bv(src), bk(dst), bv(dst), base, len, shift, smem, bar, ph);
        } else {
            if (bits) k3h_pass<K, HAS_V, NT, TILE, 8>(bk(src), bv(src), bk(dst), bv(dst), base, len, shift, smem, bar, ph);
            else k3h_pass<K, HAS_V, NT, TILE, 0>(bk(src), bv(src), bk(dst), bv(dst), base, len, shift, smem, bar, ph);
        }
        // this pass's global writes before the next pass's bulk reads (async proxy)
        asm volatile("fence.proxy.async.global;" ::: "memory");
        __syncthreads();
        src = dst;
        if (ps < 6) k3_ts(2 + ps);
    }
}

}  // namespace
}  // namespace sm
