// sm_kernels4.cuh -- two merge rounds of the merge sort in one HBM pass.
//
// Phase 2 of the sort (§3, row a9) merges pairs of runs
// in ceil(log2 p) rounds; every round reads and writes all N elements, and
// on B200 a round is bound by HBM (C5: 0.66 ms per round at 0.99 of the
// measured copy).  Here two consecutive rounds -- runs R0, R1 -> X and
// R2, R3 -> Y, then X, Y -> the run of length 4L -- happen in one pass: the
// paper's partition (L297-340) is applied to the four runs at once and every
// subproblem is merged twice inside shared memory (level 1: R0 with R1 and R2
// with R3; level 2: their results), so the intermediate runs X, Y never
// reach HBM.  The result is bit-identical to the two rounds (stable order:
// key, then run index, then position).
//
// Partition (the paper's Steps 1-2 generalised from two arrays to four):
//   every run j is cut into blocks of S elements; block start e = R_j[qS]
//   gets its rank in every other run j' -- the high rank (elements <= e)
//   when j' < j, the low rank (elements < e) when j' > j: the generalisation
//   of x̄_i = rank_low(A[x_i], B) and ȳ_j = rank_high(B[y_j], A) (L304-309,
//   ties: the earlier run first, reading R2).  e's place in the merged
//   group is f(e) = qS + the three ranks.  Sorted by f, consecutive block
//   starts delimit the subproblems: between two of them each run
//   contributes one contiguous range, of at most S elements (no block start
//   of that run lies strictly inside), so a subproblem holds at most 4S --
//   the paper's task bound (L388-393) for four arrays.  The subproblems are
//   disjoint and cover the group; their output offset is f of their first
//   block start (reading R20 in DESIGN.md).
//
//   k4_sample   the block-start keys of every run, contiguous (L2-resident)
//   k4_ranks    four lanes per block start, one per run: its three ranks, each by a
//               binary search over the other run's block-start keys (L2),
//               then one inside the block that search names (S elements,
//               HBM)
//   --  single synchronisation (PDL griddepcontrol.wait, L373-375)
//   k4_order    four lanes per block start: its place among the group's
//               block starts (three searches over the f values, L2), and
//               the group's sentinel boundaries
//   k_tasks4    K2's persistent warp-specialised TMA ring, four ranges per
//               task, two shared-memory merge levels per stage
#pragma once
#include "sm_kernels.cuh"

namespace sm {
namespace {   // internal linkage: every translation unit keeps its own kernels

#ifndef SM_K4_LOG2_NV
#define SM_K4_LOG2_NV 0       // 1: split probes sized by the stage (NV) instead of the task bound (2S)
#endif

struct Geom4 {
    int N;            // elements
    int L;            // input run length (a multiple of 16 or the whole input)
    int S;            // block size of the partition (block starts every S elements of a run)
    int cmax;         // block starts per run at most: ceil(L / S)
    int TPG;          // tasks per group: 4 * cmax + 1 (the last groups' unused ones are empty)
    int G;            // groups of four runs: ceil(N / 4L)
    int* ctr;         // k_tasks4's task counter, zeroed by k4_order
    const int4* bnd;  // [G][TPG + 1] subproblem boundaries: (rank in R0, R1, R2, R3)
    uint32_t* cover;  // SM_DEBUG builds: every output element counted here (or null)
};

__device__ __forceinline__ int64_t run_base(const Geom4& g, int grp, int j) {
    return (int64_t)grp * 4 * g.L + (int64_t)j * g.L;
}
__device__ __forceinline__ int run_len(const Geom4& g, int grp, int j) {
    const int64_t b = run_base(g, grp, j);
    return b >= g.N ? 0 : (int)min((int64_t)g.L, (int64_t)g.N - b);
}
__device__ __forceinline__ int run_starts(const Geom4& g, int len) { return (len + g.S - 1) / g.S; }

// ---- k4_sample: spl[(grp * 4 + j) * cmax + q] = R_j[qS] -------------------
template <typename K>
__global__ void __launch_bounds__(256) k4_sample(const K* __restrict__ in, Geom4 g, K* __restrict__ spl) {
    pdl_wait();                                       // the previous pass wrote `in`
    const int id = blockIdx.x * blockDim.x + threadIdx.x;
    if (id < g.G * 4 * g.cmax) {
        const int q = id % g.cmax, j = (id / g.cmax) & 3, grp = id / (4 * g.cmax);
        if ((int64_t)q * g.S < run_len(g, grp, j)) spl[id] = ldg_key(in + run_base(g, grp, j) + (int64_t)q * g.S);
    }
    pdl_launch_dependents();
}

// Count of X[0, len) before key e in the stable order: elements <= e when
// `high` (X's run precedes e's), else elements < e.  Binary, branch-light.
template <typename K>
__device__ __forceinline__ int count_before(const K* X, int len, K e, bool high) {
    int lo = 0, n = len;
    while (n > 0) {
        const int h = n >> 1;
        const K x = ldg_key(X + lo + h);
        const bool before = high ? key_le(x, e) : key_lt(x, e);
        lo = before ? lo + h + 1 : lo;
        n = before ? n - h - 1 : h;
    }
    return lo;
}

// ---- k4_ranks: Steps 1-2 for four runs ------------------------------------
// Four lanes per block start, one per run: lane jj ranks e in run jj (its own
// run: qS), so the three searches run side by side instead of one after the
// other (each is ~25 dependent loads); the quad's lane 0 writes the ranks.
template <typename K>
__global__ void __launch_bounds__(256) k4_ranks(const K* __restrict__ in, Geom4 g, const K* __restrict__ spl,
                                                int4* __restrict__ rk, int* __restrict__ fv) {
    pdl_wait();
    const int tid = blockIdx.x * blockDim.x + threadIdx.x;
    const int id = tid >> 2, jj = tid & 3;
    int r = 0;
    bool valid = false;
    if (id < g.G * 4 * g.cmax) {
        const int q = id % g.cmax, j = (id / g.cmax) & 3, grp = id / (4 * g.cmax);
        valid = (int64_t)q * g.S < run_len(g, grp, j);
        if (valid) {
            if (jj == j) {
                r = q * g.S;
            } else {
                const K e = spl[id];
                const int len = run_len(g, grp, jj);
                const bool high = jj < j;
                // the block of run jj holding the rank: c block starts lie before e
                const int c = count_before(spl + (grp * 4 + jj) * g.cmax, run_starts(g, len), e, high);
                if (c > 0) {
                    const int lo = (c - 1) * g.S + 1, hi = min(c * g.S, len);
                    r = lo + count_before(in + run_base(g, grp, jj) + lo, hi - lo, e, high);
                }
            }
        }
    }
    const int lane = threadIdx.x & 31, q0 = lane & ~3;
    const int r0 = __shfl_sync(0xffffffffu, r, q0), r1 = __shfl_sync(0xffffffffu, r, q0 + 1),
              r2 = __shfl_sync(0xffffffffu, r, q0 + 2), r3 = __shfl_sync(0xffffffffu, r, q0 + 3);
    if (valid && jj == 0) {
        rk[id] = make_int4(r0, r1, r2, r3);
        fv[id] = r0 + r1 + r2 + r3;
    }
    pdl_launch_dependents();
}

// ---- k4_order: the block starts of a group in output order ----------------
// bnd[grp][0] = (0,0,0,0); bnd[grp][1 + k] = the k-th block start by f;
// bnd[grp][1 + tot ..] = (len0, len1, len2, len3): the tasks past the
// group's last block start are empty.  Four lanes per block start as in
// k4_ranks (lane jj: the block starts of run jj before it).
__global__ void __launch_bounds__(256) k4_order(Geom4 g, const int4* __restrict__ rk, const int* __restrict__ fv,
                                                int4* __restrict__ bnd) {
    pdl_wait();
    if (g.ctr && blockIdx.x == 0 && threadIdx.x == 0) *g.ctr = 0;   // k_tasks4's counter (after the wait)
    const int tid = blockIdx.x * blockDim.x + threadIdx.x;
    const int id = tid >> 2, jj = tid & 3;
    int cntb = 0;
    bool valid = false;
    if (id < g.G * 4 * g.cmax) {
        const int q = id % g.cmax, j = (id / g.cmax) & 3, grp = id / (4 * g.cmax);
        valid = (int64_t)q * g.S < run_len(g, grp, j);
        if (valid) {
            if (jj == j) {
                cntb = q;
            } else {
                const int f = fv[id];
                const int* F = fv + (grp * 4 + jj) * g.cmax;
                int lo = 0, n = run_starts(g, run_len(g, grp, jj));
                while (n > 0) {                        // f values of distinct elements differ
                    const int h = n >> 1;
                    const bool before = __ldg(F + lo + h) < f;
                    lo = before ? lo + h + 1 : lo;
                    n = before ? n - h - 1 : h;
                }
                cntb = lo;
            }
        }
    }
    int pos = cntb;
    pos += __shfl_xor_sync(0xffffffffu, pos, 1);
    pos += __shfl_xor_sync(0xffffffffu, pos, 2);
    if (valid && jj == 0) {
        const int grp = id / (4 * g.cmax);
        bnd[(int64_t)grp * (g.TPG + 1) + 1 + pos] = rk[id];
    }
    if (tid < g.G * (g.TPG + 1)) {                    // sentinels
        const int s = tid % (g.TPG + 1), grp = tid / (g.TPG + 1);
        int len[4], tot = 0;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            len[k] = run_len(g, grp, k);
            tot += run_starts(g, len[k]);
        }
        if (s == 0) bnd[tid] = make_int4(0, 0, 0, 0);
        else if (s > tot) bnd[tid] = make_int4(len[0], len[1], len[2], len[3]);
    }
    pdl_launch_dependents();
}

// ---- k_tasks4 -------------------------------------------------------------
struct TaskDesc4 {
    int l[4];          // range lengths in R0..R3
    int s[4];          // stage key index of each range's first element
    int vs[4];         // stage payload index of each range's first payload
    int x0, xv0;       // stage key / payload index of the task region (level-1 output X | Y)
    int ob, obv;       // stage key / payload index of output element 0 (phase-aligned to C)
    int off;           // global output element index
    int pst;           // first padded diagonal of the task in the stage
    int p01;           // padded level-1 diagonals of the X half: VT * ceil((l0 + l1) / VT)
};

template <typename K, bool HAS_V, int NC, int VT, int STAGES, int MAXT>
struct K4Layout {
    static constexpr int NV = NC * VT;
    static constexpr int KB = (int)sizeof(K);
    static constexpr int EPV = 16 / KB;
    // a task's key region: four 16-byte-aligned spans (<= l*KB + 30 bytes
    // each) + 16 bytes of slack for the merges' look-ahead reads
    static constexpr int KREG = NV * KB + MAXT * 144;
    static constexpr int VREG = HAS_V ? NV * 4 + MAXT * 144 : 0;
    static constexpr int STAGE_BYTES = KREG + VREG;
    static constexpr int OFF_DESC = STAGES * STAGE_BYTES;
    static constexpr int OFF_PST = OFF_DESC + STAGES * MAXT * (int)sizeof(TaskDesc4);
    static constexpr int OFF_BAR = ((OFF_PST + STAGES * (MAXT + 2) * 4) + 15) & ~15;
    static constexpr int SMEM = OFF_BAR + 3 * STAGES * 8;
    static constexpr int THREADS = NC + 64;
    // largest task: 4S elements, padded per level-1 half (+ 2 (VT - 1))
    static constexpr int S = (NV - 2 * VT) / 4;
};

// Producer (warp 0): tasks from the launch's counter in chunks (as K2's
// dynamic assignment), each lane one task: its four ranges from the two
// boundaries around it; the longest prefix of the window that fits a stage
// is packed and its eight spans (keys, payloads) bulk-loaded.
template <typename K, bool HAS_V, int VT, int STAGES, int MAXT, typename Lay>
__device__ __forceinline__ void k4_producer(const K* __restrict__ in, const uint32_t* __restrict__ vin,
                                            const K* out, const uint32_t* vout, const Geom4& g, char* smem,
                                            TaskDesc4* desc, int* pst, uint64_t* full, uint64_t* empty) {
    constexpr int NV = Lay::NV;
    constexpr int KB = Lay::KB;
    constexpr int CH = 8;
    const int ntasks = g.G * g.TPG;
    const int lane = threadIdx.x;
    const int G = (int)gridDim.x;
    int l[4] = {0, 0, 0, 0};
    int gs[4] = {0, 0, 0, 0};                       // global element index of each range's first element
    int off = 0;
    int cnt = 0, seen = 0;
    bool more = ntasks > 0;
    int resv = 0, resv_n = 0;
    for (int it = 0;; ++it) {
        const int thr = min(33 - CH, max(16, (ntasks - seen) / G));
        if (cnt < min(8, thr) && more) {
            if (resv_n == 0) {
                resv_n = max(1, min(CH, ntasks / (2 * G)));
                if (lane == 0) resv = atomicAdd(g.ctr, resv_n);
            }
            int base = __shfl_sync(0xffffffffu, resv, 0);
            const int take = resv_n;
            seen = base + take;
            more = seen < ntasks;
            if (more) {
                resv_n = max(1, min(CH, (ntasks - seen) / (2 * G)));
                if (lane == 0) resv = atomicAdd(g.ctr, resv_n);
            }
            base -= cnt;
            const int my = base + lane;
            const bool fill = lane >= cnt && lane < cnt + take && my < ntasks;
            if (fill) {
                const int grp = my / g.TPG, t = my % g.TPG;
                const int4* b = g.bnd + (int64_t)grp * (g.TPG + 1) + t;
                const int4 lo = __ldg(b), hi = __ldg(b + 1);
                const int lo_[4] = {lo.x, lo.y, lo.z, lo.w}, hi_[4] = {hi.x, hi.y, hi.z, hi.w};
                int tot = 0;
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    // sorted runs give 0 <= l <= S (L388-393 for four arrays);
                    // clamp so that unsorted input still terminates in the stage
                    l[j] = max(0, min(hi_[j] - lo_[j], Lay::S));
                    gs[j] = (int)(run_base(g, grp, j) + lo_[j]);
                    tot += lo_[j];
                }
                off = (int)((int64_t)grp * 4 * g.L + tot);
            }
            cnt += __popc(__ballot_sync(0xffffffffu, fill));
        }
        const int st = it % STAGES;
        if (it >= STAGES) mbar_wait_sleep(&empty[st], ((it / STAGES) - 1) & 1);
        int* ps = pst + st * (MAXT + 2);
        if (cnt == 0) {
            if (lane == 0) {
                ps[MAXT + 1] = -1;
                mbar_arrive(&full[st]);
            }
            return;
        }
        const int m01 = l[0] + l[1], m23 = l[2] + l[3];
        const int p01 = ((m01 + VT - 1) / VT) * VT;
        const int P = p01 + ((m23 + VT - 1) / VT) * VT;
        int pre = lane < cnt ? P : NV + 1;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(0xffffffffu, pre, o);
            if (lane >= o) pre += t;
        }
        const unsigned taken = __ballot_sync(0xffffffffu, lane < cnt && lane < MAXT && pre <= NV);
        const bool take_me = (taken >> lane) & 1u;
        const int take = __popc(taken);
        const int pme = take_me ? P : 0;
        int kreg = 0, vreg = 0;
        if (take_me) {
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                kreg += span_bytes(in + gs[j], l[j]);
                if (HAS_V) vreg += span_bytes(vin + gs[j], l[j]);
            }
            kreg += 16;
            if (HAS_V) vreg += 16;
        }
        int incl = pme, kat = kreg, vat = vreg;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int t0 = __shfl_up_sync(0xffffffffu, incl, o);
            const int t1 = __shfl_up_sync(0xffffffffu, kat, o);
            const int t2 = __shfl_up_sync(0xffffffffu, vat, o);
            if (lane >= o) { incl += t0; kat += t1; vat += t2; }
        }
        kat -= kreg;
        vat -= vreg;
        const int last = 31 - __clz(taken);
        const int ktot = __shfl_sync(0xffffffffu, kat + kreg, last);
        const int vtot = __shfl_sync(0xffffffffu, vat + vreg, last);
        char* stage = smem + st * Lay::STAGE_BYTES;
        char* vstage = stage + Lay::KREG;
        if (take_me) {
            const int slot = __popc(taken & ((1u << lane) - 1u));
            TaskDesc4* d = desc + st * MAXT + slot;    // written in place (a local copy spills)
            int at = kat, vt = vat;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                d->l[j] = l[j];
                d->s[j] = issue_span(stage, at, in + gs[j], l[j], &full[st]);
                at += span_bytes(in + gs[j], l[j]);
                d->vs[j] = 0;
                if (HAS_V) {
                    d->vs[j] = issue_span(vstage, vt, vin + gs[j], l[j], &full[st]);
                    vt += span_bytes(vin + gs[j], l[j]);
                }
            }
            d->x0 = kat / KB;
            d->xv0 = vat / 4;
            d->ob = kat / KB + phase_of(out + off);
            d->obv = HAS_V ? vat / 4 + phase_of(vout + off) : 0;
            d->off = off;
            d->pst = incl - pme;
            d->p01 = p01;
            if (lane == last) {
                ps[take] = incl;
                ps[MAXT + 1] = take;
            }
            ps[slot] = incl - pme;
        }
        __syncwarp();
        if (lane == 0) mbar_arrive_expect_tx(&full[st], (uint32_t)(ktot - 16 * take + (HAS_V ? vtot - 16 * take : 0)));
        int sl = lane + take;
        if (sl > 31) sl = lane;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            l[j] = __shfl_sync(0xffffffffu, l[j], sl);
            gs[j] = __shfl_sync(0xffffffffu, gs[j], sl);
        }
        off = __shfl_sync(0xffffffffu, off, sl);
        cnt -= take;
    }
}

// One thread's cnt <= VT outputs of the stable merge of a[0, la) and
// b[0, lb) (stage indices sa / sb; payload indices va / vb) from diagonal d:
// ties to a.  A range may be empty (a copy).
template <typename K, bool HAS_V, int VT, int LOG2NV>
__device__ __forceinline__ void k4_merge(const K* sk, const uint32_t* sv, int sa, int la, int va, int sb, int lb,
                                         int vb, int d, K (&out)[VT], uint32_t (&v)[HAS_V ? VT : 1]) {
    constexpr int KB = (int)sizeof(K);
    if (la > 0 && lb > 0) {
        using V = typename FViewOf<K>::type;
        const uint32_t sa0 = smem_addr(sk + sa);
        const uint32_t sb0 = smem_addr(sk + sb);
        const int ai = split_smem<V, LOG2NV>(sa0, la, sb0, lb, d);
        const int bi = d - ai;
        uint32_t pa = sa0 + ai * KB, pb = sb0 + bi * KB;
        const uint32_t pae = sa0 + la * KB, pbe = sb0 + lb * KB;
        V ka = lds<V>(pa), kb = lds<V>(pb), na = lds<V>(pa + KB), nb = lds<V>(pb + KB);
        V ov[VT];
        int src[VT];
        int ia = va + ai, ib = vb + bi;
        if (__all_sync(__activemask(), ai + VT <= la && bi + VT <= lb)) {
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
            const int cnt = la + lb - d;
#pragma unroll
            for (int k = 0; k < VT; ++k)
                if (k < cnt) v[k] = sv[src[k]];
        }
    } else {
        const int ks = la ? sa : sb, vs = la ? va : vb, cnt = la + lb - d;
#pragma unroll
        for (int k = 0; k < VT; ++k) {
            if (k < cnt) {
                out[k] = sk[ks + d + k];
                if (HAS_V) v[k] = sv[vs + d + k];
            }
        }
    }
}

// k_tasks4: warp 0 producer, warp 1 storer (as K2), NC consumers: level 1
// (R0 with R1 -> X, R2 with R3 -> Y, written back in place at the task's
// region start), level 2 (X with Y, written in place phase-aligned to C).
template <typename K, bool HAS_V, int NC, int VT, int STAGES, int MAXT, int MINB>
__global__ void __launch_bounds__(K4Layout<K, HAS_V, NC, VT, STAGES, MAXT>::THREADS, MINB)
    k_tasks4(const K* __restrict__ in, const uint32_t* __restrict__ vin, K* __restrict__ out,
             uint32_t* __restrict__ vout, Geom4 g) {
    using Lay = K4Layout<K, HAS_V, NC, VT, STAGES, MAXT>;
    // merge-path splits: a level-1 range holds <= S elements, a level-2
    // range (X) <= 2S, plus the split's skew (< 2 * SM_SPLIT_SKEW_LEVEL
    // virtual candidates): 2^(LOG2+1) - 1 covers them
#if SM_K4_LOG2_NV
    constexpr int LOG2NV = 31 - __builtin_clz(Lay::NV);
#else
    constexpr int LOG2NV = 31 - __builtin_clz(2 * Lay::S + 2 * SM_SPLIT_SKEW_LEVEL);
#endif
    constexpr int EK = 2 * (Lay::EPV - 1);
    constexpr int EV = HAS_V ? 2 * 3 : 0;
    extern __shared__ __align__(128) char smem[];
    TaskDesc4* desc = (TaskDesc4*)(smem + Lay::OFF_DESC);
    int* pst = (int*)(smem + Lay::OFF_PST);
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
    pdl_wait();   // the single synchronisation (L373-375): every boundary visible

    if (threadIdx.x < 32) {
        k4_producer<K, HAS_V, VT, STAGES, MAXT, Lay>(in, vin, out, vout, g, smem, desc, pst, full, empty);
        return;
    }
    if (threadIdx.x < 64) {
        // -------------------------------------------------------- storer
        const int lane = threadIdx.x - 32;
        for (int it = 0;; ++it) {
            const int s = it % STAGES;
            mbar_wait_sleep(&written[s], (it / STAGES) & 1);
            const int nt = pst[s * (MAXT + 2) + MAXT + 1];
            if (nt < 0) break;
            const K* sk = (const K*)(smem + s * Lay::STAGE_BYTES);
            const uint32_t* sv = (const uint32_t*)(smem + s * Lay::STAGE_BYTES + Lay::KREG);
#ifdef SM_DEBUG
            for (int k = 0; k < nt; ++k) {
                const TaskDesc4& t = desc[s * MAXT + k];
                const int L = t.l[0] + t.l[1] + t.l[2] + t.l[3];
                SM_DCHECK(t.off >= 0 && L >= 0 && (long long)t.off + L <= g.N, "k_tasks4 task range outside C");
                if (g.cover)
                    for (int e = lane; e < L; e += 32) atomicAdd(&g.cover[t.off + e], 1u);
            }
#endif
            if (lane < nt) {
                const TaskDesc4& t = desc[s * MAXT + lane];
                const int L = t.l[0] + t.l[1] + t.l[2] + t.l[3];
                if (L > 0) {
                    store_middle<K>(out + t.off, sk, t.ob, L);
                    if (HAS_V) store_middle<uint32_t>(vout + t.off, sv, t.obv, L);
                }
                bulk_commit();
            }
            if constexpr (EK + EV > 0) {
                for (int e = lane; e < nt * (EK + EV); e += 32) {
                    const int k = e / (EK + EV), r = e % (EK + EV);
                    const TaskDesc4& t = desc[s * MAXT + k];
                    const int L = t.l[0] + t.l[1] + t.l[2] + t.l[3];
                    if (r < EK) store_edge<K>(out + t.off, sk, t.ob, L, r);
                    else if (HAS_V) store_edge<uint32_t>(vout + t.off, sv, t.obv, L, r - EK);
                }
            }
            bulk_wait_read<0>();
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[s]);
        }
        return;
    }

    // ---------------------------------------------------------- consumers
    const int c = threadIdx.x - 64;
    const int lane = threadIdx.x & 31;
    const int D = c * VT;
    for (int it = 0;; ++it) {
        const int s = it % STAGES;
        mbar_wait(&full[s], (it / STAGES) & 1);
        const int* ps = pst + s * (MAXT + 2);
        const int nt = ps[MAXT + 1];
        if (nt < 0) {
            if (lane == 0) mbar_arrive(&written[s]);
            break;
        }
        K* sk = (K*)(smem + s * Lay::STAGE_BYTES);
        uint32_t* sv = (uint32_t*)(smem + s * Lay::STAGE_BYTES + Lay::KREG);
        int k = -1, d = 0;
        if (D < ps[nt]) {
            int lo = 0, hi = nt - 1;
            while (lo < hi) {
                const int mid = (lo + hi + 1) >> 1;
                if (ps[mid] <= D) lo = mid;
                else hi = mid - 1;
            }
            k = lo;
            d = D - ps[lo];
        }
        const TaskDesc4* td = desc + s * MAXT + (k < 0 ? 0 : k);
        K o[VT];
        uint32_t v[HAS_V ? VT : 1];
        // level 1: X = R0 with R1, Y = R2 with R3 (ties to the earlier run),
        // written back at the task's region start; level 2: X with Y (ties
        // to X), written phase-aligned to C.  One merge call site for both
        // (a second inlined merge spills).
#pragma unroll 1
        for (int lev = 0; lev < 2; ++lev) {
            int cnt = 0, wk = 0, wv = 0;
            if (k >= 0) {
                const int m01 = td->l[0] + td->l[1], m23 = td->l[2] + td->l[3];
                int sa, la, va, sb, lb, vb, e;
                if (lev == 0) {
                    const bool hx = d < td->p01;
                    const int h = hx ? 0 : 2;
                    e = hx ? d : d - td->p01;
                    sa = td->s[h]; la = td->l[h]; va = td->vs[h];
                    sb = td->s[h + 1]; lb = td->l[h + 1]; vb = td->vs[h + 1];
                    wk = td->x0 + (hx ? 0 : m01) + e;
                    wv = td->xv0 + (hx ? 0 : m01) + e;
                } else {
                    e = d;
                    sa = td->x0; la = m01; va = td->xv0;
                    sb = td->x0 + m01; lb = m23; vb = td->xv0 + m01;
                    wk = td->ob + d;
                    wv = td->obv + d;
                }
                cnt = min(VT, la + lb - e);
                if (cnt > 0) k4_merge<K, HAS_V, VT, LOG2NV>(sk, sv, sa, la, va, sb, lb, vb, e, o, v);
            }
            named_sync(1, NC);                         // this level's inputs have been read
#pragma unroll
            for (int q = 0; q < VT; ++q) {
                if (q < cnt) {
                    sk[wk + q] = o[q];
                    if (HAS_V) sv[wv + q] = v[q];
                }
            }
            if (lev == 0) named_sync(1, NC);           // X | Y of every task written
        }
        fence_proxy_async();
        __syncwarp();
        if (lane == 0) mbar_arrive(&written[s]);
    }
}

}  // namespace
}  // namespace sm
