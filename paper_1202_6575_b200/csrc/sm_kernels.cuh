// sm_kernels.cuh -- the kernels of the B200 stable merge / merge sort.
//
//   K1  k_cross_ranks   rows a1/a2: one thread per block start, rank_low of
//                       A[x_i] in B / rank_high of B[y_j] in A  (L304-309)
//   --  stream order (or PDL griddepcontrol.wait) = the single
//       synchronisation of L373-375 (row a3)
//   K2  k_tasks         rows a4-a7: one CTA per block start (task), O(1)
//                       classification, then copy (a, e) or stable merge
//                       (b, c, d) of the task through a shared-memory tile
//   K3  k_block_sort    row a8: stable sort of one run of NT*VT elements per
//                       CTA (odd-even transposition in registers, then
//                       in-CTA merge-path merges, left run = A)
//   --  k_plan_dump     Steps 1-4 only: the task table for parity tests
//
// All in-kernel indices are 32-bit (the ABI rejects n+m or N > 2^31-1).
#pragma once
#include "sm_device.cuh"

namespace sm {

// ----------------------------------------------------------------- K1
// Rows a1/a2.  A group of G lanes performs one rank search cooperatively:
// each round the G lanes probe G evenly spaced keys of the remaining
// interval and a group ballot picks the sub-interval holding the rank, so a
// search over len keys takes ~log_{G+1}(len) dependent memory rounds instead
// of log_2(len) (the latency chain is what bounds this kernel).
//   HIGH = false: rank_low(x, X)  = #{X[t] <  x}   (L119-123)
//   HIGH = true:  rank_high(x, X) = #{X[t] <= x}   (L124-128)
template <typename K, int G>
__device__ __forceinline__ int group_rank(const K* __restrict__ X, int len, K x, bool high, bool active) {
    const int lane = threadIdx.x & 31;
    const int sub = lane % G;
    const int shift = lane - sub;
    int lo = 0, hi = active ? len : 0;     // rank in [lo, hi]; X[lo, hi) undecided
    while (__any_sync(0xffffffffu, hi > lo)) {
        const int n = hi - lo;
        int pos;
        if (n <= G) pos = lo + sub;                                   // last round: probe all
        else pos = lo + (int)(((long long)(sub + 1) * n) / (G + 1));  // G interior probes
        bool pred = false;
        if (hi > lo && (n > G || sub < n)) {
            const K v = __ldg(X + pos);
            pred = high ? (v <= x) : (v < x);
        }
        const unsigned bal = (__ballot_sync(0xffffffffu, pred) >> shift) & ((1u << G) - 1u);
        const int t = __popc(bal);   // probes passed: a prefix of the group
        if (hi > lo) {
            if (n <= G) {
                lo = lo + t;
                hi = lo;
            } else {
                const int plast = t > 0 ? lo + (int)(((long long)t * n) / (G + 1)) : lo - 1;
                const int pnext = t < G ? lo + (int)(((long long)(t + 1) * n) / (G + 1)) : hi;
                lo = plast + 1;
                hi = pnext;
            }
        }
    }
    return lo;
}

template <typename K, int G>
__global__ void __launch_bounds__(256) k_cross_ranks(const K* __restrict__ A, const K* __restrict__ B, Geom g,
                                                     int* __restrict__ xbar, int* __restrict__ ybar) {
    const int per = g.pA + g.pB + 2;
    const long long item = ((long long)blockIdx.x * blockDim.x + threadIdx.x) / G;
    const bool valid = item < (long long)g.S * per;
    int s = 0, t = 0;
    if (valid) {
        s = (int)(item / per);
        t = (int)(item % per);
    }
    const Seg sg = segment(g, s);
    const K* As = A + sg.aoff;
    const K* Bs = B + sg.boff;
    // Step 1 (t <= pA): xbar_i = rank_low(A[x_i], B), xbar_pA = m, empty block start -> m (R4)
    // Step 2 (t >  pA): ybar_j = rank_high(B[y_j], A), ybar_pB = n
    const bool sideA = t <= g.pA;
    const int idx = sideA ? t : t - g.pA - 1;
    const int plen = sideA ? g.pA : g.pB;
    const int own_len = sideA ? sg.n : sg.m;
    int start = own_len;
    if (valid && idx < plen) start = Blocks(own_len, plen).start(idx);
    const bool search = valid && start < own_len;
    K x = K(0);
    if (search) x = __ldg((sideA ? As : Bs) + start);
    const int r = group_rank<K, G>(sideA ? Bs : As, sideA ? sg.m : sg.n, x, !sideA, search);
    if (valid && (threadIdx.x % G) == 0) {
        const int v = search ? r : (sideA ? sg.m : sg.n);
        if (sideA) xbar[(size_t)s * (g.pA + 1) + idx] = v;
        else ybar[(size_t)s * (g.pB + 1) + idx] = v;
    }
    pdl_launch_dependents();
}

// Decode the task of this CTA (rows a4/a5).
__device__ __forceinline__ Task decode_task(const Geom& g, int task, const int* __restrict__ xbar,
                                            const int* __restrict__ ybar, Seg& sg) {
    const int per = g.pA + g.pB;
    const int s = task / per, t = task % per;
    sg = segment(g, s);
    const Blocks xa(sg.n, g.pA), yb(sg.m, g.pB);
    const int* xs = xbar + (size_t)s * (g.pA + 1);
    const int* ys = ybar + (size_t)s * (g.pB + 1);
    return t < g.pA ? classify_a_side(t, xa, yb, xs, ys) : classify_b_side(t - g.pA, xa, yb, xs, ys);
}

// CTA-wide copy of len elements, U loads in flight per thread (row a6).
template <typename T, int NT, int U>
__device__ __forceinline__ void cta_copy(const T* __restrict__ src, T* __restrict__ dst, int len) {
    for (int base = 0; base < len; base += NT * U) {
        T r[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int idx = base + u * NT + (int)threadIdx.x;
            if (idx < len) r[u] = ld_stream(src + idx);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int idx = base + u * NT + (int)threadIdx.x;
            if (idx < len) st_stream(dst + idx, r[u]);
        }
    }
}

// Merge-path split of diagonal d inside a shared-memory tile holding A at
// [0, la) and B at [la, la+lb): smallest i with A[i] > B[d-1-i] (reading R17:
// advance while A[mid] <= B[d-1-mid], so equal keys go to A).
template <typename K>
__device__ __forceinline__ int tile_split(const K* sk, int la, int lb, int d) {
    int lo = max(0, d - lb), hi = min(d, la);
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (sk[mid] <= sk[la + d - 1 - mid]) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

// Serial stable merge of VT outputs from the tile, starting at (ai, bi);
// A occupies [.., aend), B [.., bend) of the same tile; ties take A.
template <typename K, int VT>
__device__ __forceinline__ void serial_merge(const K* sk, int ai, int aend, int bi, int bend, K (&out)[VT],
                                             int (&src)[VT]) {
    K ka = sk[0], kb = sk[0];
    if (ai < aend) ka = sk[ai];
    if (bi < bend) kb = sk[bi];
#pragma unroll
    for (int k = 0; k < VT; ++k) {
        const bool takeA = (bi >= bend) || (ai < aend && ka <= kb);
        out[k] = takeA ? ka : kb;
        src[k] = takeA ? ai : bi;
        if (takeA) {
            ++ai;
            if (ai < aend) ka = sk[ai];
        } else {
            ++bi;
            if (bi < bend) kb = sk[bi];
        }
    }
}

// ----------------------------------------------------------------- K2
// Shared-memory tile used by K3 (block sort).
template <typename K, bool HAS_V, int NT, int VT>
struct TileSmem {
    static constexpr int NV = NT * VT;
    K keys[NV];
    uint32_t vals[HAS_V ? NV : 1];
};

// Merge-path split of diagonal d between sorted a[0,la) and b[0,lb):
// smallest i with a[i] > b[d-1-i] (reading R17: advance while
// a[mid] <= b[d-1-mid], so equal keys go to A).
template <typename K>
__device__ __forceinline__ int split_ab(const K* a, int la, const K* b, int lb, int d) {
    int lo = max(0, d - lb), hi = min(d, la);
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (a[mid] <= b[d - 1 - mid]) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

// Serial stable merge of VT outputs from (ai, bi), la >= 1 and lb >= 1;
// ties take A.  src[k] = smem payload index of output k (va + ai or vb + bi).
template <typename K, int VT, bool IDX>
__device__ __forceinline__ void merge_serial(const K* a, int ai, int la, const K* b, int bi, int lb, int va, int vb,
                                             K (&out)[VT], int (&src)[VT]) {
    K ka = a[min(ai, la - 1)];
    K kb = b[min(bi, lb - 1)];
#pragma unroll
    for (int k = 0; k < VT; ++k) {
        const bool takeA = (bi >= lb) || (ai < la && ka <= kb);
        out[k] = takeA ? ka : kb;
        if (IDX) src[k] = takeA ? va + ai : vb + bi;
        if (takeA) {
            ++ai;
            ka = a[min(ai, la - 1)];
        } else {
            ++bi;
            kb = b[min(bi, lb - 1)];
        }
    }
}

// Task descriptor handed from the producer warp to the consumers (smem).
struct TaskDesc {
    int la, lb;        // lengths of the A and B ranges
    int a_s, b_s;      // smem element index of A[a0] / B[b0] in the key region
    int va_s, vb_s;    // smem element index of the payloads in the payload region
    int off;           // global output element index (segment base + a0 + b0)
    int pad;
};

template <typename K, bool HAS_V, int NC, int VT, int STAGES>
struct K2Layout {
    static constexpr int NV = NC * VT;                    // tile capacity (max task)
    static constexpr int KPAD = 16 / (int)sizeof(K);      // elements per 16 bytes
    static constexpr int KCAP = ((NV + 4 * KPAD + KPAD - 1) / KPAD) * KPAD;
    static constexpr int VCAP = HAS_V ? ((NV + 16 + 3) / 4) * 4 : 0;
    static constexpr int STAGE_BYTES = KCAP * (int)sizeof(K) + VCAP * 4;
    static constexpr int SMEM = STAGES * STAGE_BYTES + STAGES * (int)sizeof(TaskDesc) + 2 * STAGES * 8 + 16;
};

// The 16-byte-aligned superset [g0, g0 + bytes) of src[0, len), to be
// bulk-loaded at smem byte offset `at`; `idx` = smem element index of src[0].
struct Span {
    uintptr_t g0;
    uint32_t bytes;
    int at, idx;
};

template <typename T>
__device__ __forceinline__ Span plan_range(int& at, const T* src, int len) {
    Span sp;
    const uintptr_t g = (uintptr_t)src;
    sp.g0 = g & ~(uintptr_t)15;
    sp.bytes = len > 0 ? (uint32_t)(((g + (uintptr_t)len * sizeof(T) + 15) & ~(uintptr_t)15) - sp.g0) : 0u;
    sp.at = at;
    sp.idx = (at + (int)(g - sp.g0)) / (int)sizeof(T);
    at += (int)sp.bytes;
    return sp;
}

__device__ __forceinline__ void issue_range(char* base, const Span& sp, uint64_t* bar) {
    if (sp.bytes) bulk_g2s(base + sp.at, (const void*)sp.g0, sp.bytes, bar);
}

// Store smem sbuf[ph, ph+L) (already in output order) to dst[0, L): the
// 16-byte-aligned middle with one bulk copy issued by consumer 0, the
// <= 2*(16/sizeof(T)-1) edge elements with plain stores by consumers
// edge0 .. edge0+5.
template <typename T>
__device__ __forceinline__ void store_range(T* dst, const T* sbuf, int ph, int L, int c, int edge0) {
    const uintptr_t g = (uintptr_t)dst;
    const uintptr_t gl = (g + 15) & ~(uintptr_t)15;
    const uintptr_t gh = (g + (uintptr_t)L * sizeof(T)) & ~(uintptr_t)15;
    int head = (int)((gl - g) / sizeof(T));
    if (head > L) head = L;
    const int tail0 = gh > gl ? (int)((gh - g) / sizeof(T)) : head;
    if (c == 0) {
        if (gh > gl) bulk_s2g((void*)gl, sbuf + ph + head, (uint32_t)(gh - gl));
    } else {
        const int e = c - edge0;
        if (e >= 0 && e < head) dst[e] = sbuf[ph + e];
        else if (e >= head && e - head < L - tail0) dst[tail0 + e - head] = sbuf[ph + tail0 + e - head];
    }
}

// K2 (rows a4-a7): persistent, warp-specialised.  Warp 0 lane 0 is the
// producer: it classifies task t (O(1), L310-340), and bulk-loads the task's
// A and B ranges (keys, payloads) into a STAGES-deep shared-memory ring with
// the TMA engine.  NC consumer threads merge (cases b, c, d) or realign
// (copies, cases a, e) each task and write it back with bulk stores.
template <typename K, bool HAS_V, int NC, int VT, int STAGES>
__global__ void __launch_bounds__(NC + 32) k_tasks(const K* __restrict__ A, const uint32_t* __restrict__ vA,
                                                   const K* __restrict__ B, const uint32_t* __restrict__ vB,
                                                   K* __restrict__ C, uint32_t* __restrict__ vC, Geom g,
                                                   const int* __restrict__ xbar, const int* __restrict__ ybar) {
    using Lay = K2Layout<K, HAS_V, NC, VT, STAGES>;
    extern __shared__ __align__(128) char smem[];
    TaskDesc* desc = (TaskDesc*)(smem + STAGES * Lay::STAGE_BYTES);
    uint64_t* full = (uint64_t*)(desc + STAGES);
    uint64_t* empty = full + STAGES;
    const int ntasks = g.S * (g.pA + g.pB);

    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        fence_barrier_init();
        fence_proxy_async();
    }
    __syncthreads();
    pdl_wait();   // the single synchronisation (L373-375): all ranks visible

    if (threadIdx.x < 32) {
        // ------------------------------------------------------ producer
        // The warp classifies the next 32 tasks of this CTA in parallel (one
        // per lane: the dependent rank loads overlap), then hands them to the
        // ring in order; the lane that owns a task issues its bulk loads.
        const int lane = threadIdx.x;
        for (int base = 0;; base += 32) {
            const int my_task = blockIdx.x + (base + lane) * gridDim.x;
            const bool have = my_task < ntasks;
            if (!__any_sync(0xffffffffu, have)) break;
            TaskDesc d;
            Span sa, sb, sva, svb;
            if (have) {
                Seg sg;
                const Task t = decode_task(g, my_task, xbar, ybar, sg);
                d.la = t.a1 - t.a0;
                d.lb = t.b1 - t.b0;
                d.off = sg.coff + t.a0 + t.b0;
                int at = 0, vat = 0;
                sa = plan_range(at, A + sg.aoff + t.a0, d.la);
                sb = plan_range(at, B + sg.boff + t.b0, d.lb);
                sva.bytes = svb.bytes = 0;
                sva.idx = svb.idx = 0;
                if (HAS_V) {
                    sva = plan_range(vat, vA + sg.aoff + t.a0, d.la);
                    svb = plan_range(vat, vB + sg.boff + t.b0, d.lb);
                }
                d.a_s = sa.idx; d.b_s = sb.idx; d.va_s = sva.idx; d.vb_s = svb.idx; d.pad = 0;
            }
            const unsigned owners = __ballot_sync(0xffffffffu, have);
            const int count = __popc(owners);        // tasks are a prefix of the lanes
            for (int k = 0; k < count; ++k) {
                const int it = base + k;
                const int st = it % STAGES;
                if (it >= STAGES) mbar_wait(&empty[st], ((it / STAGES) - 1) & 1);
                if (lane == k) {
                    char* stage = smem + st * Lay::STAGE_BYTES;
                    char* vstage = stage + Lay::KCAP * (int)sizeof(K);
                    desc[st] = d;   // written before the arrive (release) below
                    mbar_arrive_expect_tx(&full[st], sa.bytes + sb.bytes + sva.bytes + svb.bytes);
                    issue_range(stage, sa, &full[st]);
                    issue_range(stage, sb, &full[st]);
                    if (HAS_V) {
                        issue_range(vstage, sva, &full[st]);
                        issue_range(vstage, svb, &full[st]);
                    }
                }
                __syncwarp();
            }
        }
        return;
    }

    // ---------------------------------------------------------- consumers
    const int c = threadIdx.x - 32;
    int it = 0;
    for (int task = blockIdx.x; task < ntasks; task += gridDim.x, ++it) {
        const int s = it % STAGES;
        mbar_wait(&full[s], (it / STAGES) & 1);
        const TaskDesc d = desc[s];
        K* sk = (K*)(smem + s * Lay::STAGE_BYTES);
        uint32_t* sv = (uint32_t*)(smem + s * Lay::STAGE_BYTES + Lay::KCAP * (int)sizeof(K));
        const int L = d.la + d.lb;
        const int phC = (int)(((uintptr_t)(C + d.off) & 15) / sizeof(K));
        const int phV = HAS_V ? (int)(((uintptr_t)(vC + d.off) & 15) / 4) : 0;

        if (d.la > 0 && d.lb > 0) {
            // cases (b), (c), (d): stable merge (row a7).  Only threads whose
            // diagonal lies inside the task work (tasks average half a tile).
            const int dg = c * VT;
            const bool active = dg < L;
            K out[VT];
            int src[VT];
            uint32_t v[HAS_V ? VT : 1];
            if (active) {
                const K* a = sk + d.a_s;
                const K* b = sk + d.b_s;
                const int ai = split_ab(a, d.la, b, d.lb, dg);
                merge_serial<K, VT, HAS_V>(a, ai, d.la, b, dg - ai, d.lb, d.va_s, d.vb_s, out, src);
                if (HAS_V) {
#pragma unroll
                    for (int k = 0; k < VT; ++k) v[k] = sv[min(src[k], Lay::VCAP - 1)];
                }
            }
            named_sync(1, NC);
            if (active) {
                if (dg + VT <= L) {
#pragma unroll
                    for (int k = 0; k < VT; ++k) {
                        sk[phC + dg + k] = out[k];
                        if (HAS_V) sv[phV + dg + k] = v[k];
                    }
                } else {
#pragma unroll
                    for (int k = 0; k < VT; ++k) {
                        if (dg + k < L) {
                            sk[phC + dg + k] = out[k];
                            if (HAS_V) sv[phV + dg + k] = v[k];
                        }
                    }
                }
            }
        } else if (L > 0) {
            // cases (a), (e): copy (row a6) -- realign to the output phase
            const int ks = d.la ? d.a_s : d.b_s;
            const int vs = d.la ? d.va_s : d.vb_s;
            const bool mv = ks != phC || (HAS_V && vs != phV);
            if (mv) {
                K r[VT];
                uint32_t rv[HAS_V ? VT : 1];
#pragma unroll
                for (int k = 0; k < VT; ++k) {
                    const int t = k * NC + c;
                    if (t < L) {
                        r[k] = sk[ks + t];
                        if (HAS_V) rv[k] = sv[vs + t];
                    }
                }
                named_sync(1, NC);
#pragma unroll
                for (int k = 0; k < VT; ++k) {
                    const int t = k * NC + c;
                    if (t < L) {
                        sk[phC + t] = r[k];
                        if (HAS_V) sv[phV + t] = rv[k];
                    }
                }
            }
        }
        fence_proxy_async();
        named_sync(1, NC);
        if (L > 0) {
            store_range<K>(C + d.off, sk, phC, L, c, 1);
            if (HAS_V) store_range<uint32_t>(vC + d.off, sv, phV, L, c, 32);
        }
        if (c == 0) {
            bulk_commit();
            bulk_wait_read<1>();                 // task it-1's stores have read their stage
            if (it >= 1) mbar_arrive(&empty[(it - 1) % STAGES]);
        }
    }
    if (c == 0) bulk_wait_read<0>();
}

// ----------------------------------------------------------- plan dump
template <typename K>
__global__ void k_plan_dump(Geom g, const int* __restrict__ xbar, const int* __restrict__ ybar,
                            int64_t* __restrict__ tasks) {
    const int task = blockIdx.x * blockDim.x + threadIdx.x;
    if (task >= g.S * (g.pA + g.pB)) return;
    Seg sg;
    const Task t = decode_task(g, task, xbar, ybar, sg);
    int64_t* row = tasks + (size_t)task * 6;
    row[0] = t.side; row[1] = t.kase; row[2] = t.a0; row[3] = t.a1; row[4] = t.b0; row[5] = t.b1;
}

// ----------------------------------------------------------------- K3
// Stable block sort of runs of NT*VT elements (row a8).  A partial last run
// is padded with the maximum key AFTER the real elements: the sort is stable,
// so padding stays behind every real element and is never stored.
template <typename K>
__device__ __forceinline__ K key_max();
template <> __device__ __forceinline__ uint32_t key_max<uint32_t>() { return 0xFFFFFFFFu; }
template <> __device__ __forceinline__ int32_t key_max<int32_t>() { return 0x7FFFFFFF; }
template <> __device__ __forceinline__ uint64_t key_max<uint64_t>() { return 0xFFFFFFFFFFFFFFFFull; }
template <> __device__ __forceinline__ int64_t key_max<int64_t>() { return 0x7FFFFFFFFFFFFFFFll; }

template <typename K, bool HAS_V, int NT, int VT>
__global__ void __launch_bounds__(NT) k_block_sort(const K* __restrict__ in, const uint32_t* __restrict__ vin,
                                                   K* __restrict__ out, uint32_t* __restrict__ vout, int N) {
    constexpr int NV = NT * VT;
    __shared__ TileSmem<K, HAS_V, NT, VT> sm_;
    const int tid = threadIdx.x;
    const int base = blockIdx.x * NV;
    const int len = min(NV, N - base);

#pragma unroll
    for (int k = 0; k < VT; ++k) {
        const int idx = k * NT + tid;
        sm_.keys[idx] = idx < len ? ld_stream(in + base + idx) : key_max<K>();
        if (HAS_V) sm_.vals[idx] = idx < len ? ld_stream(vin + base + idx) : 0u;
    }
    __syncthreads();

    K k_[VT];
    uint32_t v_[HAS_V ? VT : 1];
#pragma unroll
    for (int k = 0; k < VT; ++k) {
        k_[k] = sm_.keys[tid * VT + k];
        if (HAS_V) v_[k] = sm_.vals[tid * VT + k];
    }
    // odd-even transposition sort; swapping only on strict '>' keeps it stable
#pragma unroll
    for (int pass = 0; pass < VT; ++pass) {
#pragma unroll
        for (int i = pass & 1; i + 1 < VT; i += 2) {
            if (k_[i + 1] < k_[i]) {
                K tk = k_[i]; k_[i] = k_[i + 1]; k_[i + 1] = tk;
                if (HAS_V) { uint32_t tv = v_[i]; v_[i] = v_[i + 1]; v_[i + 1] = tv; }
            }
        }
    }
    // in-CTA merge passes: groups of `coop` threads merge two sorted runs
#pragma unroll 1
    for (int coop = 2; coop <= NT; coop *= 2) {
        __syncthreads();
#pragma unroll
        for (int k = 0; k < VT; ++k) {
            sm_.keys[tid * VT + k] = k_[k];
            if (HAS_V) sm_.vals[tid * VT + k] = v_[k];
        }
        __syncthreads();
        const int run = (coop / 2) * VT;
        const int start = (tid & ~(coop - 1)) * VT;
        const int d = (tid & (coop - 1)) * VT;
        const K* sk = sm_.keys + start;
        const int ai = tile_split(sk, run, run, d);
        int src[VT];
        serial_merge<K, VT>(sk, ai, run, run + (d - ai), 2 * run, k_, src);
        if (HAS_V) {
#pragma unroll
            for (int k = 0; k < VT; ++k) v_[k] = sm_.vals[start + src[k]];
        }
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < VT; ++k) {
        sm_.keys[tid * VT + k] = k_[k];
        if (HAS_V) sm_.vals[tid * VT + k] = v_[k];
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < VT; ++k) {
        const int idx = k * NT + tid;
        if (idx < len) {
            st_stream(out + base + idx, sm_.keys[idx]);
            if (HAS_V) st_stream(vout + base + idx, sm_.vals[idx]);
        }
    }
}

}  // namespace sm
