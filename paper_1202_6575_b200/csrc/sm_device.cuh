// sm_device.cuh -- device primitives of the B200 stable merge (arXiv 1202.6575).
//
// Citations: PAPER.md line numbers.  This file is
// the CUDA side only; it shares nothing with oracle/.
#pragma once
#include <limits>
#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>

namespace sm {
namespace {   // internal linkage: every translation unit keeps its own kernels

// ---------------------------------------------------------------------------
// Row a0: block partition.
//   x_i = i*ceil(len/p)            for i <  r = len mod p
//       = i*floor(len/p) + r       otherwise;      x_p = len
//   block_of(k) = floor(k / ceil(len/p))                 if k < r*ceil(len/p)
//               = floor((k - r*ceil(len/p)) / floor(len/p)) + r   otherwise
//   block_of(len) = p  (reading R3: the virtual block after the last one)
// ---------------------------------------------------------------------------
// I: the index type -- int on the device (calls below 2^31), int64_t for the
// host's coarse partition (merges of >= 2^31 elements, host pipelines).
template <typename I>
struct BlocksT {
    I len, p, q, r;     // q = floor(len/p), r = len mod p
    __host__ __device__ __forceinline__ BlocksT(I len_, I p_) : len(len_), p(p_), q(len_ / p_), r(len_ % p_) {}
    __host__ __device__ __forceinline__ I start(I i) const { return i < r ? i * (q + 1) : i * q + r; }
    __host__ __device__ __forceinline__ I of(I k) const {
        if (k >= len) return p;
        const I big = r * (q + 1);
        return k < big ? k / (q + 1) : (k - big) / q + r;   // q > 0 whenever k >= big and k < len
    }
};
using Blocks = BlocksT<int>;

// ---------------------------------------------------------------------------
// The key order "<=" of PAPER.md L63 ("ordered by a relation <="): natural
// order for integer keys (signed for i32/i64, unsigned for u32/u64, reading
// R16) and IEEE 754 totalOrder for floating-point keys (SURVEY §8(f) row 2:
// -NaN < -inf < ... < -0.0 < +0.0 < ... < +inf < +NaN).  Every key maps
// bijectively and monotonically to an unsigned "order view" U (used by the
// radix block sort and by the floating-point compares): identity for unsigned,
// sign bit flipped for signed, sign bit flipped for non-negative floats and
// all bits flipped for negative ones.
// ---------------------------------------------------------------------------
template <typename K>
struct KeyOrd;
template <> struct KeyOrd<uint32_t> {
    using U = uint32_t;
    static constexpr bool FLOAT = false;
    static constexpr bool PTX = true;    // inline-PTX merge/split steps exist
    __device__ __host__ __forceinline__ static U to(uint32_t x) { return x; }
    __device__ __host__ __forceinline__ static uint32_t from(U u) { return u; }
};
template <> struct KeyOrd<int32_t> {
    using U = uint32_t;
    static constexpr bool FLOAT = false;
    static constexpr bool PTX = true;    // inline-PTX merge/split steps exist
    __device__ __host__ __forceinline__ static U to(int32_t x) { return (U)x ^ 0x80000000u; }
    __device__ __host__ __forceinline__ static int32_t from(U u) { return (int32_t)(u ^ 0x80000000u); }
};
template <> struct KeyOrd<uint64_t> {
    using U = uint64_t;
    static constexpr bool FLOAT = false;
    static constexpr bool PTX = true;    // inline-PTX merge/split steps exist
    __device__ __host__ __forceinline__ static U to(uint64_t x) { return x; }
    __device__ __host__ __forceinline__ static uint64_t from(U u) { return u; }
};
template <> struct KeyOrd<int64_t> {
    using U = uint64_t;
    static constexpr bool FLOAT = false;
    static constexpr bool PTX = true;    // inline-PTX merge/split steps exist
    __device__ __host__ __forceinline__ static U to(int64_t x) { return (U)x ^ 0x8000000000000000ull; }
    __device__ __host__ __forceinline__ static int64_t from(U u) { return (int64_t)(u ^ 0x8000000000000000ull); }
};
template <> struct KeyOrd<float> {
    using U = uint32_t;
    static constexpr bool FLOAT = true;
    static constexpr bool PTX = false;
    __device__ __host__ __forceinline__ static U to(float x) {
        U b;
        memcpy(&b, &x, 4);
        return b ^ ((U)((int32_t)b >> 31) | 0x80000000u);
    }
    __device__ __host__ __forceinline__ static float from(U u) {
        const U b = u ^ ((U)((int32_t)~u >> 31) | 0x80000000u);
        float x;
        memcpy(&x, &b, 4);
        return x;
    }
};
template <> struct KeyOrd<double> {
    using U = uint64_t;
    static constexpr bool FLOAT = true;
    static constexpr bool PTX = false;
    __device__ __host__ __forceinline__ static U to(double x) {
        U b;
        memcpy(&b, &x, 8);
        return b ^ ((U)((int64_t)b >> 63) | 0x8000000000000000ull);
    }
    __device__ __host__ __forceinline__ static double from(U u) {
        const U b = u ^ ((U)((int64_t)~u >> 63) | 0x8000000000000000ull);
        double x;
        memcpy(&x, &b, 8);
        return x;
    }
};
// Unsigned 128-bit keys (128-bit keys, (key, tie)
// tuples = (high, low) words in lexicographic order): native compares, no
// PTX fast path (the C++ merge over the order view, which is the identity).
typedef unsigned __int128 u128;
template <> struct KeyOrd<u128> {
    using U = u128;
    static constexpr bool FLOAT = false;
    static constexpr bool PTX = false;
    __device__ __host__ __forceinline__ static U to(u128 x) { return x; }
    __device__ __host__ __forceinline__ static u128 from(U u) { return u; }
};

// Descending order: the method for an arbitrary
// total order "<=" instantiated with the reversed one.  Desc<B>
// is a distinct key type with B's bits and the complemented order view, so
// every kernel template runs unchanged on it (ties still go to A).
template <typename B>
struct Desc {
    B v;
    Desc() = default;
    __device__ __host__ __forceinline__ constexpr explicit Desc(B x) : v(x) {}
};
template <typename B> struct KeyOrd<Desc<B>> {
    using U = typename KeyOrd<B>::U;
    static constexpr bool FLOAT = KeyOrd<B>::FLOAT;
    static constexpr bool PTX = KeyOrd<B>::PTX;
    __device__ __host__ __forceinline__ static U to(Desc<B> x) { return (U)~KeyOrd<B>::to(x.v); }
    __device__ __host__ __forceinline__ static Desc<B> from(U u) { return Desc<B>(KeyOrd<B>::from((U)~u)); }
};
template <typename K> struct IsDesc { static constexpr bool value = false; };
template <typename B> struct IsDesc<Desc<B>> { static constexpr bool value = true; };

// a <= b and a < b in the key order (native compares for integer keys)
template <typename K>
__device__ __host__ __forceinline__ bool key_le(K a, K b) {
    if constexpr (KeyOrd<K>::FLOAT || IsDesc<K>::value) return KeyOrd<K>::to(a) <= KeyOrd<K>::to(b);
    else return a <= b;
}
template <typename K>
__device__ __host__ __forceinline__ bool key_lt(K a, K b) {
    if constexpr (KeyOrd<K>::FLOAT || IsDesc<K>::value) return KeyOrd<K>::to(a) < KeyOrd<K>::to(b);
    else return a < b;
}

// A floating-point key held in registers as its totalOrder integer view I
// (int32_t / int64_t) by the PTX merge path; FViewOf maps float / double
// (and their Desc) to it.
template <typename I>
struct FView {
    I v;
};
template <typename K> struct FViewOf { using type = K; };
template <> struct FViewOf<float> { using type = FView<int32_t>; };
template <> struct FViewOf<double> { using type = FView<int64_t>; };
template <typename B> struct FViewOf<Desc<B>> { using type = Desc<typename FViewOf<B>::type>; };

// The bits of a key as an integer (for inline PTX operands).
template <typename K>
__device__ __forceinline__ K& raw_ref(K& k) { return k; }
template <typename I>
__device__ __forceinline__ I& raw_ref(FView<I>& k) { return k.v; }
template <typename B>
__device__ __forceinline__ auto& raw_ref(Desc<B>& k) { return raw_ref(k.v); }

// A merged key back from the PTX path's register form (floats: the view's
// involution, then the float bits).
template <typename K, typename V>
__device__ __forceinline__ K from_reg(V x) {
    if constexpr (sizeof(K) == sizeof(V) && !KeyOrd<K>::FLOAT) {
        return *reinterpret_cast<K*>(&x);
    } else {
        auto b = raw_ref(x);
        using I = decltype(b);
        b ^= (b >> (8 * sizeof(I) - 1)) & std::numeric_limits<I>::max();
        K k;
        memcpy(&k, &b, sizeof(K));
        return k;
    }
}

// Read-only global load of a key (u128: one 16-byte load; 16-byte aligned).
template <typename K>
__device__ __forceinline__ K ldg_key(const K* p) { return __ldg(p); }
__device__ __forceinline__ u128 ldg_key(const u128* p) {
    const ulonglong2 v = __ldg((const ulonglong2*)p);
    return ((u128)v.y << 64) | (u128)v.x;
}
template <typename B>
__device__ __forceinline__ Desc<B> ldg_key(const Desc<B>* p) { return Desc<B>(ldg_key((const B*)p)); }

// ---------------------------------------------------------------------------
// Geometry of one launch: one merge (mode 0, S = 1), one merge-sort round
// over S equal run pairs of a single array (mode 1; §3:
// "modifying the merge algorithm to work in parallel on the pairs"), or a
// batch of S independent merges of any lengths (mode 2, SURVEY §8(f) row 1:
// the same machinery exposed to callers, one segment table entry each).
// Segment s of a sort round: A = runs [2sL, 2sL+L), B = [2sL+L, 2sL+2L),
// clipped to N; the left run plays A so ties keep input order.  A pair whose
// B is empty (odd trailing run) degenerates to case-(a) copies (L409-410).
// Ranks: modes 0/1 keep xbar[s*(pA+1)..] and ybar[s*(pB+1)..]; mode 2 keeps
// one array, segment s at rbase: xbar (pA+1 entries) then ybar (pB+1).
// ---------------------------------------------------------------------------
struct SegInfo {          // mode-2 segment table entry (built by k_batch_*)
    int aoff, n, boff, m, coff;
    int pA, pB;           // block counts of this segment
    int tbase, rbase;     // first task / first rank entry of this segment
};

struct Geom {
    int S;                // segments
    int pA, pB;           // block counts per segment (modes 0, 1)
    int n, m;             // plain merge sizes (mode 0)
    int L, N;             // sort round: run length, total length (mode 1)
    int sort;             // mode: 0 merge, 1 sort round, 2 batch, 3 merge-path comparison
    int T;                // mode 2: block size
    const SegInfo* segs;  // mode 2: segment table [S]
    const int* totals;    // mode 2: [0] = tasks, [1] = rank entries
    const int* task_seg;  // mode 2: segment of every task
    const int* rank_seg;  // mode 2: segment of every rank entry
    const int4* tdesc;    // modes 1, 2: tasks classified ahead by k_classify (or null)
    uint32_t* cover;      // SM_DEBUG builds: K2 counts every output element it stores here (or null)
    int fuse;             // mode 0, few tasks per CTA: K2 computes the ranks of its own tasks (no K1 launch)
    int* ctr;             // K2's task counter (dynamic assignment): zeroed by the kernel launched before K2
    unsigned long long* ts;   // SM_K2_TSTAMP builds: per-CTA event times of K2 (or null)
};

// The kernel launched right before K2 (K1, k_classify, k_diag_splits) zeroes
// K2's task counter, after its own griddepcontrol.wait: the counter lives in
// the call's scratch, which a previous call's K2 may have used.
__device__ __forceinline__ void zero_task_counter(int* ctr) {
    if (ctr && blockIdx.x == 0 && threadIdx.x == 0) *ctr = 0;
}

// SM_DEBUG builds: device-side checks of the disjoint-write invariant of the
// paper's tasks: every store of K2 falls inside its
// task's range [off, off + L) and inside C, and (sm_debug_cover) every
// output element is stored exactly once; K3 / K3H stores stay in their run.
#ifdef SM_DEBUG
#define SM_DCHECK(cond, what)                                                                        \
    do {                                                                                             \
        if (!(cond)) {                                                                               \
            printf("SM_DEBUG check failed: %s (block %d thread %d)\n", what, blockIdx.x, threadIdx.x); \
            __trap();                                                                                \
        }                                                                                            \
    } while (0)
#else
#define SM_DCHECK(cond, what) do {} while (0)
#endif

// One segment, located: its ranges, block counts and rank arrays.
struct Seg {
    int aoff, n, boff, m, coff;
    int pA, pB;
    int* xs;              // xbar of the segment (pA+1 entries)
    int* ys;              // ybar of the segment (pB+1 entries)
};

__device__ __forceinline__ Seg segment(const Geom& g, int s, int* xbar, int* ybar) {
    Seg r;
    if (g.sort == 2) {
        const SegInfo e = g.segs[s];
        r.aoff = e.aoff; r.n = e.n; r.boff = e.boff; r.m = e.m; r.coff = e.coff; r.pA = e.pA; r.pB = e.pB;
        r.xs = xbar + e.rbase;
        r.ys = xbar + e.rbase + e.pA + 1;
        return r;
    }
    r.pA = g.pA; r.pB = g.pB;
    r.xs = xbar + (size_t)s * (g.pA + 1);
    r.ys = ybar + (size_t)s * (g.pB + 1);
    if (g.sort == 0 || g.sort == 3) {
        r.aoff = 0; r.n = g.n; r.boff = 0; r.m = g.m; r.coff = 0;
    } else {
        r.aoff = s * 2 * g.L;                       // < N < 2^31 for s < S
        r.n = min(g.L, g.N - r.aoff);
        r.boff = r.aoff + r.n;
        r.m = max(0, min(g.L, g.N - r.boff));
        r.coff = r.aoff;
    }
    return r;
}

// Number of tasks / rank entries of the launch (mode 2: from the device).
__device__ __forceinline__ int total_tasks(const Geom& g) {
    if (g.sort == 3) return (g.n + g.m + g.T - 1) / g.T;   // equal output tiles of T
    return g.sort == 2 ? g.totals[0] : g.S * (g.pA + g.pB);
}
__device__ __forceinline__ int total_rank_items(const Geom& g) {
    return g.sort == 2 ? g.totals[1] : g.S * (g.pA + g.pB + 2);
}

// Segment of global task (ranks = false) or rank entry (ranks = true) idx,
// and the index local to that segment (mode 2: O(1) through the maps).
__device__ __forceinline__ int locate(const Geom& g, int idx, bool ranks, int& local) {
    if (g.sort != 2) {
        const int per = g.pA + g.pB + (ranks ? 2 : 0);
        local = idx % per;
        return idx / per;
    }
    const int sg = ranks ? __ldg(&g.rank_seg[idx]) : __ldg(&g.task_seg[idx]);
    local = idx - (ranks ? __ldg(&g.segs[sg].rbase) : __ldg(&g.segs[sg].tbase));
    return sg;
}

// ---------------------------------------------------------------------------
// Rows a4/a5: classification of the PE at x_i (Step 3, L310-336) and at y_j
// (Step 4, L337-340).  Cases tested in the order (a), (e), (b), (d), (c)
// (reading R8); (d) takes A up to x_{i+1} (reading R1, the text's "x_{j+1}"
// is a typo).  Output offset is always a0 + b0 (x_i + xbar_i, y_j + ybar_j).
// ---------------------------------------------------------------------------
enum { CASE_A = 0, CASE_B = 1, CASE_C = 2, CASE_D = 3, CASE_E = 4 };

template <typename I>
struct TaskT {
    int side, kase;
    I a0, a1, b0, b1;
};
using Task = TaskT<int>;

// XR / YR: the rank arrays x̄, ȳ -- plain pointers, or (small merges in one
// launch) a view of the entries a CTA computed itself (LocalView).
// One implementation for the device (K2, k_classify, the small-merge
// prologue) and the host (the coarse plans of sm_plan_tasks / the pipelines).
template <typename I, typename XR, typename YR>
__host__ __device__ __forceinline__ TaskT<I> classify_a_side(I i, const BlocksT<I>& xa, const BlocksT<I>& yb,
                                                             const XR& xbar, const YR& ybar) {
    TaskT<I> t;
    t.side = 0;
    const I xi = xa.start(i), xi1 = xa.start(i + 1);
    const I xb0 = xbar[i], xb1 = xbar[i + 1];
    if (xb0 == xb1) {                                         // (a) copy A[x_i, x_{i+1})
        t.kase = CASE_A; t.a0 = xi; t.a1 = xi1; t.b0 = t.b1 = xb0; return t;
    }
    const I j = yb.of(xb0);
    const I yj = yb.start(j);
    if (xb0 == yj) {                                          // (e) copy A[x_i, ybar_j)
        t.kase = CASE_E; t.a0 = xi; t.a1 = ybar[j]; t.b0 = t.b1 = xb0; return t;
    }
    if (yb.of(xb1) == j) {                                    // (b) A block with B[xbar_i, xbar_{i+1})
        t.kase = CASE_B; t.a0 = xi; t.a1 = xi1; t.b0 = xb0; t.b1 = xb1; return t;
    }
    const I yj1 = yb.start(j + 1);
    if (xb1 == yj1) {                                         // (d) A block with B[xbar_i, y_{j+1})
        t.kase = CASE_D; t.a0 = xi; t.a1 = xi1; t.b0 = xb0; t.b1 = yj1; return t;
    }
    t.kase = CASE_C;                                          // (c) A[x_i, ybar_{j+1}) with B[xbar_i, y_{j+1})
    t.a0 = xi; t.a1 = ybar[j + 1]; t.b0 = xb0; t.b1 = yj1;
    return t;
}

template <typename I, typename XR, typename YR>
__host__ __device__ __forceinline__ TaskT<I> classify_b_side(I j, const BlocksT<I>& xa, const BlocksT<I>& yb,
                                                             const XR& xbar, const YR& ybar) {
    TaskT<I> t;
    t.side = 1;
    const I yj = yb.start(j), yj1 = yb.start(j + 1);
    const I yb0 = ybar[j], yb1 = ybar[j + 1];
    if (yb0 == yb1) {                                         // (a) copy B[y_j, y_{j+1})
        t.kase = CASE_A; t.b0 = yj; t.b1 = yj1; t.a0 = t.a1 = yb0; return t;
    }
    const I i = xa.of(yb0);
    const I xi = xa.start(i);
    if (yb0 == xi) {                                          // (e) copy B[y_j, xbar_i)
        t.kase = CASE_E; t.b0 = yj; t.b1 = xbar[i]; t.a0 = t.a1 = yb0; return t;
    }
    if (xa.of(yb1) == i) {                                    // (b) B block with A[ybar_j, ybar_{j+1})
        t.kase = CASE_B; t.b0 = yj; t.b1 = yj1; t.a0 = yb0; t.a1 = yb1; return t;
    }
    const I xi1 = xa.start(i + 1);
    if (yb1 == xi1) {                                         // (d) B block with A[ybar_j, x_{i+1})
        t.kase = CASE_D; t.b0 = yj; t.b1 = yj1; t.a0 = yb0; t.a1 = xi1; return t;
    }
    t.kase = CASE_C;                                          // (c) B[y_j, xbar_{i+1}) with A[ybar_j, x_{i+1})
    t.b0 = yj; t.b1 = xbar[i + 1]; t.a0 = yb0; t.a1 = xi1;
    return t;
}

// ---------------------------------------------------------------------------
// Streaming cache hints: inputs are read once, outputs written once.
// ---------------------------------------------------------------------------
template <typename T>
__device__ __forceinline__ T ld_stream(const T* p) { return __ldcs(p); }
template <typename T>
__device__ __forceinline__ void st_stream(T* p, T v) { __stcs(p, v); }
__device__ __forceinline__ u128 ld_stream(const u128* p) {
    const ulonglong2 v = __ldcs((const ulonglong2*)p);
    return ((u128)v.y << 64) | (u128)v.x;
}
__device__ __forceinline__ void st_stream(u128* p, u128 v) {
    __stcs((ulonglong2*)p, make_ulonglong2((unsigned long long)v, (unsigned long long)(v >> 64)));
}
template <typename B>
__device__ __forceinline__ Desc<B> ld_stream(const Desc<B>* p) { return Desc<B>(ld_stream((const B*)p)); }
template <typename B>
__device__ __forceinline__ void st_stream(Desc<B>* p, Desc<B> v) { st_stream((B*)p, v.v); }

// Programmatic dependent launch (sm_90+): wait for the producer grid's
// memory to be visible; a no-op when the launch was not programmatic.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;"); }

}  // namespace
}  // namespace sm

// ===========================================================================
// sm_90+/sm_100a asynchronous-copy primitives (inline PTX): mbarrier, 1-D
// bulk copies (TMA engine, cp.async.bulk), async-proxy fence, named barriers.
// ===========================================================================
namespace sm {
namespace {   // internal linkage: every translation unit keeps its own kernels

__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void fence_barrier_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "LAB_WAIT:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@P1 bra DONE;\n\t"
        "bra LAB_WAIT;\n"
        "DONE:\n\t}" ::"r"(smem_addr(bar)),
        "r"(parity)
        : "memory");
}

// The same for warps that are often idle (storer, producer): the suspend-time
// hint lets the hardware park the warp until the phase completes instead of
// re-polling every few hundred cycles (the polls took ~6% of issue slots).
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "LAB_WAIT:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n\t"
        "@P1 bra DONE;\n\t"
        "bra LAB_WAIT;\n"
        "DONE:\n\t}" ::"r"(smem_addr(bar)),
        "r"(parity), "r"(1000000u)
        : "memory");
}

// global -> shared bulk copy; completion counted on `bar` (bytes % 16 == 0,
// both addresses 16-byte aligned)
__device__ __forceinline__ void bulk_g2s(void* dst_smem, const void* src_gmem, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_addr(dst_smem)),
        "l"(src_gmem), "r"(bytes), "r"(smem_addr(bar))
        : "memory");
}

// shared -> global bulk copy in the current bulk group
__device__ __forceinline__ void bulk_s2g(void* dst_gmem, const void* src_smem, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst_gmem),
                 "r"(smem_addr(src_smem)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }

// L2 prefetch of the 16-byte-aligned interior of p[0, len) (a hint: no data
// lands in shared memory, nothing is written)
template <typename T>
__device__ __forceinline__ void prefetch_l2(const T* p, int len) {
    const uintptr_t a = ((uintptr_t)p + 15) & ~(uintptr_t)15, e = ((uintptr_t)(p + len)) & ~(uintptr_t)15;
    if (len > 0 && e > a)
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a), "r"((uint32_t)(e - a)) : "memory");
}

__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

template <int N>
__device__ __forceinline__ void bulk_wait_read() {
    asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}

__device__ __forceinline__ void named_sync(int id, int count) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}

}  // namespace
}  // namespace sm

// ===========================================================================
// Shared-memory merge primitives in inline PTX (rows a7, a8): branch-free,
// predicated, on 32-bit shared-window addresses, one specialisation per key
// type (signed compare for i32/i64, unsigned for u32/u64, reading R16).
// ===========================================================================
namespace sm {
namespace {   // internal linkage: every translation unit keeps its own kernels

// One binary-lifting probe of the merge-path split (reading R17): with
// sa = &a[i0], sb = &b[d-1-i0] and `rem` candidates left, if STEP <= rem and
// a[i0+STEP-1] <= b[d-1-i0-STEP+1] then advance i0 by STEP.
#ifndef SM_SPLIT_SKEW_LEVEL
#define SM_SPLIT_SKEW_LEVEL 32   // deep split levels probed in a per-thread skewed lattice (0: off)
#endif

// One output of the serial stable merge: take A when A is not exhausted and
// (B is exhausted or ka <= kb) -- ties to A.  Advances
// the taken side and loads the key after its new head (two past the end at
// most: the stage holds slack there and the value is never selected).
template <typename K>
__device__ __forceinline__ void merge_step(uint32_t& pa, uint32_t& pb, K& ka, K& kb, K& na, K& nb, uint32_t pae,
                                           uint32_t pbe, K& out);
// Same, also selecting the payload index (ia for A, ib for B).
template <typename K>
__device__ __forceinline__ void merge_step_idx(uint32_t& pa, uint32_t& pb, K& ka, K& kb, K& na, K& nb, uint32_t pae,
                                               uint32_t pbe, K& out, int& ia, int& ib, int& src);

// The same without the exhaustion checks: valid while neither input can run
// out within the thread's outputs (ai + VT <= la and bi + VT <= lb).
template <typename K>
__device__ __forceinline__ void merge_step_fast(uint32_t& pa, uint32_t& pb, K& ka, K& kb, K& na, K& nb, K& out);
template <typename K>
__device__ __forceinline__ void merge_step_idx_fast(uint32_t& pa, uint32_t& pb, K& ka, K& kb, K& na, K& nb, K& out,
                                                    int& ia, int& ib, int& src);

template <typename K>
__device__ __forceinline__ K lds(uint32_t addr);

// NAME: specialisation tag; X_LE_Y / KA_LE_KB: the operand order of the key
// compare ("x, y" / "%2, %3" ascending; reversed for the Desc<> types).
#define SM_DEF_SMEM_OPS(K, NAME, CMP, BITS, RC, SZ, X_LE_Y, KA_LE_KB, XF_XY, XF_K, XF_0, FAST_TAIL)                                \
    template <int STEP>                                                                                        \
    struct LiftProbe_##NAME {                                                                                  \
        /* v: virtual candidates left below the range (see LiftProbeV); a step */                             \
        /* taken here (STEP > v) leaves none */                                                               \
        __device__ __forceinline__ static void run(uint32_t& sa, uint32_t& sb, int& rem, int& v) {             \
            asm volatile(                                                                                      \
                "{\n\t.reg .pred p, q;\n\t.reg .b" BITS " x, y, xt;\n\t"                                          \
                "setp.le.s32 p, %4, %2;\n\t"                                                                   \
                "@p ld.shared.b" BITS " x, [%0+%5];\n\t"                                                       \
                "@p ld.shared.b" BITS " y, [%1+%6];\n\t" XF_XY                                                 \
                "setp.le.and." #CMP " q, " X_LE_Y ", p;\n\t"                                                   \
                "@q add.u32 %0, %0, %7;\n\t"                                                                   \
                "@q sub.u32 %1, %1, %7;\n\t"                                                                   \
                "@q sub.s32 %2, %2, %4;\n\t"                                                                   \
                "@q mov.s32 %3, 0;\n\t}"                                                                       \
                : "+r"(sa), "+r"(sb), "+r"(rem), "+r"(v)                                                       \
                : "n"(STEP), "n"((STEP - 1) * SZ), "n"(-(STEP - 1) * SZ), "n"(STEP * SZ)                     \
                : "memory");                                                                                   \
        }                                                                                                      \
    };                                                                                                         \
    /* The same probe in a lattice shifted down by a per-thread skew: candidates */                       \
    /* below the search range (v > 0 of them left) are "virtual" and pass without */                          \
    /* a load.  Used for the deep levels (STEP <= 32), where the unshifted */                                 \
    /* lattices of neighbouring threads share their residue mod 2*STEP and the */                             \
    /* probes of a warp pile into two or three banks (measured 6-7-way). */                                   \
    template <int STEP>                                                                                        \
    struct LiftProbeV_##NAME {                                                                                 \
        __device__ __forceinline__ static void run(uint32_t& sa, uint32_t& sb, int& rem, int& v) {             \
            asm volatile(                                                                                      \
                "{\n\t.reg .pred p, q, au;\n\t.reg .b" BITS " x, y, xt;\n\t"                                   \
                "setp.le.s32 au, %4, %3;\n\t"                                                                 \
                "setp.le.and.s32 p, %4, %2, !au;\n\t"                                                         \
                "@p ld.shared.b" BITS " x, [%0+%5];\n\t"                                                       \
                "@p ld.shared.b" BITS " y, [%1+%6];\n\t" XF_XY                                                 \
                "setp.le.and." #CMP " q, " X_LE_Y ", p;\n\t"                                                   \
                "or.pred q, q, au;\n\t"                                                                       \
                "@q add.u32 %0, %0, %7;\n\t"                                                                   \
                "@q sub.u32 %1, %1, %7;\n\t"                                                                   \
                "@q sub.s32 %2, %2, %4;\n\t"                                                                   \
                "@q sub.s32 %3, %3, %4;\n\t}"                                                                  \
                : "+r"(sa), "+r"(sb), "+r"(rem), "+r"(v)                                                       \
                : "n"(STEP), "n"((STEP - 1) * SZ), "n"(-(STEP - 1) * SZ), "n"(STEP * SZ)                     \
                : "memory");                                                                                   \
        }                                                                                                      \
    };                                                                                                         \
    template <>                                                                                                \
    __device__ __forceinline__ K lds<K>(uint32_t addr) {                                                       \
        K v;                                                                                                   \
        asm volatile("{\n\t.reg .b" BITS " xt;\n\tld.shared.b" BITS " %0, [%1];\n\t" XF_0 "}"                \
                     : "=" RC(raw_ref(v)) : "r"(addr) : "memory");                                             \
        return v;                                                                                              \
    }                                                                                                          \
    template <>                                                                                                \
    __device__ __forceinline__ void merge_step<K>(uint32_t & pa, uint32_t & pb, K & ka, K & kb, K & na, K & nb,\
                                                  uint32_t pae, uint32_t pbe, K & out) {                       \
        /* ka/kb: current heads, na/nb: the elements after them (loaded a */                                  \
        /* step ahead, so the load latency is off the compare chain); one */                                 \
        /* shared load per step, from the side just taken */                                                  \
        asm volatile(                                                                                          \
            "{\n\t.reg .pred t, u, w;\n\t.reg .b32 ad;\n\t.reg .b" BITS " k, xt;\n\t"                             \
            "setp.lt.u32 u, %0, %7;\n\t"                                                                       \
            "setp.ge.u32 w, %1, %8;\n\t"                                                                       \
            "setp.le.and." #CMP " t, " KA_LE_KB ", u;\n\t"                                                    \
            "or.pred t, t, w;\n\t"                                                                             \
            "selp.b" BITS " %6, %2, %3, t;\n\t"                                                                \
            "selp.b" BITS " %2, %4, %2, t;\n\t"                                                                \
            "selp.b" BITS " %3, %3, %5, t;\n\t"                                                                \
            "@t add.u32 %0, %0, " #SZ ";\n\t"                                                                  \
            "@!t add.u32 %1, %1, " #SZ ";\n\t"                                                                 \
            "selp.b32 ad, %0, %1, t;\n\t"                                                                      \
            "ld.shared.b" BITS " k, [ad+" #SZ "];\n\t" XF_K                                                         \
            "selp.b" BITS " %4, k, %4, t;\n\t"                                                                 \
            "selp.b" BITS " %5, %5, k, t;\n\t}"                                                                \
            : "+r"(pa), "+r"(pb), "+" RC(raw_ref(ka)), "+" RC(raw_ref(kb)), "+" RC(raw_ref(na)),              \
              "+" RC(raw_ref(nb)), "=" RC(raw_ref(out))                                                        \
            : "r"(pae), "r"(pbe)                                                                               \
            : "memory");                                                                                       \
    }                                                                                                          \
    template <>                                                                                                \
    __device__ __forceinline__ void merge_step_idx<K>(uint32_t & pa, uint32_t & pb, K & ka, K & kb, K & na,    \
                                                      K & nb, uint32_t pae, uint32_t pbe, K & out, int& ia,    \
                                                      int& ib, int& src) {                                     \
        asm volatile(                                                                                          \
            "{\n\t.reg .pred t, u, w;\n\t.reg .b32 ad;\n\t.reg .b" BITS " k, xt;\n\t"                             \
            "setp.lt.u32 u, %0, %10;\n\t"                                                                      \
            "setp.ge.u32 w, %1, %11;\n\t"                                                                      \
            "setp.le.and." #CMP " t, " KA_LE_KB ", u;\n\t"                                                    \
            "or.pred t, t, w;\n\t"                                                                             \
            "selp.b" BITS " %6, %2, %3, t;\n\t"                                                                \
            "selp.b32 %9, %7, %8, t;\n\t"                                                                      \
            "selp.b" BITS " %2, %4, %2, t;\n\t"                                                                \
            "selp.b" BITS " %3, %3, %5, t;\n\t"                                                                \
            "@t add.u32 %0, %0, " #SZ ";\n\t"                                                                  \
            "@!t add.u32 %1, %1, " #SZ ";\n\t"                                                                 \
            "@t add.s32 %7, %7, 1;\n\t"                                                                        \
            "@!t add.s32 %8, %8, 1;\n\t"                                                                       \
            "selp.b32 ad, %0, %1, t;\n\t"                                                                      \
            "ld.shared.b" BITS " k, [ad+" #SZ "];\n\t" XF_K                                                         \
            "selp.b" BITS " %4, k, %4, t;\n\t"                                                                 \
            "selp.b" BITS " %5, %5, k, t;\n\t}"                                                                \
            : "+r"(pa), "+r"(pb), "+" RC(raw_ref(ka)), "+" RC(raw_ref(kb)), "+" RC(raw_ref(na)),              \
              "+" RC(raw_ref(nb)), "=" RC(raw_ref(out)), "+r"(ia), "+r"(ib), "=r"(src)                         \
            : "r"(pae), "r"(pbe)                                                                               \
            : "memory");                                                                                       \
    }                                                                                                          \
    template <>                                                                                                \
    __device__ __forceinline__ void merge_step_fast<K>(uint32_t & pa, uint32_t & pb, K & ka, K & kb, K & na,   \
                                                       K & nb, K & out) {                                      \
        asm volatile(                                                                                          \
            "{\n\t.reg .pred t;\n\t.reg .b32 ad;\n\t.reg .b" BITS " k, xt;\n\t"                                  \
            "setp.le." #CMP " t, " KA_LE_KB ";\n\t"                                                            \
            "selp.b" BITS " %6, %2, %3, t;\n\t"                                                                \
            "selp.b" BITS " %2, %4, %2, t;\n\t"                                                                \
            "selp.b" BITS " %3, %3, %5, t;\n\t"                                                                \
            "@t add.u32 %0, %0, " #SZ ";\n\t"                                                                  \
            "@!t add.u32 %1, %1, " #SZ ";\n\t"                                                                 \
            FAST_TAIL "}"                                                                                      \
            : "+r"(pa), "+r"(pb), "+" RC(raw_ref(ka)), "+" RC(raw_ref(kb)), "+" RC(raw_ref(na)),              \
              "+" RC(raw_ref(nb)), "=" RC(raw_ref(out))                                                        \
            :                                                                                                  \
            : "memory");                                                                                       \
    }                                                                                                          \
    template <>                                                                                                \
    __device__ __forceinline__ void merge_step_idx_fast<K>(uint32_t & pa, uint32_t & pb, K & ka, K & kb,       \
                                                           K & na, K & nb, K & out, int& ia, int& ib,          \
                                                           int& src) {                                         \
        asm volatile(                                                                                          \
            "{\n\t.reg .pred t;\n\t.reg .b32 ad;\n\t.reg .b" BITS " k, xt;\n\t"                                  \
            "setp.le." #CMP " t, " KA_LE_KB ";\n\t"                                                            \
            "selp.b" BITS " %6, %2, %3, t;\n\t"                                                                \
            "selp.b32 %9, %7, %8, t;\n\t"                                                                      \
            "selp.b" BITS " %2, %4, %2, t;\n\t"                                                                \
            "selp.b" BITS " %3, %3, %5, t;\n\t"                                                                \
            "@t add.u32 %0, %0, " #SZ ";\n\t"                                                                  \
            "@!t add.u32 %1, %1, " #SZ ";\n\t"                                                                 \
            "@t add.s32 %7, %7, 1;\n\t"                                                                        \
            "@!t add.s32 %8, %8, 1;\n\t"                                                                       \
            FAST_TAIL "}"                                                                                      \
            : "+r"(pa), "+r"(pb), "+" RC(raw_ref(ka)), "+" RC(raw_ref(kb)), "+" RC(raw_ref(na)),              \
              "+" RC(raw_ref(nb)), "=" RC(raw_ref(out)), "+r"(ia), "+r"(ib), "=r"(src)                         \
            :                                                                                                  \
            : "memory");                                                                                       \
    }                                                                                                          \
    template <int STEP>                                                                                        \
    struct LiftSel<K, STEP> {                                                                                  \
        using type = LiftProbe_##NAME<STEP>;                                                                   \
        using vtype = LiftProbeV_##NAME<STEP>;                                                                 \
    };

template <typename K, int STEP>
struct LiftSel;

// The end of a fast merge step (pa / pb already advanced): integer keys
// load the next key of the side taken straight into na / nb (predicated, so
// nothing in the step waits for the load); floating-point keys load into a
// temporary, map it to the order view and select (measured: predicating the
// view as well is slower).
#define SM_TAIL_PLD(BITS, SZ) "@t ld.shared.b" BITS " %4, [%0+" #SZ "];\n\t@!t ld.shared.b" BITS " %5, [%1+" #SZ "];\n\t"
#define SM_TAIL_SEL(BITS, SZ, XF) "selp.b32 ad, %0, %1, t;\n\tld.shared.b" BITS " k, [ad+" #SZ "];\n\t" XF \
    "selp.b" BITS " %4, k, %4, t;\n\tselp.b" BITS " %5, %5, k, t;\n\t"
// The fast step's load: one load from the selected side (SEL) or two
// predicated loads, one per side (PLD: off the select's latency, but each
// costs its own shared-memory wavefronts: 4.6 per warp step against 2.9 for
// SEL on 4-byte keys, ncu r2).  SM_FAST_PLD32 / SM_FAST_PLD64 pick PLD.
#ifndef SM_FAST_PLD32
#define SM_FAST_PLD32 0
#endif
#ifndef SM_FAST_PLD64
#define SM_FAST_PLD64 1
#endif
#if SM_FAST_PLD32
#define SM_TAIL32 SM_TAIL_PLD("32", 4)
#else
#define SM_TAIL32 SM_TAIL_SEL("32", 4, "")
#endif
#if SM_FAST_PLD64
#define SM_TAIL64 SM_TAIL_PLD("64", 8)
#else
#define SM_TAIL64 SM_TAIL_SEL("64", 8, "")
#endif
SM_DEF_SMEM_OPS(uint32_t, u32, u32, "32", "r", 4, "x, y", "%2, %3", "", "", "", SM_TAIL32)
SM_DEF_SMEM_OPS(int32_t, s32, s32, "32", "r", 4, "x, y", "%2, %3", "", "", "", SM_TAIL32)
SM_DEF_SMEM_OPS(uint64_t, u64, u64, "64", "l", 8, "x, y", "%2, %3", "", "", "", SM_TAIL64)
SM_DEF_SMEM_OPS(int64_t, s64, s64, "64", "l", 8, "x, y", "%2, %3", "", "", "", SM_TAIL64)
SM_DEF_SMEM_OPS(Desc<uint32_t>, du32, u32, "32", "r", 4, "y, x", "%3, %2", "", "", "", SM_TAIL32)
SM_DEF_SMEM_OPS(Desc<int32_t>, ds32, s32, "32", "r", 4, "y, x", "%3, %2", "", "", "", SM_TAIL32)
SM_DEF_SMEM_OPS(Desc<uint64_t>, du64, u64, "64", "l", 8, "y, x", "%3, %2", "", "", "", SM_TAIL64)
SM_DEF_SMEM_OPS(Desc<int64_t>, ds64, s64, "64", "l", 8, "y, x", "%3, %2", "", "", "", SM_TAIL64)
// Floating-point keys: every shared load is followed by the totalOrder view
// (sign-magnitude -> two's complement: flip the magnitude bits of negative
// values, an involution), compared as signed integers; the merged outputs
// are mapped back by the same involution (FView below).
#define SM_XF32(R) "shr.s32 xt, " R ", 31;\n\tand.b32 xt, xt, 0x7fffffff;\n\txor.b32 " R ", " R ", xt;\n\t"
#define SM_XF64(R) "shr.s64 xt, " R ", 63;\n\tand.b64 xt, xt, 0x7fffffffffffffff;\n\txor.b64 " R ", " R ", xt;\n\t"

SM_DEF_SMEM_OPS(FView<int32_t>, fs32, s32, "32", "r", 4, "x, y", "%2, %3", SM_XF32("x") SM_XF32("y"), SM_XF32("k"),
                SM_XF32("%0"), SM_TAIL_SEL("32", 4, SM_XF32("k")))
SM_DEF_SMEM_OPS(FView<int64_t>, fs64, s64, "64", "l", 8, "x, y", "%2, %3", SM_XF64("x") SM_XF64("y"), SM_XF64("k"),
                SM_XF64("%0"), SM_TAIL_SEL("64", 8, SM_XF64("k")))
SM_DEF_SMEM_OPS(Desc<FView<int32_t>>, dfs32, s32, "32", "r", 4, "y, x", "%3, %2", SM_XF32("x") SM_XF32("y"),
                SM_XF32("k"), SM_XF32("%0"), SM_TAIL_SEL("32", 4, SM_XF32("k")))
SM_DEF_SMEM_OPS(Desc<FView<int64_t>>, dfs64, s64, "64", "l", 8, "y, x", "%3, %2", SM_XF64("x") SM_XF64("y"),
                SM_XF64("k"), SM_XF64("%0"), SM_TAIL_SEL("64", 8, SM_XF64("k")))
#undef SM_XF32
#undef SM_XF64

#undef SM_DEF_SMEM_OPS
#undef SM_TAIL_PLD
#undef SM_TAIL_SEL
#undef SM_TAIL32
#undef SM_TAIL64

template <typename K, int STEP>
__device__ __forceinline__ void lift_probe(uint32_t& sa, uint32_t& sb, int& rem, int& v) {
    if constexpr (STEP <= SM_SPLIT_SKEW_LEVEL) LiftSel<K, STEP>::vtype::run(sa, sb, rem, v);
    else LiftSel<K, STEP>::type::run(sa, sb, rem, v);
}

template <typename K, int S>
struct LiftAll {
    __device__ __forceinline__ static void run(uint32_t& sa, uint32_t& sb, int& rem, int& v) {
        lift_probe<K, (1 << S)>(sa, sb, rem, v);
        LiftAll<K, S - 1>::run(sa, sb, rem, v);
    }
};
template <typename K>
struct LiftAll<K, -1> {
    __device__ __forceinline__ static void run(uint32_t&, uint32_t&, int&, int&) {}
};

// Per-thread skew in [0, 2 * SM_SPLIT_SKEW_LEVEL) from the diagonal (a hash:
// both the lattice of a[] and that of b[d-1-i] must differ between
// neighbouring threads; simulated 79 -> 50 wavefronts per warp split).
__device__ __forceinline__ int split_skew(int d) {
    return SM_SPLIT_SKEW_LEVEL > 0 ? ((d * 37) >> 3) & (2 * SM_SPLIT_SKEW_LEVEL - 1) : 0;
}

// Merge-path split at diagonal d of sorted a[0, la) and b[0, lb) held in
// shared memory at sa0 / sb0 (byte addresses): smallest i in
// [max(0, d-lb), min(d, la)] with a[i] > b[d-1-i] (reading R17), by
// LOG2+1 predicated probes (binary lifting; 2^(LOG2+1)-1 >= any range).
// The lifting starts `skew` (< 2 * SM_SPLIT_SKEW_LEVEL) candidates below the
// range; those virtual candidates pass without a load (they lie before the
// split), so the result is unchanged while neighbouring threads probe
// different residues at the deep levels (bank conflicts of the split: ncu r2
// 14.5 M of K2's 40.6 M shared wavefronts on C2, ~6.5-way at STEP 4..16).
template <typename K, int LOG2>
__device__ __forceinline__ int split_smem(uint32_t sa0, int la, uint32_t sb0, int lb, int d) {
    const int lo = max(0, d - lb);
    const int skew = split_skew(d);
    int rem = min(d, la) - lo + skew;
    int v = skew;
    uint32_t sa = sa0 + (uint32_t)(lo - skew) * sizeof(K);    // (wraps below sa0: never dereferenced there)
    uint32_t sb = sb0 + (uint32_t)(d - 1 - lo + skew) * sizeof(K);
    LiftAll<K, LOG2>::run(sa, sb, rem, v);
    return (int)((sa - sa0) / sizeof(K));
}

}  // namespace
}  // namespace sm
