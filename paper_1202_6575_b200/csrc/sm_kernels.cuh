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
template <typename K>
__global__ void __launch_bounds__(256) k_cross_ranks(const K* __restrict__ A, const K* __restrict__ B, Geom g,
                                                     int* __restrict__ xbar, int* __restrict__ ybar) {
    const int per = g.pA + g.pB + 2;
    const long long gid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (gid < (long long)g.S * per) {
        const int s = (int)(gid / per), t = (int)(gid % per);
        const Seg sg = segment(g, s);
        const K* As = A + sg.aoff;
        const K* Bs = B + sg.boff;
        if (t <= g.pA) {                                  // Step 1: xbar_i = rank_low(A[x_i], B)
            const int i = t;
            int v = sg.m;                                 // xbar_p = m; empty block start -> m (R4)
            if (i < g.pA) {
                const int xi = Blocks(sg.n, g.pA).start(i);
                if (xi < sg.n) v = rank_low_dev(Bs, sg.m, __ldg(As + xi));
            }
            xbar[(size_t)s * (g.pA + 1) + i] = v;
        } else {                                          // Step 2: ybar_j = rank_high(B[y_j], A)
            const int j = t - g.pA - 1;
            int v = sg.n;
            if (j < g.pB) {
                const int yj = Blocks(sg.m, g.pB).start(j);
                if (yj < sg.m) v = rank_high_dev(As, sg.n, __ldg(Bs + yj));
            }
            ybar[(size_t)s * (g.pB + 1) + j] = v;
        }
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
template <typename K, bool HAS_V, int NT, int VT>
struct TileSmem {
    static constexpr int NV = NT * VT;
    K keys[NV];
    uint32_t vals[HAS_V ? NV : 1];
};

template <typename K, bool HAS_V, int NT, int VT>
__global__ void __launch_bounds__(NT) k_tasks(const K* __restrict__ A, const uint32_t* __restrict__ vA,
                                              const K* __restrict__ B, const uint32_t* __restrict__ vB,
                                              K* __restrict__ C, uint32_t* __restrict__ vC, Geom g,
                                              const int* __restrict__ xbar, const int* __restrict__ ybar) {
    constexpr int NV = NT * VT;
    __shared__ TileSmem<K, HAS_V, NT, VT> sm_;
    const int tid = threadIdx.x;

    pdl_wait();   // the single synchronisation (L373-375): all ranks visible

    Seg sg;
    const Task t = decode_task(g, blockIdx.x, xbar, ybar, sg);
    const int la = t.a1 - t.a0, lb = t.b1 - t.b0, L = la + lb;
    const int off = sg.coff + t.a0 + t.b0;
    const K* As = A + sg.aoff + t.a0;
    const K* Bs = B + sg.boff + t.b0;

    if (la == 0 || lb == 0) {                       // cases (a), (e): copy (row a6)
        const int so = la ? sg.aoff + t.a0 : sg.boff + t.b0;
        cta_copy<K, NT, 4>((la ? A : B) + so, C + off, L);
        if (HAS_V) cta_copy<uint32_t, NT, 4>((la ? vA : vB) + so, vC + off, L);
        return;
    }

    // cases (b), (c), (d): stable merge of A[a0,a1) and B[b0,b1) (row a7)
#pragma unroll
    for (int k = 0; k < VT; ++k) {
        const int idx = k * NT + tid;
        if (idx < L) {
            sm_.keys[idx] = idx < la ? ld_stream(As + idx) : ld_stream(Bs + (idx - la));
            if (HAS_V)
                sm_.vals[idx] = idx < la ? ld_stream(vA + sg.aoff + t.a0 + idx)
                                         : ld_stream(vB + sg.boff + t.b0 + (idx - la));
        }
    }
    __syncthreads();

    const int d = min(tid * VT, L);
    const int ai = tile_split(sm_.keys, la, lb, d);
    K out[VT];
    int src[VT];
    serial_merge<K, VT>(sm_.keys, ai, la, la + (d - ai), L, out, src);
    uint32_t v[HAS_V ? VT : 1];
    if (HAS_V) {
#pragma unroll
        for (int k = 0; k < VT; ++k) v[k] = sm_.vals[min(src[k], NV - 1)];
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < VT; ++k) {
        sm_.keys[tid * VT + k] = out[k];
        if (HAS_V) sm_.vals[tid * VT + k] = v[k];
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < VT; ++k) {
        const int idx = k * NT + tid;
        if (idx < L) {
            st_stream(C + off + idx, sm_.keys[idx]);
            if (HAS_V) st_stream(vC + off + idx, sm_.vals[idx]);
        }
    }
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
