// sm_host.cuh -- host drivers of the B200 stable parallel merge / merge sort
// of arXiv 1202.6575, shared by the per-key-type translation units abi_*.cu
// (the library's globals and key-type-independent C-ABI calls live in
// sm_common.cu).
//
// Call sequence of merge_stable:
//   validate -> choose p_A, p_B -> cudaMallocAsync the two rank arrays ->
//   K1 (cross ranks, PDL behind the previous kernel) -> [single
//   synchronisation: PDL griddepcontrol.wait] -> K2 (classify + copy/merge
//   every task) -> cudaFreeAsync.  No host sync.  Host buffers: staged, or
//   pipelined over three streams from 64 MB; n + m >= 2^31: a coarse
//   partition into sub-merges (one host sync).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>
#include <stdlib.h>

#include <algorithm>
#include <type_traits>
#include <vector>
#include <climits>
#include <initializer_list>
#include <mutex>

#include <nvtx3/nvToolsExt.h>

#include "stablemerge.h"
#include "sm_kernels.cuh"
#include "sm_kernels4.cuh"

namespace sm {

extern thread_local char g_err[512];
extern thread_local int64_t g_launches;

// K2 shape per element layout: NC consumer threads x VT diagonals per thread
// = NV padded diagonals per ring stage, the largest task; block size
// T = NV / 2 (task bound 2T); STAGES-deep TMA ring; MINB
// CTAs per SM requested from ptxas.  VT odd keeps the register -> shared
// write-back free of bank conflicts.  Measured on B200 (profiles/): 4-byte
// keys-only merges are bound by the consumers' shared-memory merge, and the
// best of the shapes tried is 352 x 23 (2 CTAs/SM: T = 4048, half the
// cross-rank searches of VT = 15); 8-byte elements 256 x 15 (2 CTAs/SM,
// requested: 8-byte keys-only merges of random keys +25% over 1 CTA/SM);
// 12-byte elements 320 x 17 with a 3-deep ring (1 CTA/SM; see SM_K2S12); 16-20-byte
// elements (128-bit keys) 256 x 11 (three stages fit).
template <int NC_, int VT_, int STAGES_, int MINB_ = 1>
struct K2Geo {
    static constexpr int NC = NC_, VT = VT_, STAGES = STAGES_, MINB = MINB_;
    static constexpr int NV = NC * VT;
    static constexpr int T = NV / 2;
};
// (tuning experiments override the shapes with -DSM_K2S4_NC=... etc.)
#ifndef SM_K2S4_NC
#define SM_K2S4_NC 352
#endif
#ifndef SM_K2S4_VT
#define SM_K2S4_VT 23
#endif
#ifndef SM_K2S4_ST
#define SM_K2S4_ST 3
#endif
#ifndef SM_K2S4_MINB
#define SM_K2S4_MINB 2
#endif
#ifndef SM_K2S8_NC
#define SM_K2S8_NC 256
#endif
#ifndef SM_K2S8_VT
#define SM_K2S8_VT 15
#endif
#ifndef SM_K2S8_ST
#define SM_K2S8_ST 3
#endif
#ifndef SM_K2S8_MINB
#define SM_K2S8_MINB 2
#endif
// 12-byte slots (8-byte keys + payload), one CTA per SM: 320 x 17 with three
// stages -- measured (scripts/gpu_k2s12.sh) against 256 x 15 with four: random
// i64 + payload 2^26 + 2^26 0.655 -> 0.560 ms, f64 + payload 2^25 + 2^25 0.373
// -> 0.319, C4 0.617 -> 0.612, C3 0.954 -> 0.959 (448 x 13: 0.559 / 0.318 /
// 0.613 / 0.964, spills 8 bytes; 384 x 15: 0.590 / 0.336 / 0.616 / 0.968)
#ifndef SM_K2S12_NC
#define SM_K2S12_NC 320
#endif
#ifndef SM_K2S12_VT
#define SM_K2S12_VT 17
#endif
#ifndef SM_K2S12_ST
#define SM_K2S12_ST 3
#endif
#define SM_K2S12 SM_K2S12_NC, SM_K2S12_VT, SM_K2S12_ST, 1
#define SM_K2S4 SM_K2S4_NC, SM_K2S4_VT, SM_K2S4_ST, SM_K2S4_MINB
#define SM_K2S8 SM_K2S8_NC, SM_K2S8_VT, SM_K2S8_ST, SM_K2S8_MINB
template <typename K, bool HAS_V, typename PV = uint32_t>
struct K2Shape {
    static constexpr int bytes = (int)sizeof(K) + (HAS_V ? (int)sizeof(PV) : 0);
    using type = typename std::conditional<
        bytes <= 4, K2Geo<SM_K2S4>,
        typename std::conditional<bytes <= 8, K2Geo<SM_K2S8>,
                                  typename std::conditional<bytes <= 12, K2Geo<SM_K2S12>,
                                                            K2Geo<256, 11, 3>>::type>::type>::type;
};
// Large plain merges of 8-byte slots: one CTA per SM with a larger tile
// (the split's probes amortise over 17 outputs, half the cross ranks);
// measured (scripts/gpu_k2s8.sh, ms, 256 x 15 x 2 CTAs against the large
// shape): u32 + payload 2^26 + 2^26 0.379 / 0.366 with 512 x 17, f32 +
// payload 2^25 + 2^25 0.206 / 0.198, u32 + payload 2^27 + 2^20 0.410 / 0.388,
// 2^22 + 2^22 0.0433 / 0.0402; i64 keys 2^26 + 2^26 0.429 / 0.397 with
// 448 x 17 (0.443 with 512 x 17).  Small merges keep two small CTAs per SM
// (C1, 2^20 + 2^20: 23.5 us against 26.6) and so do the sort rounds and the
// batched merges' segments.
#ifndef SM_K2_BIG_MIN
#define SM_K2_BIG_MIN (1ll << 23)     // n + m from which a default plain merge takes the large shape (from 2^22:
                                      //   u32 + payload 2^21 + 2^21 0.0219 -> 0.0229 ms, i64 keys 0.0238 -> 0.0263)
#endif
template <typename K, bool HAS_V, typename PV = uint32_t>
struct K2ShapeBig {
    static constexpr int bytes = (int)sizeof(K) + (HAS_V ? (int)sizeof(PV) : 0);
    static constexpr bool differs = bytes == 8;
    using type = typename std::conditional<
        !differs, typename K2Shape<K, HAS_V, PV>::type,
        typename std::conditional<sizeof(K) == 4, K2Geo<512, 17, 3, 1>, K2Geo<448, 17, 3, 1>>::type>::type;
};
// Tasks packed per ring stage at most.
constexpr int K2_MAXT = 16;

// Tile capacity NV (largest task) and default block size of a layout.
static int64_t tile_nv(int key_bytes, bool has_v) {
    if (key_bytes == 4) return has_v ? K2Shape<uint32_t, true>::type::NV : K2Shape<uint32_t, false>::type::NV;
    if (key_bytes == 16) return has_v ? K2Shape<u128, true>::type::NV : K2Shape<u128, false>::type::NV;
    return has_v ? K2Shape<uint64_t, true>::type::NV : K2Shape<uint64_t, false>::type::NV;
}

// 128-bit keys are loaded as one 16-byte word: their arrays must be aligned.
template <typename K>
static bool keys_aligned(std::initializer_list<const void*> ptrs) {
    if constexpr (sizeof(K) >= 16) {
        for (const void* p : ptrs)
            if ((uintptr_t)p & 15) return false;
    }
    (void)ptrs;
    return true;
}
static int64_t tile_t(int key_bytes, bool has_v) { return tile_nv(key_bytes, has_v) / 2; }
// ... of the large shape (8-byte slots; else the same)
static int64_t tile_nv_big(int key_bytes, bool has_v) {
    if (key_bytes == 4 && has_v) return K2ShapeBig<uint32_t, true>::type::NV;
    if (key_bytes == 8 && !has_v) return K2ShapeBig<uint64_t, false>::type::NV;
    return tile_nv(key_bytes, has_v);
}
// K3 shape: one run of R = k3_nt * k3_ipt elements per CTA (radix block sort),
// two CTAs per SM.  Key + payload slots of <= 8 bytes: 256 x 33 = 8448
// (>= 2^13: one merge round fewer than 256 x 17 for N = 2^28; C5 14.96 vs
// 15.92 ms); wider slots: 256 x 17 = 4352 (shared memory).
#ifndef SM_K3_NT_SMALL
#define SM_K3_NT_SMALL 256
#endif
#ifndef SM_K3_IPT_SMALL
#define SM_K3_IPT_SMALL 33
#endif
constexpr int K3_IPT = 17;
constexpr bool k3_small(int key_bytes, bool has_v) { return key_bytes + (has_v ? 4 : 0) <= 8; }
constexpr int k3_nt(int key_bytes, bool has_v) { return k3_small(key_bytes, has_v) ? SM_K3_NT_SMALL : 256; }
constexpr int k3_ipt(int key_bytes, bool has_v) { return k3_small(key_bytes, has_v) ? SM_K3_IPT_SMALL : K3_IPT; }
constexpr int64_t k3_run(int key_bytes, bool has_v) { return (int64_t)k3_nt(key_bytes, has_v) * k3_ipt(key_bytes, has_v); }
// K1: lanes per rank search (see k_cross_ranks).  Many searches: one lane
// each (the DRAM-probe traffic of wider groups costs more than it saves);
// for a plain merge the top levels come from a per-CTA shared-memory sample
// (k_cross_ranks_smp, the north_star's design; measured equal to searching
// them through L1/L2 on C2-C4, within 0.3%).  Few searches (< K1_FEW): a
// whole warp each, ~log_33 dependent rounds.
// Measured (i32 keys, n = m, ms per call, threshold 4096 / 16384): 8 M
// (4148 searches) 0.0440 / 0.0397, 12 M (6200) 0.0554 / 0.0512, 16 M (8290)
// 0.0642 / 0.0616, 24 M (12434) 0.0864 / 0.0871: a warp per search up to ~10 K
// searches (one wave of warps), the sample kernel above.
#ifndef SM_K1_FEW
#define SM_K1_FEW 10240
#endif
constexpr int K1_FEW = SM_K1_FEW;
#ifndef SM_SMALL_FUSE
#define SM_SMALL_FUSE 1          // small plain merges: one launch, each CTA ranks its own tasks (k2_local_prologue)
#endif
#ifndef SM_K1_SMP_BYTES
#define SM_K1_SMP_BYTES 8192     // the sample kernel's shared-memory sample per searched array
#endif

sm_status fail_cuda(cudaError_t e, const char* what);
sm_status fail_inval(const char* what);

// ------------------------------------------------------------ profiling
// While enabled, every kernel launch is bracketed by two CUDA events on its
// own stream; sm_profile_read() sums the durations per kernel kind.
enum { PROF_K1 = 0, PROF_K2 = 1, PROF_K3 = 2, PROF_KINDS = 3 };
struct ProfRec {
    cudaEvent_t a, b;
    int kind;
};
extern uint32_t* g_dbg_cover;  // SM_DEBUG builds: K2's coverage counters (sm_debug_cover), or null
extern unsigned long long* g_dbg_ts;   // SM_K2_TSTAMP builds: K2's per-CTA event times (sm_debug_k2_timestamps)
extern int g_k1_variant;        // test hook (sm_set_k1_variant): 0 auto, 1 warp per search, 2 sample, 3 thread per search
extern int g_sort_ways;         // sm_set_sort_ways: 0 (default) automatic, 4 -- two merge rounds per
                                //   HBM pass (k_tasks4) for keys <= 8 bytes, 2 -- one round per pass (K2)
extern int g_small_fuse;        // sm_set_small_fuse: small plain merges in one launch (default 0: measured slower
                                //   with L2 flushed between calls, C1 24.1 vs 22.9 us; back to back 21.0 vs 21.9)
extern bool g_prof_on;
extern std::vector<ProfRec> g_prof_pool;
extern size_t g_prof_used;
void prof_before(int kind, cudaStream_t st);
void prof_after(cudaStream_t st);

sm_status check_launch(const char* what);

static inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// One-time setup is per device: function attributes and memory pools belong
// to a device's context, and one process may drive several devices.  Devices
// past SM_MAX_DEV redo the setup at every call.  Concurrent first calls
// repeat idempotent work only.
constexpr int SM_MAX_DEV = 64;
static int current_device() {
    int dev = 0;
    cudaGetDevice(&dev);
    return dev;
}

// The library's scratch (rank arrays, task descriptors, the sort's auxiliary
// buffers, staging copies) comes from a private stream-ordered memory pool per
// device that keeps freed blocks (release threshold: never), so steady-state
// calls allocate nothing new -- without changing the release behaviour of the
// device's default pool for the rest of the process.
static cudaMemPool_t lib_pool() {
    static cudaMemPool_t pools[SM_MAX_DEV];
    static std::mutex mu;
    const int dev = current_device();
    if (dev < SM_MAX_DEV && pools[dev]) return pools[dev];
    std::lock_guard<std::mutex> lock(mu);
    if (dev < SM_MAX_DEV && pools[dev]) return pools[dev];
    cudaMemPoolProps props;
    memset(&props, 0, sizeof(props));
    props.allocType = cudaMemAllocationTypePinned;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = dev;
    cudaMemPool_t pool = nullptr;
    if (cudaMemPoolCreate(&pool, &props) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;                                  // dalloc falls back to the default pool
    }
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    if (dev < SM_MAX_DEV) pools[dev] = pool;
    return pool;
}
static void keep_pool(cudaStream_t) { lib_pool(); }

template <typename T>
static sm_status dalloc(T** p, int64_t count, cudaStream_t st) {
    *p = nullptr;
    if (count <= 0) return SM_OK;
    cudaMemPool_t pool = lib_pool();
    cudaError_t e = pool ? cudaMallocFromPoolAsync((void**)p, (size_t)count * sizeof(T), pool, st)
                         : cudaMallocAsync((void**)p, (size_t)count * sizeof(T), st);
    if (e != cudaSuccess) {
        cudaGetLastError();
        snprintf(g_err, sizeof(g_err), "cudaMallocAsync(%lld bytes): %s", (long long)(count * sizeof(T)),
                 cudaGetErrorString(e));
        return SM_ENOMEM;
    }
    return SM_OK;
}

static void dfree(void* p, cudaStream_t st) {
    if (p) cudaFreeAsync(p, st);
}

// ------------------------------------------------------------ launches
// K1: the cross ranks of every block start of every segment.
// Upper bounds of the launch's rank entries and tasks (exact for modes 0/1;
// mode 2 counts them on the device, the host sizes the grids by the bound).
struct GeomCounts {
    long long items, tasks;
};
static GeomCounts geom_counts(const Geom& g) {
    return {(long long)g.S * (g.pA + g.pB + 2), (long long)g.S * (g.pA + g.pB)};
}

// Launch with programmatic dependent launch (PDL) when `pdl`: the grid may
// start while the previous kernel in the stream drains; the kernel's first
// action is griddepcontrol.wait, so it reads nothing that kernel writes
// before it completes.
template <typename... KA, typename... Args>
static cudaError_t launch_maybe_pdl_smem(void (*kern)(KA...), unsigned grid, unsigned block, size_t smem,
                                         cudaStream_t st, bool pdl, Args... args) {
    cudaLaunchConfig_t cfg;
    memset(&cfg, 0, sizeof(cfg));
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = (pdl && !g_prof_on) ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kern, args...);
}
template <typename... KA, typename... Args>
static cudaError_t launch_maybe_pdl(void (*kern)(KA...), unsigned grid, unsigned block, cudaStream_t st, bool pdl,
                                    Args... args) {
    return launch_maybe_pdl_smem(kern, grid, block, 0, st, pdl, args...);
}

template <typename K>
static sm_status launch_cross_ranks(const K* A, const K* B, const Geom& g, const GeomCounts& gc, int* xbar, int* ybar,
                                    cudaStream_t st, bool pdl = false) {
    const long long items = gc.items;
    prof_before(PROF_K1, st);
    constexpr int SMP = SM_K1_SMP_BYTES / (int)sizeof(K);   // sample keys per searched array
    cudaError_t e;
    const int v = g_k1_variant;
    if (v == 1 || (v == 0 && items < K1_FEW))
        e = launch_maybe_pdl(k_cross_ranks<K, 32>, (unsigned)((items * 32 + 255) / 256), 256, st, pdl, A, B, g, xbar,
                             ybar);
    else if (g.sort == 0 && v != 3) {
        auto kern = k_cross_ranks_smp<K, SMP>;
        constexpr size_t smem = 2 * SMP * sizeof(K);
        static bool attr[SM_MAX_DEV];
        const int dev = current_device();
        if (dev >= SM_MAX_DEV || !attr[dev]) {
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            if (dev < SM_MAX_DEV) attr[dev] = true;
        }
        e = launch_maybe_pdl_smem(kern, (unsigned)((items + 255) / 256), 256, smem, st, pdl, A, B, g, xbar, ybar);
    }
    else
        e = launch_maybe_pdl(k_cross_ranks<K, 1>, (unsigned)((items + 255) / 256), 256, st, pdl, A, B, g, xbar, ybar);
    prof_after(st);
    if (e != cudaSuccess) return fail_cuda(e, "k_cross_ranks");
    return check_launch("k_cross_ranks");
}

// CTAs of K2 resident on the device at once (the persistent grid); the
// function attributes are set once per device.
template <typename K, bool HAS_V, typename Sh, typename PV = uint32_t>
static long long k2_resident() {
    using Lay = K2Layout<K, HAS_V, Sh::NC, Sh::VT, Sh::STAGES, K2_MAXT, PV>;
    auto kern = k_tasks<K, HAS_V, Sh::NC, Sh::VT, Sh::STAGES, K2_MAXT, Sh::MINB, PV>;
    static int per_sm_d[SM_MAX_DEV], n_sm_d[SM_MAX_DEV];   // 0: not yet set up on that device
    const int dev = current_device();
    int per_sm = dev < SM_MAX_DEV ? per_sm_d[dev] : 0, n_sm = dev < SM_MAX_DEV ? n_sm_d[dev] : 0;
    if (per_sm == 0) {
        cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Lay::SMEM);
        cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, Lay::THREADS, Lay::SMEM);
        if (per_sm < 1) per_sm = 1;
        if (dev < SM_MAX_DEV) {
            n_sm_d[dev] = n_sm;
            per_sm_d[dev] = per_sm;
        }
    }
    return (long long)per_sm * n_sm;
}

template <typename K, bool HAS_V, typename Sh, typename PV = uint32_t>
static sm_status launch_tasks(const K* A, const PV* vA, const K* B, const PV* vB, K* C, PV* vC,
                              const Geom& g, const GeomCounts& gc, const int* xbar, const int* ybar, cudaStream_t st,
                              bool pdl) {
    using Lay = K2Layout<K, HAS_V, Sh::NC, Sh::VT, Sh::STAGES, K2_MAXT, PV>;
    auto kern = k_tasks<K, HAS_V, Sh::NC, Sh::VT, Sh::STAGES, K2_MAXT, Sh::MINB, PV>;
    const long long resident = k2_resident<K, HAS_V, Sh, PV>();
    const long long grid = std::max(1ll, std::min<long long>(gc.tasks, resident));
    Geom gk = g;
    gk.cover = g_dbg_cover;
    gk.ts = g_dbg_ts;
    cudaLaunchConfig_t cfg;
    memset(&cfg, 0, sizeof(cfg));
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3(Lay::THREADS);
    cfg.dynamicSmemBytes = Lay::SMEM;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.numAttrs = (pdl && !g_prof_on) ? 1 : 0;
    cfg.attrs = attr;
    prof_before(PROF_K2, st);
    cudaError_t e = cudaLaunchKernelEx(&cfg, kern, A, vA, B, vB, C, vC, gk, xbar, ybar);
    prof_after(st);
    ++g_launches;
    if (e != cudaSuccess) {
        cudaGetLastError();
        return fail_cuda(e, "k_tasks");
    }
    return SM_OK;
}

// K1, (segmented modes) k_classify, K2 -- with the tile shape Sh.
template <typename K, bool HAS_V, typename Sh, typename PV>
static sm_status launch_merge_sh(const K* A, const PV* vA, const K* B, const PV* vB, K* C, PV* vC, const Geom& g0,
                                 const GeomCounts& gc, int* xbar, int* ybar, cudaStream_t st, bool pdl, int4* tdesc) {
    Geom g = g0;
    sm_status s = launch_cross_ranks<K>(A, B, g0, gc, xbar, ybar, st, pdl);
    if (s != SM_OK) return s;
    if (tdesc && gc.tasks > 0) {
        // segmented modes: classify every task once, ahead of K2 (k_classify)
        cudaLaunchConfig_t cfg;
        memset(&cfg, 0, sizeof(cfg));
        cfg.gridDim = dim3((unsigned)((gc.tasks + 255) / 256));
        cfg.blockDim = dim3(256);
        cfg.stream = st;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr;
        cfg.numAttrs = (pdl && !g_prof_on) ? 1 : 0;
        cudaError_t e = cudaLaunchKernelEx(&cfg, k_classify<Sh::NV>, g0, (const int*)xbar, (const int*)ybar, tdesc);
        if (e != cudaSuccess) return fail_cuda(e, "k_classify");
        s = check_launch("k_classify");
        if (s != SM_OK) return s;
        g.tdesc = tdesc;
    }
    return launch_tasks<K, HAS_V, Sh, PV>(A, vA, B, vB, C, vC, g, gc, xbar, ybar, st, pdl);
}

// big: the large tile shape (K2ShapeBig: large plain merges and batches of
// 8-byte slots; the caller's block counts / block size must match it).
template <typename K, bool HAS_V, typename PV = uint32_t>
static sm_status launch_merge(const K* A, const PV* vA, const K* B, const PV* vB, K* C,
                              PV* vC, const Geom& g0, int* xbar, int* ybar, cudaStream_t st, bool pdl,
                              const GeomCounts* counts = nullptr, int4* tdesc = nullptr, bool big = false) {
    const GeomCounts gc = counts ? *counts : geom_counts(g0);
    using Sh0 = typename K2Shape<K, HAS_V, PV>::type;
    if constexpr (K2ShapeBig<K, HAS_V, PV>::differs) {
        if (big && g0.sort != 1)
            return launch_merge_sh<K, HAS_V, typename K2ShapeBig<K, HAS_V, PV>::type, PV>(A, vA, B, vB, C, vC, g0, gc, xbar,
                                                                                        ybar, st, pdl, tdesc);
    }
    if (g0.sort == 0 && SM_SMALL_FUSE && g_small_fuse && g_k1_variant == 0 &&
        gc.tasks <= (long long)K2L_MAXP * k2_resident<K, HAS_V, Sh0, PV>()) {
        // a small plain merge: one launch -- each CTA of K2 computes the cross
        // ranks its own tasks read (k2_local_prologue)
        Geom g = g0;
        g.fuse = 1;
        return launch_tasks<K, HAS_V, Sh0, PV>(A, vA, B, vB, C, vC, g, gc, xbar, ybar, st, pdl);
    }
    return launch_merge_sh<K, HAS_V, Sh0, PV>(A, vA, B, vB, C, vC, g0, gc, xbar, ybar, st, pdl, tdesc);
}

// ------------------------------------------------ two rounds per pass
// The merge sort's rounds L -> 2L -> 4L in one HBM pass (sm_kernels4.cuh):
// k4_sample, k4_ranks, k4_order (the paper's Steps 1-2 and the order of the
// subproblems, for four runs), then k_tasks4; PDL between them.
struct Pass4Scratch {
    void* spl;        // block-start keys   [G * 4 * cmax]
    int4* rk;         // their ranks        [G * 4 * cmax]
    int* fv;          // their places       [G * 4 * cmax]
    int4* bnd;        // boundaries         [G * (4 * cmax + 2)]
    int* ctr;         // k_tasks4's task counter
};
#ifndef SM_K4_MIN_N
#define SM_K4_MIN_N (3 << 19)   // sorts below ~1.5 M elements keep one round per pass (2^20: 0.148 / 0.143 ms)
#endif
// k_tasks4 shapes by slot size (tuning experiments override them with
// -DSM_K4S8_NC=... etc.).  8-byte slots: one CTA of 512 x 17 per SM -- the
// split's probes amortise over 17 outputs instead of 15 and S doubles (half
// the block starts to rank and order); measured on C5 (scripts/gpu_ab.sh,
// pass / partition ms per sort): 256 x 15 x 2 CTAs 4.81 / 0.48, 288 x 13 x 2
// 4.76 / 0.48, 384 x 10 x 2 5.21 / 0.48, 512 x 15 4.83 / 0.35, 480 x 17 4.66 /
// 0.34, 576 x 15 4.67 / 0.33, 640 x 13 4.64 / 0.33, 512 x 19 with two stages
// 4.68 / 0.32, 384 x 19 4.89 / 0.35, 512 x 17 4.53 / 0.33 (C5 9.90 -> 9.45 ms;
// f32 + payload 2^28 12.24 -> 11.80 ms; i64 keys-only 2^27 unchanged, 9.23 ->
// 9.26).  12-byte slots: 448 x 13 with three stages instead of K2's 256 x 15
// with four (i64 + payload 2^27 14.11 -> 13.27 ms, f64 + payload 14.87 ->
// 14.06; scripts/gpu_k4_types.sh).  4-byte keys without payload keep K2's
// shape and one round per pass (704 x 23 at one CTA per SM: 8.29 ms against
// 8.28 for one round per pass on 2^28 u32 keys).
#ifndef SM_K4S4_NC
#define SM_K4S4_NC SM_K2S4_NC
#endif
#ifndef SM_K4S4_VT
#define SM_K4S4_VT SM_K2S4_VT
#endif
#ifndef SM_K4S4_ST
#define SM_K4S4_ST SM_K2S4_ST
#endif
#ifndef SM_K4S4_MINB
#define SM_K4S4_MINB SM_K2S4_MINB
#endif
#ifndef SM_K4S8_NC
#define SM_K4S8_NC 512
#endif
#ifndef SM_K4S8_VT
#define SM_K4S8_VT 17
#endif
#ifndef SM_K4S8_ST
#define SM_K4S8_ST 3
#endif
#ifndef SM_K4S8_MINB
#define SM_K4S8_MINB 1
#endif
#ifndef SM_K4S12_NC
#define SM_K4S12_NC 448
#endif
#ifndef SM_K4S12_VT
#define SM_K4S12_VT 13
#endif
#ifndef SM_K4S12_ST
#define SM_K4S12_ST 3
#endif
#ifndef SM_K4S12_MINB
#define SM_K4S12_MINB 1
#endif
template <typename K, bool HAS_V>
struct K4Shape {
    static constexpr int bytes = (int)sizeof(K) + (HAS_V ? 4 : 0);
    using Sh = typename std::conditional<
        bytes <= 4, K2Geo<SM_K4S4_NC, SM_K4S4_VT, SM_K4S4_ST, SM_K4S4_MINB>,
        typename std::conditional<bytes <= 8, K2Geo<SM_K4S8_NC, SM_K4S8_VT, SM_K4S8_ST, SM_K4S8_MINB>,
                                  typename std::conditional<bytes <= 12,
                                                            K2Geo<SM_K4S12_NC, SM_K4S12_VT, SM_K4S12_ST, SM_K4S12_MINB>,
                                                            typename K2Shape<K, HAS_V>::type>::type>::type>::type;
    using Lay = K4Layout<K, HAS_V, Sh::NC, Sh::VT, Sh::STAGES, K2_MAXT>;
};
template <typename K, bool HAS_V>
static Geom4 geom4(int64_t N, int64_t L) {
    Geom4 g{};
    g.N = (int)N;
    g.L = (int)L;
    g.S = K4Shape<K, HAS_V>::Lay::S;
    g.cmax = (int)ceil_div(L, g.S);
    g.TPG = 4 * g.cmax + 1;
    g.G = (int)ceil_div(N, 4 * L);
    return g;
}
template <typename K, bool HAS_V>
static sm_status launch_pass4(const K* in, const uint32_t* vin, K* out, uint32_t* vout, int64_t N, int64_t L,
                              const Pass4Scratch& sc, cudaStream_t st, bool pdl) {
    using Sh = typename K4Shape<K, HAS_V>::Sh;
    using Lay = typename K4Shape<K, HAS_V>::Lay;
    Geom4 g = geom4<K, HAS_V>(N, L);
    g.ctr = sc.ctr;
    g.bnd = sc.bnd;
    g.cover = g_dbg_cover;
    const long long ids = (long long)g.G * 4 * g.cmax;
    const long long nb = (long long)g.G * (g.TPG + 1);
    K* spl = (K*)sc.spl;
    prof_before(PROF_K1, st);
    cudaError_t e = launch_maybe_pdl(k4_sample<K>, (unsigned)ceil_div(ids, 256), 256, st, pdl, in, g, spl);
    if (e == cudaSuccess)
        e = launch_maybe_pdl(k4_ranks<K>, (unsigned)ceil_div(4 * ids, 256), 256, st, pdl, in, g, (const K*)spl, sc.rk,
                             sc.fv);
    if (e == cudaSuccess)
        e = launch_maybe_pdl(k4_order, (unsigned)ceil_div(std::max(4 * ids, nb), 256), 256, st, pdl, g,
                             (const int4*)sc.rk, (const int*)sc.fv, sc.bnd);
    prof_after(st);
    if (e != cudaSuccess) return fail_cuda(e, "k4 partition");
    g_launches += 2;
    sm_status s = check_launch("k4 partition");
    if (s != SM_OK) return s;
    auto kern = k_tasks4<K, HAS_V, Sh::NC, Sh::VT, Sh::STAGES, K2_MAXT, Sh::MINB>;
    static int per_sm_d[SM_MAX_DEV], n_sm_d[SM_MAX_DEV];
    const int dev = current_device();
    int per_sm = dev < SM_MAX_DEV ? per_sm_d[dev] : 0, n_sm = dev < SM_MAX_DEV ? n_sm_d[dev] : 0;
    if (per_sm == 0) {
        cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Lay::SMEM);
        cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, Lay::THREADS, Lay::SMEM);
        if (per_sm < 1) per_sm = 1;
        if (dev < SM_MAX_DEV) {
            n_sm_d[dev] = n_sm;
            per_sm_d[dev] = per_sm;
        }
    }
    const long long grid = std::max(1ll, std::min<long long>((long long)g.G * g.TPG, (long long)per_sm * n_sm));
    prof_before(PROF_K2, st);
    e = launch_maybe_pdl_smem(kern, (unsigned)grid, Lay::THREADS, Lay::SMEM, st, pdl, in, vin, out, vout, g);
    prof_after(st);
    if (e != cudaSuccess) return fail_cuda(e, "k_tasks4");
    return check_launch("k_tasks4");
}

// ------------------------------------------------ host-memory staging
static bool is_host_ptr(const void* p) {
    if (!p) return false;
    cudaPointerAttributes a;
    cudaError_t e = cudaPointerGetAttributes(&a, p);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return true;
    }
    return a.type == cudaMemoryTypeHost || a.type == cudaMemoryTypeUnregistered;
}

// An NVTX range for the whole C-ABI call (the kernels' own ranges nest in it)
struct NvtxCall {
    explicit NvtxCall(const char* name) { nvtxRangePushA(name); }
    ~NvtxCall() { nvtxRangePop(); }
    NvtxCall(const NvtxCall&) = delete;
    NvtxCall& operator=(const NvtxCall&) = delete;
};

// A call runs on the device of its stream, whatever the calling thread's
// current device (restored on return); the NULL, legacy and per-thread
// default streams, and a stream under graph capture, mean the current device.
struct DevGuard {
    int prev = -1;
    explicit DevGuard(void* stream) {
        cudaStream_t st = (cudaStream_t)stream;
        if (!st || st == cudaStreamLegacy || st == cudaStreamPerThread) return;
        // a stream under graph capture is not queried (the query would
        // invalidate the capture): the capturing thread's device is used
        cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
        if (cudaStreamIsCapturing(st, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) {
            cudaGetLastError();
            return;
        }
        int dev = 0, cur = 0;
        if (cudaStreamGetDevice(st, &dev) != cudaSuccess) {
            cudaGetLastError();
            return;
        }
        cudaGetDevice(&cur);
        if (dev != cur && cudaSetDevice(dev) == cudaSuccess) prev = cur;
    }
    ~DevGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
    DevGuard(const DevGuard&) = delete;
    DevGuard& operator=(const DevGuard&) = delete;
};

// One staged buffer: a device copy of a host range (in and/or out).
struct Stage {
    void* host = nullptr;
    void* dev = nullptr;
    size_t bytes = 0;
    bool out = false;
};

static sm_status stage_in(Stage& s, const void* host, size_t bytes, bool is_out, bool copy_in, cudaStream_t st) {
    s.host = (void*)host;
    s.bytes = bytes;
    s.out = is_out;
    if (!host || bytes == 0) return SM_OK;
    sm_status r = dalloc((char**)&s.dev, (int64_t)bytes, st);
    if (r != SM_OK) return r;
    if (copy_in) {
        cudaError_t e = cudaMemcpyAsync(s.dev, host, bytes, cudaMemcpyHostToDevice, st);
        if (e != cudaSuccess) return fail_cuda(e, "cudaMemcpyAsync H2D");
    }
    return SM_OK;
}

static sm_status stage_out(Stage& s, cudaStream_t st) {
    if (!s.dev) return SM_OK;
    sm_status r = SM_OK;
    if (s.out) {
        cudaError_t e = cudaMemcpyAsync(s.host, s.dev, s.bytes, cudaMemcpyDeviceToHost, st);
        if (e != cudaSuccess) r = fail_cuda(e, "cudaMemcpyAsync D2H");
    }
    dfree(s.dev, st);
    s.dev = nullptr;
    return r;
}

static bool overlaps(const void* p, size_t pb, const void* q, size_t qb) {
    if (!p || !q || pb == 0 || qb == 0) return false;
    const char *a = (const char*)p, *b = (const char*)q;
    return a < b + qb && b < a + pb;
}

// ------------------------------------------------------------ merge
// x̄ (p_A + 1), ȳ (p_B + 1) and K2's task counter
static inline int64_t merge_scratch_ints(int64_t pA, int64_t pB) { return (pA + 1) + (pB + 1) + 1; }
#ifndef SM_T_DIV
#define SM_T_DIV 2               // default block size T = tile capacity / SM_T_DIV (experiment knob)
#endif
#ifndef SM_MODE0_CLASSIFY
#define SM_MODE0_CLASSIFY 0      // 1: plain merges classify their tasks in a kernel ahead of K2 (experiment)
#endif

template <typename K, typename PV = uint32_t>
static sm_status merge_device(const K* A, const PV* vA, int64_t n, const K* B, const PV* vB, int64_t m,
                              K* C, PV* vC, cudaStream_t st, int64_t pA, int64_t pB, bool pdl,
                              int* ranks_given = nullptr, bool big = false) {
    Geom g{};
    g.S = 1; g.pA = (int)pA; g.pB = (int)pB; g.n = (int)n; g.m = (int)m; g.L = 0; g.N = 0; g.sort = 0;
    // scratch: x̄ (p_A + 1), ȳ (p_B + 1), task counter
    int* ranks = ranks_given;
    sm_status s = SM_OK;
    if (!ranks) s = dalloc(&ranks, merge_scratch_ints(pA, pB), st);
    if (s != SM_OK) return s;
    g.ctr = ranks + (pA + 1) + (pB + 1);
    int4* tdesc = nullptr;
#if SM_MODE0_CLASSIFY
    s = dalloc(&tdesc, pA + pB, st);
    if (s != SM_OK) return s;
#endif

    if (vC) s = launch_merge<K, true, PV>(A, vA, B, vB, C, vC, g, ranks, ranks + pA + 1, st, pdl, nullptr, tdesc, big);
    else s = launch_merge<K, false, PV>(A, nullptr, B, nullptr, C, nullptr, g, ranks, ranks + pA + 1, st, pdl, nullptr,
                                       tdesc, big);
    dfree(tdesc, st);
    if (!ranks_given) dfree(ranks, st);
    return s;
}

// ------------------------------------------- merge-path comparison (f4)
// Equal-output tiles of NV (one tile per ring stage), diagonal splits by
// K1mp, the same K2 -- to measure what the paper's factor-two task
// imbalance costs against perfectly balanced tiles.
template <typename K>
static sm_status merge_path_device(const K* A, const uint32_t* vA, int64_t n, const K* B, const uint32_t* vB,
                                   int64_t m, K* C, uint32_t* vC, cudaStream_t st, bool pdl) {
    const int64_t W = tile_nv((int)sizeof(K), vC != nullptr);
    const int64_t tiles = ceil_div(n + m, W);
    int* split = nullptr;
    sm_status s = dalloc(&split, tiles + 2, st);    // splits, task counter
    if (s != SM_OK) return s;
    prof_before(PROF_K1, st);
    k_diag_splits<K><<<(unsigned)((tiles + 1 + 255) / 256), 256, 0, st>>>(A, B, (int)n, (int)m, (int)W, split,
                                                                          split + tiles + 1);
    prof_after(st);
    s = check_launch("k_diag_splits");
    if (s == SM_OK) {
        Geom g{};
        g.S = 1; g.n = (int)n; g.m = (int)m; g.sort = 3; g.T = (int)W; g.pA = g.pB = 1;
        g.ctr = split + tiles + 1;
        GeomCounts gc{tiles + 2, tiles};
        if (vC) s = launch_tasks<K, true, typename K2Shape<K, true>::type>(A, vA, B, vB, C, vC, g, gc, split, split, st, pdl);
        else s = launch_tasks<K, false, typename K2Shape<K, false>::type, uint32_t>(A, nullptr, B, nullptr, C, nullptr, g,
                                                                                   gc, split, split, st, pdl);
    }
    dfree(split, st);
    return s;
}

// The host pipelines' three streams and their events belong to one device:
// one set per (host thread, device), created on first use.
struct PipeStreams {
    cudaStream_t sH = nullptr, sM = nullptr, sD = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    std::vector<cudaEvent_t> ev_a, ev_b;
};
static PipeStreams* pipe_streams() {
    thread_local PipeStreams sets[SM_MAX_DEV];
    const int dev = current_device();
    if (dev >= SM_MAX_DEV) return nullptr;
    PipeStreams& ps = sets[dev];
    if (!ps.sH) {
        if (cudaStreamCreateWithFlags(&ps.sH, cudaStreamNonBlocking) != cudaSuccess ||
            cudaStreamCreateWithFlags(&ps.sM, cudaStreamNonBlocking) != cudaSuccess ||
            cudaStreamCreateWithFlags(&ps.sD, cudaStreamNonBlocking) != cudaSuccess ||
            cudaEventCreateWithFlags(&ps.ev_fork, cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&ps.ev_join, cudaEventDisableTiming) != cudaSuccess) {
            ps.sH = nullptr;
            return nullptr;
        }
    }
    return &ps;
}

// ----------------------------------------------- pipelined host staging
// A call with HOST inputs is cut into independent sub-merges with the paper's
// own Steps 1-4 at coarse granularity (p_h blocks per array, PAPER.md
// L168-340): 2 p_h binary searches over the host arrays give the cross ranks,
// the five cases give 2 p_h disjoint tasks with their input ranges and output
// offsets.  Each task then runs the full device path (K1 + K2) on its own
// sub-ranges, and the tasks alternate between two streams so that one task's
// device->host copy overlaps the next one's host->device copy (the copy
// engines are independent); the merge itself is ~1% of the staged call.
struct SubMerge {
    int64_t a0, a1, b0, b1;
};
static void plan_from_ranks(int64_t n, int64_t m, int64_t p, const std::vector<int64_t>& xb,
                            const std::vector<int64_t>& yb, std::vector<SubMerge>& tasks);

template <typename K>
static int64_t host_pipeline_blocks(int64_t n, int64_t m, bool has_v) {
    const int64_t bytes = (n + m) * (int64_t)(sizeof(K) + (has_v ? 4 : 0));
    // p_h <= 16 blocks of >= 32 MB: fewer, larger copies (measured C2 e2e
    // +5% over p_h <= 32 of 16 MB; p_h <= 8 equal on C2, -4% on C4)
    // (and blocks of <= 2^29 elements: every sub-merge stays below 2^31)
    return std::max(std::max<int64_t>(1, std::min<int64_t>(16, bytes / (32ll << 20))),
                    ceil_div(std::max(n, m), 1ll << 29));
}

static inline int64_t hblock_start(int64_t len, int64_t p, int64_t i) {    // x_i, L168-182; x_p = len
    return BlocksT<int64_t>(len, p).start(i);
}

template <typename K>
static void host_plan(const K* A, int64_t n, const K* B, int64_t m, int64_t p, std::vector<SubMerge>& tasks) {
    std::vector<int64_t> xb(p + 1), yb(p + 1);
    for (int64_t i = 0; i < p; ++i) {      // Step 1: xbar_i = rank_low(A[x_i], B); empty block start -> m (R4)
        auto lt = [](K u, K v) { return key_lt<K>(u, v); };
        const int64_t xi = hblock_start(n, p, i), yi = hblock_start(m, p, i);
        xb[i] = xi < n ? std::lower_bound(B, B + m, A[xi], lt) - B : m;
        yb[i] = yi < m ? std::upper_bound(A, A + n, B[yi], lt) - A : n;   // Step 2: rank_high
    }
    xb[p] = m;
    yb[p] = n;
    plan_from_ranks(n, m, p, xb, yb, tasks);
}

// Steps 3-4 on the host: the p_A + p_B tasks in task
// order (A-side task i, then B-side task j) from the cross ranks
// xb[0..p_A], yb[0..p_B], by the classification the device runs
// (classify_a_side / classify_b_side, 64-bit indices).
static void plan_tasks_host(int64_t n, int64_t m, int64_t pA, int64_t pB, const std::vector<int64_t>& xb,
                            const std::vector<int64_t>& yb, std::vector<SubMerge>& tasks) {
    const BlocksT<int64_t> xa(n, pA), ybl(m, pB);
    for (int64_t i = 0; i < pA; ++i) {
        const TaskT<int64_t> t = classify_a_side<int64_t>(i, xa, ybl, xb.data(), yb.data());
        tasks.push_back({t.a0, t.a1, t.b0, t.b1});
    }
    for (int64_t j = 0; j < pB; ++j) {
        const TaskT<int64_t> t = classify_b_side<int64_t>(j, xa, ybl, xb.data(), yb.data());
        tasks.push_back({t.a0, t.a1, t.b0, t.b1});
    }
}

// Steps 3-4 at coarse granularity (p blocks per array), ordered by output offset.
static void plan_from_ranks(int64_t n, int64_t m, int64_t p, const std::vector<int64_t>& xb,
                            const std::vector<int64_t>& yb, std::vector<SubMerge>& tasks) {
    plan_tasks_host(n, m, p, p, xb, yb, tasks);
    for (SubMerge& t : tasks) {            // unsorted inputs (a precondition violation): never negative
        t.a1 = std::max(t.a0, std::min(t.a1, n));
        t.b1 = std::max(t.b0, std::min(t.b1, m));
    }
    std::sort(tasks.begin(), tasks.end(),
              [](const SubMerge& u, const SubMerge& v) { return u.a0 + u.b0 < v.a0 + v.b0; });
}


template <typename K>
static sm_status merge_host_pipelined(const K* A, const uint32_t* vA, int64_t n, const K* B, const uint32_t* vB,
                                      int64_t m, K* C, uint32_t* vC, cudaStream_t st, bool pdl) {
    // three-stage pipeline: stream sH uploads task after task without a
    // break, sM merges each task once its upload event fires, sD downloads
    // each task once its merge event fires -- the two copy engines stay busy
    // concurrently and no download waits behind the next task's kernels
    PipeStreams* ps = pipe_streams();
    if (!ps) return fail_cuda(cudaGetLastError(), "stream/event create");
    cudaStream_t sH = ps->sH, sM = ps->sM, sD = ps->sD;
    cudaEvent_t ev_fork = ps->ev_fork, ev_join = ps->ev_join;
    std::vector<cudaEvent_t>& ev_up = ps->ev_a;
    std::vector<cudaEvent_t>& ev_mg = ps->ev_b;
    std::vector<SubMerge> tasks;
    host_plan<K>(A, n, B, m, host_pipeline_blocks<K>(n, m, vC != nullptr), tasks);
    // (the two lists grow independently: the sort's host pipeline uses ev_a alone)
    for (std::vector<cudaEvent_t>* v : {&ev_up, &ev_mg}) {
        while (v->size() < tasks.size()) {
            cudaEvent_t e;
            if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess)
                return fail_cuda(cudaGetLastError(), "event create");
            v->push_back(e);
        }
    }
    const size_t kb = sizeof(K);
    const int64_t T = tile_t((int)kb, vC != nullptr);
    // every device buffer comes from `st` before the fork (stream-ordered pool)
    int64_t rank_ints = 0;
    for (const SubMerge& t : tasks)
        rank_ints += merge_scratch_ints(std::max<int64_t>(1, ceil_div(t.a1 - t.a0, T)),
                                        std::max<int64_t>(1, ceil_div(t.b1 - t.b0, T)));
    K *dA = nullptr, *dB = nullptr, *dC = nullptr;
    uint32_t *dvA = nullptr, *dvB = nullptr, *dvC = nullptr;
    int* dranks = nullptr;
    sm_status s = dalloc(&dranks, rank_ints, st);
    if (s == SM_OK) s = dalloc(&dA, n, st);
    if (s == SM_OK) s = dalloc(&dB, m, st);
    if (s == SM_OK) s = dalloc(&dC, n + m, st);
    if (s == SM_OK && vC) s = dalloc(&dvA, n, st);
    if (s == SM_OK && vC) s = dalloc(&dvB, m, st);
    if (s == SM_OK && vC) s = dalloc(&dvC, n + m, st);
    if (s == SM_OK) {
        cudaEventRecord(ev_fork, st);
        cudaStreamWaitEvent(sH, ev_fork, 0);
        cudaStreamWaitEvent(sM, ev_fork, 0);
        cudaStreamWaitEvent(sD, ev_fork, 0);
    }
    // uploads
    for (size_t k = 0; s == SM_OK && k < tasks.size(); ++k) {
        const SubMerge& t = tasks[k];
        const int64_t la = t.a1 - t.a0, lb = t.b1 - t.b0;
        cudaError_t e = cudaSuccess;
        if (la) e = cudaMemcpyAsync(dA + t.a0, A + t.a0, la * kb, cudaMemcpyDefault, sH);
        if (e == cudaSuccess && lb) e = cudaMemcpyAsync(dB + t.b0, B + t.b0, lb * kb, cudaMemcpyDefault, sH);
        if (e == cudaSuccess && vC && la) e = cudaMemcpyAsync(dvA + t.a0, vA + t.a0, la * 4, cudaMemcpyDefault, sH);
        if (e == cudaSuccess && vC && lb) e = cudaMemcpyAsync(dvB + t.b0, vB + t.b0, lb * 4, cudaMemcpyDefault, sH);
        if (e == cudaSuccess) e = cudaEventRecord(ev_up[k], sH);
        if (e != cudaSuccess) s = fail_cuda(e, "cudaMemcpyAsync H2D");
    }
    // merges and downloads
    int64_t rank_at = 0;
    for (size_t k = 0; s == SM_OK && k < tasks.size(); ++k) {
        const SubMerge& t = tasks[k];
        const int64_t la = t.a1 - t.a0, lb = t.b1 - t.b0, L = la + lb, off = t.a0 + t.b0;
        if (L == 0) continue;
        cudaStreamWaitEvent(sM, ev_up[k], 0);
        const int64_t pa = std::max<int64_t>(1, ceil_div(la, T)), pb = std::max<int64_t>(1, ceil_div(lb, T));
        s = merge_device<K>(dA + t.a0, vC ? dvA + t.a0 : nullptr, la, dB + t.b0, vC ? dvB + t.b0 : nullptr, lb,
                            dC + off, vC ? dvC + off : nullptr, sM, pa, pb, pdl, dranks + rank_at);
        rank_at += merge_scratch_ints(pa, pb);
        if (s != SM_OK) break;
        cudaEventRecord(ev_mg[k], sM);
        cudaStreamWaitEvent(sD, ev_mg[k], 0);
        cudaError_t e = cudaMemcpyAsync(C + off, dC + off, L * kb, cudaMemcpyDefault, sD);
        if (e == cudaSuccess && vC) e = cudaMemcpyAsync(vC + off, dvC + off, L * 4, cudaMemcpyDefault, sD);
        if (e != cudaSuccess) s = fail_cuda(e, "cudaMemcpyAsync D2H");
    }
    for (cudaStream_t x : {sH, sM, sD}) {          // join: st waits for the three streams
        cudaEventRecord(ev_join, x);
        cudaStreamWaitEvent(st, ev_join, 0);
    }
    for (void* q : {(void*)dA, (void*)dB, (void*)dC, (void*)dvA, (void*)dvB, (void*)dvC, (void*)dranks}) dfree(q, st);
    return s;
}

// Device merges of n + m >= 2^31 elements (the kernels index 32-bit): the
// paper's Steps 1-4 once more at coarse granularity -- p blocks of <= 2^29
// elements per array, their block-start keys ranked by the rank kernel
// (64-bit), the cases on the host -- give 2p independent sub-merges of
// < 2^31 elements, each run by the whole device path.  One host
// synchronisation (the 2p ranks).
template <typename K>
static sm_status merge_large_device(const K* A, const uint32_t* vA, int64_t n, const K* B, const uint32_t* vB,
                                    int64_t m, K* C, uint32_t* vC, cudaStream_t st, bool pdl) {
    const int64_t p = std::max<int64_t>(1, ceil_div(std::max(n, m), 1ll << 29));
    K* keys = nullptr;
    int64_t* rk = nullptr;
    sm_status s = dalloc(&keys, 2 * p, st);
    if (s == SM_OK) s = dalloc(&rk, 2 * p, st);
    const unsigned g = (unsigned)ceil_div(p, 256);
    if (s == SM_OK) {
        k_block_start_keys<K><<<g, 256, 0, st>>>(A, n, p, keys);
        k_block_start_keys<K><<<g, 256, 0, st>>>(B, m, p, keys + p);
        k_rank_keys<K><<<g, 256, 0, st>>>(B, m, keys, p, 0, rk);          // Step 1: rank_low(A[x_i], B)
        k_rank_keys<K><<<g, 256, 0, st>>>(A, n, keys + p, p, 1, rk + p);  // Step 2: rank_high(B[y_j], A)
        s = check_launch("k_rank_keys (coarse)");
    }
    std::vector<int64_t> hr(2 * p);
    if (s == SM_OK) {
        cudaError_t e = cudaMemcpyAsync(hr.data(), rk, 2 * p * sizeof(int64_t), cudaMemcpyDeviceToHost, st);
        if (e == cudaSuccess) e = cudaStreamSynchronize(st);
        if (e != cudaSuccess) s = fail_cuda(e, "coarse ranks D2H");
    }
    dfree(keys, st);
    dfree(rk, st);
    if (s != SM_OK) return s;
    std::vector<int64_t> xb(p + 1), yb(p + 1);
    for (int64_t i = 0; i < p; ++i) {              // empty block starts: the other length (R4)
        xb[i] = hblock_start(n, p, i) < n ? hr[i] : m;
        yb[i] = hblock_start(m, p, i) < m ? hr[p + i] : n;
    }
    xb[p] = m;
    yb[p] = n;
    std::vector<SubMerge> tasks;
    plan_from_ranks(n, m, p, xb, yb, tasks);
    const int64_t T = tile_t((int)sizeof(K), vC != nullptr);
    for (const SubMerge& t : tasks) {
        const int64_t la = t.a1 - t.a0, lb = t.b1 - t.b0, off = t.a0 + t.b0;
        if (la + lb == 0) continue;
        s = merge_device<K>(A + t.a0, vC ? vA + t.a0 : nullptr, la, B + t.b0, vC ? vB + t.b0 : nullptr, lb, C + off,
                            vC ? vC + off : nullptr, st, std::max<int64_t>(1, ceil_div(la, T)),
                            std::max<int64_t>(1, ceil_div(lb, T)), pdl);
        if (s != SM_OK) break;
    }
    return s;
}

// Any size, device buffers.
template <typename K>
static sm_status merge_any_device(const K* A, const uint32_t* vA, int64_t n, const K* B, const uint32_t* vB, int64_t m,
                                  K* C, uint32_t* vC, cudaStream_t st, int64_t pA, int64_t pB, bool pdl,
                                  bool big = false) {
    if (n + m > (int64_t)INT_MAX) return merge_large_device<K>(A, vA, n, B, vB, m, C, vC, st, pdl);
    return merge_device<K>(A, vA, n, B, vB, m, C, vC, st, pA, pB, pdl, nullptr, big);
}

template <typename K>
static sm_status merge_entry(const K* A, const uint32_t* vA, int64_t n, const K* B, const uint32_t* vB, int64_t m,
                             K* C, uint32_t* vC, void* stream, const sm_options* opt) {
    DevGuard dev_guard(stream);
    NvtxCall nvtx_call("sm merge_stable");
    g_launches = 0;
    g_err[0] = 0;
    cudaStream_t st = (cudaStream_t)stream;
    if (n < 0 || m < 0) return fail_inval("negative size");
    if ((n && !A) || (m && !B) || ((n + m) && !C)) return fail_inval("NULL key pointer with nonzero size");
    if (!keys_aligned<K>({A, B, C})) return fail_inval("128-bit keys must be 16-byte aligned");
    if (vC) {
        if ((n && !vA) || (m && !vB)) return fail_inval("payload pointers must be all set or all NULL");
    } else if (vA || vB) {
        return fail_inval("payload pointers must be all set or all NULL");
    }
    const bool large = n + m > (int64_t)INT_MAX;   // sub-merges below 2^31 (merge_large_device)
    if (large && opt && (opt->p_A || opt->p_B || opt->block || (opt->flags & SM_FLAG_MERGE_PATH)))
        return fail_inval("n + m > 2^31 - 1 takes no p_A / p_B / block / merge-path options");
    const size_t kb = sizeof(K);
    const size_t cb = (size_t)(n + m);
    if (overlaps(C, cb * kb, A, n * kb) || overlaps(C, cb * kb, B, m * kb) || overlaps(C, cb * kb, vA, n * 4) ||
        overlaps(C, cb * kb, vB, m * 4) || overlaps(vC, cb * 4, A, n * kb) || overlaps(vC, cb * 4, B, m * kb) ||
        overlaps(vC, cb * 4, vA, n * 4) || overlaps(vC, cb * 4, vB, m * 4) || overlaps(C, cb * kb, vC, cb * 4))
        return SM_EALIAS;

    // a default plain merge of >= SM_K2_BIG_MIN elements takes the large tile shape (8-byte slots)
    const bool big = !(opt && (opt->p_A || opt->p_B || opt->block || (opt->flags & SM_FLAG_MERGE_PATH))) && !large &&
                     n + m >= SM_K2_BIG_MIN && !g_small_fuse;
    const int64_t NV = big ? tile_nv_big((int)sizeof(K), vC != nullptr) : tile_nv((int)sizeof(K), vC != nullptr);
    int64_t pA, pB;
    if (opt && (opt->p_A || opt->p_B)) {
        if (opt->p_A < 1 || opt->p_B < 1) return fail_inval("p_A and p_B must both be >= 1");
        pA = opt->p_A; pB = opt->p_B;
        if (pA > INT_MAX / 2 || pB > INT_MAX / 2) return fail_inval("p too large");
        if (ceil_div(n, pA) + ceil_div(m, pB) > NV) return fail_inval("task bound ceil(n/p_A)+ceil(m/p_B) exceeds the tile");
    } else {
        int64_t T = (opt && opt->block) ? opt->block : NV / SM_T_DIV;
        if (T < 1 || 2 * T > NV) return fail_inval("block size T must satisfy 1 <= 2T <= tile capacity");
        pA = std::max<int64_t>(1, ceil_div(n, T));
        pB = std::max<int64_t>(1, ceil_div(m, T));
    }
    if (large) pA = pB = 1;                         // (chosen per sub-merge)
    const bool pdl = !(opt && (opt->flags & SM_FLAG_NO_PDL));
    if (n + m == 0) return SM_OK;
    keep_pool(st);
    if (opt && (opt->flags & SM_FLAG_MERGE_PATH)) {
        if (is_host_ptr(A) || is_host_ptr(B) || is_host_ptr(vA) || is_host_ptr(vB) || is_host_ptr(C) ||
            is_host_ptr(vC))
            return fail_inval("the merge-path comparison takes device pointers only");
        return merge_path_device<K>(A, vA, n, B, vB, m, C, vC, st, pdl);
    }

    const bool host = is_host_ptr(A) || is_host_ptr(B) || is_host_ptr(vA) || is_host_ptr(vB) || is_host_ptr(C) ||
                      is_host_ptr(vC);
    if (!host) return merge_any_device<K>(A, vA, n, B, vB, m, C, vC, st, pA, pB, pdl, big);

    // Host inputs large enough to pipeline: sub-merges over two streams.
    const bool host_inputs = is_host_ptr(A) && is_host_ptr(B) && (!vC || (is_host_ptr(vA) && is_host_ptr(vB)));
    if (host_inputs && host_pipeline_blocks<K>(n, m, vC != nullptr) > 1)
        return merge_host_pipelined<K>(A, vA, n, B, vB, m, C, vC, st, pdl);

    // Host buffers: stage every buffer of the call through device memory.
    Stage sA, sB, svA, svB, sC, svC;
    sm_status s = SM_OK;
    if (s == SM_OK) s = stage_in(sA, A, n * kb, false, true, st);
    if (s == SM_OK) s = stage_in(sB, B, m * kb, false, true, st);
    if (s == SM_OK && vC) s = stage_in(svA, vA, n * 4, false, true, st);
    if (s == SM_OK && vC) s = stage_in(svB, vB, m * 4, false, true, st);
    if (s == SM_OK) s = stage_in(sC, C, cb * kb, true, false, st);
    if (s == SM_OK && vC) s = stage_in(svC, vC, cb * 4, true, false, st);
    if (s == SM_OK)
        s = merge_any_device<K>((const K*)sA.dev, (const uint32_t*)svA.dev, n, (const K*)sB.dev,
                                (const uint32_t*)svB.dev, m, (K*)sC.dev, (uint32_t*)svC.dev, st, pA, pB, pdl, big);
    sm_status s2 = SM_OK;
    for (Stage* x : {&sC, &svC, &sA, &sB, &svA, &svB}) {
        if (s != SM_OK) x->out = false;
        sm_status r = stage_out(*x, st);
        if (s2 == SM_OK) s2 = r;
    }
    return s != SM_OK ? s : s2;
}

// ------------------------------------------------------------ batched merge
// S independent stable merges in one call, through the
// sort rounds' segmented machinery (§3) with a segment
// table instead of equal runs.  Device pointers only.
template <typename K, typename PV = uint32_t>
static sm_status batch_entry(const K* A, const PV* vA, int64_t n, const int64_t* a_off, const K* B,
                             const PV* vB, int64_t m, const int64_t* b_off, int64_t S, K* C, PV* vC,
                             void* stream) {
    DevGuard dev_guard(stream);
    NvtxCall nvtx_call("sm merge_stable_batched");
    g_launches = 0;
    g_err[0] = 0;
    cudaStream_t st = (cudaStream_t)stream;
    if (n < 0 || m < 0 || S < 0) return fail_inval("negative size");
    if (S > (int64_t)(INT_MAX / 8)) return fail_inval("too many segments");
    if (n + m > (int64_t)INT_MAX) return fail_inval("n + m > 2^31 - 1");
    if ((n && !A) || (m && !B) || ((n + m) && !C)) return fail_inval("NULL key pointer with nonzero size");
    if (!keys_aligned<K>({A, B, C})) return fail_inval("128-bit keys must be 16-byte aligned");
    if (S && (!a_off || !b_off)) return fail_inval("NULL segment offsets");
    if (vC) {
        if ((n && !vA) || (m && !vB)) return fail_inval("payload pointers must be all set or all NULL");
    } else if (vA || vB) {
        return fail_inval("payload pointers must be all set or all NULL");
    }
    const size_t kb = sizeof(K), cb = (size_t)(n + m), vb = sizeof(PV);
    if (overlaps(C, cb * kb, A, n * kb) || overlaps(C, cb * kb, B, m * kb) || overlaps(C, cb * kb, vA, n * vb) ||
        overlaps(C, cb * kb, vB, m * vb) || overlaps(vC, cb * vb, A, n * kb) || overlaps(vC, cb * vb, B, m * kb) ||
        overlaps(vC, cb * vb, vA, n * vb) || overlaps(vC, cb * vb, vB, m * vb) || overlaps(C, cb * kb, vC, cb * vb))
        return SM_EALIAS;
    if (S == 0 || n + m == 0) return SM_OK;
    if (is_host_ptr(A) || is_host_ptr(B) || is_host_ptr(vA) || is_host_ptr(vB) || is_host_ptr(C) || is_host_ptr(vC) ||
        is_host_ptr(a_off) || is_host_ptr(b_off))
        return fail_inval("merge_stable_batched takes device pointers only");
    keep_pool(st);
    // large batches of 8-byte slots take K2's large tile shape (C6 / B1: K2 0.338 -> 0.330 ms)
    const bool big = n + m >= SM_K2_BIG_MIN;
    const int64_t T = big ? (vC ? K2ShapeBig<K, true, PV>::type::T : K2ShapeBig<K, false>::type::T)
                          : (vC ? K2Shape<K, true, PV>::type::T : K2Shape<K, false>::type::T);
    const int nblk = (int)ceil_div(S, BATCH_NT);
    GeomCounts gc;
    gc.tasks = ceil_div(n, T) + ceil_div(m, T) + 2 * S;      // sum over segments of p_A + p_B
    gc.items = gc.tasks + 2 * S;
    const size_t seg_bytes = ((size_t)S * sizeof(SegInfo) + 15) & ~(size_t)15;
    const size_t blk_bytes = ((size_t)nblk * sizeof(int2) + 15) & ~(size_t)15;
    char* scratch = nullptr;
    const size_t td_at = (seg_bytes + blk_bytes + 16 + (size_t)(2 * gc.items + gc.tasks) * 4 + 15) & ~(size_t)15;
    sm_status s = dalloc(&scratch, (int64_t)(td_at + (size_t)gc.tasks * sizeof(int4)), st);
    if (s != SM_OK) return s;
    int4* tdesc = (int4*)(scratch + td_at);
    SegInfo* segs = (SegInfo*)scratch;
    int2* blk = (int2*)(scratch + seg_bytes);
    int* totals = (int*)(scratch + seg_bytes + blk_bytes);
    int* ranks = totals + 4;
    int* rank_seg = ranks + gc.items;
    int* task_seg = rank_seg + gc.items;
    k_batch_count<<<nblk, BATCH_NT, 0, st>>>(a_off, b_off, (int)S, n, m, (int)T, (int)(2 * T), segs, blk);
    s = check_launch("k_batch_count");
    if (s == SM_OK) {
        k_batch_scan<<<1, BATCH_NT, 0, st>>>(blk, nblk, totals);
        s = check_launch("k_batch_scan");
    }
    if (s == SM_OK) {
        k_batch_apply<<<nblk, BATCH_NT, 0, st>>>(blk, (int)S, segs, task_seg, rank_seg);
        s = check_launch("k_batch_apply");
    }
    if (s == SM_OK) {
        Geom g{};
        g.S = (int)S; g.sort = 2; g.T = (int)T; g.segs = segs; g.totals = totals;
        g.ctr = totals + 2;                           // (totals[0..1]: tasks, rank entries)
        g.task_seg = task_seg; g.rank_seg = rank_seg;
        if (vC) s = launch_merge<K, true, PV>(A, vA, B, vB, C, vC, g, ranks, ranks, st, true, &gc, tdesc, big);
        else s = launch_merge<K, false, PV>(A, nullptr, B, nullptr, C, nullptr, g, ranks, ranks, st, true, &gc, tdesc,
                                            big);
    }
    dfree(scratch, st);
    return s;
}

// ------------------------------------------------------------ rank queries
template <typename K>
static sm_status ranks_entry(const K* X, int64_t len, const K* keys, int64_t nkeys, int32_t high, int64_t* out,
                             void* stream) {
    DevGuard dev_guard(stream);
    NvtxCall nvtx_call("sm ranks_stable");
    g_launches = 0;
    g_err[0] = 0;
    cudaStream_t st = (cudaStream_t)stream;
    if (len < 0 || nkeys < 0) return fail_inval("negative size");
    if ((len && !X) || (nkeys && (!keys || !out))) return fail_inval("NULL pointer with nonzero size");
    if (!keys_aligned<K>({X, keys})) return fail_inval("128-bit keys must be 16-byte aligned");
    if (nkeys == 0) return SM_OK;
    if (is_host_ptr(X) || is_host_ptr(keys) || is_host_ptr(out)) return fail_inval("device pointers only");
    k_rank_keys<K><<<(unsigned)ceil_div(nkeys, 256), 256, 0, st>>>(X, len, keys, nkeys, high ? 1 : 0, out);
    return check_launch("k_rank_keys");
}

// ------------------------------------------------------------ plan dump
static __global__ void k_widen(const int* __restrict__ in, int64_t* __restrict__ out, int count) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < count) out[i] = in[i];
}

template <typename K>
static sm_status plan_entry(const K* A, int64_t n, const K* B, int64_t m, int64_t pA, int64_t pB, int64_t* xbar,
                            int64_t* ybar, int64_t* tasks, void* stream) {
    DevGuard dev_guard(stream);
    g_launches = 0;
    g_err[0] = 0;
    cudaStream_t st = (cudaStream_t)stream;
    if (n < 0 || m < 0 || pA < 1 || pB < 1) return fail_inval("sizes / block counts");
    if ((n && !A) || (m && !B) || !xbar || !ybar || !tasks) return fail_inval("NULL pointer");
    if (!keys_aligned<K>({A, B})) return fail_inval("128-bit keys must be 16-byte aligned");
    if (n + m > (int64_t)INT_MAX || pA > INT_MAX / 4 || pB > INT_MAX / 4) return fail_inval("too large");
    if (is_host_ptr(A) || is_host_ptr(B) || is_host_ptr(xbar) || is_host_ptr(ybar) || is_host_ptr(tasks))
        return fail_inval("merge_plan_ex takes device pointers only");
    keep_pool(st);
    Geom g{};
    g.S = 1; g.pA = (int)pA; g.pB = (int)pB; g.n = (int)n; g.m = (int)m; g.L = 0; g.N = 0; g.sort = 0;
    int* ranks = nullptr;
    sm_status s = dalloc(&ranks, (pA + 1) + (pB + 1), st);
    if (s != SM_OK) return s;
    s = launch_cross_ranks<K>(A, B, g, geom_counts(g), ranks, ranks + pA + 1, st);
    if (s == SM_OK) {
        k_widen<<<(unsigned)((pA + 1 + 255) / 256), 256, 0, st>>>(ranks, xbar, (int)(pA + 1));
        s = check_launch("k_widen");
    }
    if (s == SM_OK) {
        k_widen<<<(unsigned)((pB + 1 + 255) / 256), 256, 0, st>>>(ranks + pA + 1, ybar, (int)(pB + 1));
        s = check_launch("k_widen");
    }
    if (s == SM_OK) {
        k_plan_dump<K><<<(unsigned)((pA + pB + 127) / 128), 128, 0, st>>>(g, ranks, ranks + pA + 1, tasks);
        s = check_launch("k_plan_dump");
    }
    dfree(ranks, st);
    return s;
}

// ------------------------------------------------------------ merge sort
template <typename K, bool HAS_V>
static sm_status launch_block_sort(const K* in, const uint32_t* vin, K* out, uint32_t* vout, int64_t N,
                                   unsigned blocks, cudaStream_t st) {
    constexpr int NT = k3_nt((int)sizeof(K), HAS_V), IPT = k3_ipt((int)sizeof(K), HAS_V);
    using Lay = K3Layout<K, HAS_V, NT, IPT>;
    auto kern = k_block_sort<K, HAS_V, NT, IPT>;
    static bool attr[SM_MAX_DEV];
    const int dev = current_device();
    if (dev >= SM_MAX_DEV || !attr[dev]) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Lay::SMEM);
        if (dev < SM_MAX_DEV) attr[dev] = true;
    }
    kern<<<blocks, NT, Lay::SMEM, st>>>(in, vin, out, vout, (int)N);
    return SM_OK;
}

#ifndef SM_K3H_NT
#define SM_K3H_NT 512
#endif
#ifndef SM_K3H_TILE
#define SM_K3H_TILE (SM_K3H_GROUPS == 2 ? 4096 : 8192)
#endif
#ifndef SM_K3H_TILE12
#define SM_K3H_TILE12 4096     // 8-byte integer keys + payload
#endif
#ifndef SM_K3H_TILE12F
#define SM_K3H_TILE12F 3072    // f64 keys + payload (4096 spills more there)
#endif
#ifndef SM_K3H_TILE4
#define SM_K3H_TILE4 (SM_K3H_GROUPS == 2 ? 5120 : 8192)
#endif
// K3H (row a8 with p = the SM count): one CTA per block of the paper's
// partition, radix-sorted through global memory (k_block_sort_hbm).
template <typename K, bool HAS_V>
static sm_status launch_block_sort_hbm(K* keys, uint32_t* vals, K* aux, uint32_t* vaux, K* aux2, uint32_t* vaux2,
                                       int64_t N, int64_t L0, int final_buf, cudaStream_t st) {
    if constexpr (sizeof(K) > 8) {
        return fail_inval("K3H takes keys of <= 8 bytes");
    } else {
        constexpr int NT = SM_K3H_NT;
        // 4-byte keys: tiles of 5120 per warp group (measured, C5 K3H 4.65 -> 4.43 ms, u32 keys-only
        // 2^28 8.29 -> 8.05 ms; 3072: 5.09; 6144 spills); 8-byte keys keep 4096 (keys-only: 5120 measured
        // 6% slower, 3584 / 4608 4-7%); with a payload 4096 for integer keys and 3072 for f64 (2^27 i64 +
        // payload 13.27 ms with 2048, 12.09 with 3072, 11.77 with 4096; f64 + payload 14.07 / 12.95 / 13.30)
        constexpr int TILE = sizeof(K) == 4 ? SM_K3H_TILE4
                                            : ((int)sizeof(K) + (HAS_V ? 4 : 0) <= 8 ? SM_K3H_TILE
                                               : (KeyOrd<K>::FLOAT ? SM_K3H_TILE12F : SM_K3H_TILE12));
        using Lay = K3HLayout<K, HAS_V, NT, TILE>;
        auto kern = k_block_sort_hbm<K, HAS_V, NT, TILE>;
        static bool attr[SM_MAX_DEV];
        const int dev = current_device();
        if (dev >= SM_MAX_DEV || !attr[dev]) {
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Lay::SMEM);
            if (dev < SM_MAX_DEV) attr[dev] = true;
        }
        kern<<<(unsigned)ceil_div(N, L0), NT, Lay::SMEM, st>>>(keys, vals, aux, vaux, aux2, vaux2, N, L0, final_buf,
                                                               g_dbg_ts);
        return SM_OK;
    }
}

static int sm_count() {
    static int n_d[SM_MAX_DEV];
    const int dev = current_device();
    int n = dev < SM_MAX_DEV ? n_d[dev] : 0;
    if (n == 0) {
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        if (n < 1) n = 1;
        if (dev < SM_MAX_DEV) n_d[dev] = n;
    }
    return n;
}

// The block count p of the one-block-per-SM phase 1: the SM count times
// SM_K3H_CTAS (CTAs per SM), optionally rounded down to a power of two.
#ifndef SM_K3H_CTAS
#define SM_K3H_CTAS 1
#endif
#ifndef SM_K3H_POW2
#define SM_K3H_POW2 0
#endif
static int64_t k3h_blocks() {
    int64_t p = (int64_t)sm_count() * SM_K3H_CTAS;
    if (SM_K3H_POW2)
        while (p & (p - 1)) p &= p - 1;
    return p;
}

// Phase 1 (row a8): the initial run length of a sort of N elements.  Keys of
// <= 8 bytes: the paper's p = the processing elements -- one block per SM
// (K3H), so phase 2 takes ceil(log2 p) rounds -- when those blocks are long
// enough to amortise the radix passes (>= K3H_MIN_RUN); else (and for
// 128-bit keys, or buffers not 16-byte aligned) the shared-memory runs of K3.
// `forced` (sm_options.sort_run, tests): k3_run selects K3, any other
// multiple of 16 selects K3H with that run length.
constexpr int64_t K3H_MIN_RUN = 1 << 15;
template <typename K>
static int64_t phase1_run(int64_t N, const void* keys, const void* vals, int64_t forced) {
    const int64_t r3 = k3_run((int)sizeof(K), vals != nullptr);
    if (forced) return forced;
    if (sizeof(K) > 8 || (((uintptr_t)keys | (uintptr_t)vals) & 15)) return r3;
    const int64_t L0 = ceil_div(ceil_div(N, k3h_blocks()), 16) * 16;
    return L0 >= K3H_MIN_RUN ? L0 : r3;
}

// Phase 2 with two rounds per HBM pass?  sm_set_sort_ways: 2 never, 4
// always (keys <= 8 bytes), 0 (the default) where measured faster.
static inline bool sort_four_ways(int key_bytes, bool has_vals, int64_t N) {
    if (key_bytes > 8 || g_sort_ways == 2) return false;
    if (g_sort_ways == 4) return true;
    // measured (scripts/time_sort.py, ways 4 against 2): faster from N ~ 1.5 M on for every
    // slot size (u32 + payload 2^21 0.200 / 0.210 ms, 2^24 0.851 / 0.993; i64 + payload 2^22
    // 0.509 / 0.565; u32 keys 2^24 0.636 / 0.728, 2^27 4.12 / 4.15) except 4-byte keys without
    // a payload at 2^28 (8.36 / 8.28: their HBM pass is half as long against the same merges)
    if (key_bytes <= 4 && !has_vals && N >= (1ll << 28)) return false;
    return N >= SM_K4_MIN_N;
}

template <typename K>
static sm_status sort_device(K* keys, uint32_t* vals, int64_t N, cudaStream_t st, bool pdl, int64_t run_opt = 0) {
    const int64_t R = phase1_run<K>(N, keys, vals, run_opt);   // initial run length
    const bool hbm = R != k3_run((int)sizeof(K), vals != nullptr);
    int rounds = 0;
    for (int64_t L = R; L < N; L *= 2) ++rounds;
    // phase 2 as HBM passes: two rounds per pass (k_tasks4) where
    // sort_four_ways says so, an odd round first as a plain round (K2)
    const bool four = sort_four_ways((int)sizeof(K), vals != nullptr, N);
    const int n4 = four ? rounds / 2 : 0;
    const int passes = rounds - n4;
    // buffers: the caller's (0), aux (1) and, for the one-block-per-SM phase 1,
    // aux2 (2): phase 1 ends in aux2 whatever its pass count, and the merge
    // rounds route through aux / aux2 so that the last one writes buffer 0
    K* kb[3] = {keys, nullptr, nullptr};
    uint32_t* vb[3] = {vals, nullptr, nullptr};
    int* ranks = nullptr;
    int4* tdesc = nullptr;
    sm_status s = dalloc(&kb[1], N, st);
    if (s == SM_OK && vals) s = dalloc(&vb[1], N, st);
    if (s == SM_OK && hbm) s = dalloc(&kb[2], N, st);
    if (s == SM_OK && hbm && vals) s = dalloc(&vb[2], N, st);
    // rank arrays for the largest round: S*(pA+1) + S*(pB+1) <= 2*(N/T + 2*S) entries
    const int64_t T = tile_t((int)sizeof(K), vals != nullptr);
    const int64_t rank_ints = 2 * (ceil_div(N, T) + 2 * ceil_div(N, R) + 2);
    if (s == SM_OK) s = dalloc(&ranks, rank_ints + 1, st);     // + K2's task counter
    if (s == SM_OK) s = dalloc(&tdesc, ceil_div(N, T) + 2 * ceil_div(N, R) + 2, st);   // tasks of a round
    // scratch of the two-rounds-per-pass partition, sized for its largest pass
    Pass4Scratch sc4{};
    void* sc4_mem = nullptr;
    if (s == SM_OK && n4 > 0) {
        int64_t ids = 0, nb = 0;
        for (int64_t L = R << (rounds - 2 * n4), k = 0; k < n4; ++k, L *= 4) {
            if constexpr (sizeof(K) <= 8) {
                const Geom4 g4 = vals ? geom4<K, true>(N, L) : geom4<K, false>(N, L);
                ids = std::max(ids, (int64_t)g4.G * 4 * g4.cmax);
                nb = std::max(nb, (int64_t)g4.G * (g4.TPG + 1));
            }
        }
        const int64_t b_spl = ceil_div(ids * (int64_t)sizeof(K), 16) * 16, b_rk = ids * 16,
                      b_fv = ceil_div(ids * 4, 16) * 16, b_bnd = nb * 16;
        s = dalloc((char**)&sc4_mem, b_spl + b_rk + b_fv + b_bnd + 16, st);
        if (s == SM_OK) {
            char* p = (char*)sc4_mem;
            sc4.rk = (int4*)p;
            sc4.bnd = (int4*)(p + b_rk);
            sc4.spl = p + b_rk + b_bnd;
            sc4.fv = (int*)(p + b_rk + b_bnd + b_spl);
            sc4.ctr = (int*)(p + b_rk + b_bnd + b_spl + b_fv);
        }
    }
    if (s == SM_OK) {
        int src;
        prof_before(PROF_K3, st);
        if (hbm) {
            src = passes > 0 ? 2 : 0;
            if (vals) s = launch_block_sort_hbm<K, true>(keys, vals, kb[1], vb[1], kb[2], vb[2], N, R, src, st);
            else s = launch_block_sort_hbm<K, false>(keys, nullptr, kb[1], nullptr, kb[2], nullptr, N, R, src, st);
        } else {
            // phase 1 lands in the buffer from which the rounds, alternating
            // between 0 and 1, end in 0
            src = passes % 2;
            const unsigned blocks = (unsigned)ceil_div(N, R);
            if (vals) s = launch_block_sort<K, true>(keys, vals, kb[src], vb[src], N, blocks, st);
            else s = launch_block_sort<K, false>(keys, nullptr, kb[src], nullptr, N, blocks, st);
        }
        prof_after(st);
        if (s == SM_OK) s = check_launch(hbm ? "k_block_sort_hbm" : "k_block_sort");
        int left = passes;
        for (int64_t L = R; s == SM_OK && L < N; L *= 2) {
            --left;
            const bool pass4 = left < n4;         // the last n4 passes take two rounds each
            // this round's target: buffer 0 when an even number of rounds
            // follow, else a buffer that is neither 0 nor the source
            const int dst = left % 2 == 0 ? 0 : (src == 1 ? 2 : 1);
            if (pass4) {
                if constexpr (sizeof(K) <= 8) {
                    if (vals) s = launch_pass4<K, true>(kb[src], vb[src], kb[dst], vb[dst], N, L, sc4, st, pdl);
                    else s = launch_pass4<K, false>(kb[src], nullptr, kb[dst], nullptr, N, L, sc4, st, pdl);
                }
                src = dst;
                L *= 2;                           // (the loop doubles it again)
                continue;
            }
            Geom g{};
            g.S = (int)ceil_div(N, 2 * L);
            g.pA = g.pB = (int)ceil_div(L, T);
            g.n = g.m = 0; g.L = (int)L; g.N = (int)N; g.sort = 1;
            g.ctr = ranks + rank_ints;
            int* xbar = ranks;
            int* ybar = ranks + (int64_t)g.S * (g.pA + 1);
            if (vals)
                s = launch_merge<K, true>(kb[src], vb[src], kb[src], vb[src], kb[dst], vb[dst], g, xbar, ybar, st, pdl,
                                          nullptr, tdesc);
            else
                s = launch_merge<K, false, uint32_t>(kb[src], nullptr, kb[src], nullptr, kb[dst], nullptr, g, xbar, ybar,
                                                     st, pdl, nullptr, tdesc);
            src = dst;
        }
    }
    dfree(sc4_mem, st);
    dfree(tdesc, st);
    dfree(ranks, st);
    for (int b = 2; b >= 1; --b) {
        dfree(vb[b], st);
        dfree(kb[b], st);
    }
    return s;
}

// Sorts of N >= 2^31 elements: chunks of 2^30 sorted by the device path,
// then pairwise rounds of (large) merges, ping-ponged through one auxiliary
// array -- the paper's phase 2 at chunk granularity (L407-416).
template <typename K>
static sm_status sort_large_device(K* keys, uint32_t* vals, int64_t N, cudaStream_t st, bool pdl) {
    const int64_t CH = 1ll << 30;
    sm_status s = SM_OK;
    for (int64_t c0 = 0; s == SM_OK && c0 < N; c0 += CH)
        s = sort_device<K>(keys + c0, vals ? vals + c0 : nullptr, std::min(CH, N - c0), st, pdl);
    K* aux = nullptr;
    uint32_t* vaux = nullptr;
    if (s == SM_OK) s = dalloc(&aux, N, st);
    if (s == SM_OK && vals) s = dalloc(&vaux, N, st);
    K* src = keys;
    uint32_t* vsrc = vals;
    K* dst = aux;
    uint32_t* vdst = vaux;
    for (int64_t L = CH; s == SM_OK && L < N; L *= 2) {
        for (int64_t s0 = 0; s == SM_OK && s0 < N; s0 += 2 * L) {
            const int64_t la = std::min(L, N - s0), lb = std::max<int64_t>(0, std::min(L, N - s0 - L));
            if (lb == 0) {                         // odd trailing run: copied (L409-410)
                cudaError_t e = cudaMemcpyAsync(dst + s0, src + s0, la * sizeof(K), cudaMemcpyDeviceToDevice, st);
                if (e == cudaSuccess && vals)
                    e = cudaMemcpyAsync(vdst + s0, vsrc + s0, la * 4, cudaMemcpyDeviceToDevice, st);
                if (e != cudaSuccess) s = fail_cuda(e, "cudaMemcpyAsync D2D");
                continue;
            }
            const int64_t T = tile_t((int)sizeof(K), vals != nullptr);
            s = merge_any_device<K>(src + s0, vals ? vsrc + s0 : nullptr, la, src + s0 + la,
                                    vals ? vsrc + s0 + la : nullptr, lb, dst + s0, vals ? vdst + s0 : nullptr, st,
                                    std::max<int64_t>(1, ceil_div(la, T)), std::max<int64_t>(1, ceil_div(lb, T)), pdl);
        }
        std::swap(src, dst);
        std::swap(vsrc, vdst);
    }
    if (s == SM_OK && src != keys) {
        cudaError_t e = cudaMemcpyAsync(keys, src, N * sizeof(K), cudaMemcpyDeviceToDevice, st);
        if (e == cudaSuccess && vals) e = cudaMemcpyAsync(vals, vsrc, N * 4, cudaMemcpyDeviceToDevice, st);
        if (e != cudaSuccess) s = fail_cuda(e, "cudaMemcpyAsync D2D");
    }
    dfree(vaux, st);
    dfree(aux, st);
    return s;
}

template <typename K>
static sm_status sort_any_device(K* keys, uint32_t* vals, int64_t N, cudaStream_t st, bool pdl, int64_t run_opt = 0) {
    return N > (int64_t)INT_MAX ? sort_large_device<K>(keys, vals, N, st, pdl)
                                : sort_device<K>(keys, vals, N, st, pdl, run_opt);
}

// Sort of host buffers (both keys and payloads on the host, N <= 2^31 - 1,
// >= 64 MB): a pipeline instead of upload -> sort -> download.
//   stream sH  uploads Q chunks (multiples of the block-sort run)
//   stream sM  sorts each chunk when its upload event fires (the device sort
//              on the chunk: block sort + the merge rounds inside it), then
//              the merge rounds across chunks but the last
//   last round the paper's Steps 1-4 at coarse granularity on the two
//              sorted halves (merge_large_device's partition, one host
//              synchronisation) give independent sub-merges; sD downloads
//              each as soon as it is merged
// so the uploads overlap the chunk sorts and the downloads the last round.
template <typename K>
static sm_status sort_host_pipelined(K* keys, uint32_t* vals, int64_t N, cudaStream_t st, bool pdl) {
    PipeStreams* ps = pipe_streams();
    if (!ps) return fail_cuda(cudaGetLastError(), "stream/event create");
    cudaStream_t sH = ps->sH, sM = ps->sM, sD = ps->sD;
    cudaEvent_t ev_fork = ps->ev_fork, ev_join = ps->ev_join;
    std::vector<cudaEvent_t>& evs = ps->ev_a;
    auto event = [&](size_t k) -> cudaEvent_t {
        while (evs.size() <= k) {
            cudaEvent_t e;
            if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) return nullptr;
            evs.push_back(e);
        }
        return evs[k];
    };
    const int64_t Q = 8;                                    // chunks
    const int64_t R = k3_run((int)sizeof(K), vals != nullptr);
    const int64_t Cs = ceil_div(ceil_div(N, Q), R) * R;
    const size_t kb = sizeof(K);
    K *dk = nullptr, *dk2 = nullptr;
    uint32_t *dv = nullptr, *dv2 = nullptr;
    sm_status s = dalloc(&dk, N, st);
    if (s == SM_OK) s = dalloc(&dk2, N, st);
    if (s == SM_OK && vals) s = dalloc(&dv, N, st);
    if (s == SM_OK && vals) s = dalloc(&dv2, N, st);
    if (s != SM_OK) {
        for (void* q : {(void*)dk, (void*)dk2, (void*)dv, (void*)dv2}) dfree(q, st);
        return s;
    }
    cudaEventRecord(ev_fork, st);
    for (cudaStream_t x : {sH, sM, sD}) cudaStreamWaitEvent(x, ev_fork, 0);
    // uploads and chunk sorts
    int64_t nch = 0;
    for (int64_t c0 = 0; s == SM_OK && c0 < N; c0 += Cs, ++nch) {
        const int64_t len = std::min(Cs, N - c0);
        cudaEvent_t e_up = event(2 * nch);
        if (!e_up) { s = fail_cuda(cudaGetLastError(), "event create"); break; }
        cudaError_t e = cudaMemcpyAsync(dk + c0, keys + c0, len * kb, cudaMemcpyHostToDevice, sH);
        if (e == cudaSuccess && vals) e = cudaMemcpyAsync(dv + c0, vals + c0, len * 4, cudaMemcpyHostToDevice, sH);
        if (e == cudaSuccess) e = cudaEventRecord(e_up, sH);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(sM, e_up, 0);
        if (e != cudaSuccess) { s = fail_cuda(e, "cudaMemcpyAsync H2D"); break; }
        s = sort_device<K>(dk + c0, vals ? dv + c0 : nullptr, len, sM, pdl);
    }
    // merge rounds across chunks, all but the last (ping-pong dk <-> dk2)
    K* src = dk;
    uint32_t* vsrc = dv;
    K* dst = dk2;
    uint32_t* vdst = dv2;
    const int64_t T = tile_t((int)kb, vals != nullptr);
    int64_t L = Cs;
    for (; s == SM_OK && 2 * L < N; L *= 2) {
        for (int64_t s0 = 0; s == SM_OK && s0 < N; s0 += 2 * L) {
            const int64_t la = std::min(L, N - s0), lb = std::max<int64_t>(0, std::min(L, N - s0 - L));
            if (lb == 0) {
                cudaError_t e = cudaMemcpyAsync(dst + s0, src + s0, la * kb, cudaMemcpyDeviceToDevice, sM);
                if (e == cudaSuccess && vals) e = cudaMemcpyAsync(vdst + s0, vsrc + s0, la * 4, cudaMemcpyDeviceToDevice, sM);
                if (e != cudaSuccess) s = fail_cuda(e, "cudaMemcpyAsync D2D");
                continue;
            }
            s = merge_device<K>(src + s0, vals ? vsrc + s0 : nullptr, la, src + s0 + la, vals ? vsrc + s0 + la : nullptr,
                                lb, dst + s0, vals ? vdst + s0 : nullptr, sM, std::max<int64_t>(1, ceil_div(la, T)),
                                std::max<int64_t>(1, ceil_div(lb, T)), pdl);
        }
        std::swap(src, dst);
        std::swap(vsrc, vdst);
    }
    // the last round: halves [0, L) and [L, N) (or a single chunk: download it)
    std::vector<SubMerge> tasks;
    const int64_t n = std::min(L, N), m = N - n;
    if (s == SM_OK && m > 0) {
        const int64_t p = std::max<int64_t>(4, std::min<int64_t>(16, ceil_div(N * (int64_t)kb, 64ll << 20)));
        K* bk = nullptr;
        int64_t* rk = nullptr;
        s = dalloc(&bk, 2 * p, sM);
        if (s == SM_OK) s = dalloc(&rk, 2 * p, sM);
        if (s == SM_OK) {
            const unsigned g = (unsigned)ceil_div(p, 256);
            k_block_start_keys<K><<<g, 256, 0, sM>>>(src, n, p, bk);
            k_block_start_keys<K><<<g, 256, 0, sM>>>(src + n, m, p, bk + p);
            k_rank_keys<K><<<g, 256, 0, sM>>>(src + n, m, bk, p, 0, rk);
            k_rank_keys<K><<<g, 256, 0, sM>>>(src, n, bk + p, p, 1, rk + p);
            s = check_launch("k_rank_keys (coarse)");
        }
        std::vector<int64_t> hr(2 * p);
        if (s == SM_OK) {
            cudaError_t e = cudaMemcpyAsync(hr.data(), rk, 2 * p * sizeof(int64_t), cudaMemcpyDeviceToHost, sM);
            if (e == cudaSuccess) e = cudaStreamSynchronize(sM);
            if (e != cudaSuccess) s = fail_cuda(e, "coarse ranks D2H");
        }
        dfree(bk, sM);
        dfree(rk, sM);
        if (s == SM_OK) {
            std::vector<int64_t> xb(p + 1), yb(p + 1);
            for (int64_t i = 0; i < p; ++i) {
                xb[i] = hblock_start(n, p, i) < n ? hr[i] : m;
                yb[i] = hblock_start(m, p, i) < m ? hr[p + i] : n;
            }
            xb[p] = m;
            yb[p] = n;
            plan_from_ranks(n, m, p, xb, yb, tasks);
        }
    } else if (s == SM_OK) {
        tasks.push_back({0, N, 0, 0});                      // one chunk: sorted in place already
    }
    for (size_t k = 0; s == SM_OK && k < tasks.size(); ++k) {
        const SubMerge& t = tasks[k];
        const int64_t la = t.a1 - t.a0, lb = t.b1 - t.b0, off = t.a0 + t.b0;
        if (la + lb == 0) continue;
        if (lb == 0 && m == 0) {                            // single chunk: src holds the result
            cudaError_t e = cudaStreamWaitEvent(sD, ev_fork, 0);
            cudaEvent_t e_m = event(2 * nch + 2 * k + 1);
            if (e == cudaSuccess) e = cudaEventRecord(e_m, sM);
            if (e == cudaSuccess) e = cudaStreamWaitEvent(sD, e_m, 0);
            if (e == cudaSuccess) e = cudaMemcpyAsync(keys, src, N * kb, cudaMemcpyDeviceToHost, sD);
            if (e == cudaSuccess && vals) e = cudaMemcpyAsync(vals, vsrc, N * 4, cudaMemcpyDeviceToHost, sD);
            if (e != cudaSuccess) s = fail_cuda(e, "cudaMemcpyAsync D2H");
            continue;
        }
        s = merge_device<K>(src + t.a0, vals ? vsrc + t.a0 : nullptr, la, src + n + t.b0,
                            vals ? vsrc + n + t.b0 : nullptr, lb, dst + off, vals ? vdst + off : nullptr, sM,
                            std::max<int64_t>(1, ceil_div(la, T)), std::max<int64_t>(1, ceil_div(lb, T)), pdl);
        if (s != SM_OK) break;
        cudaEvent_t e_m = event(2 * nch + 2 * k + 1);
        cudaError_t e = e_m ? cudaEventRecord(e_m, sM) : cudaErrorUnknown;
        if (e == cudaSuccess) e = cudaStreamWaitEvent(sD, e_m, 0);
        if (e == cudaSuccess) e = cudaMemcpyAsync(keys + off, dst + off, (la + lb) * kb, cudaMemcpyDeviceToHost, sD);
        if (e == cudaSuccess && vals)
            e = cudaMemcpyAsync(vals + off, vdst + off, (la + lb) * 4, cudaMemcpyDeviceToHost, sD);
        if (e != cudaSuccess) s = fail_cuda(e, "cudaMemcpyAsync D2H");
    }
    for (cudaStream_t x : {sH, sM, sD}) {
        cudaEventRecord(ev_join, x);
        cudaStreamWaitEvent(st, ev_join, 0);
    }
    for (void* q : {(void*)dk, (void*)dk2, (void*)dv, (void*)dv2}) dfree(q, st);
    return s;
}

template <typename K>
static sm_status sort_entry(K* keys, uint32_t* vals, int64_t N, void* stream, const sm_options* opt) {
    DevGuard dev_guard(stream);
    NvtxCall nvtx_call("sm mergesort_stable");
    g_launches = 0;
    g_err[0] = 0;
    cudaStream_t st = (cudaStream_t)stream;
    if (N < 0) return fail_inval("negative size");
    if (N && !keys) return fail_inval("NULL key pointer with nonzero size");
    if (!keys_aligned<K>({keys})) return fail_inval("128-bit keys must be 16-byte aligned");
    const int64_t run_opt = opt ? opt->sort_run : 0;
    if (run_opt && run_opt != k3_run((int)sizeof(K), vals != nullptr) &&
        (sizeof(K) > 8 || run_opt < 16 || run_opt % 16 || run_opt > (int64_t)INT_MAX / 2 ||
         (((uintptr_t)keys | (uintptr_t)vals) & 15)))
        return fail_inval("sort_run: the block-sort tile (sm_sort_run), or a multiple of 16 for the one-block-per-SM "
                          "phase 1 (keys <= 8 bytes, 16-byte-aligned buffers)");
    if (overlaps(keys, N * sizeof(K), vals, N * 4)) return SM_EALIAS;
    const bool pdl = !(opt && (opt->flags & SM_FLAG_NO_PDL));
    if (N <= 1) return SM_OK;
    keep_pool(st);
    if (!is_host_ptr(keys) && !is_host_ptr(vals)) return sort_any_device<K>(keys, vals, N, st, pdl, run_opt);
    if (is_host_ptr(keys) && (!vals || is_host_ptr(vals)) && N <= (int64_t)INT_MAX &&
        N * (int64_t)(sizeof(K) + (vals ? 4 : 0)) >= (64ll << 20))
        return sort_host_pipelined<K>(keys, vals, N, st, pdl);
    Stage sk, sv;
    sm_status s = stage_in(sk, keys, N * sizeof(K), true, true, st);
    if (s == SM_OK && vals) s = stage_in(sv, vals, N * 4, true, true, st);
    if (s == SM_OK) s = sort_any_device<K>((K*)sk.dev, (uint32_t*)sv.dev, N, st, pdl, run_opt);
    if (s != SM_OK) { sk.out = false; sv.out = false; }
    sm_status r1 = stage_out(sk, st), r2 = stage_out(sv, st);
    return s != SM_OK ? s : (r1 != SM_OK ? r1 : r2);
}

// ------------------------------------------------------------ wide payloads
// payload rows of vbytes bytes (any width: structs,
// 64-bit, ...).  The method runs unchanged with a uint32 index payload (the
// position of each element in A||B), then one gather moves the rows.
// Device pointers only.
static const int64_t WIDE_MAX_BYTES = 4096;

static sm_status gather_rows(const uint32_t* idx, const void* PA, int64_t n, const void* PB, void* out, int64_t rows,
                             int64_t vbytes, cudaStream_t st) {
    if (rows == 0) return SM_OK;
    const uintptr_t al = (uintptr_t)PA | (uintptr_t)PB | (uintptr_t)out | (uintptr_t)vbytes;
    const int64_t blocks = std::min<int64_t>(ceil_div(rows * vbytes / 4 + 1, 256), 148 * 16);
    const unsigned grid = (unsigned)std::max<int64_t>(1, blocks);
#define SM_GATHER(W)                                                                                            \
    k_gather_rows<W><<<grid, 256, 0, st>>>(idx, (const W*)PA, n, (const W*)PB, (W*)out, rows,                 \
                                           (int)(vbytes / (int64_t)sizeof(W)))
    if ((al & 15) == 0) SM_GATHER(uint4);
    else if ((al & 7) == 0) SM_GATHER(uint2);
    else if ((al & 3) == 0) SM_GATHER(uint32_t);
    else if ((al & 1) == 0) SM_GATHER(uint16_t);
    else SM_GATHER(uint8_t);
#undef SM_GATHER
    return check_launch("k_gather_rows");
}

static sm_status iota(uint32_t* out, int64_t count, cudaStream_t st) {
    if (count == 0) return SM_OK;
    k_iota<<<(unsigned)std::min<int64_t>(ceil_div(count, 256), 148 * 16), 256, 0, st>>>(out, count);
    return check_launch("k_iota");
}

static sm_status wide_check(int64_t vbytes, std::initializer_list<const void*> ptrs) {
    if (vbytes < 1 || vbytes > WIDE_MAX_BYTES) return fail_inval("payload row bytes must be in [1, 4096]");
    for (const void* p : ptrs)
        if (is_host_ptr(p)) return fail_inval("the wide-payload calls take device pointers only");
    return SM_OK;
}

template <typename K>
static sm_status merge_wide_entry(const K* A, const void* vA, int64_t n, const K* B, const void* vB, int64_t m, K* C,
                                  void* vC, int64_t vbytes, void* stream) {
    DevGuard dev_guard(stream);
    NvtxCall nvtx_call("sm merge_stable_wide");
    g_launches = 0;
    g_err[0] = 0;
    cudaStream_t st = (cudaStream_t)stream;
    if (n < 0 || m < 0) return fail_inval("negative size");
    if ((n && (!A || !vA)) || (m && (!B || !vB)) || ((n + m) && (!C || !vC)))
        return fail_inval("NULL pointer with nonzero size");
    if (!keys_aligned<K>({A, B, C})) return fail_inval("128-bit keys must be 16-byte aligned");
    if (n + m > (int64_t)INT_MAX) return fail_inval("n + m > 2^31 - 1");
    sm_status s = wide_check(vbytes, {A, B, C, vA, vB, vC});
    if (s != SM_OK) return s;
    const size_t kb = sizeof(K), cb = (size_t)(n + m), vb = (size_t)vbytes;
    if (overlaps(C, cb * kb, A, n * kb) || overlaps(C, cb * kb, B, m * kb) || overlaps(C, cb * kb, vA, n * vb) ||
        overlaps(C, cb * kb, vB, m * vb) || overlaps(vC, cb * vb, A, n * kb) || overlaps(vC, cb * vb, B, m * kb) ||
        overlaps(vC, cb * vb, vA, n * vb) || overlaps(vC, cb * vb, vB, m * vb) || overlaps(C, cb * kb, vC, cb * vb))
        return SM_EALIAS;
    if (n + m == 0) return SM_OK;
    keep_pool(st);
    if (vbytes == 8 && (((uintptr_t)vA | (uintptr_t)vB | (uintptr_t)vC) & 7) == 0) {
        // 8-byte rows (int64 / double / pairs of 32-bit): the fused path -- K2
        // moves them as its payload type, no index payload and no gather
        using Sh8 = typename K2Shape<K, true, uint64_t>::type;
        return merge_device<K, uint64_t>(A, (const uint64_t*)vA, n, B, (const uint64_t*)vB, m, C, (uint64_t*)vC, st,
                                         std::max<int64_t>(1, ceil_div(n, Sh8::T)),
                                         std::max<int64_t>(1, ceil_div(m, Sh8::T)), true);
    }
    uint32_t* idx = nullptr;
    s = dalloc(&idx, 2 * (n + m), st);
    if (s != SM_OK) return s;
    const int64_t NV = tile_nv((int)sizeof(K), true);
    s = iota(idx, n + m, st);
    if (s == SM_OK)
        s = merge_device<K>(A, idx, n, B, idx + n, m, C, idx + n + m, st, std::max<int64_t>(1, ceil_div(n, NV / 2)),
                            std::max<int64_t>(1, ceil_div(m, NV / 2)), true);
    if (s == SM_OK) s = gather_rows(idx + n + m, vA, n, vB, vC, n + m, vbytes, st);
    dfree(idx, st);
    return s;
}

template <typename K>
static sm_status batch_wide_entry(const K* A, const void* vA, int64_t n, const int64_t* a_off, const K* B,
                                  const void* vB, int64_t m, const int64_t* b_off, int64_t S, K* C, void* vC,
                                  int64_t vbytes, void* stream) {
    DevGuard dev_guard(stream);
    cudaStream_t st = (cudaStream_t)stream;
    g_launches = 0;
    g_err[0] = 0;
    if (n < 0 || m < 0 || S < 0) return fail_inval("negative size");
    if ((n && !vA) || (m && !vB) || ((n + m) && !vC)) return fail_inval("NULL payload pointer with nonzero size");
    if (n + m > (int64_t)INT_MAX) return fail_inval("n + m > 2^31 - 1");
    sm_status s = wide_check(vbytes, {vA, vB, vC});
    if (s != SM_OK) return s;
    const size_t kb = sizeof(K), cb = (size_t)(n + m), vb = (size_t)vbytes;
    if (overlaps(vC, cb * vb, A, n * kb) || overlaps(vC, cb * vb, B, m * kb) || overlaps(vC, cb * vb, vA, n * vb) ||
        overlaps(vC, cb * vb, vB, m * vb) || overlaps(C, cb * kb, vC, cb * vb) || overlaps(C, cb * kb, vA, n * vb) ||
        overlaps(C, cb * kb, vB, m * vb))
        return SM_EALIAS;
    if (S == 0 || n + m == 0)
        return batch_entry<K, uint32_t>(A, nullptr, n, a_off, B, nullptr, m, b_off, S, C, nullptr, stream);
    if (vbytes == 8 && (((uintptr_t)vA | (uintptr_t)vB | (uintptr_t)vC) & 7) == 0)   // fused 64-bit payload
        return batch_entry<K, uint64_t>(A, (const uint64_t*)vA, n, a_off, B, (const uint64_t*)vB, m, b_off, S, C,
                                        (uint64_t*)vC, stream);
    keep_pool(st);
    uint32_t* idx = nullptr;
    s = dalloc(&idx, 2 * (n + m), st);
    if (s != SM_OK) return s;
    s = iota(idx, n + m, st);
    const int64_t l0 = g_launches;
    if (s == SM_OK) s = batch_entry<K>(A, idx, n, a_off, B, idx + n, m, b_off, S, C, idx + n + m, stream);
    g_launches += l0;
    if (s == SM_OK) s = gather_rows(idx + n + m, vA, n, vB, vC, n + m, vbytes, st);
    dfree(idx, st);
    return s;
}

template <typename K>
static sm_status sort_wide_entry(K* keys, void* vals, int64_t N, int64_t vbytes, void* stream) {
    DevGuard dev_guard(stream);
    NvtxCall nvtx_call("sm mergesort_stable_wide");
    g_launches = 0;
    g_err[0] = 0;
    cudaStream_t st = (cudaStream_t)stream;
    if (N < 0) return fail_inval("negative size");
    if (N && (!keys || !vals)) return fail_inval("NULL pointer with nonzero size");
    if (!keys_aligned<K>({keys})) return fail_inval("128-bit keys must be 16-byte aligned");
    if (N > (int64_t)INT_MAX) return fail_inval("N > 2^31 - 1");
    sm_status s = wide_check(vbytes, {keys, vals});
    if (s != SM_OK) return s;
    if (overlaps(keys, N * sizeof(K), vals, (size_t)(N * vbytes))) return SM_EALIAS;
    if (N <= 1) return SM_OK;
    keep_pool(st);
    uint32_t* idx = nullptr;
    char* tmp = nullptr;
    s = dalloc(&idx, N, st);
    if (s == SM_OK) s = dalloc(&tmp, N * vbytes, st);
    if (s == SM_OK) s = iota(idx, N, st);
    if (s == SM_OK) s = sort_device<K>(keys, idx, N, st, true);
    if (s == SM_OK) s = gather_rows(idx, vals, N, nullptr, tmp, N, vbytes, st);
    if (s == SM_OK) {
        cudaError_t e = cudaMemcpyAsync(vals, tmp, (size_t)(N * vbytes), cudaMemcpyDeviceToDevice, st);
        if (e != cudaSuccess) s = fail_cuda(e, "cudaMemcpyAsync");
    }
    dfree(tmp, st);
    dfree(idx, st);
    return s;
}

}  // namespace sm

// ================================================================ C ABI
// (instantiated per key type in abi_*.cu)

// K: the key type the kernels see; C: its bits as the ABI type (C = K, or
// the base type of Desc<C> for the descending-order entries).
#define SM_DEFINE_ABI(SUF, K, C)                                                                                \
    sm_status merge_stable_##SUF(const C* keys_A, const uint32_t* vals_A, int64_t n, const C* keys_B,          \
                                 const uint32_t* vals_B, int64_t m, C* out_keys, uint32_t* out_vals,          \
                                 void* stream) {                                                               \
        return sm::merge_entry<K>((const K*)keys_A, vals_A, n, (const K*)keys_B, vals_B, m, (K*)out_keys,      \
                                  out_vals, stream, nullptr);                                                  \
    }                                                                                                           \
    sm_status merge_stable_ex_##SUF(const C* keys_A, const uint32_t* vals_A, int64_t n, const C* keys_B,       \
                                    const uint32_t* vals_B, int64_t m, C* out_keys, uint32_t* out_vals,       \
                                    void* stream, const sm_options* opt) {                                     \
        return sm::merge_entry<K>((const K*)keys_A, vals_A, n, (const K*)keys_B, vals_B, m, (K*)out_keys,      \
                                  out_vals, stream, opt);                                                      \
    }                                                                                                           \
    sm_status merge_plan_ex_##SUF(const C* keys_A, int64_t n, const C* keys_B, int64_t m, int64_t p_A,         \
                                  int64_t p_B, int64_t* xbar, int64_t* ybar, int64_t* tasks, void* stream) {   \
        return sm::plan_entry<K>((const K*)keys_A, n, (const K*)keys_B, m, p_A, p_B, xbar, ybar, tasks,        \
                                 stream);                                                                      \
    }                                                                                                           \
    sm_status merge_stable_batched_##SUF(const C* keys_A, const uint32_t* vals_A, int64_t n,                   \
                                         const int64_t* a_offsets, const C* keys_B, const uint32_t* vals_B,    \
                                         int64_t m, const int64_t* b_offsets, int64_t S, C* out_keys,          \
                                         uint32_t* out_vals, void* stream) {                                   \
        return sm::batch_entry<K>((const K*)keys_A, vals_A, n, a_offsets, (const K*)keys_B, vals_B, m,        \
                                  b_offsets, S, (K*)out_keys, out_vals, stream);                               \
    }                                                                                                           \
    sm_status ranks_stable_##SUF(const C* X, int64_t len, const C* keys, int64_t nkeys, int32_t high,        \
                                 int64_t* out, void* stream) {                                                 \
        return sm::ranks_entry<K>((const K*)X, len, (const K*)keys, nkeys, high, out, stream);                  \
    }                                                                                                           \
    sm_status mergesort_stable_##SUF(C* keys, uint32_t* vals, int64_t N, void* stream) {                       \
        return sm::sort_entry<K>((K*)keys, vals, N, stream, nullptr);                                           \
    }                                                                                                           \
    sm_status mergesort_stable_ex_##SUF(C* keys, uint32_t* vals, int64_t N, void* stream,                      \
                                        const sm_options* opt) {                                               \
        return sm::sort_entry<K>((K*)keys, vals, N, stream, opt);                                               \
    }                                                                                                           \
    sm_status merge_stable_wide_##SUF(const C* keys_A, const void* vals_A, int64_t n, const C* keys_B,         \
                                      const void* vals_B, int64_t m, C* out_keys, void* out_vals,             \
                                      int64_t val_bytes, void* stream) {                                       \
        return sm::merge_wide_entry<K>((const K*)keys_A, vals_A, n, (const K*)keys_B, vals_B, m, (K*)out_keys, \
                                       out_vals, val_bytes, stream);                                           \
    }                                                                                                           \
    sm_status merge_stable_batched_wide_##SUF(const C* keys_A, const void* vals_A, int64_t n,                  \
                                              const int64_t* a_offsets, const C* keys_B, const void* vals_B,   \
                                              int64_t m, const int64_t* b_offsets, int64_t S, C* out_keys,     \
                                              void* out_vals, int64_t val_bytes, void* stream) {               \
        return sm::batch_wide_entry<K>((const K*)keys_A, vals_A, n, a_offsets, (const K*)keys_B, vals_B, m,   \
                                       b_offsets, S, (K*)out_keys, out_vals, val_bytes, stream);               \
    }                                                                                                           \
    sm_status mergesort_stable_wide_##SUF(C* keys, void* vals, int64_t N, int64_t val_bytes, void* stream) {   \
        return sm::sort_wide_entry<K>((K*)keys, vals, N, val_bytes, stream);                                    \
    }
