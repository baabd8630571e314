// sm_common.cu -- the library's globals (per-thread error text and launch
// count, the CUDA-event profiler) and the C-ABI calls that do not depend on
// the key type (include/stablemerge.h).
#include "sm_host.cuh"
#include <nvtx3/nvToolsExt.h>

namespace sm {

thread_local char g_err[512] = "";
thread_local int64_t g_launches = 0;

sm_status fail_cuda(cudaError_t e, const char* what) {
    snprintf(g_err, sizeof(g_err), "%s: %s", what, cudaGetErrorString(e));
    return SM_ECUDA;
}

sm_status fail_inval(const char* what) {
    snprintf(g_err, sizeof(g_err), "invalid argument: %s", what);
    return SM_EINVAL;
}

int g_k1_variant = 0;
int g_small_fuse = 0;
int g_sort_ways = 0;
uint32_t* g_dbg_cover = nullptr;
unsigned long long* g_dbg_ts = nullptr;
bool g_prof_on = false;
std::vector<ProfRec> g_prof_pool;
size_t g_prof_used = 0;

// NVTX ranges around the launches of the method's kernels (host side; a
// tool such as nsys / ncu --nvtx shows them, otherwise a pointer test each)
static const char* const kKernelRange[PROF_KINDS] = {"sm K1 cross ranks (Steps 1-2)",
                                                     "sm K2 tasks (Steps 3-4, copy / merge)",
                                                     "sm K3 block sort (phase 1)"};
void prof_before(int kind, cudaStream_t st) {
    nvtxRangePushA(kind >= 0 && kind < PROF_KINDS ? kKernelRange[kind] : "sm kernel");
    if (!g_prof_on) return;
    if (g_prof_used == g_prof_pool.size()) {
        ProfRec r;
        cudaEventCreate(&r.a);
        cudaEventCreate(&r.b);
        g_prof_pool.push_back(r);
    }
    g_prof_pool[g_prof_used].kind = kind;
    cudaEventRecord(g_prof_pool[g_prof_used].a, st);
}

void prof_after(cudaStream_t st) {
    nvtxRangePop();
    if (!g_prof_on) return;
    cudaEventRecord(g_prof_pool[g_prof_used].b, st);
    ++g_prof_used;
}

sm_status check_launch(const char* what) {
    ++g_launches;
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? SM_OK : fail_cuda(e, what);
}

}  // namespace sm

extern "C" {

sm_status sm_debug_cover(uint32_t* cover, int64_t len) {
#ifdef SM_DEBUG
    if (cover && len <= 0) return sm::fail_inval("sm_debug_cover: length");
    sm::g_dbg_cover = cover;
    return SM_OK;
#else
    (void)cover;
    (void)len;
    return sm::fail_inval("sm_debug_cover: not an SM_DEBUG build");
#endif
}

#ifdef SM_K2_TSTAMP
// experiment builds only (not in the header): later K2 launches record their
// per-CTA event times into ts[8 * CTA + slot] (device memory; NULL stops)
void sm_debug_k2_timestamps(unsigned long long* ts) { sm::g_dbg_ts = ts; }
#endif

int32_t sm_is_debug_build(void) {
#ifdef SM_DEBUG
    return 1;
#else
    return 0;
#endif
}

void sm_set_k1_variant(int32_t variant) { sm::g_k1_variant = (variant >= 0 && variant <= 3) ? variant : 0; }

void sm_set_small_fuse(int32_t on) { sm::g_small_fuse = on != 0; }

void sm_set_sort_ways(int32_t ways) { sm::g_sort_ways = (ways == 2 || ways == 4) ? ways : 0; }

sm_status sm_plan_from_ranks(int64_t n, int64_t m, int64_t p, const int64_t* xbar, const int64_t* ybar,
                             int64_t* tasks) {
    if (n < 0 || m < 0 || p < 1 || !xbar || !ybar || !tasks) return sm::fail_inval("sm_plan_from_ranks arguments");
    std::vector<int64_t> xb(xbar, xbar + p + 1), yb(ybar, ybar + p + 1);
    std::vector<sm::SubMerge> t;
    sm::plan_from_ranks(n, m, p, xb, yb, t);
    for (size_t k = 0; k < t.size(); ++k) {
        tasks[4 * k] = t[k].a0;
        tasks[4 * k + 1] = t[k].a1;
        tasks[4 * k + 2] = t[k].b0;
        tasks[4 * k + 3] = t[k].b1;
    }
    return SM_OK;
}

sm_status sm_plan_tasks(int64_t n, int64_t m, int64_t pA, int64_t pB, const int64_t* xbar, const int64_t* ybar,
                        int64_t* tasks) {
    if (n < 0 || m < 0 || pA < 1 || pB < 1 || !xbar || !ybar || !tasks) return sm::fail_inval("sm_plan_tasks arguments");
    std::vector<int64_t> xb(xbar, xbar + pA + 1), yb(ybar, ybar + pB + 1);
    std::vector<sm::SubMerge> t;
    sm::plan_tasks_host(n, m, pA, pB, xb, yb, t);
    for (size_t k = 0; k < t.size(); ++k) {
        tasks[4 * k] = t[k].a0;
        tasks[4 * k + 1] = t[k].a1;
        tasks[4 * k + 2] = t[k].b0;
        tasks[4 * k + 3] = t[k].b1;
    }
    return SM_OK;
}

int64_t sm_tile_capacity(int32_t key_bytes, int32_t has_vals) {
    return sm::tile_nv(key_bytes, has_vals != 0);
}

int64_t sm_sort_run(int32_t key_bytes, int32_t has_vals) {
    return sm::k3_run(key_bytes, has_vals != 0);
}

int64_t sm_sort_run_n(int32_t key_bytes, int32_t has_vals, int64_t n) {
    // phase1_run's rule for 16-byte-aligned buffers, on the current device
    const int64_t r3 = sm::k3_run(key_bytes, has_vals != 0);
    if (key_bytes > 8 || n <= 0) return r3;
    const int64_t L0 = sm::ceil_div(sm::ceil_div(n, sm::k3h_blocks()), 16) * 16;
    return L0 >= sm::K3H_MIN_RUN ? L0 : r3;
}

int32_t sm_sort_merge_passes(int32_t key_bytes, int32_t has_vals, int64_t n) {
    // sort_device's phase-2 plan: ceil(log2(n / R)) rounds, two per pass
    // where sort_four_ways holds (an odd round on its own)
    const int64_t R = sm_sort_run_n(key_bytes, has_vals, n);
    int32_t rounds = 0;
    for (int64_t L = R; L < n; L *= 2) ++rounds;
    return sm::sort_four_ways(key_bytes, has_vals != 0, n) ? rounds - rounds / 2 : rounds;
}

const char* sm_status_string(sm_status s) {
    switch (s) {
        case SM_OK: return "SM_OK";
        case SM_EINVAL: return "SM_EINVAL: invalid argument";
        case SM_EALIAS: return "SM_EALIAS: output overlaps an input";
        case SM_ENOMEM: return "SM_ENOMEM: scratch allocation failed";
        case SM_ECUDA: return "SM_ECUDA: CUDA error";
    }
    return "unknown status";
}

const char* sm_last_error(void) { return sm::g_err; }

int64_t sm_last_launch_count(void) { return sm::g_launches; }

void sm_profile_enable(int on) {
    sm::g_prof_on = on != 0;
    sm::g_prof_used = 0;
}

sm_status sm_profile_read(int kind, double* total_ms, int64_t* launches) {
    double t = 0.0;
    int64_t c = 0;
    for (size_t i = 0; i < sm::g_prof_used; ++i) {
        const sm::ProfRec& r = sm::g_prof_pool[i];
        if (r.kind != kind) continue;
        cudaError_t e = cudaEventSynchronize(r.b);
        if (e != cudaSuccess) return sm::fail_cuda(e, "cudaEventSynchronize");
        float ms = 0.f;
        e = cudaEventElapsedTime(&ms, r.a, r.b);
        if (e != cudaSuccess) return sm::fail_cuda(e, "cudaEventElapsedTime");
        t += ms;
        ++c;
    }
    if (total_ms) *total_ms = t;
    if (launches) *launches = c;
    return SM_OK;
}

}  // extern "C"
