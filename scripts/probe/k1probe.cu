// Probe: where the time of the cross-rank searches goes (C2 shape: 33158
// searches of random keys in a sorted 2^26 int array).
#include <cuda_runtime.h>
#include <stdio.h>
#include "sm_device.cuh"
#include "sm_kernels.cuh"
using namespace sm;

template <int MODE>
__global__ void __launch_bounds__(256) k_probe(const int* __restrict__ X, int len, const int* __restrict__ keys, int nk,
                                               int* out, int depth) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nk) return;
    const int x = keys[i];
    int r = 0;
    if (MODE == 0) r = rank_kary<int, 4>(X, len, x, false);
    if (MODE == 1) {   // binary search
        int lo = 0, n = len;
        while (n > 0) { const int h = n >> 1; const bool right = __ldg(X + lo + h) < x; lo = right ? lo + h + 1 : lo; n = right ? n - h - 1 : h; }
        r = lo;
    }
    if (MODE == 2) {   // `depth` dependent random loads only (no search)
        int a = (int)(((unsigned)x * 2654435761u) % (unsigned)len);
        for (int k = 0; k < depth; ++k) { const int v = __ldg(X + a); a = (int)(((unsigned)(v + k) * 2654435761u) % (unsigned)len); }
        r = a;
    }
    if (MODE == 3) {   // 8-ary
        r = rank_kary<int, 8>(X, len, x, false);
    }
    out[i] = r;
}

int main() {
    const int len = 1 << 26, nk = 33158;
    int *X, *keys, *out;
    cudaMalloc(&X, (size_t)len * 4); cudaMalloc(&keys, nk * 4); cudaMalloc(&out, nk * 4);
    int* h = (int*)malloc((size_t)len * 4);
    for (int i = 0; i < len; ++i) h[i] = 2 * i;
    cudaMemcpy(X, h, (size_t)len * 4, cudaMemcpyHostToDevice);
    unsigned s = 1;
    for (int i = 0; i < nk; ++i) { s = s * 1664525u + 1013904223u; h[i] = (int)(s % (2u * len)); }
    // sorted keys like block starts
    for (int i = 0; i < nk; ++i) h[i] = (int)((long long)i * (2ll * len) / nk) + 1;
    cudaMemcpy(keys, h, nk * 4, cudaMemcpyHostToDevice);
    char* flush; cudaMalloc(&flush, 512 << 20);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    auto timeit = [&](auto launch, const char* name) {
        float best = 1e9;
        for (int rep = 0; rep < 5; ++rep) {
            cudaMemset(flush, rep, 512 << 20);
            cudaEventRecord(e0); launch(); cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1); best = ms < best ? ms : best;
        }
        printf("%-28s %8.2f us\n", name, best * 1e3);
    };
    const unsigned g = (nk + 255) / 256;
    timeit([&] { k_probe<0><<<g, 256>>>(X, len, keys, nk, out, 0); }, "4-ary + window tail");
    timeit([&] { k_probe<3><<<g, 256>>>(X, len, keys, nk, out, 0); }, "8-ary + window tail");
    timeit([&] { k_probe<1><<<g, 256>>>(X, len, keys, nk, out, 0); }, "binary");
    for (int d : {1, 2, 4, 8, 13, 26}) {
        char nm[64]; snprintf(nm, 64, "%d dependent random loads", d);
        timeit([&] { k_probe<2><<<g, 256>>>(X, len, keys, nk, out, d); }, nm);
    }
    timeit([&] { k_probe<2><<<1, 32>>>(X, len, keys, 32, out, 26); }, "26 dep loads, 32 threads");
    return 0;
}
