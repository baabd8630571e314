// Probe: do H2D and D2H overlap across two non-blocking streams forked from the legacy stream?
#include <cuda_runtime.h>
#include <stdio.h>
#include <chrono>
int main(int argc, char** argv) {
    const size_t n = 256ull << 20;   // bytes per direction
    const int P = 16;
    char *ha, *hc, *da, *dc;
    cudaHostAlloc(&ha, n, 0); cudaHostAlloc(&hc, n, 0);
    cudaMalloc(&da, n); cudaMalloc(&dc, n);
    cudaStream_t s[2];
    for (int k = 0; k < 2; ++k) cudaStreamCreateWithFlags(&s[k], cudaStreamNonBlocking);
    cudaEvent_t fork, join[2];
    cudaEventCreateWithFlags(&fork, cudaEventDisableTiming);
    for (int k = 0; k < 2; ++k) cudaEventCreateWithFlags(&join[k], cudaEventDisableTiming);
    for (int mode = 0; mode < 6; ++mode) {
        cudaMemcpyKind h2d = (mode & 1) ? cudaMemcpyDefault : cudaMemcpyHostToDevice;
        cudaMemcpyKind d2h = (mode & 1) ? cudaMemcpyDefault : cudaMemcpyDeviceToHost;
        cudaStream_t st = (mode & 2) ? s[0] : (cudaStream_t)0;
        const bool pool = mode >= 4;
        auto run = [&]() {
            char *pa = da, *pc = dc;
            if (pool) { cudaMallocAsync((void**)&pa, n, st); cudaMallocAsync((void**)&pc, n, st); }
            char *da = pa, *dc = pc;
            cudaEventRecord(fork, st);
            cudaStreamWaitEvent(s[0], fork, 0); cudaStreamWaitEvent(s[1], fork, 0);
            const size_t ch = n / P;
            for (int k = 0; k < P; ++k) {
                cudaStream_t ss = s[k & 1];
                cudaMemcpyAsync(da + k * ch, ha + k * ch, ch, h2d, ss);
                cudaMemcpyAsync(hc + k * ch, dc + k * ch, ch, d2h, ss);
            }
            for (int j = 0; j < 2; ++j) { cudaEventRecord(join[j], s[j]); cudaStreamWaitEvent(st, join[j], 0); }
            if (pool) { cudaFreeAsync(pa, st); cudaFreeAsync(pc, st); }
        };
        run(); cudaDeviceSynchronize();
        auto t0 = std::chrono::steady_clock::now();
        for (int r = 0; r < 5; ++r) run();
        cudaStreamSynchronize(st); cudaDeviceSynchronize();
        double dt = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() / 5;
        printf("mode %d (kind %s, st %s, pool %d): %.2f ms, %.1f GB/s aggregate\n", mode, (mode & 1) ? "Default" : "explicit",
               (mode & 2) ? "side" : "legacy", (int)pool, dt * 1e3, 2 * n / dt / 1e9);
    }
    return 0;
}
