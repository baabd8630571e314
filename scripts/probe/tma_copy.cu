// Probe: TMA bulk-copy streaming through shared memory -- what DRAM rate a
// K2-like pipeline (producer bulk loads -> stage -> storer bulk stores) reaches
// for different access patterns, with no compute.  Experiment tool only.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_copy tma_copy.cu
//   ./tma_copy <pattern 1|2|3> <chunk KB> <stages> <ctas/SM> [strided 1|0]
// pattern 1: C[i-chunk] <- A[i-chunk]                     (one read stream)
// pattern 2: C[i-chunk] <- A[half chunk] ++ B[half chunk]  (two read streams, like a merge task)
// pattern 3: like 2, but B's half from a place 1/3 of the array away (unrelated windows)
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(b)), "r"(c)); }
__device__ __forceinline__ void expect(uint64_t* b, uint32_t bytes) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(b)), "r"(bytes) : "memory"); }
__device__ __forceinline__ void arrive(uint64_t* b) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(b)) : "memory"); }
__device__ __forceinline__ void wait(uint64_t* b, uint32_t ph) {
    asm volatile("{\n.reg .pred P;\nW: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n@!P bra W;\n}" ::"r"(sa(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void g2s(void* d, const void* s, uint32_t n, uint64_t* b) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(sa(d)), "l"(s), "r"(n), "r"(sa(b)) : "memory");
}
__device__ __forceinline__ void s2g(void* d, const void* s, uint32_t n) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(d), "r"(sa(s)), "r"(n) : "memory");
}

__global__ void __launch_bounds__(64) k(const char* A, const char* B, char* C, long long chunks, int chunk, int stages,
                                       int pattern, int strided, long long bshift) {
    extern __shared__ __align__(128) char sm[];
    uint64_t* full = (uint64_t*)(sm + (size_t)stages * chunk);
    uint64_t* empty = full + stages;
    if (threadIdx.x == 0) {
        for (int s = 0; s < stages; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    const long long per = (chunks + gridDim.x - 1) / gridDim.x;
    auto chunk_of = [&](long long it) -> long long {
        return strided ? blockIdx.x + it * (long long)gridDim.x : blockIdx.x * per + it;
    };
    const long long nit = strided ? (chunks - blockIdx.x + gridDim.x - 1) / gridDim.x : min(per, chunks - blockIdx.x * per);
    if (threadIdx.x == 0) {                       // producer
        for (long long it = 0; it < nit; ++it) {
            const int s = it % stages;
            if (it >= stages) wait(&empty[s], ((it / stages) - 1) & 1);
            const long long c = chunk_of(it);
            char* st = sm + (size_t)s * chunk;
            expect(&full[s], chunk);
            if (pattern == 1) g2s(st, A + c * chunk, chunk, &full[s]);
            else {
                const int h = chunk / 2;
                g2s(st, A + c * h, h, &full[s]);
                const long long bc = pattern == 3 ? (c + bshift) % chunks : c;
                g2s(st + h, B + bc * h, h, &full[s]);
            }
        }
    } else if (threadIdx.x == 32) {               // storer
        for (long long it = 0; it < nit; ++it) {
            const int s = it % stages;
            wait(&full[s], (it / stages) & 1);
            s2g(C + chunk_of(it) * chunk, sm + (size_t)s * chunk, chunk);
            asm volatile("cp.async.bulk.commit_group;");
            asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
            arrive(&empty[s]);
        }
        asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
}

int main(int argc, char** argv) {
    const int pattern = argc > 1 ? atoi(argv[1]) : 1, ckb = argc > 2 ? atoi(argv[2]) : 32;
    const int stages = argc > 3 ? atoi(argv[3]) : 3, per_sm = argc > 4 ? atoi(argv[4]) : 2;
    const int strided = argc > 5 ? atoi(argv[5]) : 1;
    const long long bytes = 1ll << 30;            // 1 GiB output per step (C2: 0.5 GiB in + 0.5 out)
    const int chunk = ckb * 1024;
    const long long chunks = bytes / chunk;
    char *A, *B, *C;
    cudaMalloc(&A, bytes); cudaMalloc(&B, bytes); cudaMalloc(&C, bytes);
    cudaMemset(A, 1, bytes); cudaMemset(B, 2, bytes);
    const int smem = stages * chunk + 2 * stages * 8;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    const int grid = nsm * per_sm;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int w = 0; w < 3; ++w) k<<<grid, 64, smem>>>(A, B, C, chunks, chunk, stages, pattern, strided, chunks / 3);
    cudaEventRecord(e0);
    const int reps = 20;
    for (int r = 0; r < reps; ++r) k<<<grid, 64, smem>>>(A, B, C, chunks, chunk, stages, pattern, strided, chunks / 3);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    const cudaError_t e = cudaGetLastError();
    printf("pattern %d chunk %3d KB stages %d ctas/SM %d %s: %.3f ms/step  %.0f GB/s (read+write)  %s\n", pattern, ckb, stages,
           per_sm, strided ? "strided" : "blocked", ms / reps, 2.0 * bytes / (ms / reps * 1e-3) / 1e9, cudaGetErrorString(e));
    return 0;
}
