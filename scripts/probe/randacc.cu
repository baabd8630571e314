// Probe: random-access DRAM rate on B200 for different access granularities
// (the bottom levels of the cross-rank searches are private random probes).
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdint.h>

__device__ __forceinline__ uint64_t mix(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}

// G lanes read G*W contiguous 4-byte words (W per lane, W in {1,4,8}) at a
// random GW-aligned location; R rounds of dependent accesses per group.
template <int G, int W>
__global__ void k_rand(const uint32_t* __restrict__ buf, uint64_t words, int rounds, uint32_t* out) {
    const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const uint64_t grp = tid / G;
    const int sub = threadIdx.x % G;
    uint32_t acc = 0;
    uint64_t st = grp * 0x9e3779b97f4a7c15ull;
    const uint64_t slots = words / (G * W);
    for (int r = 0; r < rounds; ++r) {
        st = mix(st + acc);                         // dependent on the previous round
        const uint64_t base = (st % slots) * (G * W) + sub * W;
        if (W == 1) acc += __ldg(buf + base);
        else if (W == 4) { uint4 v = __ldg((const uint4*)(buf + base)); acc += v.x ^ v.y ^ v.z ^ v.w; }
        else { uint4 v = __ldg((const uint4*)(buf + base)); uint4 u = __ldg((const uint4*)(buf + base + 4)); acc += v.x ^ v.y ^ u.z ^ u.w; }
        if (G > 1) acc = __shfl_sync(0xffffffffu, acc, (threadIdx.x & 31) & ~(G - 1));   // one address per group
    }
    if (acc == 0x12345678u) out[0] = acc;
}

template <int G, int W>
void run(const uint32_t* buf, uint64_t words, long long groups, int rounds, uint32_t* out, const char* name) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    const long long threads = groups * G;
    const int bs = 256;
    const unsigned grid = (unsigned)((threads + bs - 1) / bs);
    k_rand<G, W><<<grid, bs>>>(buf, words, rounds, out);
    cudaEventRecord(e0);
    k_rand<G, W><<<grid, bs>>>(buf, words, rounds, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    const double acc = (double)groups * rounds;
    printf("%-22s groups %8lld rounds %3d  %8.3f us  %6.3f us/round  %7.1f G accesses/s  %7.1f GB/s\n", name, groups, rounds,
           ms * 1e3, ms * 1e3 / rounds, acc / (ms * 1e-3) / 1e9, acc * G * W * 4 / (ms * 1e-3) / 1e9);
}

int main() {
    const uint64_t words = 1ull << 30;   // 4 GiB
    uint32_t* buf; uint32_t* out;
    cudaMalloc(&buf, words * 4); cudaMalloc(&out, 64);
    cudaMemset(buf, 1, words * 4);
    for (long long groups : {33158ll, 132632ll, 1ll << 20}) {
        run<1, 1>(buf, words, groups, 16, out, "4B/thread");
        run<1, 8>(buf, words, groups, 16, out, "32B/thread");
        run<2, 8>(buf, words, groups, 16, out, "64B/2 lanes");
        run<4, 8>(buf, words, groups, 16, out, "128B/4 lanes");
        run<8, 8>(buf, words, groups, 16, out, "256B/8 lanes");
        run<32, 8>(buf, words, groups, 16, out, "1KB/warp");
    }
    return 0;
}
