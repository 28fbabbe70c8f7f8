// Latency of dependent random 4-byte atomicOr / loads over buffers of growing size, with
// the whole GPU busy (148 x 1024 threads) or one warp: does the 5 GB bit-matrix footprint
// of config 4 cost TLB misses compared with an L2-resident table?
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t mix(uint64_t x) {
    x ^= x >> 33; x *= 0xff51afd7ed558ccdull; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ull; x ^= x >> 33;
    return x;
}

__global__ void chase(uint32_t* buf, uint64_t words, int steps, int atomic, unsigned long long* out) {
    uint64_t x = mix(blockIdx.x * 1024ull + threadIdx.x + 1);
    uint32_t acc = 0;
    long long t0 = clock64();
    for (int s = 0; s < steps; ++s) {
        uint64_t w = (x + acc) % words;
        uint32_t v = atomic ? atomicOr(buf + w, 1u << (x & 31)) : __ldcg(buf + w);
        acc = v & 1u;    // dependent chain
        x = mix(x + s);
    }
    long long t1 = clock64();
    if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = (unsigned long long)(t1 - t0);
    if (acc == 12345) out[1] = acc;
}

int main() {
    const size_t sizes_mb[] = {16, 48, 96, 256, 1024, 5120};
    unsigned long long* out;
    cudaMalloc(&out, 16);
    for (size_t mb : sizes_mb) {
        uint32_t* buf;
        size_t bytes = mb << 20;
        if (cudaMalloc(&buf, bytes) != cudaSuccess) { printf("alloc %zu MB failed\n", mb); return 1; }
        cudaMemset(buf, 0, bytes);
        for (int atomic = 0; atomic < 2; ++atomic)
            for (int full = 0; full < 2; ++full) {
                int blocks = full ? 148 : 1, threads = full ? 1024 : 32, steps = 256;
                chase<<<blocks, threads>>>(buf, bytes / 4, 16, atomic, out);
                cudaEvent_t a, b;
                cudaEventCreate(&a); cudaEventCreate(&b);
                cudaEventRecord(a);
                chase<<<blocks, threads>>>(buf, bytes / 4, steps, atomic, out);
                cudaEventRecord(b);
                cudaEventSynchronize(b);
                float ms; cudaEventElapsedTime(&ms, a, b);
                unsigned long long cyc; cudaMemcpy(&cyc, out, 8, cudaMemcpyDeviceToHost);
                printf("%6zu MB %-6s %-9s  %.1f ns/step (event)  %.0f cycles/step (clock)  %.2f Gop/s\n", mb,
                       atomic ? "atomic" : "load", full ? "148x1024" : "1 warp", ms * 1e6 / steps, (double)cyc / steps,
                       (double)blocks * threads * steps / (ms * 1e6));
            }
        cudaFree(buf);
    }
    return 0;
}
