// Throughput of hashed-cell-set inserts (64-bit atomicCAS, linear probing) vs random
// 4-byte atomicOr into a 5 GB bit matrix, whole GPU, keys drawn from a universe of 3M.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t mix(uint64_t x) {
    x ^= x >> 33; x *= 0xff51afd7ed558ccdull; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ull; x ^= x >> 33;
    return x;
}

__global__ void hash_ins(unsigned long long* tab, int shift, unsigned long long mask, int steps, uint64_t universe,
                         int mode, unsigned long long* out) {
    uint64_t x = mix(blockIdx.x * 1024ull + threadIdx.x + 7);
    unsigned long long probes = 0, news = 0;
    for (int s = 0; s < steps; ++s) {
        uint64_t key = mix(x % universe) & 0x3fffffffffffffull;   // a "cell"
        if (mode == 0) {
            unsigned long long h = (key * 0x9E3779B97F4A7C15ull) >> shift;
            for (int q = 0; q < 4096; ++q) {
                ++probes;
                unsigned long long old = atomicCAS(tab + h, ~0ull, key);
                if (old == ~0ull) { ++news; break; }
                if (old == key) break;
                h = (h + 1) & mask;
            }
        } else if (mode == 1) {   // load first, CAS only if not found in the probe run
            unsigned long long h = (key * 0x9E3779B97F4A7C15ull) >> shift;
            for (int q = 0; q < 4096; ++q) {
                ++probes;
                unsigned long long cur = __ldcg(tab + h);
                if (cur == key) break;
                if (cur == ~0ull) {
                    unsigned long long old = atomicCAS(tab + h, ~0ull, key);
                    if (old == ~0ull) { ++news; break; }
                    if (old == key) break;
                }
                h = (h + 1) & mask;
            }
        } else {                  // bitmap: 10 x 512 MB, random word
            uint32_t* bm = (uint32_t*)tab;
            uint64_t w = key % (mask + 1);
            uint32_t old = atomicOr(bm + w, 1u << (key >> 58));
            probes++;
            news += !(old & (1u << (key >> 58)));
        }
        x = mix(x + s);
    }
    for (int o = 16; o > 0; o >>= 1) {
        probes += __shfl_xor_sync(0xffffffffu, probes, o);
        news += __shfl_xor_sync(0xffffffffu, news, o);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(out, probes);
        atomicAdd(out + 1, news);
    }
}

int main() {
    unsigned long long* out;
    cudaMalloc(&out, 16);
    struct Cfg { int lg; int mode; const char* name; };
    Cfg cfgs[] = {{21, 0, "cas 2^21 (16MB)"}, {22, 0, "cas 2^22 (32MB)"}, {23, 0, "cas 2^23 (64MB)"},
                  {24, 0, "cas 2^24 (128MB)"}, {23, 1, "ld+cas 2^23 (64MB)"}, {22, 1, "ld+cas 2^22 (32MB)"},
                  {30, 2, "bitmap atomicOr 4GB"}, {23, 2, "bitmap atomicOr 32MB"}};
    for (auto c : cfgs) {
        size_t slots = 1ull << c.lg;
        size_t bytes = c.mode == 2 ? slots * 4 : slots * 8;
        unsigned long long* tab;
        if (cudaMalloc(&tab, bytes) != cudaSuccess) { printf("alloc failed\n"); return 1; }
        for (int rep = 0; rep < 2; ++rep) {
            cudaMemset(tab, c.mode == 2 ? 0 : 0xff, bytes);
            cudaMemset(out, 0, 16);
            int steps = 256;
            cudaEvent_t a, b;
            cudaEventCreate(&a); cudaEventCreate(&b);
            cudaEventRecord(a);
            hash_ins<<<148, 1024>>>(tab, 64 - c.lg, slots - 1, steps, c.mode == 2 ? 3000000ull : (uint64_t)(0.45 * slots), c.mode, out);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b);
            unsigned long long h[2]; cudaMemcpy(h, out, 16, cudaMemcpyDeviceToHost);
            double ops = 148.0 * 1024 * steps;
            if (rep == 1)
                printf("%-24s %.3f ms  %.1f G inserts/s  %.2f probes/insert  new %llu\n", c.name, ms, ops / (ms * 1e6),
                       h[0] / ops, h[1]);
        }
        cudaFree(tab);
    }
    return 0;
}
