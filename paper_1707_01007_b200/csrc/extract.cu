// Result extraction: R_A = {(i,j) | A ∈ T^cf_ij} (Theorem 2) as sorted pairs,
// per-NT counts and single-path lengths, read from the derived-cell log.
#include <cub/cub.cuh>

#include "cfpq_internal.cuh"

namespace cfpq {

// Per-NT cell counts: block-private shared-memory histogram, one global atomic per
// (block, NT) — a single global counter per NT serialises millions of atomics.
__global__ void nt_histogram_kernel(const uint64_t* __restrict__ log, unsigned long long n,
                                    unsigned long long* counts, int n_nt) {
    extern __shared__ unsigned int hist[];
    for (int t = threadIdx.x; t < n_nt; t += blockDim.x) hist[t] = 0u;
    __syncthreads();
    for (unsigned long long e = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; e < n;
         e += (unsigned long long)gridDim.x * blockDim.x) {
        atomicAdd(hist + cell_nt(__ldg((const unsigned long long*)log + e)), 1u);
    }
    __syncthreads();
    for (int t = threadIdx.x; t < n_nt; t += blockDim.x)
        if (hist[t]) atomicAdd(counts + t, (unsigned long long)hist[t]);
}

__global__ void filter_nt_kernel(const uint64_t* __restrict__ log, unsigned long long n, uint32_t A,
                                 uint64_t* keys, unsigned long long* count) {
    for (unsigned long long e = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; e < n;
         e += (unsigned long long)gridDim.x * blockDim.x) {
        uint64_t c = __ldg((const unsigned long long*)log + e);
        if (cell_nt(c) == A) {
            unsigned long long at = atomicAdd(count, 1ull);
            keys[at] = c & ((1ull << (2 * kNodeBits)) - 1ull);   // (i << 27) | j
        }
    }
}

__global__ void unpack_pairs_kernel(const uint64_t* __restrict__ keys, unsigned long long n, int32_t* pairs) {
    for (unsigned long long e = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; e < n;
         e += (unsigned long long)gridDim.x * blockDim.x) {
        uint64_t k = keys[e];
        pairs[2 * e] = (int32_t)cell_i(k);
        pairs[2 * e + 1] = (int32_t)cell_j(k);
    }
}

__global__ void gather_lengths_kernel(const uint64_t* __restrict__ keys, unsigned long long n,
                                      const uint64_t* __restrict__ K, int64_t n_nodes, uint32_t* out) {
    for (unsigned long long e = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; e < n;
         e += (unsigned long long)gridDim.x * blockDim.x) {
        uint64_t k = keys[e];
        uint32_t l = 1;   // preterminal cells: length 1 (P:393 seed)
        if (K) l = (uint32_t)(K[(size_t)cell_i(k) * (size_t)n_nodes + cell_j(k)] & 0xffffffffull);
        out[e] = l;
    }
}

static int grid_for(unsigned long long work) {
    unsigned long long g = (work + 255) / 256;
    if (g < 1) g = 1;
    if (g > 148 * 16) g = 148 * 16;
    return (int)g;
}

cudaError_t launch_nt_histogram(const uint64_t* log, unsigned long long n, unsigned long long* counts, int n_nt,
                                cudaStream_t s) {
    if (n) nt_histogram_kernel<<<grid_for(n), 256, n_nt * sizeof(unsigned int), s>>>(log, n, counts, n_nt);
    return cudaGetLastError();
}

cudaError_t launch_filter_nt(const uint64_t* log, unsigned long long n, uint32_t A, uint64_t* keys,
                             unsigned long long* count, cudaStream_t s) {
    if (n) filter_nt_kernel<<<grid_for(n), 256, 0, s>>>(log, n, A, keys, count);
    return cudaGetLastError();
}

// Sort (i<<27 | j) keys ascending -> (i,j) lexicographic order.  Result in `keys`.
cudaError_t sort_keys(uint64_t* keys, uint64_t* keys_alt, unsigned long long n, int end_bit, void* temp,
                      size_t* temp_bytes, cudaStream_t s) {
    cub::DoubleBuffer<unsigned long long> db((unsigned long long*)keys, (unsigned long long*)keys_alt);
    cudaError_t e = cub::DeviceRadixSort::SortKeys(temp, *temp_bytes, db, (int)n, 0, end_bit, s);
    if (e != cudaSuccess || temp == nullptr) return e;
    if (db.Current() != (unsigned long long*)keys)
        e = cudaMemcpyAsync(keys, db.Current(), n * sizeof(uint64_t), cudaMemcpyDeviceToDevice, s);
    return e;
}

cudaError_t launch_unpack_pairs(const uint64_t* keys, unsigned long long n, int32_t* pairs, cudaStream_t s) {
    if (n) unpack_pairs_kernel<<<grid_for(n), 256, 0, s>>>(keys, n, pairs);
    return cudaGetLastError();
}

cudaError_t launch_gather_lengths(const uint64_t* keys, unsigned long long n, const uint64_t* K, int64_t n_nodes,
                                  uint32_t* out, cudaStream_t s) {
    if (n) gather_lengths_kernel<<<grid_for(n), 256, 0, s>>>(keys, n, K, n_nodes, out);
    return cudaGetLastError();
}

cudaError_t launch_scan(const int32_t* in, int32_t* out, int64_t n, void* temp, size_t* temp_bytes,
                        cudaStream_t s) {
    return cub::DeviceScan::ExclusiveSum(temp, *temp_bytes, in, out, (int)n, s);
}

}  // namespace cfpq
