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

// A's cells as compact keys (i << bits) | j (bits = ceil(log2 n)), so the radix sort runs
// over 2*bits key bits only; uint32 keys when 2*bits <= 32.  Each block filters a tile of
// kFilterTile entries and appends its hits with ONE atomic (same-address atomics per warp
// would serialise on the counter).
constexpr int kFilterThreads = 256, kFilterPer = 8, kFilterTile = kFilterThreads * kFilterPer;

__global__ void __launch_bounds__(kFilterThreads) filter_nt_kernel(const uint64_t* __restrict__ log,
                                                                   unsigned long long n, uint32_t A, void* keys,
                                                                   unsigned long long* count, int bits, int k32) {
    __shared__ int wcnt[kFilterThreads / 32];
    __shared__ unsigned long long s_base;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (unsigned long long tile = (unsigned long long)blockIdx.x * kFilterTile; tile < n;
         tile += (unsigned long long)gridDim.x * kFilterTile) {
        uint64_t c[kFilterPer];
        unsigned hitm = 0;
#pragma unroll
        for (int q = 0; q < kFilterPer; ++q) {
            const unsigned long long e = tile + (unsigned long long)q * kFilterThreads + threadIdx.x;
            c[q] = e < n ? __ldg((const unsigned long long*)log + e) : ~0ull;
            if (e < n && cell_nt(c[q]) == A) hitm |= 1u << q;
        }
        const int mine = __popc(hitm);
        int incl = mine;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int v = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += v;
        }
        if (lane == 31) wcnt[warp] = incl;
        __syncthreads();
        int before = 0, total = 0;
#pragma unroll
        for (int w = 0; w < kFilterThreads / 32; ++w) {
            if (w < warp) before += wcnt[w];
            total += wcnt[w];
        }
        if (threadIdx.x == 0) s_base = total ? atomicAdd(count, (unsigned long long)total) : 0ull;
        __syncthreads();
        unsigned long long at = s_base + (unsigned long long)(before + incl - mine);
#pragma unroll
        for (int q = 0; q < kFilterPer; ++q)
            if (hitm & (1u << q)) {
                const uint64_t key = ((uint64_t)cell_i(c[q]) << bits) | cell_j(c[q]);
                if (k32) reinterpret_cast<uint32_t*>(keys)[at] = (uint32_t)key;
                else reinterpret_cast<uint64_t*>(keys)[at] = key;
                ++at;
            }
        __syncthreads();
    }
}

__global__ void unpack_pairs_kernel(const void* __restrict__ keys, unsigned long long n, int32_t* pairs,
                                    int bits, int k32) {
    for (unsigned long long e = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; e < n;
         e += (unsigned long long)gridDim.x * blockDim.x) {
        uint64_t k = k32 ? (uint64_t)reinterpret_cast<const uint32_t*>(keys)[e] : reinterpret_cast<const uint64_t*>(keys)[e];
        pairs[2 * e] = (int32_t)(k >> bits);
        pairs[2 * e + 1] = (int32_t)(k & ((1ull << bits) - 1ull));
    }
}

__global__ void gather_lengths_kernel(const void* __restrict__ keys, unsigned long long n,
                                      const uint64_t* __restrict__ K, int64_t n_nodes, uint32_t* out, int bits,
                                      int k32) {
    for (unsigned long long e = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; e < n;
         e += (unsigned long long)gridDim.x * blockDim.x) {
        uint64_t k = k32 ? (uint64_t)reinterpret_cast<const uint32_t*>(keys)[e] : reinterpret_cast<const uint64_t*>(keys)[e];
        uint32_t l = 1;   // preterminal cells: length 1 (P:393 seed)
        if (K) l = (uint32_t)(K[(size_t)(k >> bits) * (size_t)n_nodes + (k & ((1ull << bits) - 1ull))] & 0xffffffffull);
        out[e] = l;
    }
}

// ---- bit-matrix extraction (results of the dense engine, which keeps no cell log) ----
// one warp per row: popcount of row i -> rowcnt[i]
__global__ void bitmap_rowcount_kernel(const uint32_t* __restrict__ T, int32_t n, int64_t wn, int64_t Wp,
                                       int32_t* rowcnt, unsigned long long* total) {
    const int lane = threadIdx.x & 31;
    unsigned long long acc = 0;
    for (int64_t row = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; row < n;
         row += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        int c = 0;
        for (int64_t w = lane; w < wn; w += 32) c += __popc(__ldg(T + (size_t)row * Wp + w));
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
        if (lane == 0) {
            if (rowcnt) rowcnt[row] = c;
            acc += (unsigned long long)c;
        }
    }
    if (lane == 0 && acc) atomicAdd(total, acc);
}

// one warp per row: write (i,j) of the set bits of row i, ascending, from rowoff[i]
// cols_only: write j into pairs[at] (the column array of the CSR form) instead of (i, j)
__global__ void bitmap_pairs_kernel(const uint32_t* __restrict__ T, int32_t n, int64_t wn, int64_t Wp,
                                    const int32_t* __restrict__ rowoff, int32_t* pairs, int cols_only) {
    const int lane = threadIdx.x & 31;
    for (int64_t row = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; row < n;
         row += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        int64_t base = rowoff[row];
        for (int64_t w0 = 0; w0 < wn; w0 += 32) {
            int64_t w = w0 + lane;
            uint32_t bits = w < wn ? __ldg(T + (size_t)row * Wp + w) : 0u;
            int c = __popc(bits);
            int incl = c;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                int v = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += v;
            }
            int64_t at = base + incl - c;
            while (bits) {
                int b = __ffs(bits) - 1;
                bits &= bits - 1u;
                if (cols_only) {
                    pairs[at] = (int32_t)(w * 32 + b);
                } else {
                    pairs[2 * at] = (int32_t)row;
                    pairs[2 * at + 1] = (int32_t)(w * 32 + b);
                }
                ++at;
            }
            base += __shfl_sync(0xffffffffu, incl, 31);
        }
    }
}

cudaError_t launch_bitmap_rowcount(const uint32_t* T, int32_t n, int64_t Wp, int32_t* rowcnt,
                                   unsigned long long* total, cudaStream_t s) {
    if (n) {
        int64_t blocks = ((int64_t)n * 32 + 255) / 256;
        if (blocks > 148 * 16) blocks = 148 * 16;
        bitmap_rowcount_kernel<<<(int)blocks, 256, 0, s>>>(T, n, (n + 31) / 32, Wp, rowcnt, total);
    }
    return cudaGetLastError();
}

cudaError_t launch_bitmap_pairs(const uint32_t* T, int32_t n, int64_t Wp, const int32_t* rowoff, int32_t* pairs,
                                cudaStream_t s, int cols_only) {
    if (n) {
        int64_t blocks = ((int64_t)n * 32 + 255) / 256;
        if (blocks > 148 * 16) blocks = 148 * 16;
        bitmap_pairs_kernel<<<(int)blocks, 256, 0, s>>>(T, n, (n + 31) / 32, Wp, rowoff, pairs, cols_only);
    }
    return cudaGetLastError();
}

// CSR of sorted compact keys (i << bits | j): cols[t] = j; row_ptr[r] = first t with row >= r
// (every row written exactly once: by the entry that opens it or, past the last entry, by it).
__global__ void keys_to_csr_kernel(const void* __restrict__ keys, unsigned long long m, int bits, int k32, int64_t n,
                                   int64_t* row_ptr, int32_t* cols) {
    for (unsigned long long t = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; t < m;
         t += (unsigned long long)gridDim.x * blockDim.x) {
        auto key = [&](unsigned long long e) -> uint64_t {
            return k32 ? (uint64_t)reinterpret_cast<const uint32_t*>(keys)[e] : reinterpret_cast<const uint64_t*>(keys)[e];
        };
        const uint64_t k = key(t);
        const int64_t i = (int64_t)(k >> bits);
        CFPQ_DASSERT(i < n);
        cols[t] = (int32_t)(k & ((1ull << bits) - 1ull));
        const int64_t prev = t ? (int64_t)(key(t - 1) >> bits) : -1;
        for (int64_t r = prev + 1; r <= i; ++r) row_ptr[r] = (int64_t)t;
        if (t == m - 1)
            for (int64_t r = i + 1; r <= n; ++r) row_ptr[r] = (int64_t)m;
    }
}

__global__ void rowoff_to_ptr_kernel(const int32_t* __restrict__ rowoff, int64_t n1, int64_t* row_ptr) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n1; t += (int64_t)gridDim.x * blockDim.x)
        row_ptr[t] = rowoff[t];
}

static int grid_for(unsigned long long work);

cudaError_t launch_keys_to_csr(const void* keys, unsigned long long m, int bits, int k32, int64_t n, int64_t* row_ptr,
                               int32_t* cols, cudaStream_t s) {
    if (m == 0) return cudaMemsetAsync(row_ptr, 0, (size_t)(n + 1) * sizeof(int64_t), s);
    keys_to_csr_kernel<<<grid_for(m), 256, 0, s>>>(keys, m, bits, k32, n, row_ptr, cols);
    return cudaGetLastError();
}

cudaError_t launch_rowoff_to_ptr(const int32_t* rowoff, int64_t n, int64_t* row_ptr, cudaStream_t s) {
    rowoff_to_ptr_kernel<<<grid_for((unsigned long long)n + 1), 256, 0, s>>>(rowoff, n + 1, row_ptr);
    return cudaGetLastError();
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

cudaError_t launch_filter_nt(const uint64_t* log, unsigned long long n, uint32_t A, void* keys,
                             unsigned long long* count, int bits, int k32, cudaStream_t s) {
    if (n) {
        unsigned long long tiles = (n + kFilterTile - 1) / kFilterTile;
        int g = (int)std::min<unsigned long long>(tiles, 148ull * 8);
        filter_nt_kernel<<<g, kFilterThreads, 0, s>>>(log, n, A, keys, count, bits, k32);
    }
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

// 32-bit variant of sort_keys (compact keys of graphs with n <= 65,536)
cudaError_t sort_keys32(uint32_t* keys, uint32_t* keys_alt, unsigned long long n, int end_bit, void* temp,
                        size_t* temp_bytes, cudaStream_t s) {
    cub::DoubleBuffer<unsigned int> db(keys, keys_alt);
    cudaError_t e = cub::DeviceRadixSort::SortKeys(temp, *temp_bytes, db, (int)n, 0, end_bit, s);
    if (e != cudaSuccess || temp == nullptr) return e;
    if (db.Current() != keys) e = cudaMemcpyAsync(keys, db.Current(), n * sizeof(uint32_t), cudaMemcpyDeviceToDevice, s);
    return e;
}

cudaError_t launch_unpack_pairs(const void* keys, unsigned long long n, int32_t* pairs, int bits, int k32,
                                cudaStream_t s) {
    if (n) unpack_pairs_kernel<<<grid_for(n), 256, 0, s>>>(keys, n, pairs, bits, k32);
    return cudaGetLastError();
}

cudaError_t launch_gather_lengths(const void* keys, unsigned long long n, const uint64_t* K, int64_t n_nodes,
                                  uint32_t* out, int bits, int k32, cudaStream_t s) {
    if (n) gather_lengths_kernel<<<grid_for(n), 256, 0, s>>>(keys, n, K, n_nodes, out, bits, k32);
    return cudaGetLastError();
}

cudaError_t launch_scan(const int32_t* in, int32_t* out, int64_t n, void* temp, size_t* temp_bytes,
                        cudaStream_t s) {
    return cub::DeviceScan::ExclusiveSum(temp, *temp_bytes, in, out, (int)n, s);
}

}  // namespace cfpq
