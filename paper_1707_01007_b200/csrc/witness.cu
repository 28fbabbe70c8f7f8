// Single-path witness extraction on the GPU ("a path can be
// found by a simple search").  Given the single-path lengths recorded by the
// closure (l_A = l_B + l_C, first write wins), a path of exactly l_A(i,j) edges whose
// word A derives is rebuilt top-down (Lemma 4):
//   l = 1  -> an edge (i, x, j) with A -> x (the seed of the cell);
//   l > 1  -> the first (rule A -> B C in grammar order, node r ascending) with both
//             sub-cells recorded and l_B(i,r) + l_C(r,j) = l; recurse into (B,i,r), (C,r,j).
// Both parts are shorter than l, so the recursion ends; every recorded length is realised
// by induction.  One CTA walks the derivation with an explicit stack in global memory
// (left part on top, so edges come out in path order); each split is a CTA-wide scan of
// |rules of A| x n candidates reduced with a shared atomicMin, each leaf a scan of the
// out-edges of i.
#include "cfpq_internal.cuh"

namespace cfpq {

struct WFrame {
    uint32_t A, i, j, len;
};

constexpr int kWBlock = 1024;

__device__ __forceinline__ uint32_t w_len(const EngineParams& p, uint32_t X, uint32_t a, uint32_t b) {
    const NTInfo& t = p.nt[X];
    if (t.K) {
        uint64_t v = t.K[(size_t)a * p.n + b];
        return v == kEmptyKey ? 0u : (uint32_t)(v & 0xffffffffull);
    }
    // preterminal: present iff its bit is set (length 1, a seed)
    return (t.T[(size_t)a * p.Wp + (b >> 5)] >> (b & 31)) & 1u;
}

__global__ void __launch_bounds__(kWBlock) witness_kernel(EngineParams p, const int32_t* __restrict__ rules,
                                                          const int32_t* __restrict__ rule_ptr,
                                                          const int32_t* __restrict__ rule_ids,
                                                          const int32_t* __restrict__ e_ptr,
                                                          const int32_t* __restrict__ e_idx,
                                                          const int32_t* __restrict__ edges,
                                                          const int32_t* __restrict__ lab_ptr,
                                                          const int32_t* __restrict__ lab_nt, int32_t n_labels,
                                                          WFrame* stack, int64_t stack_cap, WFrame root, int32_t* out,
                                                          int64_t out_cap, long long* result) {
    __shared__ WFrame top;
    __shared__ unsigned long long best;
    __shared__ long long sp, pos;
    __shared__ int err, quit;
    if (threadIdx.x == 0) {
        stack[0] = root;
        sp = 1;
        pos = 0;
        err = 0;
    }
    __syncthreads();
    for (;;) {
        if (threadIdx.x == 0) {
            quit = (sp == 0 || err) ? 1 : 0;
            if (!quit) top = stack[--sp];
            best = ~0ull;
        }
        __syncthreads();
        if (quit) break;
        const WFrame f = top;
        if (f.len == 1u) {
            // leaf: an edge (i, x, j) with A -> x
            for (int t = e_ptr[f.i] + threadIdx.x; t < e_ptr[f.i + 1]; t += kWBlock) {
                const int e = e_idx[t];
                const int x = edges[3 * e + 1];
                if ((uint32_t)edges[3 * e + 2] != f.j || x < 0 || x >= n_labels) continue;
                for (int q = lab_ptr[x]; q < lab_ptr[x + 1]; ++q)
                    if ((uint32_t)lab_nt[q] == f.A) {
                        atomicMin(&best, (unsigned long long)e);
                        break;
                    }
            }
        } else {
            // split: first (rule of A, r) with l_B(i,r) + l_C(r,j) = l
            const int rb = rule_ptr[f.A], re = rule_ptr[f.A + 1];
            const long long total = (long long)(re - rb) * p.n;
            for (long long t = threadIdx.x; t < total; t += kWBlock) {
                const int q = (int)(t / p.n);
                const uint32_t r = (uint32_t)(t - (long long)q * p.n);
                const int rl = rule_ids[rb + q];
                const uint32_t B = (uint32_t)rules[3 * rl + 1], C = (uint32_t)rules[3 * rl + 2];
                const uint32_t lb = w_len(p, B, f.i, r);
                if (lb == 0u || lb >= f.len) continue;
                const uint32_t lc = w_len(p, C, r, f.j);
                if (lc != 0u && (uint64_t)lb + lc == f.len) atomicMin(&best, (unsigned long long)t);
            }
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            if (best == ~0ull || f.len == 0u) {
                err = 1;   // no seed edge / no split: not a recorded derivation
            } else if (f.len == 1u) {
                const int e = (int)best;
                if (pos < out_cap) {
                    out[3 * pos + 0] = edges[3 * e + 0];
                    out[3 * pos + 1] = edges[3 * e + 1];
                    out[3 * pos + 2] = edges[3 * e + 2];
                }
                ++pos;
            } else {
                const long long t = (long long)best;
                const int q = (int)(t / p.n);
                const uint32_t r = (uint32_t)(t - (long long)q * p.n);
                const int rl = rule_ids[rule_ptr[f.A] + q];
                const uint32_t B = (uint32_t)rules[3 * rl + 1], C = (uint32_t)rules[3 * rl + 2];
                const uint32_t lb = w_len(p, B, f.i, r);
                if (sp + 2 > stack_cap) {
                    err = 2;
                } else {
                    stack[sp++] = WFrame{C, r, f.j, f.len - lb};   // right part below
                    stack[sp++] = WFrame{B, f.i, r, lb};           // left part on top
                }
            }
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) result[0] = err ? -(long long)err : pos;
}

// out-degree count / fill of the edge list by source (CSR of edge ids)
__global__ void edge_count_kernel(const int32_t* __restrict__ edges, int64_t n_edges, int32_t n, int32_t* deg) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n_edges; e += (int64_t)gridDim.x * blockDim.x) {
        const int s = edges[3 * e];
        if (s >= 0 && s < n) atomicAdd(deg + s, 1);
    }
}

__global__ void edge_fill_kernel(const int32_t* __restrict__ edges, int64_t n_edges, int32_t n, int32_t* cursor,
                                 int32_t* idx) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n_edges; e += (int64_t)gridDim.x * blockDim.x) {
        const int s = edges[3 * e];
        if (s >= 0 && s < n) idx[atomicAdd(cursor + s, 1)] = (int32_t)e;
    }
}

static int wgrid(int64_t work) {
    int64_t g = (work + 255) / 256;
    return (int)std::max<int64_t>(1, std::min<int64_t>(g, 148 * 16));
}

cudaError_t launch_edge_csr(const int32_t* edges, int64_t n_edges, int32_t n, int32_t* deg, int32_t* ptr,
                            int32_t* cursor, int32_t* idx, void* temp, size_t* temp_bytes, cudaStream_t s) {
    cudaError_t e = cudaMemsetAsync(deg, 0, (size_t)(n + 1) * 4, s);
    if (e != cudaSuccess) return e;
    if (n_edges) edge_count_kernel<<<wgrid(n_edges), 256, 0, s>>>(edges, n_edges, n, deg);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    if ((e = launch_scan(deg, ptr, (int64_t)n + 1, temp, temp_bytes, s)) != cudaSuccess) return e;
    if ((e = cudaMemcpyAsync(cursor, ptr, (size_t)n * 4, cudaMemcpyDeviceToDevice, s)) != cudaSuccess) return e;
    if (n_edges) edge_fill_kernel<<<wgrid(n_edges), 256, 0, s>>>(edges, n_edges, n, cursor, idx);
    return cudaGetLastError();
}

cudaError_t launch_witness(const EngineParams& p, const int32_t* rules, const int32_t* rule_ptr,
                           const int32_t* rule_ids, const int32_t* e_ptr, const int32_t* e_idx, const int32_t* edges,
                           const int32_t* lab_ptr, const int32_t* lab_nt, int32_t n_labels, void* stack,
                           int64_t stack_cap, uint32_t A, uint32_t i, uint32_t j, uint32_t len, int32_t* out,
                           int64_t out_cap, long long* result, cudaStream_t s) {
    witness_kernel<<<1, kWBlock, 0, s>>>(p, rules, rule_ptr, rule_ids, e_ptr, e_idx, edges, lab_ptr, lab_nt, n_labels,
                                         (WFrame*)stack, stack_cap, WFrame{A, i, j, len}, out, out_cap, result);
    return cudaGetLastError();
}

size_t witness_frame_bytes() { return sizeof(WFrame); }

}  // namespace cfpq
