// Sparse (index-list, semi-naive) closure engine for sm_100a.
//
// Algorithm 1 loop body k computes T_k = T_{k-1} ∪ (T_{k-1} × T_{k-1})
// (P:222).  Because T only grows, T_{k-1} × T_{k-1} = T_{k-2} × T_{k-2}
// ∪ Δ_{k-1} × T_{k-1} ∪ T_{k-1} × Δ_{k-1} with Δ_{k-1} = T_{k-1} \ T_{k-2}, and
// T_{k-2} × T_{k-2} ⊆ T_{k-1}; so expanding only Δ_{k-1} yields exactly T_k
// (semi-naive evaluation, SURVEY V-1).  Per rule A -> B C (one Boolean
// product per rule):
//   Δ_B entry (i,r)  -> (i,j) for every j with C ∈ T_{k-1}[r][j]
//   Δ_C entry (r,j)  -> (i,j) for every i with B ∈ T_{k-1}[i][r]
// Preterminals (LHS of no binary rule) never change after seeding, so their rows
// and columns come from CSR/CSC built once; only rules whose two operands both
// change need row/column snapshots of T_{k-1}.
//
// One persistent cooperative kernel runs the whole fixpoint loop (no host round
// trip per iteration): one grid barrier per iteration, the last CTA to arrive
// closes the iteration (changed <=> Δ_k non-empty).  When |Δ| is small the
// iteration is run by CTA 0 alone with __syncthreads() only (the a^n b^n worst
// case adds one cell per iteration for 2pq+1 iterations, SURVEY V-2).
#include <cooperative_groups.h>
#include <cub/cub.cuh>

#include "cfpq_internal.cuh"

namespace cfpq {

constexpr int kBlock = 512;
constexpr int kWarps = kBlock / 32;
constexpr unsigned kFull = 0xffffffffu;

// ------------------------------------------------------------------------------------------
// small device helpers
// ------------------------------------------------------------------------------------------
__device__ __forceinline__ uint64_t ldcg64(const uint64_t* p) {
    uint64_t v;
    asm volatile("ld.global.cg.u64 %0, [%1];" : "=l"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ uint32_t ldcg32(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.global.cg.u32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ unsigned long long ld_volatile_u64(const unsigned long long* p) {
    return *(volatile const unsigned long long*)p;
}

struct WarpScratch {
    int32_t off[33];
    int32_t beg[32];
    uint32_t A[32];
    uint32_t fixed[32];   // bit 31 set: the fixed coordinate is j (R kinds), else i (L kinds)
    uint32_t len[32];
};

// Length of an existing cell (X,i,j): preterminal cells have length 1 (P:393 seed),
// others read their key (final for every cell of T_{k-1}).
__device__ __forceinline__ uint64_t cell_len(const EngineParams& p, uint32_t X, uint32_t i, uint32_t j) {
    const uint64_t* K = p.nt[X].K;
    if (K == nullptr) return 1;
    return ldcg64(K + (size_t)i * (size_t)p.n + j) & 0xffffffffull;
}

// Warp-uniform: every lane calls with its optional candidate (A,i,j,len).
// A candidate is new iff it flips its bit (relational) or turns its key from EMPTY
// (lengths); new cells are appended to the log (Δ_k) with one atomic per warp.
__device__ __forceinline__ void emit(const EngineParams& p, bool has, uint32_t A, uint32_t i, uint32_t j,
                                     uint64_t len, long long k, int lane) {
    bool disc = false;
    uint32_t* word = nullptr;
    uint32_t bit = 0;
    uint64_t* key = nullptr;
    if (has) {
        word = p.nt[A].T + (size_t)i * (size_t)p.Wp + (j >> 5);
        bit = 1u << (j & 31);
        if (p.lengths && p.nt[A].K != nullptr) {
            if (len > 0xffffffffull) {
                p.st->status = ST_LEN_OVERFLOW;   // reported at the next barrier
                len = 0xffffffffull;
            }
            key = p.nt[A].K + (size_t)i * (size_t)p.n + j;
            uint64_t kv = ((uint64_t)k << 32) | len;
            uint64_t old = atomicMin((unsigned long long*)key, (unsigned long long)kv);
            disc = (old == kEmptyKey);
        } else {
            uint32_t old = atomicOr(word, bit);
            disc = !(old & bit);
        }
    }
    unsigned mask = __ballot_sync(kFull, disc);
    if (mask == 0) return;
    int leader = __ffs(mask) - 1;
    unsigned long long base = 0;
    if (lane == leader) base = atomicAdd(&p.st->log_size, (unsigned long long)__popc(mask));
    base = __shfl_sync(kFull, base, leader);
    if (disc) {
        unsigned long long idx = base + __popc(mask & ((1u << lane) - 1u));
        if (idx < p.log_cap) {
            p.log[idx] = pack_cell(A, i, j);
            if (key != nullptr) atomicOr(word, bit);
            if (p.rowc != nullptr) {
                atomicAdd(p.rowc + (size_t)A * p.n + i, 1u);
                atomicAdd(p.colc + (size_t)A * p.n + j, 1u);
            }
        } else {
            // roll back: a re-run of this iteration (after the host grows the log)
            // rediscovers the cell; appended cells stay set and are not re-appended.
            if (key != nullptr) atomicExch((unsigned long long*)key, (unsigned long long)kEmptyKey);
            else atomicAnd(word, ~bit);
            *(volatile int*)&p.st->overflow = 1;
        }
    }
}

// ------------------------------------------------------------------------------------------
// Seeding (Alg. 1 lines 6-7): T_ij ∪= {A | A -> x} for every (i,x,j) ∈ E.
// Parallel edges accumulate; duplicate edges dedupe through the bit test.
// ------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(256) seed_kernel(EngineParams p, const int32_t* __restrict__ edges,
                                                   int64_t n_edges, const int32_t* __restrict__ lab_ptr,
                                                   const int32_t* __restrict__ lab_nt, int32_t n_labels,
                                                   int32_t max_rules) {
    const int lane = threadIdx.x & 31;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < n_edges; base += stride) {
        int64_t e = base + threadIdx.x;
        bool valid = e < n_edges;
        int32_t s = 0, x = 0, d = 0, rb = 0, re = 0;
        if (valid) {
            s = __ldg(edges + 3 * e);
            x = __ldg(edges + 3 * e + 1);
            d = __ldg(edges + 3 * e + 2);
            if (s < 0 || s >= p.n || d < 0 || d >= p.n || x < 0 || x >= n_labels) {
                p.st->bad_edge = 1;
                valid = false;
            } else {
                rb = __ldg(lab_ptr + x);
                re = __ldg(lab_ptr + x + 1);
            }
        }
        for (int t = 0; t < max_rules; ++t) {
            bool has = valid && (rb + t < re);
            uint32_t A = has ? (uint32_t)__ldg(lab_nt + rb + t) : 0u;
            emit(p, has, A, (uint32_t)s, (uint32_t)d, 1, 0, lane);
        }
    }
}

// CSR / CSC of preterminals from the seed cells Δ_0 = log[0, n_seed).
// slot_row[X] / slot_col[X] = offset (in units of (n+1)) of X's CSR / CSC pointer
// array inside the concatenated count array, or -1.
__global__ void adj_count_kernel(EngineParams p, const int32_t* __restrict__ slot_row,
                                 const int32_t* __restrict__ slot_col, int32_t* counts) {
    const unsigned long long n_seed = ld_volatile_u64(&p.st->hi);
    for (unsigned long long e = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; e < n_seed;
         e += (unsigned long long)gridDim.x * blockDim.x) {
        uint64_t c = p.log[e];
        uint32_t X = cell_nt(c);
        int32_t sr = __ldg(slot_row + X), sc = __ldg(slot_col + X);
        if (sr >= 0) atomicAdd(counts + (size_t)sr * (p.n + 1) + cell_i(c), 1);
        if (sc >= 0) atomicAdd(counts + (size_t)sc * (p.n + 1) + cell_j(c), 1);
    }
}

__global__ void adj_fill_kernel(EngineParams p, const int32_t* __restrict__ slot_row,
                                const int32_t* __restrict__ slot_col, int32_t* cursor, int32_t* idx) {
    const unsigned long long n_seed = ld_volatile_u64(&p.st->hi);
    for (unsigned long long e = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; e < n_seed;
         e += (unsigned long long)gridDim.x * blockDim.x) {
        uint64_t c = p.log[e];
        uint32_t X = cell_nt(c);
        int32_t sr = __ldg(slot_row + X), sc = __ldg(slot_col + X);
        if (sr >= 0) idx[atomicAdd(cursor + (size_t)sr * (p.n + 1) + cell_i(c), 1)] = (int32_t)cell_j(c);
        if (sc >= 0) idx[atomicAdd(cursor + (size_t)sc * (p.n + 1) + cell_j(c), 1)] = (int32_t)cell_i(c);
    }
}

// Clear the cells of a previous run (bitmaps, snapshots, keys, counters) in O(|log|).
__global__ void clear_log_kernel(EngineParams p, unsigned long long n_cells) {
    for (unsigned long long e = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; e < n_cells;
         e += (unsigned long long)gridDim.x * blockDim.x) {
        uint64_t c = p.log[e];
        uint32_t A = cell_nt(c), i = cell_i(c), j = cell_j(c);
        const NTInfo& nt = p.nt[A];
        nt.T[(size_t)i * p.Wp + (j >> 5)] = 0u;
        if (nt.S) nt.S[(size_t)i * p.Wp + (j >> 5)] = 0u;
        if (nt.ST) nt.ST[(size_t)j * p.Wp + (i >> 5)] = 0u;
        if (nt.K) nt.K[(size_t)i * p.n + j] = kEmptyKey;
        if (p.rowc) {
            p.rowc[(size_t)A * p.n + i] = 0u;
            p.colc[(size_t)A * p.n + j] = 0u;
        }
    }
}

// ------------------------------------------------------------------------------------------
// Closure kernel pieces
// ------------------------------------------------------------------------------------------

// Expand the Δ entries log[lo,hi) of iteration k.  Work unit = a chunk of 32
// consecutive entries per warp; warps [warp0, warp0+nwarps) stride over chunks.
__device__ void expand(const EngineParams& p, unsigned long long lo, unsigned long long hi, long long k,
                       int warp, int nwarps, int lane, WarpScratch* ws) {
    unsigned long long cand = 0;
    for (unsigned long long cbase = lo + (unsigned long long)warp * 32ull; cbase < hi;
         cbase += (unsigned long long)nwarps * 32ull) {
        unsigned long long e = cbase + lane;
        bool valid = e < hi;
        uint64_t cell = valid ? ldcg64(p.log + e) : 0ull;
        uint32_t X = cell_nt(cell), ci = cell_i(cell), cj = cell_j(cell);
        int eb = 0, ee = 0;
        if (valid) {
            eb = __ldg(&p.nt[X].exp_begin);
            ee = __ldg(&p.nt[X].exp_end);
        }
        int nexp = ee - eb;
        {
            int tot = nexp;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) tot += __shfl_xor_sync(kFull, tot, o);
            if (lane == 0 && tot) atomicAdd(&p.st->expansions, (unsigned long long)tot);
        }
        uint32_t len_e = 0;
        if (p.lengths && nexp > 0) len_e = (uint32_t)cell_len(p, X, ci, cj);
        int maxexp = nexp;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) maxexp = max(maxexp, __shfl_xor_sync(kFull, maxexp, o));
        unsigned var_mask = 0;   // bit x: this lane's expansion x is a var kind
        for (int x = 0; x < maxexp; ++x) {
            int32_t beg = 0, deg = 0;
            uint32_t A = 0, fixed = 0;
            if (x < nexp) {
                Expansion ex = p.exps[eb + x];
                if (ex.kind == EXP_L_CONST) {
                    const int32_t* ptr = p.nt[ex.other].csr_ptr;   // C's row r = cj
                    beg = __ldg(ptr + cj);
                    deg = __ldg(ptr + cj + 1) - beg;
                    fixed = ci;
                    A = ex.A;
                } else if (ex.kind == EXP_R_CONST) {
                    const int32_t* ptr = p.nt[ex.other].csc_ptr;   // B's column r = ci
                    beg = __ldg(ptr + ci);
                    deg = __ldg(ptr + ci + 1) - beg;
                    fixed = cj | 0x80000000u;
                    A = ex.A;
                } else if (x < 32) {
                    var_mask |= 1u << x;
                }
            }
            // warp-wide exclusive scan of the degrees: a load-balanced expansion of all
            // 32 lanes' neighbour lists (hub rows are spread over the warp)
            int incl = deg;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                int v = __shfl_up_sync(kFull, incl, o);
                if (lane >= o) incl += v;
            }
            int total = __shfl_sync(kFull, incl, 31);
            if (total == 0) continue;
            ws->off[lane] = incl - deg;
            ws->beg[lane] = beg;
            ws->A[lane] = A;
            ws->fixed[lane] = fixed;
            ws->len[lane] = len_e;
            if (lane == 0) ws->off[32] = total;
            __syncwarp();
            if (lane == 0) cand += (unsigned long long)total;
            for (int tb = 0; tb < total; tb += 32) {
                int t = tb + lane;
                bool has = t < total;
                uint32_t cA = 0, oi = 0, oj = 0;
                uint64_t clen = 0;
                if (has) {
                    int l = 0;
#pragma unroll
                    for (int step = 16; step > 0; step >>= 1)
                        if (ws->off[l + step] <= t) l += step;
                    int32_t nb = __ldg(p.adj_idx + ws->beg[l] + (t - ws->off[l]));
                    uint32_t fx = ws->fixed[l];
                    cA = ws->A[l];
                    if (fx & 0x80000000u) {
                        oi = (uint32_t)nb;
                        oj = fx & 0x7fffffffu;
                    } else {
                        oi = fx;
                        oj = (uint32_t)nb;
                    }
                    clen = (uint64_t)ws->len[l] + 1ull;   // the preterminal operand has length 1
                }
                emit(p, has, cA, oi, oj, clen, k, lane);
            }
            __syncwarp();
        }
        // rules whose other operand also changes: scan the snapshot row, warp-cooperative
        unsigned any_var = __ballot_sync(kFull, var_mask != 0);
        while (any_var) {
            int src = __ffs(any_var) - 1;
            any_var &= any_var - 1;
            unsigned vm = __shfl_sync(kFull, var_mask, src);
            uint32_t sX = __shfl_sync(kFull, X, src);
            uint32_t si = __shfl_sync(kFull, ci, src);
            uint32_t sj = __shfl_sync(kFull, cj, src);
            uint32_t slen = __shfl_sync(kFull, len_e, src);
            int seb = __shfl_sync(kFull, eb, src);
            (void)sX;
            while (vm) {
                int x = __ffs(vm) - 1;
                vm &= vm - 1;
                Expansion ex = p.exps[seb + x];
                const uint32_t* row;
                bool left = ex.kind == EXP_L_VAR;
                if (left) row = p.nt[ex.other].S + (size_t)sj * p.Wp;    // S_C row r = sj
                else row = p.nt[ex.other].ST + (size_t)si * p.Wp;        // ST_B row r = si
                const int64_t wn = (p.n + 31) >> 5;
                for (int64_t w0 = 0; w0 < wn; w0 += 32) {
                    int64_t w = w0 + lane;
                    uint32_t bits = (w < wn) ? ldcg32(row + w) : 0u;
                    while (__any_sync(kFull, bits != 0u)) {
                        bool has = bits != 0u;
                        uint32_t oi = 0, oj = 0;
                        uint64_t clen = 0;
                        if (has) {
                            int b = __ffs(bits) - 1;
                            bits &= bits - 1u;
                            uint32_t v = (uint32_t)(w * 32 + b);
                            if (left) {
                                oi = si;
                                oj = v;
                                if (p.lengths) clen = (uint64_t)slen + cell_len(p, ex.other, sj, v);
                            } else {
                                oi = v;
                                oj = sj;
                                if (p.lengths) clen = cell_len(p, ex.other, v, si) + (uint64_t)slen;
                            }
                            ++cand;
                        }
                        emit(p, has, (uint32_t)ex.A, oi, oj, clen, k, lane);
                    }
                }
            }
        }
    }
    if (cand) atomicAdd(&p.st->candidates, cand);
}

// Fold Δ_k = log[lo,hi) into the snapshots S (row) and ST (transposed).
__device__ void apply_snapshots(const EngineParams& p, unsigned long long lo, unsigned long long hi, long long tid,
                                long long nthreads) {
    for (unsigned long long e = lo + (unsigned long long)tid; e < hi; e += (unsigned long long)nthreads) {
        uint64_t c = ldcg64(p.log + e);
        uint32_t A = cell_nt(c), i = cell_i(c), j = cell_j(c);
        uint32_t* S = p.nt[A].S;
        uint32_t* ST = p.nt[A].ST;
        if (S) atomicOr(S + (size_t)i * p.Wp + (j >> 5), 1u << (j & 31));
        if (ST) atomicOr(ST + (size_t)j * p.Wp + (i >> 5), 1u << (i & 31));
    }
}

// Jacobi work of iteration k (account mode): Σ_rules Σ_r |col r of T_B| · |row r of T_C|,
// the AND-true triples of T_{k-1} × T_{k-1}.
__device__ void account(const EngineParams& p, long long k, long long tid, long long nthreads) {
    unsigned long long acc = 0;
    long long total = (long long)p.n_rules * p.n;
    for (long long t = tid; t < total; t += nthreads) {
        int rl = (int)(t / p.n);
        int r = (int)(t - (long long)rl * p.n);
        int B = p.rules[3 * rl + 1], C = p.rules[3 * rl + 2];
        acc += (unsigned long long)ldcg32(p.colc + (size_t)B * p.n + r) *
               (unsigned long long)ldcg32(p.rowc + (size_t)C * p.n + r);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(kFull, acc, o);
    if ((threadIdx.x & 31) == 0 && acc && k < p.iter_off_cap) atomicAdd(p.jac + k, acc);
}

// Close iteration k (single thread): Δ_k = log[hi, log_size).
__device__ void finalize(const EngineParams& p, long long k) {
    EngineState* st = p.st;
    __threadfence();
    unsigned long long ls = ld_volatile_u64(&st->log_size);
    int ov = *(volatile int*)&st->overflow;
    int status = *(volatile int*)&st->status;
    if (status == ST_LEN_OVERFLOW) return;
    if (ov) {
        st->status = ST_OVERFLOW;   // keep lo/hi/iter: the host grows the log and re-runs k
        return;
    }
    unsigned long long new_lo = st->hi;
    st->lo = new_lo;
    st->hi = ls;
    st->iter = k;
    if (k < p.iter_off_cap) {
        p.iter_off[k] = new_lo;
        if (p.iter_time) {
            unsigned long long t;
            asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
            p.iter_time[k] = t;
        }
    }
    if (k + 1 < p.iter_off_cap) p.iter_off[k + 1] = ls;
    if (ls == new_lo) st->status = ST_DONE;             // T_k = T_{k-1}: fixpoint
    else if (k >= p.max_iter) st->status = ST_CAP;      // Theorem 3 cap
    __threadfence();
}

// Grid barrier; the last CTA to arrive runs finalize(k) (if k >= 0) before release.
__device__ bool grid_barrier(const EngineParams& p, long long k) {
    __syncthreads();
    __shared__ int s_timeout;
    if (threadIdx.x == 0) {
        s_timeout = 0;
        EngineState* st = p.st;
        volatile unsigned* gen = &st->bar_gen;
        unsigned my = *gen;
        __threadfence();
        unsigned arrived = atomicAdd(&st->bar_count, 1u);
        if (arrived == (unsigned)p.nblocks - 1u) {
            if (k >= 0) finalize(p, k);
            st->bar_count = 0u;
            __threadfence();
            atomicAdd(&st->bar_gen, 1u);
        } else {
            long long t0 = clock64();
            while (*gen == my) {
                __nanosleep(64);
                if (clock64() - t0 > 40000000000ll) {   // ~20 s watchdog: never hang the GPU
                    s_timeout = 1;
                    break;
                }
            }
        }
        __threadfence();
    }
    __syncthreads();
    return s_timeout == 0;
}

__global__ void __launch_bounds__(kBlock) closure_kernel(EngineParams p) {
    __shared__ WarpScratch ws[kWarps];
    __shared__ unsigned long long s_lo, s_hi;
    __shared__ long long s_iter;
    __shared__ int s_status;
    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    EngineState* st = p.st;
    for (;;) {
        if (threadIdx.x == 0) {
            s_lo = ld_volatile_u64(&st->lo);
            s_hi = ld_volatile_u64(&st->hi);
            s_iter = *(volatile long long*)&st->iter;
            s_status = *(volatile int*)&st->status;
        }
        __syncthreads();
        unsigned long long lo = s_lo, hi = s_hi;
        long long k = s_iter + 1;
        if (s_status != ST_RUNNING) break;
        __syncthreads();
        if ((long long)(hi - lo) <= (long long)p.solo_max) {
            // ---------------- single-CTA iterations ----------------
            if (blockIdx.x == 0) {
                for (;;) {
                    if (p.jac) {
                        account(p, k, threadIdx.x, kBlock);
                        __syncthreads();
                    }
                    expand(p, lo, hi, k, wib, kWarps, lane, &ws[wib]);
                    __syncthreads();
                    if (threadIdx.x == 0) {
                        finalize(p, k);
                        st->solo_iters += 1;
                        s_lo = st->lo;
                        s_hi = st->hi;
                        s_status = st->status;
                    }
                    __syncthreads();
                    if (s_status != ST_RUNNING) break;
                    lo = s_lo;
                    hi = s_hi;
                    if (p.has_snapshots) {
                        apply_snapshots(p, lo, hi, threadIdx.x, kBlock);
                        __syncthreads();
                    }
                    ++k;
                    if ((long long)(hi - lo) > (long long)p.solo_max) break;
                }
            }
            if (!grid_barrier(p, -1)) return;
            continue;
        }
        // ---------------- grid-wide iteration k ----------------
        const long long gtid = (long long)blockIdx.x * kBlock + threadIdx.x;
        const long long gthreads = (long long)gridDim.x * kBlock;
        if (p.jac) {
            account(p, k, gtid, gthreads);
            if (!grid_barrier(p, -1)) return;
        }
        expand(p, lo, hi, k, blockIdx.x * kWarps + wib, gridDim.x * kWarps, lane, &ws[wib]);
        if (!grid_barrier(p, k)) return;
        if (p.has_snapshots) {
            if (threadIdx.x == 0) {
                s_lo = ld_volatile_u64(&st->lo);
                s_hi = ld_volatile_u64(&st->hi);
                s_status = *(volatile int*)&st->status;
            }
            __syncthreads();
            if (s_status == ST_RUNNING) apply_snapshots(p, s_lo, s_hi, gtid, gthreads);
            if (!grid_barrier(p, -1)) return;
        }
    }
}

// After seeding: Δ_0 = log[0, log_size) (T_0), iteration 0 complete.
__global__ void begin_kernel(EngineParams p) {
    EngineState* st = p.st;
    unsigned long long n0 = ld_volatile_u64(&st->log_size);
    st->lo = 0;
    st->hi = n0;
    st->iter = 0;
    if (p.iter_off_cap > 0) p.iter_off[0] = 0;
    if (p.iter_off_cap > 1) p.iter_off[1] = n0;
    if (p.iter_time) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
        p.iter_time[0] = t;
    }
    if (n0 == 0) st->status = ST_RUNNING;   // iteration 1 still runs: no change -> 1 iteration
}

// Δ_0 into the snapshots (one launch after seeding).
__global__ void seed_snapshots_kernel(EngineParams p) {
    apply_snapshots(p, 0, ld_volatile_u64(&p.st->hi), (long long)blockIdx.x * blockDim.x + threadIdx.x,
                    (long long)gridDim.x * blockDim.x);
}

// ------------------------------------------------------------------------------------------
// launchers
// ------------------------------------------------------------------------------------------
static int grid_for(int64_t work, int block) {
    int64_t g = (work + block - 1) / block;
    if (g < 1) g = 1;
    if (g > 148 * 32) g = 148 * 32;
    return (int)g;
}

cudaError_t launch_seed(const int32_t* edges, int64_t n_edges, int32_t n_nodes, const int32_t* lab_ptr,
                        const int32_t* lab_nt, int32_t n_labels, int32_t max_rules_per_label,
                        const EngineParams& p, cudaStream_t s) {
    (void)n_nodes;
    if (n_edges > 0 && max_rules_per_label > 0)
        seed_kernel<<<grid_for(n_edges, 256), 256, 0, s>>>(p, edges, n_edges, lab_ptr, lab_nt, n_labels,
                                                            max_rules_per_label);
    return cudaGetLastError();
}

cudaError_t launch_adj_count(const EngineParams& p, const int32_t* slot_row, const int32_t* slot_col,
                             int32_t* counts, unsigned long long n_seed, cudaStream_t s) {
    if (n_seed) adj_count_kernel<<<grid_for((int64_t)n_seed, 256), 256, 0, s>>>(p, slot_row, slot_col, counts);
    return cudaGetLastError();
}

cudaError_t launch_adj_fill(const EngineParams& p, const int32_t* slot_row, const int32_t* slot_col,
                            int32_t* cursor, int32_t* idx, unsigned long long n_seed, cudaStream_t s) {
    if (n_seed)
        adj_fill_kernel<<<grid_for((int64_t)n_seed, 256), 256, 0, s>>>(p, slot_row, slot_col, cursor, idx);
    return cudaGetLastError();
}

cudaError_t launch_clear_log(const EngineParams& p, unsigned long long n_cells, cudaStream_t s) {
    if (n_cells) clear_log_kernel<<<grid_for((int64_t)n_cells, 256), 256, 0, s>>>(p, n_cells);
    return cudaGetLastError();
}

cudaError_t launch_seed_snapshots(const EngineParams& p, unsigned long long n_seed, cudaStream_t s) {
    if (n_seed) seed_snapshots_kernel<<<grid_for((int64_t)n_seed, 256), 256, 0, s>>>(p);
    return cudaGetLastError();
}

cudaError_t launch_begin(const EngineParams& p, cudaStream_t s) {
    begin_kernel<<<1, 1, 0, s>>>(p);
    return cudaGetLastError();
}

int closure_kernel_block_size() { return kBlock; }

int closure_kernel_blocks_per_sm() {
    int nb = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, closure_kernel, kBlock, 0) != cudaSuccess) return 0;
    return nb;
}

cudaError_t launch_closure(const EngineParams& p, int grid, cudaStream_t s) {
    void* args[] = {(void*)&p};
    return cudaLaunchCooperativeKernel((const void*)closure_kernel, dim3(grid), dim3(kBlock), args, 0, s);
}

}  // namespace cfpq
