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
// and columns come from adjacency lists built once (ELL head {beg, deg, nb0, nb1}
// + CSR tail); only rules whose two operands both change need row/column
// snapshots of T_{k-1}.
//
// One persistent cooperative kernel runs the whole fixpoint loop (no host round
// trip per iteration): one grid barrier per iteration, the last CTA to arrive
// closes the iteration (changed <=> Δ_k non-empty).  When |Δ| is small the
// iteration is run by CTA 0 alone with __syncthreads() only (the a^n b^n worst
// case adds one cell per iteration for 2pq+1 iterations, SURVEY V-2).
//
// Latency structure of one 32-entry chunk (one warp): load the entries, load the
// ELL heads of all their rule occurrences, issue all bit/key atomics, then stage
// the new cells in a per-warp shared-memory buffer that is appended to the global
// log with one atomic per <= kBuf cells.
#include <cooperative_groups.h>
#include <cub/cub.cuh>

#include "cfpq_internal.cuh"

namespace cfpq {

constexpr int kBlock = 512;
constexpr int kWarps = kBlock / 32;
constexpr int kSeedBlock = 256;
constexpr int kBuf = 64;             // per-warp staging capacity (cells)
constexpr int kSoloMax = 1024;       // max |Δ| mirrored in shared memory by the single-CTA path
constexpr int kSmemNT = 64;          // NT / expansion tables cached in shared memory
constexpr int kSmemExp = 256;
constexpr int kPre = 2;              // rule occurrences prefetched per entry
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
__device__ __forceinline__ unsigned long long globaltimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ unsigned lanemask_lt(int lane) { return (1u << lane) - 1u; }

// Where new cells go: the log append counter and the error flags live in global memory
// for grid-wide iterations and in shared memory for single-CTA iterations; the single-
// CTA path also mirrors Δ_k into shared memory (mirror[idx - mirror_base]).
struct Sink {
    unsigned long long* counter;
    int* overflow;
    int* len_overflow;
    uint64_t* mirror;
    unsigned long long mirror_base;
    unsigned long long mirror_cap;
};

struct __align__(16) WarpScratch {
    uint64_t buf[kBuf];   // staged new cells
    int32_t off[33];
    int32_t beg[32];
    uint32_t A[32];
    uint32_t fixed[32];   // bit 31 set: the fixed coordinate is j (R kinds), else i (L kinds)
    uint32_t len[32];
    int32_t nbuf;
};

// Length of an existing cell (X,i,j): preterminal cells have length 1 (P:393 seed),
// others read their key (final for every cell of T_{k-1}).
__device__ __forceinline__ uint64_t cell_len(const EngineParams& p, const NTInfo* nt, uint32_t X, uint32_t i,
                                             uint32_t j) {
    const uint64_t* K = nt[X].K;
    if (K == nullptr) return 1;
    return ldcg64(K + (size_t)i * (size_t)p.n + j) & 0xffffffffull;
}

// Insert candidate (A,i,j) of length len into T_k; true iff the cell is new:
// relational -> the bit flips; single-path -> the key leaves EMPTY (atomicMin on
// (iteration<<32 | length): first write wins across iterations, min within one).
__device__ __forceinline__ bool try_insert(const EngineParams& p, const NTInfo* nt, const Sink& sk, bool has,
                                           uint32_t A, uint32_t i, uint32_t j, uint64_t len, long long k) {
    if (!has) return false;
    uint64_t* K = nt[A].K;
    if (p.lengths && K != nullptr) {
        if (len > 0xffffffffull) {
            *(volatile int*)sk.len_overflow = 1;   // reported when the iteration closes
            len = 0xffffffffull;
        }
        uint64_t kv = ((uint64_t)k << 32) | len;
        uint64_t old = atomicMin((unsigned long long*)(K + (size_t)i * (size_t)p.n + j), (unsigned long long)kv);
        return old == kEmptyKey;
    }
    uint32_t bit = 1u << (j & 31);
    uint32_t old = atomicOr(nt[A].T + (size_t)i * (size_t)p.Wp + (j >> 5), bit);
    return !(old & bit);
}

// Append the warp's staged cells to the log (one atomic per flush).  A cell that
// does not fit is rolled back so that a re-run of the iteration (after the host
// grows the log) rediscovers it; appended cells stay set and are not re-appended.
__device__ __forceinline__ void flush(const EngineParams& p, const NTInfo* nt, const Sink& sk, WarpScratch* ws,
                                      int lane) {
    int nb = ws->nbuf;
    if (nb == 0) return;
    unsigned long long base = 0;
    if (lane == 0) base = atomicAdd(sk.counter, (unsigned long long)nb);
    base = __shfl_sync(kFull, base, 0);
    for (int t = lane; t < nb; t += 32) {
        uint64_t c = ws->buf[t];
        unsigned long long idx = base + (unsigned long long)t;
        uint32_t A = cell_nt(c), i = cell_i(c), j = cell_j(c);
        uint64_t* K = p.lengths ? nt[A].K : nullptr;
        uint32_t* word = nt[A].T + (size_t)i * (size_t)p.Wp + (j >> 5);
        uint32_t bit = 1u << (j & 31);
        if (idx < p.log_cap) {
            p.log[idx] = c;
            if (sk.mirror != nullptr && idx - sk.mirror_base < sk.mirror_cap) sk.mirror[idx - sk.mirror_base] = c;
            if (K != nullptr) atomicOr(word, bit);   // the bit matrix mirrors the keys
            if (p.rowc != nullptr) {
                atomicAdd(p.rowc + (size_t)A * p.n + i, 1u);
                atomicAdd(p.colc + (size_t)A * p.n + j, 1u);
            }
        } else {
            if (K != nullptr) atomicExch((unsigned long long*)(K + (size_t)i * (size_t)p.n + j),
                                         (unsigned long long)kEmptyKey);
            else atomicAnd(word, ~bit);
            *(volatile int*)sk.overflow = 1;
        }
    }
    __syncwarp();
    if (lane == 0) ws->nbuf = 0;
    __syncwarp();
}

// Warp-uniform: stage the lanes' new cells (disc) in the warp buffer.
__device__ __forceinline__ void stage(const EngineParams& p, const NTInfo* nt, const Sink& sk, WarpScratch* ws,
                                      int lane, bool disc, uint32_t A, uint32_t i, uint32_t j) {
    unsigned mask = __ballot_sync(kFull, disc);
    if (mask == 0) return;
    int cnt = __popc(mask);
    int nb = ws->nbuf;
    if (nb + cnt > kBuf) {
        flush(p, nt, sk, ws, lane);
        nb = 0;
    }
    if (disc) ws->buf[nb + __popc(mask & lanemask_lt(lane))] = pack_cell(A, i, j);
    __syncwarp();
    if (lane == 0) ws->nbuf = nb + cnt;
    __syncwarp();
}

__device__ __forceinline__ void emit(const EngineParams& p, const NTInfo* nt, const Sink& sk, WarpScratch* ws,
                                     int lane, bool has, uint32_t A, uint32_t i, uint32_t j, uint64_t len,
                                     long long k) {
    bool d = try_insert(p, nt, sk, has, A, i, j, len, k);
    stage(p, nt, sk, ws, lane, d, A, i, j);
}

__device__ __forceinline__ Sink global_sink(const EngineParams& p) {
    Sink sk;
    sk.counter = &p.st->log_size;
    sk.overflow = &p.st->overflow;
    sk.len_overflow = &p.st->len_overflow;
    sk.mirror = nullptr;
    sk.mirror_base = 0;
    sk.mirror_cap = 0;
    return sk;
}

// ------------------------------------------------------------------------------------------
// Seeding (Alg. 1 lines 6-7): T_ij ∪= {A | A -> x} for every (i,x,j) ∈ E.
// Parallel edges accumulate; duplicate edges dedupe through the bit test.
// ------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(kSeedBlock) seed_kernel(EngineParams p, const int32_t* __restrict__ edges,
                                                          int64_t n_edges, const int32_t* __restrict__ lab_ptr,
                                                          const int32_t* __restrict__ lab_nt, int32_t n_labels,
                                                          int32_t max_rules) {
    __shared__ WarpScratch wsa[kSeedBlock / 32];
    const int lane = threadIdx.x & 31;
    WarpScratch* ws = &wsa[threadIdx.x >> 5];
    const Sink sk = global_sink(p);
    if (lane == 0) ws->nbuf = 0;
    __syncwarp();
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
            emit(p, p.nt, sk, ws, lane, has, A, (uint32_t)s, (uint32_t)d, 1, 0);
        }
    }
    flush(p, p.nt, sk, ws, lane);
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

// ELL heads: ell[s][r] = {beg, deg, first neighbour, second neighbour} of slot s, row r.
__global__ void adj_ell_kernel(const int32_t* __restrict__ ptr, const int32_t* __restrict__ idx, int4* ell,
                               int64_t n_rows_total, int32_t n) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n_rows_total;
         t += (int64_t)gridDim.x * blockDim.x) {
        int64_t s = t / n, r = t - s * n;
        const int32_t* pp = ptr + s * (int64_t)(n + 1);
        int32_t b = pp[r], e = pp[r + 1];
        int4 v;
        v.x = b;
        v.y = e - b;
        v.z = e - b > 0 ? idx[b] : -1;
        v.w = e - b > 1 ? idx[b + 1] : -1;
        ell[t] = v;
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

__device__ __forceinline__ void cand_coords(uint32_t fx, int32_t nb, uint32_t& i, uint32_t& j) {
    if (fx & 0x80000000u) {
        i = (uint32_t)nb;
        j = fx & 0x7fffffffu;
    } else {
        i = fx;
        j = (uint32_t)nb;
    }
}

// Neighbours beyond the ELL head (deg > 2): warp-wide exclusive scan of the tail
// lengths, load-balanced over the 32 lanes (hub rows are spread over the warp).
__device__ void expand_tail(const EngineParams& p, const NTInfo* nt, const Sink& sk, WarpScratch* ws, int lane, int4 el,
                            uint32_t A, uint32_t fx, uint32_t len_e, long long k) {
    int32_t beg = el.x + 2;
    int32_t deg = el.y > 2 ? el.y - 2 : 0;
    int incl = deg;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int v = __shfl_up_sync(kFull, incl, o);
        if (lane >= o) incl += v;
    }
    int total = __shfl_sync(kFull, incl, 31);
    if (total == 0) return;
    ws->off[lane] = incl - deg;
    ws->beg[lane] = beg;
    ws->A[lane] = A;
    ws->fixed[lane] = fx;
    ws->len[lane] = len_e;
    if (lane == 0) ws->off[32] = total;
    __syncwarp();
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
            int32_t nbv = __ldg(p.adj_idx + ws->beg[l] + (t - ws->off[l]));
            cA = ws->A[l];
            cand_coords(ws->fixed[l], nbv, oi, oj);
            clen = (uint64_t)ws->len[l] + 1ull;   // the preterminal operand has length 1
        }
        emit(p, nt, sk, ws, lane, has, cA, oi, oj, clen, k);
    }
    __syncwarp();
}

// ELL head of expansion ex for entry (ci, cj).
__device__ __forceinline__ int4 load_head(const NTInfo* nt, const Expansion& ex, uint32_t ci, uint32_t cj,
                                          uint32_t& A, uint32_t& fx) {
    A = (uint32_t)ex.A;
    if (ex.kind == EXP_L_CONST) {          // Δ_B entry (i, r=cj): row r of preterminal C
        fx = ci;
        return __ldg(nt[ex.other].csr_ell + cj);
    }
    fx = cj | 0x80000000u;                 // Δ_C entry (r=ci, j): column r of preterminal B
    return __ldg(nt[ex.other].csc_ell + ci);
}

// Expand the Δ entries log[lo,hi) of iteration k.  Work unit = a chunk of 32
// consecutive entries per warp; warps [warp, warp+nwarps) stride over chunks.
// `src` = shared-memory copy of log[lo,hi) (single-CTA path) or null (read the log).
__device__ void expand(const EngineParams& p, const NTInfo* nt, const Expansion* exps, const Sink& sk,
                       const uint64_t* src, unsigned long long lo, unsigned long long hi, long long k, int warp,
                       int nwarps, int lane, WarpScratch* ws, unsigned long long& dcand, unsigned long long& dexp) {
    for (unsigned long long cbase = lo + (unsigned long long)warp * 32ull; cbase < hi;
         cbase += (unsigned long long)nwarps * 32ull) {
        unsigned long long e = cbase + lane;
        bool valid = e < hi;
        uint64_t cell = 0ull;
        if (valid) cell = src ? src[e - lo] : ldcg64(p.log + e);
        uint32_t X = cell_nt(cell), ci = cell_i(cell), cj = cell_j(cell);
        int eb = 0, nexp = 0;
        if (valid) {
            eb = nt[X].exp_begin;
            nexp = nt[X].exp_end - eb;
        }
        dexp += (unsigned long long)nexp;
        uint32_t len_e = 0;
        if (p.lengths && nexp > 0) len_e = (uint32_t)cell_len(p, nt, X, ci, cj);
        int maxexp = nexp;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) maxexp = max(maxexp, __shfl_xor_sync(kFull, maxexp, o));
        if (maxexp == 0) continue;

        // ---- preterminal-operand occurrences 0..kPre-1: all loads, then all atomics ----
        unsigned var_mask = 0;
        int4 el[kPre];
        uint32_t eA[kPre], efx[kPre];
#pragma unroll
        for (int x = 0; x < kPre; ++x) {
            el[x] = make_int4(0, 0, -1, -1);
            eA[x] = 0;
            efx[x] = 0;
            if (x < nexp) {
                Expansion ex = exps[eb + x];
                if (ex.kind == EXP_L_CONST || ex.kind == EXP_R_CONST) el[x] = load_head(nt, ex, ci, cj, eA[x], efx[x]);
                else var_mask |= 1u << x;
            }
        }
        bool d0[kPre], d1[kPre];
        uint32_t ci0[kPre], cj0[kPre], ci1[kPre], cj1[kPre];
#pragma unroll
        for (int x = 0; x < kPre; ++x) {
            cand_coords(efx[x], el[x].z, ci0[x], cj0[x]);
            cand_coords(efx[x], el[x].w, ci1[x], cj1[x]);
            d0[x] = try_insert(p, nt, sk, el[x].y > 0, eA[x], ci0[x], cj0[x], (uint64_t)len_e + 1ull, k);
            d1[x] = try_insert(p, nt, sk, el[x].y > 1, eA[x], ci1[x], cj1[x], (uint64_t)len_e + 1ull, k);
            dcand += (unsigned long long)el[x].y;
        }
        bool any_tail = false;
#pragma unroll
        for (int x = 0; x < kPre; ++x) {
            if (x < maxexp) {
                stage(p, nt, sk, ws, lane, d0[x], eA[x], ci0[x], cj0[x]);
                stage(p, nt, sk, ws, lane, d1[x], eA[x], ci1[x], cj1[x]);
                any_tail |= el[x].y > 2;
            }
        }
        if (__any_sync(kFull, any_tail)) {
#pragma unroll
            for (int x = 0; x < kPre; ++x)
                if (x < maxexp) expand_tail(p, nt, sk, ws, lane, el[x], eA[x], efx[x], len_e, k);
        }
        // ---- occurrences kPre.. (rare: NTs on the RHS of many rules) ----
        for (int x = kPre; x < maxexp; ++x) {
            int4 h = make_int4(0, 0, -1, -1);
            uint32_t A = 0, fx = 0;
            if (x < nexp) {
                Expansion ex = exps[eb + x];
                if (ex.kind == EXP_L_CONST || ex.kind == EXP_R_CONST) h = load_head(nt, ex, ci, cj, A, fx);
                else if (x < 32) var_mask |= 1u << x;
            }
            uint32_t a0, b0, a1, b1;
            cand_coords(fx, h.z, a0, b0);
            cand_coords(fx, h.w, a1, b1);
            bool q0 = try_insert(p, nt, sk, h.y > 0, A, a0, b0, (uint64_t)len_e + 1ull, k);
            bool q1 = try_insert(p, nt, sk, h.y > 1, A, a1, b1, (uint64_t)len_e + 1ull, k);
            dcand += (unsigned long long)h.y;
            stage(p, nt, sk, ws, lane, q0, A, a0, b0);
            stage(p, nt, sk, ws, lane, q1, A, a1, b1);
            if (__any_sync(kFull, h.y > 2)) expand_tail(p, nt, sk, ws, lane, h, A, fx, len_e, k);
        }
        // ---- rules whose other operand also changes: scan the snapshot row, warp-cooperative ----
        unsigned any_var = __ballot_sync(kFull, var_mask != 0);
        while (any_var) {
            int src = __ffs(any_var) - 1;
            any_var &= any_var - 1;
            unsigned vm = __shfl_sync(kFull, var_mask, src);
            uint32_t si = __shfl_sync(kFull, ci, src);
            uint32_t sj = __shfl_sync(kFull, cj, src);
            uint32_t slen = __shfl_sync(kFull, len_e, src);
            int seb = __shfl_sync(kFull, eb, src);
            while (vm) {
                int x = __ffs(vm) - 1;
                vm &= vm - 1;
                Expansion ex = exps[seb + x];
                const uint32_t* row;
                bool left = ex.kind == EXP_L_VAR;
                if (left) row = nt[ex.other].S + (size_t)sj * p.Wp;    // S_C row r = sj
                else row = nt[ex.other].ST + (size_t)si * p.Wp;        // ST_B row r = si
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
                                if (p.lengths) clen = (uint64_t)slen + cell_len(p, nt, ex.other, sj, v);
                            } else {
                                oi = v;
                                oj = sj;
                                if (p.lengths) clen = cell_len(p, nt, ex.other, v, si) + (uint64_t)slen;
                            }
                            ++dcand;
                        }
                        emit(p, nt, sk, ws, lane, has, (uint32_t)ex.A, oi, oj, clen, k);
                    }
                }
            }
        }
    }
    flush(p, nt, sk, ws, lane);
}

// Fold Δ_k = log[lo,hi) into the snapshots S (row) and ST (transposed).
__device__ void apply_snapshots(const EngineParams& p, const NTInfo* nt, const uint64_t* src, unsigned long long lo,
                                unsigned long long hi, long long tid, long long nthreads) {
    for (unsigned long long e = lo + (unsigned long long)tid; e < hi; e += (unsigned long long)nthreads) {
        uint64_t c = src ? src[e - lo] : ldcg64(p.log + e);
        uint32_t A = cell_nt(c), i = cell_i(c), j = cell_j(c);
        uint32_t* S = nt[A].S;
        uint32_t* ST = nt[A].ST;
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

struct LoopState {
    unsigned long long lo, hi;
    long long iter;
    int status;
};

// Close iteration k: Δ_k = log[hi, ls).  Single thread; `s` is updated and the caller
// publishes it (fenced) when other CTAs must see it.
__device__ void close_iteration(const EngineParams& p, long long k, LoopState& s, unsigned long long ls, int ov,
                                int lov) {
    if (lov) {
        s.status = ST_LEN_OVERFLOW;
        return;
    }
    if (ov) {
        s.status = ST_OVERFLOW;   // keep lo/hi/iter: the host grows the log and re-runs k
        return;
    }
    s.lo = s.hi;
    s.hi = ls;
    s.iter = k;
    if (k < p.iter_off_cap) {
        p.iter_off[k] = s.lo;
        if (p.iter_time) p.iter_time[k] = globaltimer();
    }
    if (k + 1 < p.iter_off_cap) p.iter_off[k + 1] = ls;
    if (ls == s.lo) s.status = ST_DONE;             // T_k = T_{k-1}: fixpoint
    else if (k >= p.max_iter) s.status = ST_CAP;    // Theorem 3 cap
}

__device__ void publish(const EngineParams& p, const LoopState& s) {
    EngineState* st = p.st;
    st->lo = s.lo;
    st->hi = s.hi;
    st->iter = s.iter;
    *(volatile int*)&st->status = s.status;
    __threadfence();
}

// Grid barrier; the last CTA to arrive closes iteration k (if k >= 0) before release.
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
            if (k >= 0) {
                LoopState s;
                s.lo = ld_volatile_u64(&st->lo);
                s.hi = ld_volatile_u64(&st->hi);
                s.iter = *(volatile long long*)&st->iter;
                s.status = *(volatile int*)&st->status;
                close_iteration(p, k, s, ld_volatile_u64(&st->log_size), *(volatile int*)&st->overflow,
                                *(volatile int*)&st->len_overflow);
                publish(p, s);
            }
            st->bar_count = 0u;
            __threadfence();
            atomicAdd(&st->bar_gen, 1u);
        } else {
            long long t0 = clock64();
            while (*gen == my) {
                __nanosleep(64);
                if (clock64() - t0 > 60000000000ll) {   // ~30 s watchdog: never hang the GPU
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

__global__ void __launch_bounds__(kBlock, 2) closure_kernel(EngineParams p) {
    __shared__ WarpScratch ws[kWarps];
    __shared__ NTInfo s_nt[kSmemNT];
    __shared__ Expansion s_exp[kSmemExp];
    __shared__ uint64_t s_delta[2][kSoloMax];
    __shared__ LoopState s_state;
    __shared__ unsigned long long s_ls;
    __shared__ int s_ov, s_lov;
    __shared__ long long s_solo;
    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    EngineState* st = p.st;
    // NT / expansion tables into shared memory (fences invalidate L1 every iteration)
    const bool small = p.n_nt <= kSmemNT && p.n_exps <= kSmemExp;
    if (small) {
        for (int t = threadIdx.x; t < p.n_nt; t += kBlock) s_nt[t] = p.nt[t];
        for (int t = threadIdx.x; t < p.n_exps; t += kBlock) s_exp[t] = p.exps[t];
    }
    const NTInfo* nt = small ? s_nt : p.nt;
    const Expansion* exps = small ? s_exp : p.exps;
    const Sink gsink = global_sink(p);
    if (lane == 0) ws[wib].nbuf = 0;
    if (threadIdx.x == 0) s_solo = 0;
    __syncthreads();
    unsigned long long dcand = 0, dexp = 0;
    for (;;) {
        if (threadIdx.x == 0) {
            s_state.lo = ld_volatile_u64(&st->lo);
            s_state.hi = ld_volatile_u64(&st->hi);
            s_state.iter = *(volatile long long*)&st->iter;
            s_state.status = *(volatile int*)&st->status;
        }
        __syncthreads();
        LoopState s = s_state;
        __syncthreads();
        if (s.status != ST_RUNNING) break;
        long long k = s.iter + 1;
        if ((long long)(s.hi - s.lo) <= (long long)p.solo_max) {
            // ------------- single-CTA iterations: Δ, counter and flags in shared memory -------------
            if (blockIdx.x == 0) {
                int cur = 0;
                if (threadIdx.x == 0) {
                    s_ls = ld_volatile_u64(&st->log_size);
                    s_ov = 0;
                    s_lov = 0;
                }
                if (s.hi - s.lo <= (unsigned long long)kSoloMax)
                    for (unsigned long long e = s.lo + threadIdx.x; e < s.hi; e += kBlock)
                        s_delta[cur][e - s.lo] = ldcg64(p.log + e);
                __syncthreads();
                for (;;) {
                    if (p.jac) {
                        account(p, k, threadIdx.x, kBlock);
                        __syncthreads();
                    }
                    Sink sk;
                    sk.counter = &s_ls;
                    sk.overflow = &s_ov;
                    sk.len_overflow = &s_lov;
                    sk.mirror = s_delta[cur ^ 1];
                    sk.mirror_base = s.hi;
                    sk.mirror_cap = kSoloMax;
                    const uint64_t* src = (s.hi - s.lo <= (unsigned long long)kSoloMax) ? s_delta[cur] : nullptr;
                    expand(p, nt, exps, sk, src, s.lo, s.hi, k, wib, kWarps, lane, &ws[wib], dcand, dexp);
                    __syncthreads();
                    if (threadIdx.x == 0) {
                        close_iteration(p, k, s_state, s_ls, s_ov, s_lov);
                        s_solo += 1;
                    }
                    __syncthreads();
                    s = s_state;
                    if (s.status != ST_RUNNING) break;
                    cur ^= 1;
                    if (p.has_snapshots) {
                        const uint64_t* sn = (s.hi - s.lo <= (unsigned long long)kSoloMax) ? s_delta[cur] : nullptr;
                        apply_snapshots(p, nt, sn, s.lo, s.hi, threadIdx.x, kBlock);
                        __syncthreads();
                    }
                    ++k;
                    if ((long long)(s.hi - s.lo) > (long long)p.solo_max) break;
                }
                if (threadIdx.x == 0) {
                    st->log_size = s_ls;   // the other CTAs are parked at the grid barrier
                    if (s_ov) st->overflow = 1;
                    if (s_lov) st->len_overflow = 1;
                    publish(p, s_state);
                    atomicAdd((unsigned long long*)&st->solo_iters, (unsigned long long)s_solo);
                    s_solo = 0;
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
        expand(p, nt, exps, gsink, nullptr, s.lo, s.hi, k, blockIdx.x * kWarps + wib, gridDim.x * kWarps, lane,
               &ws[wib], dcand, dexp);
        if (!grid_barrier(p, k)) return;
        if (p.has_snapshots) {
            if (threadIdx.x == 0) {
                s_state.lo = ld_volatile_u64(&st->lo);
                s_state.hi = ld_volatile_u64(&st->hi);
                s_state.status = *(volatile int*)&st->status;
            }
            __syncthreads();
            if (s_state.status == ST_RUNNING)
                apply_snapshots(p, nt, nullptr, s_state.lo, s_state.hi, gtid, gthreads);
            if (!grid_barrier(p, -1)) return;
        }
    }
    // diagnostics: one atomic per warp per launch
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        dcand += __shfl_xor_sync(kFull, dcand, o);
        dexp += __shfl_xor_sync(kFull, dexp, o);
    }
    if (lane == 0) {
        if (dcand) atomicAdd(&st->candidates, dcand);
        if (dexp) atomicAdd(&st->expansions, dexp);
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
    if (p.iter_time) p.iter_time[0] = globaltimer();
}

// Δ_0 into the snapshots (one launch after seeding).
__global__ void seed_snapshots_kernel(EngineParams p) {
    apply_snapshots(p, p.nt, nullptr, 0, ld_volatile_u64(&p.st->hi), (long long)blockIdx.x * blockDim.x + threadIdx.x,
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
        seed_kernel<<<grid_for(n_edges, kSeedBlock), kSeedBlock, 0, s>>>(p, edges, n_edges, lab_ptr, lab_nt, n_labels,
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

cudaError_t launch_adj_ell(const int32_t* ptr, const int32_t* idx, int4* ell, int64_t n_slots, int32_t n,
                           cudaStream_t s) {
    int64_t rows = n_slots * (int64_t)n;
    if (rows) adj_ell_kernel<<<grid_for(rows, 256), 256, 0, s>>>(ptr, idx, ell, rows, n);
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
