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

constexpr int kBlock = 1024;
constexpr int kWarps = kBlock / 32;
constexpr int kSeedBlock = 256;
constexpr int kBuf = 128;            // per-warp staging capacity (cells)
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
    uint64_t tag;                  // OR-ed into every appended entry (asynchronous schedule: valid flag)
    unsigned long long* counter;
    int* overflow;
    int* len_overflow;
    uint64_t* mirror;
    unsigned long long mirror_base;
    unsigned long long mirror_cap;
    // peer-memory exchange (xr_P > 0): every append goes to every rank's log
    int32_t xr_P;
    EngineState* const* xr_st;
    uint64_t* const* xr_log;
};

// Peer-memory exchange: reserve nb entries in rank q's log (system scope: q may be another GPU).
__device__ __forceinline__ unsigned long long xr_reserve(const Sink& sk, int q, unsigned long long nb) {
    return atomicAdd_system(&sk.xr_st[q]->log_size, nb);
}
// An append that does not fit flags this rank only; the cross-rank barrier sums the flags of
// every rank into the iteration's outcome (every rank then restarts with larger logs).
__device__ __forceinline__ void xr_flag_overflow(const Sink& sk) { *(volatile int*)sk.overflow = 1; }

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

// Warp-level deduplication of candidates: lanes holding the same cell (e.g. the hub
// cell (owl:Class, owl:Class) reached from thousands of classes) elect the lowest lane,
// which carries the minimum length; same-address atomics would serialise in L2.
__device__ __forceinline__ bool warp_dedup(const EngineParams& p, const Sink& sk, bool has, uint32_t A, uint32_t i,
                                           uint32_t j, uint64_t& len, int lane) {
    uint64_t key = has ? pack_cell(A, i, j) : ~0ull;   // ~0 is never a cell (node ids < 2^27 - 1)
    unsigned peers = __match_any_sync(kFull, key);
    if (p.lengths) {
        if (has && len > 0xffffffffull) *(volatile int*)sk.len_overflow = 1;
        uint32_t l = (uint32_t)(len > 0xffffffffull ? 0xffffffffull : len);
        len = __reduce_min_sync(peers, l);
    }
    return has && (__ffs(peers) - 1 == lane);
}

// Insert candidate (A,i,j) of length len into T_k; true iff the cell is new:
// relational -> the bit flips; single-path -> the key leaves EMPTY (atomicMin on
// (iteration<<32 | length): first write wins across iterations, min within one).
// ------------------------------------------------------------------------------------------
// Hashed cell set.  At config-4 scale the bit matrices are |N| x 512 MiB and every candidate
// is a random 4-byte atomic into them: the DRAM page / TLB misses cap the whole GPU at
// ~20 G atomics/s (scripts/tlb_probe.cu).  The cells themselves are few (2.9 M at config 4),
// so for relational runs whose rules all have a preterminal operand (no row scans of T)
// the set of derived cells lives in an open-addressing table of packed cells sized
// 2x the log (~64 MiB, L2-resident: ~130 G CAS/s).  Insert = atomicCAS(EMPTY -> cell)
// along a linear probe run; "new" iff this CAS filled the slot.  No deletions: a cell
// rolled back at log overflow stays in the table, and the host rebuilds the table from
// the log's valid prefix (launch_rehash) before the iteration is re-run.
// ------------------------------------------------------------------------------------------
__device__ __forceinline__ bool hash_insert(const EngineParams& p, uint64_t c, int* ovf,
                                            unsigned long long max_probe = kHashMaxProbe) {
    unsigned long long h = (c * 0x9E3779B97F4A7C15ull) >> p.hshift;
    for (unsigned long long probe = 0; probe < max_probe; ++probe) {
        unsigned long long old = atomicCAS(p.hset + h, kHashEmpty, (unsigned long long)c);
        if (old == kHashEmpty) return true;
        if (old == c) return false;
        h = (h + 1) & p.hmask;
    }
    *(volatile int*)ovf = 1;   // table too full: the host grows log + table and re-runs
    return false;
}

// need_flag: asynchronous-schedule logs mark written entries with bit 63 (kValid)
// N inserts with their home-slot CASes issued back to back (N round trips overlap, like
// the N independent atomicOr of the bit-matrix path); collisions (~20% at load 1/2)
// continue probing one by one.
template <int N>
__device__ __forceinline__ void hash_insert_n(const EngineParams& p, const uint64_t (&c)[N], const bool (&has)[N],
                                              bool (&fresh)[N], int* ovf) {
    unsigned long long h[N], old[N];
#pragma unroll
    for (int q = 0; q < N; ++q) {
        h[q] = (c[q] * 0x9E3779B97F4A7C15ull) >> p.hshift;
        const bool own = cell_i(c[q]) >= p.row_lo && cell_i(c[q]) < p.row_hi;
        old[q] = has[q] && own ? atomicCAS(p.hset + h[q], kHashEmpty, (unsigned long long)c[q]) : (unsigned long long)c[q];
    }
#pragma unroll
    for (int q = 0; q < N; ++q) {
        fresh[q] = old[q] == kHashEmpty;
        if (!fresh[q] && old[q] != c[q]) {
            unsigned long long hh = h[q];
            fresh[q] = false;
            for (int probe = 1; probe < kHashMaxProbe; ++probe) {
                hh = (hh + 1) & p.hmask;
                unsigned long long o = atomicCAS(p.hset + hh, kHashEmpty, (unsigned long long)c[q]);
                if (o == kHashEmpty) {
                    fresh[q] = true;
                    break;
                }
                if (o == c[q]) break;
                if (probe == kHashMaxProbe - 1) *(volatile int*)ovf = 1;
            }
        }
    }
}

__device__ __forceinline__ void hash_pair(const EngineParams& p, bool has0, uint64_t c0, bool has1, uint64_t c1,
                                          bool& n0, bool& n1, int* ovf) {
    const uint64_t c[2] = {c0, c1};
    const bool has[2] = {has0, has1};
    bool f[2];
    hash_insert_n<2>(p, c, has, f, ovf);
    n0 = f[0];
    n1 = f[1];
}

__global__ void rehash_kernel(EngineParams p, unsigned long long n_cells, uint64_t cell_mask, int need_flag) {
    int dummy = 0;
    for (unsigned long long e = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; e < n_cells;
         e += (unsigned long long)gridDim.x * blockDim.x) {
        const uint64_t c = ldcg64(p.log + e);
        if (need_flag && !(c >> 63)) continue;
        hash_insert(p, c & cell_mask, &dummy, p.hmask + 1);
    }
}

__global__ void log_to_bitmap_kernel(const uint64_t* __restrict__ log, unsigned long long n_cells, uint32_t A,
                                     uint32_t* dst, int64_t stride) {
    for (unsigned long long e = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; e < n_cells;
         e += (unsigned long long)gridDim.x * blockDim.x) {
        uint64_t c = log[e];
        if (cell_nt(c) == A) atomicOr(dst + (size_t)cell_i(c) * stride + (cell_j(c) >> 5), 1u << (cell_j(c) & 31));
    }
}

__device__ __forceinline__ bool try_insert(const EngineParams& p, const NTInfo* nt, const Sink& sk, bool has,
                                           uint32_t A, uint32_t i, uint32_t j, uint64_t len, long long k) {
    if (!has || i < p.row_lo || i >= p.row_hi) return false;   // rows owned by this shard only
    CFPQ_DASSERT(A < (uint32_t)p.n_nt && i < (uint32_t)p.n && j < (uint32_t)p.n);
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
    // seeding (k = 0) may probe the whole table: it holds >= 2x the seed bound, so it ends
    if (p.hset) return hash_insert(p, pack_cell(A, i, j), sk.overflow, k == 0 ? p.hmask + 1 : kHashMaxProbe);
    uint32_t bit = 1u << (j & 31);
    uint32_t* word = nt[A].T + (size_t)i * (size_t)p.Wp + (j >> 5);
    if (p.precheck && (ldcg32(word) & bit)) return false;   // already set: no RMW on a hot word
    uint32_t old = atomicOr(word, bit);
    return !(old & bit);
}

// Append the warp's staged cells to the log (one atomic per flush).  A cell that
// does not fit is rolled back so that a re-run of the iteration (after the host
// grows the log) rediscovers it; appended cells stay set and are not re-appended.
__device__ __forceinline__ void flush(const EngineParams& p, const NTInfo* nt, const Sink& sk, WarpScratch* ws,
                                      int lane) {
    int nb = ws->nbuf;
    if (nb == 0) return;
    if (sk.xr_P) {
        // peer-memory exchange: the warp's cells into every rank's log (relational only)
        for (int q = 0; q < sk.xr_P; ++q) {
            unsigned long long base = 0;
            if (lane == 0) base = xr_reserve(sk, q, (unsigned long long)nb);
            base = __shfl_sync(kFull, base, 0);
            uint64_t* lg = sk.xr_log[q];
            for (int t = lane; t < nb; t += 32) {
                const unsigned long long idx = base + (unsigned long long)t;
                if (idx < p.log_cap) lg[idx] = ws->buf[t];
                else xr_flag_overflow(sk);
            }
        }
        if (lane == 0) atomicAdd(&p.st->xr_new, (unsigned long long)nb);   // this rank's new cells
        __syncwarp();
        if (lane == 0) ws->nbuf = 0;
        __syncwarp();
        return;
    }
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
            p.log[idx] = c | sk.tag;
            if (sk.mirror != nullptr && idx - sk.mirror_base < sk.mirror_cap) sk.mirror[idx - sk.mirror_base] = c;
            if (sk.tag) {   // asynchronous schedule: snapshots are live (any state <= T^cf is sound)
                if (nt[A].S) atomicOr(nt[A].S + (size_t)i * p.Wp + (j >> 5), 1u << (j & 31));
                if (nt[A].ST) atomicOr(nt[A].ST + (size_t)j * p.Wp + (i >> 5), 1u << (i & 31));
            }
            if (K != nullptr) atomicOr(word, bit);   // the bit matrix mirrors the keys
            if (p.rowc != nullptr) {
                atomicAdd(p.rowc + (size_t)A * p.n + i, 1u);
                atomicAdd(p.colc + (size_t)A * p.n + j, 1u);
            }
        } else {
            if (K != nullptr) atomicExch((unsigned long long*)(K + (size_t)i * (size_t)p.n + j),
                                         (unsigned long long)kEmptyKey);
            else if (!p.hset) atomicAnd(word, ~bit);
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
    bool keep = warp_dedup(p, sk, has, A, i, j, len, lane);
    bool d = try_insert(p, nt, sk, keep, A, i, j, len, k);
    stage(p, nt, sk, ws, lane, d, A, i, j);
}

__device__ __forceinline__ Sink global_sink(const EngineParams& p) {
    Sink sk;
    sk.tag = 0;
    sk.counter = &p.st->log_size;
    sk.overflow = &p.st->overflow;
    sk.len_overflow = &p.st->len_overflow;
    sk.mirror = nullptr;
    sk.mirror_base = 0;
    sk.mirror_cap = 0;
    sk.xr_P = 0;
    sk.xr_st = nullptr;
    sk.xr_log = nullptr;
    return sk;
}

// End of a grid-wide expansion: the CTA appends all warps' staged cells with ONE global
// atomic (thousands of warps ending the iteration together would otherwise serialise on
// the log counter).
// Peer-memory exchange variant: one reservation per rank's log per CTA (warp 0, lane q),
// then every warp writes its cells into every rank's log.
template <int NW>
__device__ void cta_flush_xr(const EngineParams& p, const Sink& sk, WarpScratch* ws_all, int wib, int lane,
                             unsigned long long* s_bases, int32_t* s_prefix) {
    __syncthreads();
    if (wib == 0) {
        int nb = lane < NW ? ws_all[lane].nbuf : 0;
        int incl = nb;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int v = __shfl_up_sync(kFull, incl, o);
            if (lane >= o) incl += v;
        }
        if (lane < NW) s_prefix[lane] = incl - nb;
        const int tot = __shfl_sync(kFull, incl, 31);
        if (lane < sk.xr_P) s_bases[lane] = tot ? xr_reserve(sk, lane, (unsigned long long)tot) : 0ull;
        if (lane == 0 && tot) atomicAdd(&p.st->xr_new, (unsigned long long)tot);   // this rank's new cells
    }
    __syncthreads();
    WarpScratch* ws = &ws_all[wib];
    const int nb = ws->nbuf;
    for (int q = 0; q < sk.xr_P; ++q) {
        const unsigned long long base = s_bases[q] + (unsigned long long)s_prefix[wib];
        uint64_t* lg = sk.xr_log[q];
        for (int t = lane; t < nb; t += 32) {
            const unsigned long long idx = base + (unsigned long long)t;
            if (idx < p.log_cap) lg[idx] = ws->buf[t];
            else xr_flag_overflow(sk);
        }
    }
    __syncwarp();
    if (lane == 0) ws->nbuf = 0;
    __syncwarp();
}

template <int NW>
__device__ void cta_flush_n(const EngineParams& p, const NTInfo* nt, const Sink& sk, WarpScratch* ws_all, int wib,
                            int lane, unsigned long long* s_base, int32_t* s_prefix) {
    __syncthreads();
    if (wib == 0) {
        int nb = lane < NW ? ws_all[lane].nbuf : 0;
        int incl = nb;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int v = __shfl_up_sync(kFull, incl, o);
            if (lane >= o) incl += v;
        }
        if (lane < NW) s_prefix[lane] = incl - nb;
        int tot = __shfl_sync(kFull, incl, 31);
        unsigned long long b = 0;
        if (lane == 0 && tot) b = atomicAdd(sk.counter, (unsigned long long)tot);
        if (lane == 0) *s_base = b;
    }
    __syncthreads();
    WarpScratch* ws = &ws_all[wib];
    const int nb = ws->nbuf;
    const unsigned long long base = *s_base + (unsigned long long)s_prefix[wib];
    for (int t = lane; t < nb; t += 32) {
        uint64_t c = ws->buf[t];
        unsigned long long idx = base + (unsigned long long)t;
        uint32_t A = cell_nt(c), i = cell_i(c), j = cell_j(c);
        uint64_t* K = p.lengths ? nt[A].K : nullptr;
        uint32_t* word = nt[A].T + (size_t)i * (size_t)p.Wp + (j >> 5);
        uint32_t bit = 1u << (j & 31);
        if (idx < p.log_cap) {
            p.log[idx] = c;
            if (K != nullptr) atomicOr(word, bit);
            if (p.rowc != nullptr) {
                atomicAdd(p.rowc + (size_t)A * p.n + i, 1u);
                atomicAdd(p.colc + (size_t)A * p.n + j, 1u);
            }
        } else {
            if (K != nullptr) atomicExch((unsigned long long*)(K + (size_t)i * (size_t)p.n + j),
                                         (unsigned long long)kEmptyKey);
            else if (!p.hset) atomicAnd(word, ~bit);
            *(volatile int*)sk.overflow = 1;
        }
    }
    __syncwarp();
    if (lane == 0) ws->nbuf = 0;
    __syncwarp();
}

__device__ __forceinline__ void cta_flush(const EngineParams& p, const NTInfo* nt, const Sink& sk, WarpScratch* ws_all,
                                          int wib, int lane, unsigned long long* s_base, int32_t* s_prefix) {
    cta_flush_n<kWarps>(p, nt, sk, ws_all, wib, lane, s_base, s_prefix);
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
    // one log atomic per CTA (thousands of warps ending together would serialise on it)
    __shared__ unsigned long long s_base;
    __shared__ int32_t s_prefix[kSeedBlock / 32];
    cta_flush_n<kSeedBlock / 32>(p, p.nt, sk, wsa, threadIdx.x >> 5, lane, &s_base, s_prefix);
}

// CSR / CSC of preterminals from the seed cells Δ_0 = log[0, n_seed).
// slot_row[X] / slot_col[X] = offset (in units of (n+1)) of X's CSR / CSC pointer
// array inside the concatenated count array, or -1.
// Degree counts of the preterminal slots over the seed cells Δ_0 = log[0, n_seed); block 0
// also opens iteration 1 (the work of begin_kernel: Δ_0 = [0, n_seed)).
__global__ void adj_count_kernel(EngineParams p, const int32_t* __restrict__ slot_row,
                                 const int32_t* __restrict__ slot_col, int32_t* counts) {
    const unsigned long long n_seed = ld_volatile_u64(&p.st->log_size);
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        p.st->lo = 0;
        p.st->hi = n_seed;
        p.st->iter = 0;
        if (p.iter_off_cap > 0) p.iter_off[0] = 0;
        if (p.iter_off_cap > 1) p.iter_off[1] = n_seed;
        if (p.iter_time) p.iter_time[0] = globaltimer();
        p.st->gs_ring[1] = n_seed;   // L_1 (Gauss-Seidel windows)
        p.st->gs_slot = 1;
        p.st->gs_stage = 0;
        p.st->gs_round = 0;
    }
    for (unsigned long long e = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; e < n_seed;
         e += (unsigned long long)gridDim.x * blockDim.x) {
        uint64_t c = p.log[e];
        uint32_t X = cell_nt(c);
        int32_t sr = __ldg(slot_row + X), sc = __ldg(slot_col + X);
        if (sr >= 0) atomicAdd(counts + (size_t)sr * (p.n + 1) + cell_i(c), 1);
        if (sc >= 0) atomicAdd(counts + (size_t)sc * (p.n + 1) + cell_j(c), 1);
    }
}

// Scatter the neighbours into CSR order and write the ELL heads in the same pass: the
// counts are consumed (atomicSub: slot ptr[r] + old - 1, so they end at zero), the entry
// that lands in a row's first slot writes {beg, deg, nb0}, the second one nb1 (ell was
// zeroed: deg 0 rows read {0, 0, 0, 0}).
__device__ __forceinline__ void adj_place(const int32_t* __restrict__ ptr, int32_t* counts, int32_t* idx, int4* ell,
                                          size_t slot_off, size_t ell_off, uint32_t row, int32_t nb) {
    const int32_t beg = ptr[slot_off + row];
    const int32_t old = atomicSub(counts + slot_off + row, 1);
    const int32_t pos = beg + old - 1;
    idx[pos] = nb;
    int* e = reinterpret_cast<int*>(ell + ell_off + row);
    if (old == 1) {
        e[0] = beg;
        e[1] = ptr[slot_off + row + 1] - beg;
        e[2] = nb;
    } else if (old == 2) {
        e[3] = nb;
    }
}

__global__ void adj_fill_kernel(EngineParams p, const int32_t* __restrict__ slot_row,
                                const int32_t* __restrict__ slot_col, const int32_t* __restrict__ ptr,
                                int32_t* counts, int32_t* idx, int4* ell) {
    const unsigned long long n_seed = ld_volatile_u64(&p.st->hi);
    for (unsigned long long e = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; e < n_seed;
         e += (unsigned long long)gridDim.x * blockDim.x) {
        uint64_t c = p.log[e];
        uint32_t X = cell_nt(c);
        int32_t sr = __ldg(slot_row + X), sc = __ldg(slot_col + X);
        if (sr >= 0)
            adj_place(ptr, counts, idx, ell, (size_t)sr * (p.n + 1), (size_t)sr * p.n, cell_i(c), (int32_t)cell_j(c));
        if (sc >= 0)
            adj_place(ptr, counts, idx, ell, (size_t)sc * (p.n + 1), (size_t)sc * p.n, cell_j(c), (int32_t)cell_i(c));
    }
}

// Reset the bit word of a cell by zeroing its whole aligned 32-byte sector: every bit of the
// matrices is being reset (all of them belong to logged cells), and a full-sector store needs
// no DRAM read-modify-write of a partial sector.
__device__ __forceinline__ void zero_sector(uint32_t* w) {
    uint4* sct = reinterpret_cast<uint4*>(reinterpret_cast<uintptr_t>(w) & ~uintptr_t(31));
    sct[0] = make_uint4(0u, 0u, 0u, 0u);
    sct[1] = make_uint4(0u, 0u, 0u, 0u);
}

// Clear the cells of a previous run (bitmaps, snapshots, keys, counters) in O(|log|).
__global__ void clear_log_kernel(EngineParams p, unsigned long long n_cells) {
    for (unsigned long long e = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; e < n_cells;
         e += (unsigned long long)gridDim.x * blockDim.x) {
        uint64_t c = p.log[e];
        uint32_t A = cell_nt(c), i = cell_i(c), j = cell_j(c);
        const NTInfo& nt = p.nt[A];
        if (nt.T) zero_sector(nt.T + (size_t)i * p.Wp + (j >> 5));
        if (nt.S) zero_sector(nt.S + (size_t)i * p.Wp + (j >> 5));
        if (nt.ST) zero_sector(nt.ST + (size_t)j * p.Wp + (i >> 5));
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

// Gauss-Seidel schedule: step k applies only the rules of stage (k-1) mod S.
__device__ __forceinline__ bool stage_ok(const EngineParams& p, const Expansion& ex, int stage) {
    return p.gs_stages == 0 || ex.stage == stage;
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
            CFPQ_DASSERT((long long)ws->beg[l] + (t - ws->off[l]) < p.adj_cap);
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
    CFPQ_DASSERT(ci < 0x7fffffffu && cj < 0x7fffffffu && ex.other >= 0 && ex.A >= 0);
    if (ex.kind == EXP_L_CONST) {          // Δ_B entry (i, r=cj): row r of preterminal C
        fx = ci;
        return __ldg(nt[ex.other].csr_ell + cj);
    }
    fx = cj | 0x80000000u;                 // Δ_C entry (r=ci, j): column r of preterminal B
    return __ldg(nt[ex.other].csc_ell + ci);
}

// Expand one 32-entry chunk (one entry per lane, `valid` lanes only) of iteration k.
__device__ __forceinline__ void expand_chunk(const EngineParams& p, const NTInfo* nt, const Expansion* exps,
                                             const Sink& sk, uint64_t cell, bool valid, long long k, int gstage, int lane,
                                             WarpScratch* ws, unsigned long long& dcand, unsigned long long& dexp) {
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
    if (maxexp == 0) return;

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
            if (!stage_ok(p, ex, gstage)) continue;
            // row shards: an L expansion derives cells in the entry's row only
            if (ex.kind == EXP_L_CONST && (ci < p.row_lo || ci >= p.row_hi)) continue;
            if (ex.kind == EXP_L_CONST || ex.kind == EXP_R_CONST) el[x] = load_head(nt, ex, ci, cj, eA[x], efx[x]);
            else var_mask |= 1u << x;
        }
    }
    bool d0[kPre], d1[kPre];
    uint32_t ci0[kPre], cj0[kPre], ci1[kPre], cj1[kPre];
    if (p.hset) {
        // hashed cell set: all 2*kPre home-slot CASes in flight together
        uint64_t hc[2 * kPre];
        bool hk[2 * kPre], hf[2 * kPre];
#pragma unroll
        for (int x = 0; x < kPre; ++x) {
            cand_coords(efx[x], el[x].z, ci0[x], cj0[x]);
            cand_coords(efx[x], el[x].w, ci1[x], cj1[x]);
            uint64_t l0 = 1ull, l1 = 1ull;
            hk[2 * x] = warp_dedup(p, sk, el[x].y > 0, eA[x], ci0[x], cj0[x], l0, lane);
            hk[2 * x + 1] = warp_dedup(p, sk, el[x].y > 1, eA[x], ci1[x], cj1[x], l1, lane);
            hc[2 * x] = pack_cell(eA[x], ci0[x], cj0[x]);
            hc[2 * x + 1] = pack_cell(eA[x], ci1[x], cj1[x]);
            dcand += (unsigned long long)el[x].y;
        }
        hash_insert_n<2 * kPre>(p, hc, hk, hf, sk.overflow);
#pragma unroll
        for (int x = 0; x < kPre; ++x) {
            d0[x] = hf[2 * x];
            d1[x] = hf[2 * x + 1];
        }
    } else {
#pragma unroll
        for (int x = 0; x < kPre; ++x) {
            cand_coords(efx[x], el[x].z, ci0[x], cj0[x]);
            cand_coords(efx[x], el[x].w, ci1[x], cj1[x]);
            uint64_t l0 = (uint64_t)len_e + 1ull, l1 = l0;
            bool k0 = warp_dedup(p, sk, el[x].y > 0, eA[x], ci0[x], cj0[x], l0, lane);
            bool k1 = warp_dedup(p, sk, el[x].y > 1, eA[x], ci1[x], cj1[x], l1, lane);
            d0[x] = try_insert(p, nt, sk, k0, eA[x], ci0[x], cj0[x], l0, k);
            d1[x] = try_insert(p, nt, sk, k1, eA[x], ci1[x], cj1[x], l1, k);
            dcand += (unsigned long long)el[x].y;
        }
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
            if (!stage_ok(p, ex, gstage) || (ex.kind == EXP_L_CONST && (ci < p.row_lo || ci >= p.row_hi))) {
            } else if (ex.kind == EXP_L_CONST || ex.kind == EXP_R_CONST) {
                h = load_head(nt, ex, ci, cj, A, fx);
            } else if (x < 32) {
                var_mask |= 1u << x;
            }
        }
        uint32_t a0, b0, a1, b1;
        cand_coords(fx, h.z, a0, b0);
        cand_coords(fx, h.w, a1, b1);
        uint64_t l0 = (uint64_t)len_e + 1ull, l1 = l0;
        bool k0 = warp_dedup(p, sk, h.y > 0, A, a0, b0, l0, lane);
        bool k1 = warp_dedup(p, sk, h.y > 1, A, a1, b1, l1, lane);
        bool q0, q1;
        if (p.hset) {
            hash_pair(p, k0, pack_cell(A, a0, b0), k1, pack_cell(A, a1, b1), q0, q1, sk.overflow);
        } else {
            q0 = try_insert(p, nt, sk, k0, A, a0, b0, l0, k);
            q1 = try_insert(p, nt, sk, k1, A, a1, b1, l1, k);
        }
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

// Expand the Δ entries log[lo,hi) of iteration k.  Work unit = a chunk of 32
// consecutive entries per warp; warps [warp, warp+nwarps) stride over chunks.
// `src` = shared-memory copy of log[lo,hi) (single-CTA path) or null (read the log).
__device__ void expand(const EngineParams& p, const NTInfo* nt, const Expansion* exps, const Sink& sk,
                       const uint64_t* src, unsigned long long lo, unsigned long long hi, long long k, int gstage, int warp,
                       int nwarps, int lane, WarpScratch* ws, unsigned long long& dcand, unsigned long long& dexp,
                       bool final_flush = true) {
    for (unsigned long long cbase = lo + (unsigned long long)warp * 32ull; cbase < hi;
         cbase += (unsigned long long)nwarps * 32ull) {
        unsigned long long e = cbase + lane;
        bool valid = e < hi;
        uint64_t cell = 0ull;
        if (valid) cell = src ? src[e - lo] : ldcg64(p.log + e);
        expand_chunk(p, nt, exps, sk, cell, valid, k, gstage, lane, ws, dcand, dexp);
    }
    if (final_flush) flush(p, nt, sk, ws, lane);
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
    int gs_stage, gs_slot;   // Gauss-Seidel: stage of the next step, ring slot of its L (EngineState)
    long long gs_round;
};

// ---- memory-model primitives for the grid barrier (release/acquire at gpu scope) ----
__device__ __forceinline__ unsigned atom_add_acq_rel(unsigned* p, unsigned v) {
    unsigned old;
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
    return old;
}
__device__ __forceinline__ void red_add_release(unsigned* p, unsigned v) {
    asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void fence_acq_rel() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
__device__ __forceinline__ unsigned long long ld_acquire_word(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_word(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
constexpr int kBarGenShift = 40;
constexpr unsigned long long kBarLsMask = (1ull << 38) - 1;
// The released barrier word of the last arriver: next generation | flags | log size.
__device__ __forceinline__ unsigned long long bar_release_word(EngineState* st, unsigned long long gen, long long k) {
    unsigned long long f = 0, ls = 0;
    if (k >= 0) {
        f = (*(volatile int*)&st->overflow ? 1ull : 0ull) | (*(volatile int*)&st->len_overflow ? 2ull : 0ull);
        ls = ld_volatile_u64(&st->log_size) & kBarLsMask;
    }
    return (((gen + 1) & 0xFFFFFFull) << kBarGenShift) | (f << 38) | ls;
}

// Close iteration k from the log size `ls` and the error flags: Δ_k = log[hi, ls).
// Every CTA runs this on identical inputs and reaches the identical state.
__device__ __forceinline__ void close_iteration(const EngineParams& p, long long k, LoopState& s, unsigned long long ls,
                                                int flags, bool record, unsigned long long* gs_ring = nullptr) {
    if (flags & 2) {
        s.status = ST_LEN_OVERFLOW;
        return;
    }
    if (flags & 1) {
        s.status = ST_OVERFLOW;   // keep lo/hi/iter: the host grows the log and re-runs k
        return;
    }
    if (p.gs_stages > 0) {
        // Gauss-Seidel: step k+1 expands log[L_{k+1-S}, L_{k+1}) (everything derived since its
        // stage last ran); slots and stages advance incrementally (R = S+1, so the slot of
        // L_{k+1-S} is the one after L_{k+1}'s); fixpoint test and records per round of S steps
        const int S = p.gs_stages, R = S + 1;
        unsigned long long* ring = gs_ring ? gs_ring : p.st->gs_ring;   // warp-solo: a shared copy
        const int slot = s.gs_slot + 1 == R ? 0 : s.gs_slot + 1;        // (k+1) mod R
        const int lo_slot = slot + 1 == R ? 0 : slot + 1;               // (k+1-S) mod R
        const unsigned long long lo = k + 1 - S >= 1 ? *(volatile unsigned long long*)&ring[lo_slot] : 0ull;
        if (record) ring[slot] = ls;   // read S steps later; never the slot read above
        s.lo = lo;
        s.hi = ls;
        s.iter = k;
        s.gs_slot = slot;
        s.gs_stage = s.gs_stage + 1 == S ? 0 : s.gs_stage + 1;
        if (s.gs_stage != 0) return;   // a round ends when the next step is stage 0 again
        const long long rd = ++s.gs_round;
        if (record) {
            if (rd < p.iter_off_cap) {
                p.iter_off[rd] = lo;
                if (p.iter_time) p.iter_time[rd] = globaltimer();
            }
            if (rd + 1 < p.iter_off_cap) p.iter_off[rd + 1] = ls;
        }
        if (ls == lo) s.status = ST_DONE;                // a whole round added nothing
        else if (rd >= p.max_iter) s.status = ST_CAP;
        return;
    }
    s.lo = s.hi;
    s.hi = ls;
    s.iter = k;
    if (record) {
        if (k < p.iter_off_cap) {
            p.iter_off[k] = s.lo;
            if (p.iter_time) p.iter_time[k] = globaltimer();
        }
        if (k + 1 < p.iter_off_cap) p.iter_off[k + 1] = ls;
    }
    if (ls == s.lo) s.status = ST_DONE;             // T_k = T_{k-1}: fixpoint
    else if (k >= p.max_iter) s.status = ST_CAP;    // Theorem 3 cap
    else if (p.switch_cells && ls - s.lo > p.switch_cells) s.status = ST_SWITCH;   // dense Δ: tensor engine
}

__device__ void publish(const EngineParams& p, const LoopState& s) {
    EngineState* st = p.st;
    st->lo = s.lo;
    st->hi = s.hi;
    st->iter = s.iter;
    st->status = s.status;
    st->gs_stage = s.gs_stage;
    st->gs_slot = s.gs_slot;
    st->gs_round = s.gs_round;
    fence_acq_rel();
}

// ---- clearing the other bank's cells with otherwise idle barrier time ----
constexpr unsigned long long kClrChunk = 2048;

// Reset one claimed chunk of the previous run's cells (same work as clear_log_kernel).
__device__ __forceinline__ void clear_chunk(const EngineParams& p, unsigned long long base) {
    const unsigned long long end = min(base + kClrChunk, p.clr_n);
    for (unsigned long long e = base + threadIdx.x; e < end; e += kBlock) {
        const uint64_t c = ldcg64(p.clr_log + e);
        const uint32_t A = cell_nt(c), i = cell_i(c), j = cell_j(c);
        CFPQ_DASSERT(A < (uint32_t)p.n_nt && i < (uint32_t)p.n && j < (uint32_t)p.n);
        const NTInfo& t = p.clr_nt[A];
        if (t.T) zero_sector(t.T + (size_t)i * p.Wp + (j >> 5));
        if (t.S) zero_sector(t.S + (size_t)i * p.Wp + (j >> 5));
        if (t.ST) zero_sector(t.ST + (size_t)j * p.Wp + (i >> 5));
        if (t.K) t.K[(size_t)i * p.n + j] = kEmptyKey;
        if (p.clr_rowc) {
            p.clr_rowc[(size_t)A * p.n + i] = 0u;
            p.clr_colc[(size_t)A * p.n + j] = 0u;
        }
    }
}

// Whole CTA: claim and clear chunks until none is left (kernel end).
__device__ void clear_drain(const EngineParams& p) {
    __shared__ unsigned long long s_base;
    if (p.clr_n == 0) return;
    for (;;) {
        __syncthreads();
        if (threadIdx.x == 0) s_base = atomicAdd(&p.st->clr_cursor, kClrChunk);
        __syncthreads();
        if (s_base >= p.clr_n) break;
        clear_chunk(p, s_base);
    }
}

// Grid barrier (generation counter, release/acquire).  If k >= 0 the last CTA to arrive
// publishes the log size and error flags of iteration k in the released word; every CTA
// closes the iteration from it (`word`, valid in thread 0 after the barrier).
__device__ bool grid_barrier(const EngineParams& p, long long k, unsigned long long* word = nullptr) {
    __shared__ int s_timeout;
    __shared__ unsigned long long s_word;
    if (p.clr_n) {
        // CTAs that are not the last to arrive clear chunks of the other bank while they
        // wait; the release is checked between chunks
        __shared__ int s_go;
        __shared__ unsigned long long s_my;
        __shared__ unsigned long long s_base;
        __syncthreads();
        if (threadIdx.x == 0) {
            s_timeout = 0;
            s_go = 0;
            EngineState* st = p.st;
            s_my = ld_volatile_u64(&st->bar_word) >> kBarGenShift;
            unsigned arrived = atom_add_acq_rel(&st->bar_count, 1u);
            if (arrived == (unsigned)p.nblocks - 1u) {
                const unsigned long long w = bar_release_word(st, s_my, k);
                st->bar_count = 0u;
                st_release_word(&st->bar_word, w);
                s_word = w;
                s_go = 1;
            }
        }
        __syncthreads();
        while (!s_go) {
            if (threadIdx.x == 0)
                s_base = ld_volatile_u64(&p.st->clr_cursor) < p.clr_n ? atomicAdd(&p.st->clr_cursor, kClrChunk)
                                                                       : ~0ull;
            __syncthreads();
            const bool work = s_base < p.clr_n;
            if (work) clear_chunk(p, s_base);
            if (threadIdx.x == 0) {
                unsigned long long w = ld_acquire_word(&p.st->bar_word);
                if ((w >> kBarGenShift) != s_my) {
                    s_word = w;
                    s_go = 1;
                } else if (!work) {
                    // nothing left to clear: plain wait
                    long long t0 = clock64();
                    unsigned ns = 0;
                    while (((w = ld_acquire_word(&p.st->bar_word)) >> kBarGenShift) == s_my) {
                        if (ns) __nanosleep(ns);
                        if (clock64() - t0 > 40000) ns = ns ? (ns < 2048u ? ns * 2u : 2048u) : 64u;
                        if (clock64() - t0 > 60000000000ll) {
                            s_timeout = 1;
                            break;
                        }
                    }
                    s_word = w;
                    s_go = 1;
                }
            }
            __syncthreads();
        }
        if (word && threadIdx.x == 0) *word = s_word;
        return s_timeout == 0;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        s_timeout = 0;
        EngineState* st = p.st;
        const unsigned long long my = ld_volatile_u64(&st->bar_word) >> kBarGenShift;
        unsigned arrived = atom_add_acq_rel(&st->bar_count, 1u);
        unsigned long long w;
        if (arrived == (unsigned)p.nblocks - 1u) {
            w = bar_release_word(st, my, k);
            st->bar_count = 0u;
            st_release_word(&st->bar_word, w);
        } else {
            long long t0 = clock64();
            unsigned ns = 0;
            while (((w = ld_acquire_word(&st->bar_word)) >> kBarGenShift) == my) {
                // poll at L2 latency for ~20 µs (grid iterations), then back off (a
                // single-CTA phase can park the other CTAs for a long time)
                if (ns) __nanosleep(ns);
                if (clock64() - t0 > 40000) ns = ns ? (ns < 2048u ? ns * 2u : 2048u) : 64u;
                if (clock64() - t0 > 60000000000ll) {   // ~30 s watchdog: never hang the GPU
                    s_timeout = 1;
                    break;
                }
            }
        }
        if (word) *word = w;
    }
    __syncthreads();
    return s_timeout == 0;
}

// ------------------------------------------------------------------------------------------
// Seeding inside the closure kernel (fused_seed; one-GPU sparse runs).  Alg. 1 lines 6-7
// as in seed_kernel, but a NEW seed cell of a preterminal also counts itself into
// the ELL head of its row (CSR) / column (CSC) slot and claims the first two neighbour slots;
// the CSR tails (exclusive scan of the degrees + fill) are built only when some head has
// more than two entries.  Replaces 5-8 launches of the seed phase by grid barriers.
// ------------------------------------------------------------------------------------------
__device__ __forceinline__ void ell_add(const EngineParams& p, int sl, uint32_t row, int32_t nb) {
    int* e = reinterpret_cast<int*>(p.ell + (size_t)sl * p.n + row);
    const int old = atomicAdd(e + 1, 1);
    if (old == 0) e[2] = nb;
    else if (old == 1) e[3] = nb;
    else if (old == 2) *(volatile int*)&p.st->adj_tail = 1;
}

__device__ __forceinline__ void ell_place(const EngineParams& p, int sl, uint32_t row, int32_t nb) {
    const size_t x = (size_t)sl * p.n + row;
    int* e = reinterpret_cast<int*>(p.ell + x);
    const int k = atomicAdd(p.adj_cursor + x, 1);
    CFPQ_DASSERT((long long)e[0] + k < p.adj_cap && row < (uint32_t)p.n);
    p.adj_idx_w[e[0] + k] = nb;
    if (k == 0) e[2] = nb;          // the ELL copies are the first two CSR entries
    else if (k == 1) e[3] = nb;
}

// Block-wide exclusive scan of one value per thread (kBlock threads); returns the prefix,
// *total = the block's sum.
__device__ unsigned long long block_exclusive_scan(unsigned long long v, unsigned long long* total) {
    __shared__ unsigned long long s_w[kWarps];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    unsigned long long incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long t = __shfl_up_sync(kFull, incl, o);
        if (lane >= o) incl += t;
    }
    if (lane == 31) s_w[wib] = incl;
    __syncthreads();
    if (wib == 0) {
        unsigned long long w = lane < kWarps ? s_w[lane] : 0ull;
        unsigned long long wi = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned long long t = __shfl_up_sync(kFull, wi, o);
            if (lane >= o) wi += t;
        }
        if (lane < kWarps) s_w[lane] = wi - w;
        if (lane == kWarps - 1) *total = wi;
    }
    __syncthreads();
    const unsigned long long r = s_w[wib] + incl - v;
    __syncthreads();
    return r;
}

__device__ bool fused_seed_phase(const EngineParams& p, const NTInfo* nt, WarpScratch* ws_all, int wib, int lane,
                                 unsigned long long* s_base, int32_t* s_prefix, LoopState& s) {
    __shared__ unsigned long long s_nseed, s_total, s_off;
    __shared__ int s_tail;
    const long long gtid = (long long)blockIdx.x * kBlock + threadIdx.x;
    const long long gthreads = (long long)gridDim.x * kBlock;
    const size_t ne = (size_t)p.n_slots * (size_t)p.n;
    for (size_t t = (size_t)gtid; t < ne; t += (size_t)gthreads) {
        p.ell[t] = make_int4(0, 0, 0, 0);
        p.adj_cursor[t] = 0;
    }
    if (!grid_barrier(p, -1)) return false;
    // ---- T_0 ----
    const Sink sk = global_sink(p);
    WarpScratch* ws = &ws_all[wib];
    for (int64_t base = (int64_t)blockIdx.x * kBlock; base < p.n_edges; base += gthreads) {
        const int64_t e = base + threadIdx.x;
        bool valid = e < p.n_edges;
        int32_t sv = 0, x = 0, dv = 0, rb = 0, re = 0;
        if (valid) {
            sv = __ldg(p.edges + 3 * e);
            x = __ldg(p.edges + 3 * e + 1);
            dv = __ldg(p.edges + 3 * e + 2);
            if (sv < 0 || sv >= p.n || dv < 0 || dv >= p.n || x < 0 || x >= p.n_labels) {
                p.st->bad_edge = 1;
                valid = false;
            } else {
                rb = __ldg(p.lab_ptr + x);
                re = __ldg(p.lab_ptr + x + 1);
            }
        }
        for (int t = 0; t < p.max_rules; ++t) {
            const bool has = valid && (rb + t < re);
            const uint32_t A = has ? (uint32_t)__ldg(p.lab_nt + rb + t) : 0u;
            uint64_t len = 1;
            const bool keep = warp_dedup(p, sk, has, A, (uint32_t)sv, (uint32_t)dv, len, lane);
            const bool nw = try_insert(p, nt, sk, keep, A, (uint32_t)sv, (uint32_t)dv, len, 0);
            if (nw) {
                const int sr = __ldg(p.slot_row + A), sc = __ldg(p.slot_col + A);
                if (sr >= 0) ell_add(p, sr, (uint32_t)sv, dv);
                if (sc >= 0) ell_add(p, sc, (uint32_t)dv, sv);
            }
            stage(p, nt, sk, ws, lane, nw, A, (uint32_t)sv, (uint32_t)dv);
        }
    }
    cta_flush(p, nt, sk, ws_all, wib, lane, s_base, s_prefix);
    unsigned long long bw = 0;
    if (!grid_barrier(p, 0, &bw)) return false;
    if (threadIdx.x == 0) {
        s_nseed = bw & kBarLsMask;
        s_tail = *(volatile int*)&p.st->adj_tail;
    }
    __syncthreads();
    const unsigned long long n_seed = s_nseed;
    if (s_tail) {
        // ---- CSR tails: begins = exclusive scan of the degrees, then the fill ----
        const size_t per = (ne + gridDim.x - 1) / gridDim.x;
        const size_t lo = min(ne, (size_t)blockIdx.x * per), hi = min(ne, lo + per);
        const size_t sub = (hi - lo + kBlock - 1) / kBlock;
        const size_t a = min(hi, lo + (size_t)threadIdx.x * sub), b = min(hi, a + sub);
        unsigned long long mine = 0;
        for (size_t x = a; x < b; ++x) mine += (unsigned long long)p.ell[x].y;
        const unsigned long long excl = block_exclusive_scan(mine, &s_total);
        if (threadIdx.x == 0) p.scan_tot[blockIdx.x] = s_total;
        if (!grid_barrier(p, -1)) return false;
        if (wib == 0) {
            unsigned long long acc = 0;
            for (int q = lane; q < (int)blockIdx.x; q += 32) acc += ld_volatile_u64(&p.scan_tot[q]);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(kFull, acc, o);
            if (lane == 0) s_off = acc;
        }
        __syncthreads();
        unsigned long long run = s_off + excl;
        for (size_t x = a; x < b; ++x) {
            reinterpret_cast<int*>(p.ell + x)[0] = (int)run;
            run += (unsigned long long)p.ell[x].y;
        }
        if (!grid_barrier(p, -1)) return false;
        for (unsigned long long e = (unsigned long long)gtid; e < n_seed; e += (unsigned long long)gthreads) {
            const uint64_t c = ldcg64(p.log + e);
            const uint32_t X = cell_nt(c);
            const int sr = __ldg(p.slot_row + X), sc = __ldg(p.slot_col + X);
            if (sr >= 0) ell_place(p, sr, cell_i(c), (int32_t)cell_j(c));
            if (sc >= 0) ell_place(p, sc, cell_j(c), (int32_t)cell_i(c));
        }
        if (!grid_barrier(p, -1)) return false;
    }
    // ---- open iteration 1: Δ_0 = log[0, n_seed) (T_0) ----
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        EngineState* st = p.st;
        st->lo = 0;
        st->hi = n_seed;
        st->iter = 0;
        if (p.iter_off_cap > 0) p.iter_off[0] = 0;
        if (p.iter_off_cap > 1) p.iter_off[1] = n_seed;
        if (p.iter_time) p.iter_time[0] = globaltimer();
        st->gs_ring[1] = n_seed;
        st->gs_slot = 1;
        st->gs_stage = 0;
        st->gs_round = 0;
    }
    s.lo = 0;
    s.hi = n_seed;
    s.iter = 0;
    s.status = ST_RUNNING;
    s.gs_stage = 0;
    s.gs_slot = 1;
    s.gs_round = 0;
    if (p.has_snapshots) {
        apply_snapshots(p, nt, nullptr, 0, n_seed, gtid, gthreads);
        if (!grid_barrier(p, -1)) return false;
    }
    return true;
}

// Single-CTA iterations (|Δ| <= solo_max): one thread per Δ entry, Δ mirrored in
// shared memory, appends counted in shared memory.  Counters and error flags rotate
// over three slots (k mod 3) so that ONE __syncthreads() per iteration suffices: every
// thread reads slot k after the barrier and closes the iteration itself; slot k+1 is
// reset by thread 0 during iteration k, after every thread has read it (at iteration
// k-2's close, before the barrier of k-1).
struct SoloShared {
    uint64_t delta[2][kSoloMax];
    unsigned cnt[3];
    int ov[3], lov[3];
    long long solo;
};

__device__ __forceinline__ void solo_append(const EngineParams& p, const NTInfo* nt, SoloShared& so, int slot,
                                            unsigned long long base, uint64_t* mirror, uint32_t A, uint32_t i,
                                            uint32_t j) {
    unsigned long long idx = base + atomicAdd(&so.cnt[slot], 1u);
    uint64_t c = pack_cell(A, i, j);
    uint64_t* K = p.lengths ? nt[A].K : nullptr;
    uint32_t* word = nt[A].T + (size_t)i * (size_t)p.Wp + (j >> 5);
    uint32_t bit = 1u << (j & 31);
    if (idx < p.log_cap) {
        p.log[idx] = c;
        if (idx - base < (unsigned long long)kSoloMax) mirror[idx - base] = c;
        if (K != nullptr) atomicOr(word, bit);
        if (p.rowc != nullptr) {
            atomicAdd(p.rowc + (size_t)A * p.n + i, 1u);
            atomicAdd(p.colc + (size_t)A * p.n + j, 1u);
        }
    } else {
        if (K != nullptr) atomicExch((unsigned long long*)(K + (size_t)i * (size_t)p.n + j), (unsigned long long)kEmptyKey);
        else if (!p.hset) atomicAnd(word, ~bit);
        so.ov[slot] = 1;
    }
}

// Issue the bit/key atomic of a candidate; returns whether the cell is new.
__device__ __forceinline__ bool solo_try(const EngineParams& p, const NTInfo* nt, SoloShared& so, int slot, uint32_t A,
                                         uint32_t i, uint32_t j, uint64_t len, long long k) {
    if (i < p.row_lo || i >= p.row_hi) return false;
    uint64_t* K = nt[A].K;
    if (p.lengths && K != nullptr) {
        if (len > 0xffffffffull) {
            so.lov[slot] = 1;
            len = 0xffffffffull;
        }
        uint64_t old = atomicMin((unsigned long long*)(K + (size_t)i * (size_t)p.n + j),
                                 (unsigned long long)(((uint64_t)k << 32) | len));
        return old == kEmptyKey;
    }
    if (p.hset) return hash_insert(p, pack_cell(A, i, j), &so.ov[slot]);
    uint32_t bit = 1u << (j & 31);
    return !(atomicOr(nt[A].T + (size_t)i * (size_t)p.Wp + (j >> 5), bit) & bit);
}

// Prefetch into L1 the ELL head that the next iteration reads for candidate (A,i,j)
// if it becomes new (its first two rule occurrences); overlaps with the bit atomic.
__device__ __forceinline__ void prefetch_next(const NTInfo* nt, const Expansion* exps, uint32_t A, uint32_t i,
                                              uint32_t j) {
    int eb = nt[A].exp_begin, ee = nt[A].exp_end;
    for (int x = eb; x < ee && x < eb + 2; ++x) {
        Expansion ex = exps[x];
        const int4* a = nullptr;
        if (ex.kind == EXP_L_CONST) a = nt[ex.other].csr_ell + j;
        else if (ex.kind == EXP_R_CONST) a = nt[ex.other].csc_ell + i;
        if (a) asm volatile("prefetch.global.L1 [%0];" ::"l"(a));
    }
}

// ------------------------------------------------------------------------------------------
// Warp-solo iterations (|Δ| <= 32): warp 0 of CTA 0 alone, one Δ entry per lane, no CTA
// barrier (__syncwarp only), appends positioned by a shared counter of this warp only.
// The a^n b^n worst case (one new cell per iteration, 2pq+1 iterations) lives here.
// ------------------------------------------------------------------------------------------
struct WarpSoloShared {
    uint64_t nxt[32];
    uint64_t win[64];                        // Gauss-Seidel: log entries by position mod 64
    unsigned long long ring[kMaxStages + 1]; // Gauss-Seidel: shared copy of EngineState::gs_ring
    int cnt;
    int ov, lov;
    LoopState cs;                            // single-cell chain: the state it hands back
    int cm;                                  //   cells it leaves in nxt for the warp (0: stopped)
    int stuck;                               //   1: nxt[0] is a cell the chain cannot expand
};

// Single-cell chains (the a^n b^n worst case: one new cell per iteration for 2pq+1 iterations).
// While Δ is one cell whose rule occurrences are all ELL walks of preterminal operands, lane 0
// runs the iterations alone in registers: the candidates' bits are set by atomics issued
// together, and the ELL heads of every candidate's own occurrences are loaded before those
// atomics return, so the next iteration starts without waiting for its heads — one dependent
// L2 round trip per iteration instead of two, and no warp barrier or shared staging.  A cell
// it cannot expand, several new cells, or a log that might run out hand the step back to the
// warp path (w.cm cells in w.nxt), with identical per-iteration states.
__device__ void solo_chain(const EngineParams& p, const NTInfo* nt, const Expansion* exps, WarpSoloShared& w,
                           LoopState& s, long long& k, uint64_t cell, long long& iters, unsigned long long& dcand,
                           unsigned long long& dexp) {
    int4 pre[2] = {make_int4(0, 0, -1, -1), make_int4(0, 0, -1, -1)};
    unsigned pv = 0;
    // single-path lengths: the chain's cell's length (read once, then carried: every candidate
    // of a one-cell Δ has length l + 1 through its preterminal operand)
    uint64_t clen = p.lengths ? cell_len(p, nt, cell_nt(cell), cell_i(cell), cell_j(cell)) : 0;
    for (;;) {
        const uint32_t X = cell_nt(cell), ci = cell_i(cell), cj = cell_j(cell);
        const int eb = nt[X].exp_begin, ne = nt[X].exp_end - eb;
        bool ok = ne <= 2 && s.hi + 4 <= p.log_cap && clen < 0xffffffffull;
        int4 h[2];
        uint32_t hA[2] = {0, 0}, hf[2] = {0, 0};
#pragma unroll
        for (int x = 0; x < 2; ++x) {
            h[x] = make_int4(0, 0, -1, -1);
            if (ok && x < ne) {
                const Expansion ex = exps[eb + x];
                if (ex.kind != EXP_L_CONST && ex.kind != EXP_R_CONST) {
                    ok = false;
                } else if ((pv >> x) & 1u) {
                    h[x] = pre[x];
                    hA[x] = (uint32_t)ex.A;
                    hf[x] = ex.kind == EXP_L_CONST ? ci : (cj | 0x80000000u);
                } else {
                    h[x] = load_head(nt, ex, ci, cj, hA[x], hf[x]);
                }
            }
        }
        if (ok)
#pragma unroll
            for (int x = 0; x < 2; ++x) ok = ok && h[x].y <= 2;
        if (!ok) {   // the warp path expands this cell
            w.nxt[0] = cell;
            w.cm = 1;
            w.stuck = 1;
            return;
        }
        uint32_t cA[4], ca[4], cb[4];
        bool has[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int x = q >> 1, m = q & 1;
            cand_coords(hf[x], m ? h[x].w : h[x].z, ca[q], cb[q]);
            cA[q] = hA[x];
            has[q] = x < ne && h[x].y > m && ca[q] >= p.row_lo && ca[q] < p.row_hi;
        }
        // the candidates' own heads (they are the next Δ if new), before the atomics return
        int4 sp[4][2];
        unsigned spv[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            spv[q] = 0;
            sp[q][0] = sp[q][1] = make_int4(0, 0, -1, -1);
            if (!has[q]) continue;
            const int qb = nt[cA[q]].exp_begin, qn = nt[cA[q]].exp_end - qb;
#pragma unroll
            for (int x = 0; x < 2; ++x)
                if (x < qn) {
                    const Expansion ex = exps[qb + x];
                    if (ex.kind == EXP_L_CONST) {
                        sp[q][x] = __ldg(nt[ex.other].csr_ell + cb[q]);
                        spv[q] |= 1u << x;
                    } else if (ex.kind == EXP_R_CONST) {
                        sp[q][x] = __ldg(nt[ex.other].csc_ell + ca[q]);
                        spv[q] |= 1u << x;
                    }
                }
        }
        bool fresh[4];
        if (p.lengths) {
            // keys (iteration << 32 | length): new iff the atomicMin leaves EMPTY (first write wins)
            const unsigned long long kv = ((unsigned long long)k << 32) | (clen + 1ull);
            unsigned long long old64[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                old64[q] = 0ull;
                if (has[q]) {
                    CFPQ_DASSERT(cA[q] < (uint32_t)p.n_nt && ca[q] < (uint32_t)p.n && cb[q] < (uint32_t)p.n);
                    old64[q] = atomicMin((unsigned long long*)(nt[cA[q]].K + (size_t)ca[q] * (size_t)p.n + cb[q]), kv);
                }
            }
#pragma unroll
            for (int q = 0; q < 4; ++q) fresh[q] = has[q] && old64[q] == kEmptyKey;
        } else {
            uint32_t old[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                old[q] = ~0u;
                if (has[q]) {
                    CFPQ_DASSERT(cA[q] < (uint32_t)p.n_nt && ca[q] < (uint32_t)p.n && cb[q] < (uint32_t)p.n);
                    old[q] = atomicOr(nt[cA[q]].T + (size_t)ca[q] * (size_t)p.Wp + (cb[q] >> 5), 1u << (cb[q] & 31));
                }
            }
#pragma unroll
            for (int q = 0; q < 4; ++q) fresh[q] = has[q] && !(old[q] & (1u << (cb[q] & 31)));
        }
        dexp += (unsigned long long)ne;
        dcand += (unsigned long long)(h[0].y + (ne > 1 ? h[1].y : 0));
        int n_new = 0, last = 0;
#pragma unroll
        for (int q = 0; q < 4; ++q)
            if (fresh[q]) {
                const uint64_t c = pack_cell(cA[q], ca[q], cb[q]);
                p.log[s.hi + (unsigned long long)n_new] = c;
                if (p.lengths)   // the bit matrix mirrors the keys
                    atomicOr(nt[cA[q]].T + (size_t)ca[q] * (size_t)p.Wp + (cb[q] >> 5), 1u << (cb[q] & 31));
                w.nxt[n_new] = c;
                ++n_new;
                last = q;
            }
        close_iteration(p, k, s, s.hi + (unsigned long long)n_new, 0, true);
        ++iters;
        ++k;
        if (s.status != ST_RUNNING || n_new != 1) {   // done, capped, or several cells: the warp path
            w.cm = s.status == ST_RUNNING ? n_new : 0;
            w.stuck = 0;
            return;
        }
        cell = w.nxt[0];
        pre[0] = sp[last][0];
        pre[1] = sp[last][1];
        pv = spv[last];
        clen += 1ull;
    }
}

__device__ __forceinline__ bool ws_try(const EngineParams& p, const NTInfo* nt, uint32_t A, uint32_t i, uint32_t j,
                                       uint64_t len, long long k, int* lov, int* ovf) {
    if (i < p.row_lo || i >= p.row_hi) return false;
    CFPQ_DASSERT(A < (uint32_t)p.n_nt && i < (uint32_t)p.n && j < (uint32_t)p.n);
    uint64_t* K = nt[A].K;
    if (p.lengths && K != nullptr) {
        if (len > 0xffffffffull) {
            *(volatile int*)lov = 1;
            len = 0xffffffffull;
        }
        uint64_t old = atomicMin((unsigned long long*)(K + (size_t)i * (size_t)p.n + j),
                                 (unsigned long long)(((uint64_t)k << 32) | len));
        return old == kEmptyKey;
    }
    if (p.hset) return hash_insert(p, pack_cell(A, i, j), ovf);
    uint32_t bit = 1u << (j & 31);
    return !(atomicOr(nt[A].T + (size_t)i * (size_t)p.Wp + (j >> 5), bit) & bit);
}

__device__ __forceinline__ void ws_append(const EngineParams& p, const NTInfo* nt, WarpSoloShared& w,
                                          unsigned long long base, uint32_t A, uint32_t i, uint32_t j) {
    const int pos = atomicAdd(&w.cnt, 1);
    const unsigned long long idx = base + (unsigned long long)pos;
    const uint64_t c = pack_cell(A, i, j);
    uint64_t* K = p.lengths ? nt[A].K : nullptr;
    uint32_t* word = nt[A].T + (size_t)i * (size_t)p.Wp + (j >> 5);
    const uint32_t bit = 1u << (j & 31);
    if (idx < p.log_cap) {
        p.log[idx] = c;
        if (pos < 32) w.nxt[pos] = c;
        if (p.gs_stages) w.win[idx & 63] = c;
        if (K != nullptr) atomicOr(word, bit);
        if (p.rowc != nullptr) {
            atomicAdd(p.rowc + (size_t)A * p.n + i, 1u);
            atomicAdd(p.colc + (size_t)A * p.n + j, 1u);
        }
    } else {
        if (K != nullptr) atomicExch((unsigned long long*)(K + (size_t)i * (size_t)p.n + j), (unsigned long long)kEmptyKey);
        else if (!p.hset) atomicAnd(word, ~bit);
        w.ov = 1;
    }
}

// Runs iterations while |Δ| <= 32; returns with `s` closed at the last iteration run.
__device__ void warp_solo(const EngineParams& p, const NTInfo* nt, const Expansion* exps, WarpSoloShared& w,
                          LoopState& s, long long& iters, unsigned long long& dcand, unsigned long long& dexp) {
    const int lane = threadIdx.x & 31;
    long long k = s.iter + 1;
    int m = (int)(s.hi - s.lo);
    uint64_t cell = lane < m ? ldcg64(p.log + s.lo + lane) : 0ull;
    unsigned long long* ring = nullptr;
    if (p.gs_stages) {
        // Gauss-Seidel windows span S steps: keep the ring and the latest 64 log entries in
        // shared memory (a window of <= 32 entries lies inside them)
        for (int q = lane; q <= p.gs_stages; q += 32) w.ring[q] = ld_volatile_u64(&p.st->gs_ring[q]);
        if (lane < m) w.win[(s.lo + lane) & 63] = cell;
        ring = w.ring;
        __syncwarp();
    }
    // single-cell chains need the plain Jacobi path (no hashed set, stages or snapshots);
    // cfpq diag_flags bit 13 disables them (A/B)
    const bool chains = !p.hset && !p.gs_stages && !p.has_snapshots && !p.jac && !p.no_chain;
    bool stuck = false;
    for (;;) {
        if (chains && m == 1 && !stuck) {
            if (lane == 0) {
                w.cs = s;
                long long kk = k;
                solo_chain(p, nt, exps, w, w.cs, kk, cell, iters, dcand, dexp);
            }
            __syncwarp();
            s = w.cs;
            k = s.iter + 1;
            m = w.cm;
            stuck = w.stuck != 0;
            if (s.status != ST_RUNNING || m == 0) break;
            if (m > p.solo_max) break;   // the CTA / grid paths take Δ from the log
            cell = lane < m ? w.nxt[lane] : 0ull;
            __syncwarp();
            continue;
        }
        stuck = false;
        if (lane == 0) {
            w.cnt = 0;
            w.ov = 0;
            w.lov = 0;
        }
        __syncwarp();
        const unsigned long long base = s.hi;
        if (lane < m) {
            const uint32_t X = cell_nt(cell), ci = cell_i(cell), cj = cell_j(cell);
            const int eb = nt[X].exp_begin, ee = nt[X].exp_end;
            dexp += (unsigned long long)(ee - eb);
            const uint64_t len_e = (p.lengths && ee > eb) ? cell_len(p, nt, X, ci, cj) : 0;
            for (int x = eb; x < ee; ++x) {
                const Expansion ex = exps[x];
                if (!stage_ok(p, ex, s.gs_stage)) continue;
                if (ex.kind == EXP_L_CONST || ex.kind == EXP_R_CONST) {
                    uint32_t A, fx;
                    const int4 h = load_head(nt, ex, ci, cj, A, fx);
                    dcand += (unsigned long long)h.y;
                    uint32_t a0, b0, a1, b1;
                    cand_coords(fx, h.z, a0, b0);
                    cand_coords(fx, h.w, a1, b1);
                    bool n0, n1;
                    if (p.hset) {
                        hash_pair(p, h.y > 0, pack_cell(A, a0, b0), h.y > 1, pack_cell(A, a1, b1), n0, n1, &w.ov);
                    } else {
                        n0 = h.y > 0 && ws_try(p, nt, A, a0, b0, len_e + 1, k, &w.lov, &w.ov);
                        n1 = h.y > 1 && ws_try(p, nt, A, a1, b1, len_e + 1, k, &w.lov, &w.ov);
                    }
                    if (n0) ws_append(p, nt, w, base, A, a0, b0);
                    if (n1) ws_append(p, nt, w, base, A, a1, b1);
                    for (int t = 2; t < h.y; ++t) {
                        uint32_t a, b;
                        CFPQ_DASSERT((long long)h.x + t < p.adj_cap);
                        CFPQ_DASSERT((long long)h.x + t < p.adj_cap);
                    cand_coords(fx, __ldg(p.adj_idx + h.x + t), a, b);
                        if (ws_try(p, nt, A, a, b, len_e + 1, k, &w.lov, &w.ov)) ws_append(p, nt, w, base, A, a, b);
                    }
                } else {
                    const bool left = ex.kind == EXP_L_VAR;
                    const uint32_t* row = left ? nt[ex.other].S + (size_t)cj * p.Wp : nt[ex.other].ST + (size_t)ci * p.Wp;
                    const int64_t wn = (p.n + 31) >> 5;
                    for (int64_t wd = 0; wd < wn; ++wd) {
                        uint32_t bits = ldcg32(row + wd);
                        while (bits) {
                            const int b = __ffs(bits) - 1;
                            bits &= bits - 1u;
                            const uint32_t v = (uint32_t)(wd * 32 + b);
                            const uint32_t oi = left ? ci : v, oj = left ? v : cj;
                            uint64_t clen = 0;
                            if (p.lengths)
                                clen = left ? len_e + cell_len(p, nt, ex.other, cj, v) : cell_len(p, nt, ex.other, v, ci) + len_e;
                            ++dcand;
                            if (ws_try(p, nt, (uint32_t)ex.A, oi, oj, clen, k, &w.lov, &w.ov))
                                ws_append(p, nt, w, base, (uint32_t)ex.A, oi, oj);
                        }
                    }
                }
            }
        }
        __syncwarp();
        const int total = *(volatile int*)&w.cnt;
        const int f = (*(volatile int*)&w.ov ? 1 : 0) | (*(volatile int*)&w.lov ? 2 : 0);
        close_iteration(p, k, s, base + (unsigned long long)total, f, lane == 0, ring);
        ++iters;
        if (s.status != ST_RUNNING) break;
        if (p.has_snapshots) {
            for (int q = lane; q < total; q += 32) {
                const uint64_t c = q < 32 ? w.nxt[q] : ldcg64(p.log + base + q);
                const uint32_t A = cell_nt(c), i = cell_i(c), j = cell_j(c);
                if (nt[A].S) atomicOr(nt[A].S + (size_t)i * p.Wp + (j >> 5), 1u << (j & 31));
                if (nt[A].ST) atomicOr(nt[A].ST + (size_t)j * p.Wp + (i >> 5), 1u << (i & 31));
            }
            __syncwarp();
        }
        ++k;
        const long long mw = (long long)(s.hi - s.lo);   // the next step's entries (Jacobi: = total)
        if (mw > 32 || mw > p.solo_max) break;           // hand over to the CTA or grid paths
        m = (int)mw;
        __syncwarp();
        // Gauss-Seidel windows span several steps: read them from the shared log mirror
        cell = lane < m ? (p.gs_stages ? w.win[(s.lo + lane) & 63] : w.nxt[lane]) : 0ull;
        __syncwarp();
    }
    if (p.gs_stages) {
        __syncwarp();
        for (int q = lane; q <= p.gs_stages; q += 32) p.st->gs_ring[q] = w.ring[q];
        __syncwarp();
    }
}

__device__ void solo_expand(const EngineParams& p, const NTInfo* nt, const Expansion* exps, SoloShared& so,
                            const uint64_t* src, unsigned long long lo, unsigned long long hi, long long k, int gstage,
                            int slot,
                            uint64_t* mirror, unsigned long long& dcand, unsigned long long& dexp,
                            long long* pacc = nullptr) {
    long long t0 = pacc ? clock64() : 0;
    for (unsigned long long e = lo + threadIdx.x; e < hi; e += kBlock) {
        uint64_t cell = src ? src[e - lo] : ldcg64(p.log + e);
        uint32_t X = cell_nt(cell), ci = cell_i(cell), cj = cell_j(cell);
        int eb = nt[X].exp_begin, ee = nt[X].exp_end;
        dexp += (unsigned long long)(ee - eb);
        uint64_t len_e = (p.lengths && ee > eb) ? cell_len(p, nt, X, ci, cj) : 0;
        for (int x = eb; x < ee; ++x) {
            Expansion ex = exps[x];
            if (!stage_ok(p, ex, gstage)) continue;
            if (ex.kind == EXP_L_CONST || ex.kind == EXP_R_CONST) {
                uint32_t A, fx;
                int4 h = load_head(nt, ex, ci, cj, A, fx);
                dcand += (unsigned long long)h.y;
                uint32_t a0, b0, a1, b1;
                cand_coords(fx, h.z, a0, b0);
                cand_coords(fx, h.w, a1, b1);
                if (pacc) {
                    long long t = clock64() + (h.y < -1 ? 1 : 0);   // depends on the head: waits for it
                    pacc[5] += t - t0;
                    t0 = t;
                }
                bool n0, n1;
                if (p.hset) {
                    hash_pair(p, h.y > 0, pack_cell(A, a0, b0), h.y > 1, pack_cell(A, a1, b1), n0, n1, &so.ov[slot]);
                } else {
                    n0 = h.y > 0 && solo_try(p, nt, so, slot, A, a0, b0, len_e + 1, k);
                    n1 = h.y > 1 && solo_try(p, nt, so, slot, A, a1, b1, len_e + 1, k);
                }
                if (pacc) {
                    long long t = clock64() + (n0 ? 1 : 0) + (n1 ? 1 : 0);
                    pacc[6] += t - t0;
                    t0 = t;
                }
                if (h.y > 0) prefetch_next(nt, exps, A, a0, b0);
                if (h.y > 1) prefetch_next(nt, exps, A, a1, b1);
                if (n0) solo_append(p, nt, so, slot, hi, mirror, A, a0, b0);
                if (n1) solo_append(p, nt, so, slot, hi, mirror, A, a1, b1);
                for (int t = 2; t < h.y; ++t) {
                    uint32_t a, b;
                    CFPQ_DASSERT((long long)h.x + t < p.adj_cap);
                    cand_coords(fx, __ldg(p.adj_idx + h.x + t), a, b);
                    if (solo_try(p, nt, so, slot, A, a, b, len_e + 1, k)) solo_append(p, nt, so, slot, hi, mirror, A, a, b);
                }
            } else {
                const bool left = ex.kind == EXP_L_VAR;
                const uint32_t* row = left ? nt[ex.other].S + (size_t)cj * p.Wp : nt[ex.other].ST + (size_t)ci * p.Wp;
                const int64_t wn = (p.n + 31) >> 5;
                for (int64_t w = 0; w < wn; ++w) {
                    uint32_t bits = ldcg32(row + w);
                    while (bits) {
                        int b = __ffs(bits) - 1;
                        bits &= bits - 1u;
                        uint32_t v = (uint32_t)(w * 32 + b);
                        uint32_t oi = left ? ci : v, oj = left ? v : cj;
                        uint64_t clen = 0;
                        if (p.lengths)
                            clen = left ? len_e + cell_len(p, nt, ex.other, cj, v) : cell_len(p, nt, ex.other, v, ci) + len_e;
                        ++dcand;
                        if (solo_try(p, nt, so, slot, (uint32_t)ex.A, oi, oj, clen, k))
                            solo_append(p, nt, so, slot, hi, mirror, (uint32_t)ex.A, oi, oj);
                    }
                }
            }
        }
    }
}

// Dynamic shared memory of the closure kernel.
struct ClosureShared {
    WarpSoloShared wsolo;
    unsigned long long flush_base;
    int32_t flush_prefix[kWarps];
    WarpScratch ws[kWarps];
    NTInfo nt[kSmemNT];
    Expansion exp[kSmemExp];
    SoloShared solo;
    LoopState state;
};

__global__ void __launch_bounds__(kBlock, 1) closure_kernel(EngineParams p) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    ClosureShared& S = *reinterpret_cast<ClosureShared*>(smem_raw);
    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    EngineState* st = p.st;
    // NT / expansion tables into shared memory (loads stay on-chip across iterations)
    const bool small = p.n_nt <= kSmemNT && p.n_exps <= kSmemExp;
    if (small) {
        for (int t = threadIdx.x; t < p.n_nt; t += kBlock) S.nt[t] = p.nt[t];
        for (int t = threadIdx.x; t < p.n_exps; t += kBlock) S.exp[t] = p.exps[t];
    }
    const NTInfo* nt = small ? S.nt : p.nt;
    const Expansion* exps = small ? S.exp : p.exps;
    const Sink gsink = global_sink(p);
    if (lane == 0) S.ws[wib].nbuf = 0;
    if (threadIdx.x == 0) {
        S.solo.solo = 0;
        S.state.lo = ld_volatile_u64(&st->lo);
        S.state.hi = ld_volatile_u64(&st->hi);
        S.state.iter = *(volatile long long*)&st->iter;
        S.state.status = *(volatile int*)&st->status;
        S.state.gs_stage = *(volatile int*)&st->gs_stage;
        S.state.gs_slot = *(volatile int*)&st->gs_slot;
        S.state.gs_round = *(volatile long long*)&st->gs_round;
    }
    __syncthreads();
    LoopState s = S.state;   // identical in every CTA
    __syncthreads();         // every thread holds it before warp-solo may rewrite S.state
    unsigned long long dcand = 0, dexp = 0;
    bool aborted = false;
    if (p.fused_seed) {
        if (!fused_seed_phase(p, nt, S.ws, wib, lane, &S.flush_base, S.flush_prefix, s)) aborted = true;
        __syncthreads();
        if (threadIdx.x == 0) S.state = s;   // the solo paths re-read the loop state from here
        __syncthreads();
    }
    while (!aborted && s.status == ST_RUNNING) {
        long long k = s.iter + 1;
        if ((long long)(s.hi - s.lo) <= (long long)p.solo_max) {
            // ------------- single-CTA iterations (see SoloShared) -------------
            if (blockIdx.x == 0) {
                // warp-solo first while |Δ| <= 32 (not on the re-run of an overflowed iteration)
                if (wib == 0 && s.hi - s.lo <= 32 && !p.jac && ld_volatile_u64(&st->log_size) == s.hi) {
                    long long wi = 0;
                    warp_solo(p, nt, exps, S.wsolo, s, wi, dcand, dexp);
                    if (lane == 0) {
                        unsigned long long ls = s.hi;
                        if (s.status == ST_OVERFLOW || s.status == ST_LEN_OVERFLOW) {
                            // s still holds iteration k's range; the counter went past the log
                            ls = s.hi + (unsigned long long)S.wsolo.cnt;
                            if (S.wsolo.ov) st->overflow = 1;
                            if (S.wsolo.lov) st->len_overflow = 1;
                        }
                        st->log_size = ls;
                        atomicAdd((unsigned long long*)&st->solo_iters, (unsigned long long)wi);
                        S.state = s;
                    }
                }
                __syncthreads();
                s = S.state;
                k = s.iter + 1;
            }
            if (blockIdx.x == 0 && s.status == ST_RUNNING && (long long)(s.hi - s.lo) <= (long long)p.solo_max) {
                SoloShared& so = S.solo;
                int cur = 0;
                const unsigned long long ls0 = ld_volatile_u64(&st->log_size);
                if (s.hi - s.lo <= (unsigned long long)kSoloMax)
                    for (unsigned long long e = s.lo + threadIdx.x; e < s.hi; e += kBlock)
                        so.delta[cur][e - s.lo] = ldcg64(p.log + e);
                {
                    // cells of Δ_k appended before a log-overflow re-run of iteration k
                    unsigned long long end = ls0 < s.hi + kSoloMax ? ls0 : s.hi + kSoloMax;
                    for (unsigned long long e = s.hi + threadIdx.x; e < end; e += kBlock)
                        so.delta[cur ^ 1][e - s.hi] = ldcg64(p.log + e);
                }
                if (threadIdx.x == 0) {
                    for (int q = 0; q < 3; ++q) {
                        so.cnt[q] = 0u;
                        so.ov[q] = 0;
                        so.lov[q] = 0;
                    }
                    so.cnt[k % 3] = (unsigned)(ls0 - s.hi);
                }
                __syncthreads();
                unsigned long long last_ls = ls0;
                long long tp = clock64();
                long long pacc[7] = {0, 0, 0, 0, 0, 0, 0};
                const bool prof = p.profile && threadIdx.x == 0;
                int slot = (int)(k % 3);
                for (;;) {
                    const int nx = slot == 2 ? 0 : slot + 1;
                    if (p.jac) {
                        account(p, k, threadIdx.x, kBlock);
                        __syncthreads();
                    }
                    if (prof) {
                        long long t = clock64();
                        pacc[0] += t - tp;   // loop overhead
                        tp = t;
                    }
                    const uint64_t* src =
                        (s.hi - s.lo <= (unsigned long long)kSoloMax && !p.gs_stages) ? so.delta[cur] : nullptr;
                    solo_expand(p, nt, exps, so, src, s.lo, s.hi, k, s.gs_stage, slot, so.delta[cur ^ 1], dcand, dexp,
                                prof ? pacc : nullptr);
                    if (threadIdx.x == 0) {
                        so.cnt[nx] = 0u;
                        so.ov[nx] = 0;
                        so.lov[nx] = 0;
                        so.solo += 1;
                    }
                    if (prof) {
                        long long t = clock64();
                        pacc[1] += t - tp;   // expand (thread 0's share)
                        tp = t;
                    }
                    __syncthreads();
                    if (prof) {
                        long long t = clock64();
                        pacc[2] += t - tp;   // the barrier
                        tp = t;
                    }
                    const unsigned long long ls = s.hi + so.cnt[slot];
                    const unsigned long long old_hi = s.hi;
                    const int f = (so.ov[slot] ? 1 : 0) | (so.lov[slot] ? 2 : 0);
                    last_ls = ls;
                    close_iteration(p, k, s, ls, f, threadIdx.x == 0);
                    if (prof) {
                        long long t = clock64();
                        pacc[3] += t - tp;   // close
                        tp = t;
                    }
                    if (s.status != ST_RUNNING) break;
                    cur ^= 1;
                    if (p.has_snapshots) {
                        if (p.gs_stages) {   // this step's cells only (the window spans S steps)
                            apply_snapshots(p, nt, nullptr, old_hi, s.hi, threadIdx.x, kBlock);
                        } else {
                            const uint64_t* sn = (s.hi - s.lo <= (unsigned long long)kSoloMax) ? so.delta[cur] : nullptr;
                            apply_snapshots(p, nt, sn, s.lo, s.hi, threadIdx.x, kBlock);
                        }
                        __syncthreads();
                    }
                    ++k;
                    slot = nx;
                    if ((long long)(s.hi - s.lo) > (long long)p.solo_max) break;
                }
                if (prof)
                    for (int q = 0; q < 7; ++q) st->prof[q] += pacc[q];
                if (threadIdx.x == 0) {
                    st->log_size = last_ls;   // the other CTAs are parked at the grid barrier
                    if (so.ov[slot]) st->overflow = 1;
                    if (so.lov[slot]) st->len_overflow = 1;
                    atomicAdd((unsigned long long*)&st->solo_iters, (unsigned long long)so.solo);
                    so.solo = 0;
                    publish(p, s);
                }
            } else if (blockIdx.x == 0 && threadIdx.x == 0) {
                publish(p, s);   // warp-solo ended the phase (done, or Δ grew past the CTA path)
            }
            if (!grid_barrier(p, -1)) {
                aborted = true;
                break;
            }
            if (threadIdx.x == 0) {
                S.state.lo = ld_volatile_u64(&st->lo);
                S.state.hi = ld_volatile_u64(&st->hi);
                S.state.iter = *(volatile long long*)&st->iter;
                S.state.status = *(volatile int*)&st->status;
        S.state.gs_stage = *(volatile int*)&st->gs_stage;
        S.state.gs_slot = *(volatile int*)&st->gs_slot;
        S.state.gs_round = *(volatile long long*)&st->gs_round;
            }
            __syncthreads();
            s = S.state;
            __syncthreads();
            continue;
        }
        // ---------------- grid-wide iteration k ----------------
        const long long gtid = (long long)blockIdx.x * kBlock + threadIdx.x;
        const long long gthreads = (long long)gridDim.x * kBlock;
        if (p.jac) {
            account(p, k, gtid, gthreads);
            if (!grid_barrier(p, -1)) {
                aborted = true;
                break;
            }
        }
        // diagnostics (p.phase): per iteration, max over CTAs of [0] expand, [1] CTA flush,
        // [3] close; [2] = ~(min over CTAs of the barrier wait) = the last arriver's release
        const bool ph = p.phase != nullptr && k < p.iter_off_cap;
        long long c0 = ph ? clock64() : 0, c1 = 0, c2 = 0, c3 = 0;
        // chunk c -> CTA c mod grid (interleaved): a Δ of ~3k chunks spreads over every SM
        // instead of filling the first ~100 CTAs (diag_flags bit 8: CTA-major, round 1)
        const int vwarp = p.cta_major ? (int)blockIdx.x * kWarps + wib : wib * (int)gridDim.x + (int)blockIdx.x;
        expand(p, nt, exps, gsink, nullptr, s.lo, s.hi, k, s.gs_stage, vwarp, gridDim.x * kWarps, lane,
               &S.ws[wib], dcand, dexp, p.warp_flush != 0);
        if (ph) {
            __syncthreads();
            c1 = clock64();
        }
        if (!p.warp_flush) cta_flush(p, nt, gsink, S.ws, wib, lane, &S.flush_base, S.flush_prefix);
        if (ph) c2 = clock64();
        unsigned long long bw = 0;
        if (!grid_barrier(p, k, &bw)) {
            aborted = true;
            break;
        }
        if (ph) c3 = clock64();
        if (threadIdx.x == 0) {
            LoopState t = s;
            close_iteration(p, k, t, bw & kBarLsMask, (int)((bw >> 38) & 3ull), blockIdx.x == 0);
            S.state = t;
        }
        __syncthreads();
        LoopState prev = s;
        s = S.state;
        __syncthreads();
        if (ph && threadIdx.x == 0) {
            unsigned long long* q = p.phase + 4 * k;
            atomicMax(q + 0, (unsigned long long)(c1 - c0));
            atomicMax(q + 1, (unsigned long long)(c2 - c1));
            atomicMax(q + 2, ~(unsigned long long)(c3 - c2));
            atomicMax(q + 3, (unsigned long long)(clock64() - c3));
        }
        if (s.status == ST_OVERFLOW || s.status == ST_LEN_OVERFLOW) {
            // keep the pre-iteration range for the host's re-run
            s.lo = prev.lo;
            s.hi = prev.hi;
            s.iter = prev.iter;
        }
        if (p.has_snapshots && s.status == ST_RUNNING) {
            apply_snapshots(p, nt, nullptr, p.gs_stages ? prev.hi : s.lo, s.hi, gtid, gthreads);
            if (!grid_barrier(p, -1)) {
                aborted = true;
                break;
            }
        }
    }
    if (!aborted && blockIdx.x == 0 && threadIdx.x == 0) publish(p, s);
    if (!aborted) clear_drain(p);   // the other bank is clean when this launch ends
    if (!aborted && p.self_clear && (s.status == ST_DONE || s.status == ST_CAP)) {
        // the relations are in the log: reset the bit words of every logged cell while they
        // are still hot in L2, so the next run starts on clean matrices (no clear pass)
        __syncthreads();
        const unsigned long long n_cells = s.hi;
        for (unsigned long long e = (unsigned long long)blockIdx.x * kBlock + threadIdx.x; e < n_cells;
             e += (unsigned long long)gridDim.x * kBlock) {
            const uint64_t c = ldcg64(p.log + e);
            const uint32_t A = cell_nt(c), i = cell_i(c), j = cell_j(c);
            const NTInfo& t = nt[A];
            zero_sector(t.T + (size_t)i * p.Wp + (j >> 5));
            if (t.S) zero_sector(t.S + (size_t)i * p.Wp + (j >> 5));
            if (t.ST) zero_sector(t.ST + (size_t)j * p.Wp + (i >> 5));
            if (p.rowc) {
                p.rowc[(size_t)A * p.n + i] = 0u;
                p.colc[(size_t)A * p.n + j] = 0u;
            }
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

// ------------------------------------------------------------------------------------------
// Row-sharded sparse engine with a device-resident peer-memory exchange (exchange = 1; §8(e),
// P:572).  Each rank runs this persistent kernel over the whole fixpoint: it expands all of
// Δ_{k-1} (its own copy in its own log), inserts only the cells of its rows, and appends every
// new cell to EVERY rank's log (system-scope reservations and stores; NVLink peer mappings on
// real GPUs), so the exchange overlaps the expansion instead of following it.  Iteration end:
// the rank's CTAs meet at a rank-local barrier whose last CTA fences system-wide, adds its
// rank's new-cell count and overflow flag to every rank's slot of this iteration (xr_slot) and
// waits for all P arrivals; after that its own log holds Δ_k of every rank (the same set on
// every rank) and it releases its CTAs with the log size hi + Σ counts.  An emulated launch runs P virtual ranks as CTA groups of one grid.
// ------------------------------------------------------------------------------------------
__device__ bool xr_barrier(const EngineParams& p, const XrParams& x, long long k, unsigned long long hi,
                           unsigned long long* word) {
    __shared__ int s_timeout;
    __threadfence_system();   // this CTA's appends to peer logs are visible system-wide first
    __syncthreads();
    if (threadIdx.x == 0) {
        s_timeout = 0;
        EngineState* st = p.st;
        const unsigned long long my = ld_volatile_u64(&st->bar_word) >> kBarGenShift;
        const unsigned arrived = atom_add_acq_rel(&st->bar_count, 1u);
        unsigned long long w;
        if (arrived == (unsigned)p.nblocks - 1u) {
            // every CTA of this rank has appended (acq_rel chain): its iteration-k contribution
            // is its new-cell count and its overflow flag, which no other rank writes
            __threadfence();
            const unsigned long long nk = ld_volatile_u64(&st->xr_new);
            const unsigned long long ov = *(volatile int*)&st->overflow ? 1ull : 0ull;
            st->xr_new = 0ull;
            __threadfence_system();
            const int sl = (int)(k & 1);
            const unsigned long long add = (nk << 32) | (ov << 16) | 1ull;
            for (int q = 0; q < x.P; ++q) atomicAdd_system(&x.st[q]->xr_slot[sl], add);
            // Δ_k of THIS log = the sum of every rank's new cells, read from the slot once all P
            // ranks arrived — not from the log counter, which a rank already released from
            // iteration k may be advancing with its iteration-(k+1) appends.  The slot is next
            // used at iteration k+2, whose arrivals need this rank's arrival at k+1 first.
            long long t0 = clock64();
            unsigned ns = 0;
            unsigned long long v;
            while (((v = ld_volatile_u64(&st->xr_slot[sl])) & 0xFFFFull) < (unsigned long long)x.P) {
                if (ns) __nanosleep(ns);
                if (clock64() - t0 > 40000) ns = ns ? (ns < 1024u ? ns * 2u : 1024u) : 64u;
                if (clock64() - t0 > 60000000000ll) {
                    s_timeout = 1;
                    break;
                }
            }
            __threadfence_system();
            st->xr_slot[sl] = 0ull;
            const unsigned long long f = ((v >> 16) & 0xFFFFull) ? 1ull : 0ull;
            w = (((my + 1) & 0xFFFFFFull) << kBarGenShift) | (f << 38) | ((hi + (v >> 32)) & kBarLsMask);
            st->bar_count = 0u;
            st_release_word(&st->bar_word, w);
        } else {
            long long t0 = clock64();
            unsigned ns = 0;
            while (((w = ld_acquire_word(&st->bar_word)) >> kBarGenShift) == my) {
                if (ns) __nanosleep(ns);
                if (clock64() - t0 > 40000) ns = ns ? (ns < 2048u ? ns * 2u : 2048u) : 64u;
                if (clock64() - t0 > 60000000000ll) {
                    s_timeout = 1;
                    break;
                }
            }
        }
        *word = w;
    }
    __syncthreads();
    return s_timeout == 0;
}

__global__ void __launch_bounds__(kBlock, 1) xr_closure_kernel(EngineParams p0, XrParams x) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    ClosureShared& S = *reinterpret_cast<ClosureShared*>(smem_raw);
    __shared__ unsigned long long s_bases[kMaxXrRanks];
    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    const int rank = x.my_rank >= 0 ? x.my_rank : (int)blockIdx.x / x.cpr;
    const int lb = x.my_rank >= 0 ? (int)blockIdx.x : (int)blockIdx.x % x.cpr;
    EngineParams p = p0;
    p.st = x.st[rank];
    p.log = x.log[rank];
    p.row_lo = x.row_lo[rank];
    p.row_hi = x.row_hi[rank];
    p.nblocks = x.cpr;
    EngineState* st = p.st;
    const bool small = p.n_nt <= kSmemNT && p.n_exps <= kSmemExp;
    if (small) {
        for (int t = threadIdx.x; t < p.n_nt; t += kBlock) S.nt[t] = p.nt[t];
        for (int t = threadIdx.x; t < p.n_exps; t += kBlock) S.exp[t] = p.exps[t];
    }
    const NTInfo* nt = small ? S.nt : p.nt;
    const Expansion* exps = small ? S.exp : p.exps;
    Sink sk = global_sink(p);
    sk.xr_P = x.P;
    sk.xr_st = x.st;
    sk.xr_log = x.log;
    if (lane == 0) S.ws[wib].nbuf = 0;
    if (threadIdx.x == 0) {
        S.state.lo = ld_volatile_u64(&st->lo);
        S.state.hi = ld_volatile_u64(&st->hi);
        S.state.iter = *(volatile long long*)&st->iter;
        S.state.status = *(volatile int*)&st->status;
        S.state.gs_stage = 0;
        S.state.gs_slot = 1;
        S.state.gs_round = 0;
    }
    __syncthreads();
    LoopState s = S.state;
    __syncthreads();
    unsigned long long dcand = 0, dexp = 0;
    bool aborted = false;
    while (s.status == ST_RUNNING) {
        const long long k = s.iter + 1;
        expand(p, nt, exps, sk, nullptr, s.lo, s.hi, k, 0, wib * x.cpr + lb, x.cpr * kWarps, lane, &S.ws[wib], dcand,
               dexp, false);
        cta_flush_xr<kWarps>(p, sk, S.ws, wib, lane, s_bases, S.flush_prefix);
        unsigned long long bw = 0;
        if (!xr_barrier(p, x, k, s.hi, &bw)) {
            aborted = true;
            break;
        }
        if (threadIdx.x == 0) {
            LoopState t = s;
            close_iteration(p, k, t, bw & kBarLsMask, (int)((bw >> 38) & 3ull), lb == 0);
            S.state = t;
        }
        __syncthreads();
        s = S.state;
        __syncthreads();
    }
    if (lb == 0 && threadIdx.x == 0) {
        if (aborted) s.status = ST_TIMEOUT;
        publish(p, s);
    }
    if (!aborted && p.self_clear && (s.status == ST_DONE || s.status == ST_CAP)) {
        // reset the bit words of the cells of this rank's rows (the relations stay in the log)
        __syncthreads();
        const unsigned long long n_cells = s.hi;
        for (unsigned long long e = (unsigned long long)lb * kBlock + threadIdx.x; e < n_cells;
             e += (unsigned long long)x.cpr * kBlock) {
            const uint64_t c = ldcg64(p.log + e);
            const uint32_t i = cell_i(c);
            if (i < p.row_lo || i >= p.row_hi) continue;
            zero_sector(nt[cell_nt(c)].T + (size_t)i * p.Wp + (cell_j(c) >> 5));
        }
    }
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

static int grid_for(int64_t work, int block);
size_t closure_kernel_smem() { return sizeof(ClosureShared); }

// ------------------------------------------------------------------------------------------
// Asynchronous (chaotic) schedule, relational semantics only (schedule 2).
// T ↦ T ∪ T×T is monotone, so ANY fair order of applying it reaches the same least
// fixpoint T^cf; the per-iteration states of Alg. 1 are not reproduced.  Every warp claims
// 32 log slots at a time and expands each entry as soon as it has been appended (entries
// carry a valid flag, bit 63); no grid barrier at all.  Quiescence: a warp counts its
// entries as done only after flushing the cells they produced, so done == appended (read
// in that order) means nothing is pending or in flight.
// ------------------------------------------------------------------------------------------
constexpr uint64_t kValid = 1ull << 63;

__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__global__ void __launch_bounds__(kBlock, 1) async_kernel(EngineParams p) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    ClosureShared& S = *reinterpret_cast<ClosureShared*>(smem_raw);
    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    EngineState* st = p.st;
    const bool small = p.n_nt <= kSmemNT && p.n_exps <= kSmemExp;
    if (small) {
        for (int t = threadIdx.x; t < p.n_nt; t += kBlock) S.nt[t] = p.nt[t];
        for (int t = threadIdx.x; t < p.n_exps; t += kBlock) S.exp[t] = p.exps[t];
    }
    const NTInfo* nt = small ? S.nt : p.nt;
    const Expansion* exps = small ? S.exp : p.exps;
    Sink sk = global_sink(p);
    sk.tag = kValid;
    WarpScratch* ws = &S.ws[wib];
    if (lane == 0) ws->nbuf = 0;
    __syncthreads();
    unsigned long long dcand = 0, dexp = 0;
    bool finished = false;
    while (!finished) {
        unsigned long long c = 0;
        if (lane == 0) c = atomicAdd(&st->async_head, 32ull);
        c = __shfl_sync(kFull, c, 0);
        unsigned pending = kFull;
        unsigned ns = 0;
        while (pending) {
            const unsigned long long e = c + lane;
            bool ok = false;
            uint64_t cell = 0;
            if ((pending >> lane) & 1u) {
                if (e < p.log_cap) {
                    uint64_t v = ldcg64(p.log + e);
                    ok = (v & kValid) != 0;
                    cell = v & ~kValid;
                }
            }
            const unsigned okm = __ballot_sync(kFull, ok);
            if (okm) {
                expand_chunk(p, nt, exps, sk, cell, ok, 0, 0, lane, ws, dcand, dexp);
                flush(p, nt, sk, ws, lane);   // produced cells are appended before ours count as done
                if (lane == 0) {
                    __threadfence();
                    atomicAdd(&st->async_done, (unsigned long long)__popc(okm));
                }
                pending &= ~okm;
                ns = 0;
            } else {
                int fin = 0;
                if (lane == 0) {
                    const unsigned long long d = ld_acquire_u64(&st->async_done);
                    const unsigned long long t = ld_acquire_u64(&st->log_size);
                    fin = (d == t) || *(volatile int*)&st->overflow || *(volatile int*)&st->bad_edge;
                }
                fin = __shfl_sync(kFull, fin, 0);
                if (fin) {
                    finished = true;
                    break;
                }
                if (ns) __nanosleep(ns);
                ns = ns ? (ns < 1024u ? ns * 2u : 1024u) : 64u;
            }
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        dcand += __shfl_xor_sync(kFull, dcand, o);
        dexp += __shfl_xor_sync(kFull, dexp, o);
    }
    if (lane == 0) {
        if (dcand) atomicAdd(&st->candidates, dcand);
        if (dexp) atomicAdd(&st->expansions, dexp);
    }
    if (p.self_clear) {
        // quiescence is global and stable (done == appended): every CTA passes one grid
        // barrier, then one pass over the log strips the valid flags and resets the bit
        // words of every cell while they are hot in L2 (the relations stay in the log; the
        // next run starts on clean matrices).  After an overflow the host re-runs instead.
        __syncthreads();
        if (!grid_barrier(p, -1)) return;
        if (*(volatile int*)&st->overflow || *(volatile int*)&st->bad_edge) return;
        const unsigned long long n_cells = ld_volatile_u64(&st->log_size);
        for (unsigned long long e = (unsigned long long)blockIdx.x * kBlock + threadIdx.x; e < n_cells;
             e += (unsigned long long)gridDim.x * kBlock) {
            const uint64_t c = ldcg64(p.log + e) & ~kValid;
            p.log[e] = c;
            const uint32_t A = cell_nt(c), i = cell_i(c), j = cell_j(c);
            const NTInfo& t = nt[A];
            zero_sector(t.T + (size_t)i * p.Wp + (j >> 5));
            if (t.S) zero_sector(t.S + (size_t)i * p.Wp + (j >> 5));
            if (t.ST) zero_sector(t.ST + (size_t)j * p.Wp + (i >> 5));
        }
    }
}

__global__ void flag_seeds_kernel(EngineParams p) {
    const unsigned long long n0 = ld_volatile_u64(&p.st->log_size);
    for (unsigned long long e = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; e < n0;
         e += (unsigned long long)gridDim.x * blockDim.x)
        p.log[e] |= kValid;
}

__global__ void strip_flags_kernel(uint64_t* log, unsigned long long lo, unsigned long long hi) {
    for (unsigned long long e = lo + blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; e < hi;
         e += (unsigned long long)gridDim.x * blockDim.x)
        log[e] &= ~kValid;
}

cudaError_t launch_async(const EngineParams& p, int grid, cudaStream_t s, bool flag_seeds,
                         unsigned long long seeds_upper) {
    if (flag_seeds && seeds_upper) flag_seeds_kernel<<<grid_for((int64_t)seeds_upper, 256), 256, 0, s>>>(p);
    async_kernel<<<grid, kBlock, sizeof(ClosureShared), s>>>(p);
    return cudaGetLastError();
}

cudaError_t launch_strip_flags(uint64_t* log, unsigned long long lo, unsigned long long hi, cudaStream_t s) {
    if (hi > lo) strip_flags_kernel<<<grid_for((int64_t)(hi - lo), 256), 256, 0, s>>>(log, lo, hi);
    return cudaGetLastError();
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
    st->gs_ring[1] = n0;   // L_1 (Gauss-Seidel windows)
    st->gs_slot = 1;
    st->gs_stage = 0;
    st->gs_round = 0;
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
        seed_kernel<<<std::min(grid_for(n_edges, kSeedBlock), 148 * 8), kSeedBlock, 0, s>>>(p, edges, n_edges, lab_ptr, lab_nt, n_labels,
                                                                          max_rules_per_label);
    return cudaGetLastError();
}

cudaError_t launch_adj_count(const EngineParams& p, const int32_t* slot_row, const int32_t* slot_col,
                             int32_t* counts, unsigned long long n_seed, cudaStream_t s) {
    adj_count_kernel<<<grid_for((int64_t)std::max<unsigned long long>(n_seed, 1), 256), 256, 0, s>>>(p, slot_row,
                                                                                                  slot_col, counts);
    return cudaGetLastError();
}

cudaError_t launch_adj_fill(const EngineParams& p, const int32_t* slot_row, const int32_t* slot_col,
                            const int32_t* ptr, int32_t* counts, int32_t* idx, int4* ell, unsigned long long n_seed,
                            cudaStream_t s) {
    if (n_seed)
        adj_fill_kernel<<<grid_for((int64_t)n_seed, 256), 256, 0, s>>>(p, slot_row, slot_col, ptr, counts, idx, ell);
    return cudaGetLastError();
}

cudaError_t launch_clear_log(const EngineParams& p, unsigned long long n_cells, cudaStream_t s) {
    if (n_cells) clear_log_kernel<<<grid_for((int64_t)n_cells, 256), 256, 0, s>>>(p, n_cells);
    return cudaGetLastError();
}

cudaError_t launch_rehash(const EngineParams& p, unsigned long long n_cells, uint64_t cell_mask, int need_flag,
                          cudaStream_t s) {
    if (n_cells) rehash_kernel<<<grid_for((int64_t)n_cells, 256), 256, 0, s>>>(p, n_cells, cell_mask, need_flag);
    return cudaGetLastError();
}

cudaError_t launch_log_to_bitmap(const uint64_t* log, unsigned long long n_cells, uint32_t A, uint32_t* dst,
                                 int64_t stride_words, cudaStream_t s) {
    if (n_cells)
        log_to_bitmap_kernel<<<grid_for((int64_t)n_cells, 256), 256, 0, s>>>(log, n_cells, A, dst, stride_words);
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
    const size_t smem = sizeof(ClosureShared);
    if (cudaFuncSetAttribute(closure_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
        return 0;
    if (cudaFuncSetAttribute(async_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
        return 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, closure_kernel, kBlock, smem) != cudaSuccess) return 0;
    return nb;
}

cudaError_t launch_xr_closure(const EngineParams& p, const XrParams& x, int grid, cudaStream_t s) {
    const size_t smem = sizeof(ClosureShared);
    cudaError_t c = cudaFuncSetAttribute(xr_closure_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (c != cudaSuccess) return c;
    void* args[] = {(void*)&p, (void*)&x};
    return cudaLaunchCooperativeKernel((const void*)xr_closure_kernel, dim3(grid), dim3(kBlock), args, smem, s);
}

cudaError_t launch_closure(const EngineParams& p, int grid, cudaStream_t s) {
    void* args[] = {(void*)&p};
    return cudaLaunchCooperativeKernel((const void*)closure_kernel, dim3(grid), dim3(kBlock), args,
                                       sizeof(ClosureShared), s);
}

}  // namespace cfpq
