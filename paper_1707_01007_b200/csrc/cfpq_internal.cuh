// Internal declarations of libcfpq (not part of the C-ABI).
//
// Layout in HBM:
//   T      : per NT A, an n x Wp bit matrix, uint32 words, row-major; bit j of row i
//            is word j>>5, bit j&31.  Wp = words per row, padded to a multiple of 32
//            (128-byte rows).  T_A = T + A*n*Wp.  The set-valued matrix of P:94/P:157 is
//            exactly the bundle of these |N| bit matrices (Valiant's |N|^2 BMM view).
//   log    : append-only list of derived cells, packed uint64 (A:10 | i:27 | j:27).
//            Δ_0 = seeds, then Δ_1, Δ_2, ... (Δ_k = T_k \ T_{k-1}); iter_off[k] = start
//            of Δ_k.  Iteration k expands exactly Δ_{k-1} (semi-naive, exact per
//            iteration: T_k = T_{k-1} ∪ Δ_B×T_C ∪ T_B×Δ_C).
//   adj    : CSR (rows) / CSC (columns) of preterminal NTs (LHS of no binary rule,
//            constant after seeding), one concatenated index array.
//   S, ST  : row / transposed snapshots of NTs that are operands of a rule whose two
//            operands both change (needed to read T_{k-1} exactly while T_k is written).
//   K      : single-path keys, uint64 per cell of non-preterminal NTs:
//            (iteration << 32) | length; EMPTY = ~0.  atomicMin on the key gives
//            first-write-wins across iterations (smaller stamp) and the minimum length
//            within the discovery iteration (P:393 + reading c7), order-independently.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <string>
#include <vector>

#include "../../include/cfpq.h"

// Checked build (libcfpq_checked.so, `build(checked=True)`): device-side bounds assertions on
// the computed indices of the hot kernels (matrix words, log slots, adjacency entries); a
// failed one prints its site and traps.  The product build compiles them out.
#ifdef CFPQ_CHECKED
#include <cstdio>
#define CFPQ_DASSERT(c)                                                                    \
    do {                                                                                   \
        if (!(c)) {                                                                        \
            printf("CFPQ_DASSERT failed %s:%d: %s\n", __FILE__, __LINE__, #c);           \
            __trap();                                                                      \
        }                                                                                  \
    } while (0)
#else
#define CFPQ_DASSERT(c) \
    do {                \
    } while (0)
#endif

namespace cfpq {

constexpr int kMaxNT = 1024;
constexpr int kNodeBits = 27;
constexpr uint64_t kNodeMask = (1ull << kNodeBits) - 1;
constexpr uint64_t kEmptyKey = ~0ull;
constexpr unsigned long long kHashEmpty = ~0ull;   // no cell packs to it (hashed mode needs |N| < 1024)
constexpr int kHashMaxProbe = 4096;                // a longer run reports overflow: the host regrows

__host__ __device__ inline uint64_t pack_cell(uint32_t A, uint32_t i, uint32_t j) {
    return ((uint64_t)A << (2 * kNodeBits)) | ((uint64_t)i << kNodeBits) | (uint64_t)j;
}
__host__ __device__ inline uint32_t cell_nt(uint64_t c) { return (uint32_t)(c >> (2 * kNodeBits)); }
__host__ __device__ inline uint32_t cell_i(uint64_t c) { return (uint32_t)((c >> kNodeBits) & kNodeMask); }
__host__ __device__ inline uint32_t cell_j(uint64_t c) { return (uint32_t)(c & kNodeMask); }

// Expansion of one Δ entry of NT X through one rule A -> B C in which X occurs.
enum ExpKind : int32_t {
    EXP_L_CONST = 0,  // X = B, C preterminal : (i,r) -> (i, j) for j in CSR_C.row(r)
    EXP_R_CONST = 1,  // X = C, B preterminal : (r,j) -> (i, j) for i in CSC_B.col(r)
    EXP_L_VAR = 2,    // X = B, C changes     : (i,r) -> (i, j) for j in S_C row r
    EXP_R_VAR = 3,    // X = C, B changes     : (r,j) -> (i, j) for i in ST_B row r
};

struct Expansion {
    int32_t kind;
    int32_t A;      // LHS
    int32_t other;  // the other operand NT (C for L kinds, B for R kinds)
    int32_t stage;  // Gauss-Seidel schedule: the stage of the LHS A (LHS NTs in id order)
};

constexpr int kMaxStages = 64;   // Gauss-Seidel stages (distinct LHS NTs) supported

// Per-NT device table (read through the read-only path).
struct NTInfo {
    uint32_t* T;          // bit matrix
    uint32_t* S;          // row snapshot (or null)
    uint32_t* ST;         // transposed snapshot (or null)
    uint64_t* K;          // single-path keys (or null: preterminal -> length 1)
    const int32_t* csr_ptr;  // n+1 (or null)
    const int32_t* csc_ptr;  // n+1 (or null)
    const int4* csr_ell;     // n ELL heads {beg, deg, nb0, nb1} of the CSR rows (or null)
    const int4* csc_ell;     // n ELL heads of the CSC columns (or null)
    int32_t exp_begin, exp_end;   // expansions of Δ entries of this NT
    int32_t is_const;
    int32_t needs_snapshot;       // S and/or ST present
};

// Global state of one closure run (device memory).
struct EngineState {
    unsigned long long log_size;   // append counter (may exceed cap on overflow)
    unsigned long long lo, hi;     // Δ_{k-1} = log[lo, hi)
    long long iter;                // iterations completed
    int status;                    // ST_*
    int overflow;                  // set by a failed append
    int len_overflow;              // set by a single-path length > 2^32-1
    int bad_edge;                  // seed saw an out-of-range edge
    unsigned long long candidates; // expanded candidates = semi-naive AND-true triples
    unsigned long long expansions; // (Δ entry, rule occurrence) pairs expanded
    long long solo_iters;          // iterations run by the single-CTA path
    unsigned long long prof[7];    // single-CTA phase cycle counters (record_times diagnostics)
    unsigned long long async_head; // asynchronous schedule: next log slot to claim
    unsigned long long async_done; // asynchronous schedule: log entries fully expanded
    unsigned bar_count;            // grid-barrier words, on their own 128-byte line
    unsigned bar_pad;
    // released by the last CTA to arrive: generation (bits 63-40) | error flags of the
    // iteration it closes (bits 39-38: overflow, length overflow) | log size (bits 37-0), so
    // a waiting CTA gets the iteration's outcome with the same load that releases it
    unsigned long long bar_word;
    unsigned long long pad_snap[2];
    unsigned pad1[20];
    unsigned long long clr_cursor; // in-kernel clear of the other bank: next cell to claim
    // Gauss-Seidel schedule: gs_ring[t mod (S+1)] = L_t, the log size when step t starts
    // (L_1 = |Δ_0|); step t expands log[L_{t-S}, L_t) through the rules of stage (t-1) mod S
    unsigned long long gs_ring[kMaxStages + 1];
    // peer-memory exchange: xr_slot[k & 1] collects, on every rank, the iteration-k arrival of
    // every rank's last CTA as (its new cells << 32) | (its overflow << 16) | 1; xr_new counts
    // this rank's new cells of the current iteration (appended to every rank's log)
    unsigned long long xr_slot[2];
    unsigned long long xr_new;
    int adj_tail;                  // fused seeding: some adjacency row has > 2 entries
    int gs_stage;                  // stage of the next step ((k) mod S after step k closed)
    int gs_slot;                   // ring slot of L_{k+1} ((k+1) mod (S+1))
    long long gs_round;            // rounds completed (k / S)
};

enum : int { ST_RUNNING = 0, ST_DONE = 1, ST_OVERFLOW = 2, ST_CAP = 3, ST_LEN_OVERFLOW = 4, ST_SWITCH = 5,
              ST_TIMEOUT = 6 };

// Peer-memory exchange of the row-sharded sparse engine (exchange = 1): every rank's engine
// state and log, reachable from every rank (NVLink peer mappings on real GPUs; plain device
// pointers of the virtual ranks of an emulated launch).
constexpr int kMaxXrRanks = 32;
struct XrParams {
    int32_t P;                     // ranks
    int32_t my_rank;               // >= 0: one launch per GPU; -1: emulated, rank = blockIdx.x / cpr
    int32_t cpr;                   // CTAs per rank
    EngineState* const* st;        // [P]
    uint64_t* const* log;          // [P]
    const uint32_t* row_lo;        // [P] rows each rank derives
    const uint32_t* row_hi;
};

struct EngineParams {
    int32_t n;
    int32_t n_nt;
    int64_t Wp;                    // words per bit-matrix row
    const NTInfo* nt;              // [n_nt]
    const Expansion* exps;
    int32_t n_exps;
    const int32_t* adj_idx;        // concatenated CSR/CSC index array
    long long adj_cap;             // its capacity (checked build)
    uint64_t* log;
    unsigned long long log_cap;
    EngineState* st;
    unsigned long long* iter_off;  // [iter_off_cap]
    long long iter_off_cap;
    unsigned long long* jac;       // per-iteration Jacobi triple counts (account mode) or null
    unsigned long long* iter_time; // per-iteration %globaltimer stamps (ns) at finalize, [iter_off_cap]
    unsigned long long* phase;     // diagnostics: per grid iteration [k][4] SM cycles (see closure_kernel)
    uint32_t* rowc;                // account mode: per NT row / column nnz of T (n_nt*n each)
    uint32_t* colc;
    const int32_t* rules;          // [n_rules][3] (account mode)
    int32_t n_rules;
    int32_t lengths;               // single-path semantics
    long long max_iter;
    int32_t solo_max;              // |Δ| <= solo_max -> single-CTA iterations
    int32_t has_snapshots;
    int32_t nblocks;
    int32_t profile;               // accumulate single-CTA phase cycles into EngineState::prof
    unsigned long long switch_cells;  // |Δ_k| above which the loop stops for the dense engine (0 = never)
    int32_t precheck;              // read a candidate's word before its atomicOr (hot cells)
    int32_t cta_major;             // diagnostics (diag_flags bit 8): chunk c -> warp c (CTA-major)
    int32_t no_chain;              // diagnostics (diag_flags bit 13): no single-cell chains in warp-solo
    int32_t warp_flush;            // each warp appends its own cells at the end of its expansion (default;
                                   // diag_flags bit 3 = one CTA-level append instead)
                                   // (one log atomic per warp) instead of the CTA-level flush
    int32_t self_clear;            // relational runs: at the fixpoint the kernel resets the words
                                   // of all logged cells in T/S/ST (the results stay in the log)
    // hashed cell set (relational sparse runs without var x var rules): open addressing,
    // linear probing over 64-bit packed cells, replaces the T bit matrices as the
    // membership structure (see engine.cu, "Hashed cell set")
    unsigned long long* hset;      // [hmask + 1] or null (bit matrices)
    unsigned long long hmask;
    int32_t hshift;                // 64 - log2(hmask + 1)
    // row-block sharding of the sparse engine: this launch derives only cells whose row
    // i lies in [row_lo, row_hi) (the rows its rank owns); [0, n) when unsharded
    uint32_t row_lo, row_hi;
    // the previous run's cells in the other workspace bank, cleared by CTAs that wait at
    // a grid barrier (and drained at kernel end): clr_n = 0 when there is nothing to clear
    const uint64_t* clr_log;
    unsigned long long clr_n;
    const NTInfo* clr_nt;
    uint32_t* clr_rowc;
    uint32_t* clr_colc;
    unsigned long long async_init; // asynchronous schedule: log entries < this are valid unflagged
    int32_t gs_stages;             // > 0: Gauss-Seidel schedule with that many stages (0: Jacobi)
    // seeding folded into the closure kernel (fused_seed = 1 on the first launch of a
    // one-GPU sparse run): T_0 from the edges, the preterminal ELL heads counted on the fly,
    // CSR tails (scan + fill) only when some adjacency row has more than two entries
    int32_t fused_seed;
    const int32_t* edges;
    int64_t n_edges;
    const int32_t* lab_ptr;
    const int32_t* lab_nt;
    int32_t n_labels;
    int32_t max_rules;
    const int32_t* slot_row;
    const int32_t* slot_col;
    int32_t n_slots;
    int32_t* adj_cursor;           // [n_slots * n] CSR fill cursors (zeroed in the kernel)
    int32_t* adj_idx_w;            // adj_idx, writable
    int4* ell;                     // [n_slots * n] ELL heads {beg, deg, nb0, nb1}
    unsigned long long* scan_tot;  // [grid + 1] per-CTA totals of the in-kernel scan
};

// ------------------------------------------------------------------------------------------
// Host-side objects behind the opaque C handles
// ------------------------------------------------------------------------------------------
struct Rule3 { int32_t A, B, C; };

}  // namespace cfpq

struct cfpq_grammar {
    int32_t n_nt = 0, n_labels = 0;
    std::vector<cfpq::Rule3> rules;              // distinct binary rules
    std::vector<std::pair<int32_t, int32_t>> term;  // distinct (A, x)
    std::vector<int32_t> is_const;               // LHS of no binary rule
};

struct cfpq_graph {
    int64_t n_nodes = 0;
    int64_t n_edges = 0;
    int64_t cap_edges = 0;
    int32_t* d_edges = nullptr;    // device [cap][3]
};

struct cfpq_result;   // defined in api.cu

namespace cfpq {

// error plumbing
void set_error(const std::string& msg);
#define CFPQ_CUDA_TRY(expr)                                                               \
    do {                                                                                  \
        cudaError_t _e = (expr);                                                          \
        if (_e != cudaSuccess) {                                                          \
            (void)cudaGetLastError(); /* a non-sticky error must not leak into later calls */ \
            ::cfpq::set_error(std::string(#expr) + ": " + cudaGetErrorString(_e));        \
            return CFPQ_E_CUDA;                                                           \
        }                                                                                 \
    } while (0)

// kernels/launchers implemented in the .cu files
cudaError_t launch_seed(const int32_t* edges, int64_t n_edges, int32_t n_nodes, const int32_t* lab_ptr,
                        const int32_t* lab_nt, int32_t n_labels, int32_t max_rules_per_label,
                        const EngineParams& p, cudaStream_t s);
cudaError_t launch_adj_count(const EngineParams& p, const int32_t* slot_row, const int32_t* slot_col,
                             int32_t* counts, unsigned long long n_seed_upper, cudaStream_t s);
cudaError_t launch_adj_fill(const EngineParams& p, const int32_t* slot_row, const int32_t* slot_col,
                            const int32_t* ptr, int32_t* counts, int32_t* idx, int4* ell, unsigned long long n_seed,
                            cudaStream_t s);
cudaError_t launch_rehash(const EngineParams& p, unsigned long long n_cells, uint64_t cell_mask, int need_flag,
                          cudaStream_t s);
cudaError_t launch_log_to_bitmap(const uint64_t* log, unsigned long long n_cells, uint32_t A, uint32_t* dst,
                                 int64_t stride_words, cudaStream_t s);
cudaError_t launch_clear_log(const EngineParams& p, unsigned long long n_cells, cudaStream_t s);
cudaError_t launch_begin(const EngineParams& p, cudaStream_t s);
cudaError_t launch_async(const EngineParams& p, int grid, cudaStream_t s, bool flag_seeds,
                         unsigned long long seeds_upper);
cudaError_t launch_strip_flags(uint64_t* log, unsigned long long lo, unsigned long long hi, cudaStream_t s);

cudaError_t launch_seed_snapshots(const EngineParams& p, unsigned long long n_seed_upper, cudaStream_t s);
int closure_kernel_blocks_per_sm();
int closure_kernel_block_size();
cudaError_t launch_closure(const EngineParams& p, int grid, cudaStream_t s);
cudaError_t launch_xr_closure(const EngineParams& p, const XrParams& x, int grid, cudaStream_t s);

cudaError_t launch_nt_histogram(const uint64_t* log, unsigned long long n, unsigned long long* counts, int n_nt,
                                cudaStream_t s);
cudaError_t launch_filter_nt(const uint64_t* log, unsigned long long n, uint32_t A, void* keys,
                             unsigned long long* count, int bits, int k32, cudaStream_t s);
cudaError_t sort_keys32(uint32_t* keys, uint32_t* keys_alt, unsigned long long n, int end_bit, void* temp,
                        size_t* temp_bytes, cudaStream_t s);
cudaError_t sort_keys(uint64_t* keys, uint64_t* keys_alt, unsigned long long n, int end_bit, void* temp,
                      size_t* temp_bytes, cudaStream_t s);
cudaError_t launch_unpack_pairs(const void* keys, unsigned long long n, int32_t* pairs, int bits, int k32,
                                cudaStream_t s);
cudaError_t launch_gather_lengths(const void* keys, unsigned long long n, const uint64_t* K, int64_t n_nodes,
                                  uint32_t* out, int bits, int k32, cudaStream_t s);
cudaError_t launch_scan(const int32_t* in, int32_t* out, int64_t n, void* temp, size_t* temp_bytes,
                        cudaStream_t s);
cudaError_t launch_edge_csr(const int32_t* edges, int64_t n_edges, int32_t n, int32_t* deg, int32_t* ptr,
                            int32_t* cursor, int32_t* idx, void* temp, size_t* temp_bytes, cudaStream_t s);
cudaError_t launch_witness(const EngineParams& p, const int32_t* rules, const int32_t* rule_ptr,
                           const int32_t* rule_ids, const int32_t* e_ptr, const int32_t* e_idx, const int32_t* edges,
                           const int32_t* lab_ptr, const int32_t* lab_nt, int32_t n_labels, void* stack,
                           int64_t stack_cap, uint32_t A, uint32_t i, uint32_t j, uint32_t len, int32_t* out,
                           int64_t out_cap, long long* result, cudaStream_t s);
size_t witness_frame_bytes();
cudaError_t launch_bitmap_rowcount(const uint32_t* T, int32_t n, int64_t Wp, int32_t* rowcnt,
                                   unsigned long long* total, cudaStream_t s);
cudaError_t launch_bitmap_pairs(const uint32_t* T, int32_t n, int64_t Wp, const int32_t* rowoff, int32_t* pairs,
                                cudaStream_t s, int cols_only = 0);
cudaError_t launch_keys_to_csr(const void* keys, unsigned long long m, int bits, int k32, int64_t n, int64_t* row_ptr,
                               int32_t* cols, cudaStream_t s);
cudaError_t launch_rowoff_to_ptr(const int32_t* rowoff, int64_t n, int64_t* row_ptr, cudaStream_t s);

// dense (tcgen05) engine, dense.cu
struct DenseEngine;
DenseEngine* dense_create(int32_t n, int32_t n_nt, int64_t Wp, const std::vector<Rule3>& rules,
                          const std::vector<int32_t>& is_const, cudaStream_t s, std::string* err, bool tensor,
                          bool fp4, int64_t dlist_cap, int32_t launch_mode);
bool dense_is_fp4(const DenseEngine* e);
void dense_destroy(DenseEngine* e);
void dense_set_rgather_variant(DenseEngine* e, int v);   // diagnostics (diag_flags bits 4-6)
cudaError_t dense_begin(DenseEngine* e, uint32_t* const* T, uint32_t* const* Tn, bool first, cudaStream_t s,
                        int* launches, bool pack_operands);
// Bit-row (full-operand Jacobi) iteration: nt = the device NT table (is_const, CSR rows of
// preterminals), adj_idx = CSR index array, log[0, n_seeds) = the seed cells (read at the
// first iteration only).
cudaError_t rows_product(DenseEngine* e, uint32_t* const* T, uint32_t* const* Tn, const NTInfo* nt,
                         const int32_t* adj_idx, const uint64_t* log, unsigned long long n_seeds, bool first,
                         cudaStream_t s, int* launches);
// T_k rows of row tiles [i_lo, i_hi) (128 rows) x column tiles [j_lo, j_hi) (256 columns;
// j_hi < 0: all) of every output.
cudaError_t dense_product(DenseEngine* e, int64_t i_lo, int64_t i_hi, cudaStream_t s, int* launches, int64_t j_lo = 0,
                          int64_t j_hi = -1);
// 2-D block exchange: copy the bit block rows [r_lo, r_hi) x words [w_lo, w_hi) of T between
// the matrix and a contiguous staging buffer (to_buf 1: matrix -> buffer).
cudaError_t bit_block_copy(uint32_t* T, int64_t Wp, int64_t r_lo, int64_t r_hi, int64_t w_lo, int64_t w_hi,
                           uint32_t* buf, int to_buf, cudaStream_t s);
// Row-block sharded bit-row iterations: begin (T_k := T_{k-1}), per shard plan + products of
// rows [row_lo, row_hi), settle (list length; rebuilt from T_k minus T_{k-1} on overflow), the
// exchange of the word lists (caller), then apply every rank's words to T_k.
cudaError_t rows_begin(DenseEngine* e, const NTInfo* nt, const int32_t* adj_idx, const uint64_t* log,
                       unsigned long long n_seeds, bool first, cudaStream_t s, int* launches);
cudaError_t rows_shard(DenseEngine* e, int64_t row_lo, int64_t row_hi, cudaStream_t s, int* launches);
// After a sync: grow what overflowed; *redo = re-run the shard (chunk lists); check_list:
// also handle a Δ word-list overflow (unsharded runs; sharded runs rebuild the list instead)
cudaError_t rows_shard_check(DenseEngine* e, cudaStream_t s, bool* redo, bool check_list);
cudaError_t rows_list_settle(DenseEngine* e, int64_t row_lo, int64_t row_hi, unsigned long long keep, cudaStream_t s,
                             unsigned long long* count);
cudaError_t rows_list(DenseEngine* e, unsigned long long want, void** list, unsigned long long* cap);
cudaError_t rows_apply_all(DenseEngine* e, unsigned long long total, cudaStream_t s, int* launches);
cudaError_t dense_finish(DenseEngine* e, cudaStream_t s, unsigned long long* new_total);
// pipelined bit-row iterations (unsharded compact mode; dense.cu)
bool rows_pipe_eligible(DenseEngine* e);
cudaError_t rows_pipe_begin(DenseEngine* e, uint32_t* const* T, uint32_t* const* Tn, cudaStream_t s);
void rows_pipe_end(DenseEngine* e);
void rows_set_first(DenseEngine* e, bool first);
cudaError_t rows_pipe_clear_stop(DenseEngine* e, cudaStream_t s);
cudaError_t dense_set_tables(DenseEngine* e, uint32_t* const* T, uint32_t* const* Tn, cudaStream_t s);
cudaError_t rows_pipe_iteration(DenseEngine* e, const NTInfo* nt, const int32_t* adj_idx, const uint64_t* log,
                                unsigned long long n_seeds, bool first, long long k, long long cap_iter, int slot,
                                cudaEvent_t done, cudaStream_t s, int* launches);
void rows_pipe_result(DenseEngine* e, int slot, unsigned long long* nw, int* stop, unsigned long long* list_words);
cudaError_t rows_grow_list(DenseEngine* e, unsigned long long words);
unsigned long long dense_list_capacity(const DenseEngine* e);
unsigned long long* dense_total_counter(DenseEngine* e);
int64_t dense_row_tiles(const DenseEngine* e);

// multi-GPU plumbing, comm.cu
bool nccl_unique_id(void* out, std::string* err);
size_t nccl_unique_id_bytes();
void* nccl_comm_create(const void* id_bytes, int world, int rank, std::string* err);
void nccl_comm_destroy(void* comm);
bool nccl_allgather_u64(void* comm, uint64_t* buf, size_t count, int rank, cudaStream_t s, std::string* err);
bool nccl_exchange_rows(void* comm, uint32_t* const* mats, int n_mats, size_t block_words, int rank,
                        unsigned long long* counter, cudaStream_t s, std::string* err);
void dense_partition(int64_t n, int world, int rank, int64_t* tile_lo, int64_t* tile_hi, int64_t* block_rows);
// 2-D process grid gr x gc: shard (a, b) owns row tiles [ti_lo, ti_hi) (128 rows) and column
// tiles [tj_lo, tj_hi) (256 columns) of every T_A.
void dense_partition2(int64_t n, int gr, int gc, int a, int b, int64_t* ti_lo, int64_t* ti_hi, int64_t* tj_lo,
                      int64_t* tj_hi);
void* nccl_comm_split(void* comm, int color, int key, std::string* err);
bool nccl_allgather_u32(void* comm, uint32_t* buf, size_t count, int rank, cudaStream_t s, std::string* err);
bool nccl_allreduce_sum_u64(void* comm, unsigned long long* buf, size_t count, cudaStream_t s, std::string* err);
bool nccl_group(bool start, std::string* err);
const std::vector<int32_t>& dense_outputs(const DenseEngine* e);
unsigned long long dense_kblocks(DenseEngine* e, bool reset);
cudaError_t dense_account(DenseEngine* e, uint32_t* const* T, const std::vector<Rule3>& rules, cudaStream_t s,
                          unsigned long long* out);

}  // namespace cfpq
