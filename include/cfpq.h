/*
 * libcfpq — B200 (sm_100a) context-free path querying by matrix closure.
 *
 * Implements the hot path of Azimov & Grigorev, "Context-Free Path Querying by
 * Matrix Multiplication" (arXiv 1707.01007); P:n cites PAPER.md line n.
 *
 *   seed     a_ij = {A_k | (i,x,j) ∈ E ∧ (A_k -> x) ∈ P}            (Alg. 1 lines 6-7)
 *   closure  while T changes: T <- T ∪ (T × T)                        (Alg. 1 lines 8-9)
 *            (T × T)_ij = ∪_k T_ik · T_kj,
 *            N1 · N2 = {A | ∃B∈N1, ∃C∈N2, (A -> B C) ∈ P}
 *   result   R_A = {(i,j) | A ∈ T^cf_ij}                              (Theorem 2)
 *   lengths  single-path semantics: seed (A,1); a cell first added in iteration p
 *            through A->BC gets l_A = l_B + l_C and is never overwritten.
 *            Within one iteration the minimum candidate wins (reading c7).
 *
 * Conventions for every call:
 *   - Return value: CFPQ_OK (0) or a negative cfpq_status.  On error the thread-local
 *     message from cfpq_last_error() says why; outputs are left untouched unless the
 *     call documents otherwise.
 *   - Handles are opaque, created and destroyed by the library; the caller owns them
 *     and must destroy them (destroy(NULL) is a no-op).  Handles are not thread-safe:
 *     use one handle from one thread at a time.
 *   - Input arrays are copied (host or device memory as flagged).  Grammar arrays may be
 *     freed as soon as the call returns.  Edge arrays (cfpq_graph_create/set_edges) are
 *     copied on cuda_stream: pageable host memory may be freed on return; device memory
 *     and page-locked host memory are copied asynchronously and must stay valid and
 *     unmodified until the stream has passed the copy (cfpq_closure synchronises the
 *     stream before it returns).  Output buffers are caller-allocated; query sizes first
 *     (two-call pattern via cfpq_result_count).
 *   - Node ids are dense 0..n_nodes-1 ("We enumerate the nodes ... from 0 to
 *     (|V|-1)"); NT ids dense 0..n_nt-1; label ids dense 0..n_labels-1.
 *   - Limits: n_nodes < 2^27, n_nt <= 1024.
 *   - All device work runs on the stream given in cfpq_options.cuda_stream (NULL =
 *     the legacy default stream) of the current CUDA device.  Calls that return host
 *     data synchronise that stream.
 */
#ifndef CFPQ_H
#define CFPQ_H

#include <stdint.h>

#if defined(__GNUC__)
#define CFPQ_API __attribute__((visibility("default")))
#else
#define CFPQ_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    CFPQ_OK = 0,
    CFPQ_E_INVAL = -1,          /* bad argument: out-of-range id, NULL pointer, size mismatch */
    CFPQ_E_NOMEM = -2,          /* device or host allocation failed */
    CFPQ_E_CUDA = -3,           /* a CUDA runtime error (message has cudaGetErrorString) */
    CFPQ_E_NCCL = -4,           /* multi-GPU exchange failed */
    CFPQ_E_NOT_CONVERGED = -5,  /* max_iterations reached before the fixpoint; the
                                   result holds the (sound, monotone) partial T */
    CFPQ_E_OVERFLOW = -6,       /* a single-path length exceeded 2^32-1 */
    CFPQ_E_UNSUPPORTED = -7     /* option combination not implemented */
} cfpq_status;

typedef struct cfpq_grammar cfpq_grammar;
typedef struct cfpq_graph cfpq_graph;
typedef struct cfpq_result cfpq_result;

/* ---------------------------------------------------------------------------------------
 * Grammar: CNF without a start symbol: rules A -> B C and A -> x only.
 *   bin  : host int32 [n_bin][3]  = (A, B, C) for A -> B C, ids in [0, n_nt)
 *   term : host int32 [n_term][2] = (A, x)    for A -> x,   A in [0,n_nt), x in [0,n_labels)
 * P is a set: duplicate rules collapse.  n_bin or n_term may be 0.
 * Errors: CFPQ_E_INVAL on any out-of-range id or n_nt outside [1,1024].
 * ------------------------------------------------------------------------------------- */
CFPQ_API cfpq_status cfpq_grammar_create(int32_t n_nt, int32_t n_labels,
                                const int32_t* bin, int64_t n_bin,
                                const int32_t* term, int64_t n_term,
                                cfpq_grammar** out);
CFPQ_API void cfpq_grammar_destroy(cfpq_grammar* g);

/* ---------------------------------------------------------------------------------------
 * Graph D = (V, E), E ⊆ V × Σ × V.
 *   edges: int32 [n_edges][3] = (src, label, dst); host memory if edges_on_device == 0,
 *          else device memory of the current device.  0 <= src,dst < n_nodes.
 *   Duplicate edges collapse (E is a set); parallel edges with different labels
 *   accumulate; labels without a terminal rule seed nothing.
 *   Edge validity (ranges) is checked on the device by the seed kernel for host and
 *   device input alike: cfpq_closure returns CFPQ_E_INVAL for an out-of-range edge.
 * cfpq_graph_set_edges replaces the edge list of an existing graph (same n_nodes),
 * reusing its device buffer when it is large enough (the host->device copy of a
 * per-query upload).
 * ------------------------------------------------------------------------------------- */
CFPQ_API cfpq_status cfpq_graph_create(int64_t n_nodes, const int32_t* edges, int64_t n_edges,
                              int32_t edges_on_device, void* cuda_stream, cfpq_graph** out);
CFPQ_API cfpq_status cfpq_graph_set_edges(cfpq_graph* g, const int32_t* edges, int64_t n_edges,
                                 int32_t edges_on_device, void* cuda_stream);
CFPQ_API void cfpq_graph_destroy(cfpq_graph* g);

/* ---------------------------------------------------------------------------------------
 * Closure options.  Zero-initialise and set what you need (cfpq_options_default).
 * ------------------------------------------------------------------------------------- */
typedef struct {
    int32_t semantics;       /* 0 relational; 1 single-path lengths. Lengths need
                                8*n^2 bytes of device memory per non-preterminal NT.     */
    int32_t schedule;        /* 0 jacobi: per-iteration states equal Alg. 1's T_k;
                                1 seminaive: same states, same as 0 in this library;
                                2 asynchronous: cells are expanded as soon as they appear,
                                no iteration barriers; same fixpoint T^cf (monotone
                                operator), no per-iteration states (iterations = 0);
                                relational semantics, sparse engine, |N| <= 512;
                                3 Gauss-Seidel: an iteration applies the rules stage by
                                stage (LHS NTs in id order), each stage reading T with the
                                cells of the earlier stages of the same iteration (in-place
                                update of P:222); same fixpoint, fewer iterations (a^n b^n:
                                pq + 1 instead of 2pq + 1); relational, sparse engine, one
                                GPU, no account_work, <= 64 LHS NTs                         */
    int32_t path_policy;     /* 0 auto: sparse, switching to tensor when Δ turns dense and a
                                rule has two changing operands; 1 sparse (index-list semi-
                                naive); 2 tensor (tcgen05 dense, tensor_format); 3 rows (bit-row full-
                                operand, paper-faithful)                                     */
    int32_t account_work;    /* 1: also record per-iteration Jacobi AND-true triple counts
                                (the work of Alg. 1 line 9 on sparse operands); slower     */
    int64_t max_iterations;  /* 0 = |V|^2 |N| + 1 (Theorem 3)                   */
    void*   cuda_stream;     /* cudaStream_t to run on (NULL = default stream)             */
    int32_t world_size;      /* > 1: this process is `rank` of world_size GPUs; every T_A is
                                row-block sharded (cfpq_shard_rows): each rank derives the
                                cells of its rows and the ranks exchange every iteration over
                                NCCL — Δ_k cells as index lists (sparse engine, path_policy
                                0/1), Δ_k word lists (bit-row engine, 3), row blocks or 2-D
                                blocks of T_k (tensor engine, 2).  Every rank passes identical
                                inputs.                                                       */
    int32_t rank;
    const void* nccl_unique_id;  /* world_size > 1: the 128-byte ncclUniqueId from
                                cfpq_nccl_unique_id on one rank, broadcast to all ranks      */
    int64_t log_capacity;    /* initial capacity (cells) of the derived-cell log; 0 = auto */
    int32_t solo_threshold;  /* |Δ| at or below which one CTA runs iterations alone; -1 =
                                auto (1024), 0 = only for an empty Δ                       */
    int32_t record_times;    /* 1: record a device timestamp per iteration (diagnostics,
                                cfpq_result_iteration_stats2)                              */
    int32_t max_ctas;        /* diagnostics: limit the closure kernel's grid (0 = full)    */
    int32_t reserved_emulate;/* testing: > 1 runs that many row-block shards in this process
                                on one GPU (the multi-GPU partition without NCCL)           */
    int32_t cell_set;        /* membership structure of the sparse engine: 0 auto (hashed
                                where allowed and the bit matrices would exceed 1/4 of free
                                HBM), 1 bit matrices, 2 hashed cell set (relational,
                                path_policy 0/1, no rule whose two operands both change,
                                |N| < 1024; else CFPQ_E_UNSUPPORTED)                         */
    int32_t tensor_format;   /* operand format of the tensor engine (path_policy 0/2):
                                0 auto (= 2), 1 int8 (tcgen05 kind::i8, s32 accumulator),
                                2 fp4 (tcgen05 kind::mxf4: 0/1 as e2m1 nibbles, every block
                                scale 1.0, f32 accumulator; all terms are >= 0, so the
                                threshold P > 0 is exact)                           */
    int32_t dense_launch;    /* CTA layout of the tensor engine: 0 auto (= 1), 1 CTA pairs
                                (tcgen05.mma.cta_group::2, M = 256 per pair), 2 one CTA per
                                SM (cta_group::1), 3 CTA pairs of one-SM MMAs sharing the B
                                tile by TMA multicast                                        */
    int32_t diag_flags;      /* diagnostics, 0 = defaults: bit 0 no bit pre-check before the
                                atomic, bit 1 clear the other workspace bank on a side
                                stream, bit 2 no reset of the bit words at the fixpoint,
                                bit 3 one CTA-level log append per iteration instead of
                                each warp appending its own cells (0.49 vs 0.48 ms, config 4),
                                bits 4-6 bit-row R-form kernel variant (0 = default), bit 7
                                reset the bit words at the fixpoint instead of rotating two
                                workspace banks (the default clears the other bank inside
                                the next closure, during its grid-barrier waits), bit 8
                                map Δ chunks to warps CTA-major instead of interleaved, bit 9
                                seed with separate kernels instead of inside the closure
                                kernel, bit 11 bit-row iterations without pipelining (the host
                                reads each iteration's outcome before enqueueing the next),
                                bit 13 no single-cell chains in the one-warp iterations      */
    int32_t grid_rows;       /* tensor engine, world_size (or reserved_emulate) > 1: 2-D
                                process grid grid_rows x grid_cols (SUMMA-style blocks
                                (I_a, J_b) of every T_A); 0 = 1-D row blocks.
                                grid_rows * grid_cols must equal the number of shards        */
    int32_t grid_cols;
    int64_t rows_list_capacity; /* bit-row engine: initial capacity (words) of the Δ_k word
                                list; 0 = 2^20.  Grown on overflow (tests use tiny values)    */
    int32_t exchange;        /* row-sharded sparse engine (world_size or reserved_emulate > 1):
                                0 NCCL, host-driven iterations (all-gather of counts + padded
                                cells per iteration); 1 peer memory, device-resident: one
                                persistent kernel per GPU appends every new cell to every
                                rank's log over NVLink (CUDA IPC mappings) and meets the other
                                ranks at a cross-GPU barrier each iteration (emulated shards:
                                virtual ranks = CTA groups of one launch)                    */
} cfpq_options;

CFPQ_API void cfpq_options_default(cfpq_options* o);

/* ---------------------------------------------------------------------------------------
 * Run seed + closure to the fixpoint.
 *   cfpq_closure        allocates a new result (device workspace sized for this grammar
 *                       and graph) and runs.
 *   cfpq_closure_reuse  re-runs into an existing result created with the same grammar
 *                       shape, n_nodes and options (its workspace is cleared first, in
 *                       O(previous result size)); for repeated queries / benchmarking.
 * Both block until the closure finished (the stream is synchronised).
 * Returns CFPQ_E_NOT_CONVERGED when max_iterations is reached first (the result is
 * then valid and holds the partial T), CFPQ_E_OVERFLOW for a length > 2^32-1.
 * ------------------------------------------------------------------------------------- */
CFPQ_API cfpq_status cfpq_closure(const cfpq_grammar* g, const cfpq_graph* d, const cfpq_options* o,
                         cfpq_result** out);
CFPQ_API cfpq_status cfpq_closure_reuse(const cfpq_grammar* g, const cfpq_graph* d, const cfpq_options* o,
                               cfpq_result* r);
CFPQ_API void cfpq_result_destroy(cfpq_result* r);

/* Loop bodies executed, including the final no-change pass ("k = 6 since T6 = T5"). */
CFPQ_API cfpq_status cfpq_result_iterations(const cfpq_result* r, int64_t* out);

/* |R_A| (Table 1/2 "#results" for the start NT). */
CFPQ_API cfpq_status cfpq_result_count(cfpq_result* r, int32_t nt, int64_t* out);

/* |{(i,j) : A ∈ T_k[i][j]}| and the pairs of T_k for iteration k (0 = seed T_0, up to
 * iterations): the per-iteration states of Alg. 1, for golden tests. */
CFPQ_API cfpq_status cfpq_result_count_at(cfpq_result* r, int32_t nt, int64_t k, int64_t* out);

/* R_A as (i,j) int32 pairs in ascending (i,j) order into dst_pairs[2*capacity].
 * *written = |R_A|; CFPQ_E_INVAL if capacity < |R_A|.  dst on host or device. */
CFPQ_API cfpq_status cfpq_result_pairs(cfpq_result* r, int32_t nt, int32_t* dst_pairs, int64_t capacity,
                              int32_t dst_is_device, int64_t* written);
CFPQ_API cfpq_status cfpq_result_pairs_at(cfpq_result* r, int32_t nt, int64_t k, int32_t* dst_pairs,
                                 int64_t capacity, int32_t dst_is_device, int64_t* written);

/* R_A in compressed-row form (Theorem 2): row_ptr[0..n] int64 with row i's columns in
 * cols[row_ptr[i] .. row_ptr[i+1]) (int32, ascending: the order of cfpq_result_pairs), cols of
 * capacity entries.  *written = |R_A|; CFPQ_E_INVAL if capacity < |R_A| (nothing written then).
 * Both buffers on the host or both on the device (dst_is_device).  Half the bytes of the pair
 * form (4 B per pair + 8(n+1) B) for reading a large relation back. */
CFPQ_API cfpq_status cfpq_result_csr(cfpq_result* r, int32_t nt, int64_t* row_ptr, int32_t* cols, int64_t capacity,
                                     int32_t dst_is_device, int64_t* written);

/* The bit matrix of A: row i, bit j = word j>>5, bit j&31 (LSB first); dst rows are
 * row_stride_words uint32 apart (>= ceil(n/32)); n rows.  dst on host or device. */
CFPQ_API cfpq_status cfpq_result_matrix(cfpq_result* r, int32_t nt, uint32_t* dst, int64_t row_stride_words,
                               int32_t dst_is_device);

/* Single-path lengths of A in the order of cfpq_result_pairs: dst_len[capacity] uint32
 * (only for semantics = 1).  *written = |R_A|. */
CFPQ_API cfpq_status cfpq_result_lengths(cfpq_result* r, int32_t nt, uint32_t* dst_len, int64_t capacity,
                                int32_t dst_is_device, int64_t* written);

/* Single-path witness ("a path can be found by a simple search"), rebuilt on
 * the GPU from the recorded lengths (semantics = 1 only): out_edges[3*t .. 3*t+2] =
 * (src, label, dst) of the t-th edge of a path i -> j of exactly *written = l_A(i,j) edges
 * whose word A derives.  Split choice: the first binary rule A -> B C in (B, C) ascending
 * order (rules are kept deduplicated and sorted, "P is a set") and the
 * smallest node r with l_B(i,r) + l_C(r,j) = l; a length-1 cell takes the lowest-index edge
 * (i, x, j) with A -> x.  d = the graph of the closure (its edges).  CFPQ_E_INVAL if (A,i,j)
 * is not in R_A or capacity < l (*written still holds l for a second call).  dst on host
 * or device. */
CFPQ_API cfpq_status cfpq_result_witness(cfpq_result* r, const cfpq_graph* d, int32_t nt, int32_t i, int32_t j,
                                         int32_t* out_edges, int64_t capacity, int32_t dst_is_device,
                                         int64_t* written);

/* Diagnostics (all optional):
 *   stats[0] iterations, [1] total derived cells incl. seeds, [2] log capacity used,
 *   [3] overflow regrows, [4] kernel launches of the last closure, [5] iterations run
 *   in single-CTA mode, [6] candidates expanded (semi-naive AND-true triples),
 *   [7] (Δ entry, rule occurrence) expansions, [8] device time of the seed phase (seed,
 *   adjacency build, snapshot seeding) in ns, [9] device time of the fixpoint-loop
 *   kernel launches in ns (CUDA events on the closure stream), [10] CTAs of the closure
 *   kernel, [11..17] single-CTA phase cycle counters (only with record_times), [18] tcgen05
 *   MMA work issued by the dense engine, in units of 128 x 32 x 128 multiply-adds = 2^20 ops (an
 *   M=128 x N=256 x K=128 int8 k-block counts 8; fp4 k-blocks are 256 deep),
 *   [19] 1 if the last closure finished on the dense engine (path_policy 2, or the auto
 *   policy switched to it once Δ became dense), [20] 1 if the cells were kept in the
 *   hashed cell set (cell_set), [21] its capacity in slots.
 * Per-iteration arrays (length = iterations) via cfpq_result_iteration_stats:
 *   new_cells[k-1] = |T_k \ T_{k-1}|, jacobi_triples[k-1] (only with account_work). */
CFPQ_API cfpq_status cfpq_result_stats(const cfpq_result* r, int64_t* stats, int32_t n_stats);
CFPQ_API cfpq_status cfpq_result_iteration_stats(cfpq_result* r, int64_t* new_cells, int64_t* jacobi_triples,
                                        int64_t capacity);
/* As above plus end_ns[k-1] = device time (ns, %globaltimer) from the end of seeding to
 * the end of iteration k (iterations past 2^22 are not recorded). */
CFPQ_API cfpq_status cfpq_result_iteration_stats2(cfpq_result* r, int64_t* new_cells, int64_t* jacobi_triples,
                                                  int64_t* end_ns, int64_t capacity);

/* Diagnostics of a run with record_times = 1: cycles[(k-1)*4 + q] for grid-wide iteration k
 * (SM clock cycles; 0 for iterations run by one CTA or warp):
 *   q = 0  expansion of Δ_{k-1}, max over CTAs     q = 1  CTA flush of staged cells, max
 *   q = 2  grid-barrier wait of the last CTA to arrive (min over CTAs)
 *   q = 3  close of the iteration (range / flag update), max over CTAs
 * capacity = number of iterations the caller's buffer holds (4 entries each). */
CFPQ_API cfpq_status cfpq_result_iteration_phases(cfpq_result* r, int64_t* cycles, int64_t capacity);

/* Multi-GPU bootstrap: write a fresh ncclUniqueId (128 bytes) into out[bytes].  NCCL is
 * loaded at run time (libnccl.so.2); CFPQ_E_NCCL if it is unavailable. */
CFPQ_API cfpq_status cfpq_nccl_unique_id(void* out, int64_t bytes);

/* Rows [row_lo, row_hi) of every T_A that `rank` of world_size computes under row-block
 * sharding (blocks of 128-row tiles; "matrix multiplication in the main loop ... may
 * be performed on different GPGPU independently").  Pure host function. */
CFPQ_API cfpq_status cfpq_shard_rows(int64_t n_nodes, int32_t world_size, int32_t rank, int64_t* row_lo,
                                     int64_t* row_hi);

/* Block [row_lo, row_hi) x [col_lo, col_hi) of every T_A that shard `rank` (row-major in the
 * grid: a = rank / grid_cols, b = rank % grid_cols) derives under 2-D block sharding of the
 * tensor engine (grid_rows x grid_cols grid; 128-row and 256-column tiles).  Pure host
 * function; CFPQ_E_INVAL on a bad grid or rank. */
CFPQ_API cfpq_status cfpq_shard_block(int64_t n_nodes, int32_t grid_rows, int32_t grid_cols, int32_t rank,
                                      int64_t* row_lo, int64_t* row_hi, int64_t* col_lo, int64_t* col_hi);

/* Thread-local message describing the last non-OK status. */
CFPQ_API const char* cfpq_last_error(void);

/* Library build/version string ("libcfpq <ver> sm_100a ..."). */
CFPQ_API const char* cfpq_version(void);

#ifdef __cplusplus
}
#endif
#endif /* CFPQ_H */
