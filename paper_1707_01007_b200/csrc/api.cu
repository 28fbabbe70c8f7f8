// C-ABI of libcfpq (include/cfpq.h): handles, workspace planning, the closure driver
// and result extraction.  All arithmetic of the method runs in the kernels of
// engine.cu / extract.cu; this file only validates, allocates and launches.
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <set>
#include <string>
#include <tuple>
#include <vector>

#include "cfpq_internal.cuh"

namespace cfpq {
static thread_local std::string g_last_error;
void set_error(const std::string& msg) { g_last_error = msg; }
}  // namespace cfpq

using namespace cfpq;

#define CFPQ_CHECK_ARG(cond, msg)          \
    do {                                   \
        if (!(cond)) {                     \
            set_error(msg);                \
            return CFPQ_E_INVAL;           \
        }                                  \
    } while (0)

// ------------------------------------------------------------------------------------------
// device buffer helper
// ------------------------------------------------------------------------------------------
template <typename T>
static cfpq_status dalloc(T** p, size_t count, const char* what) {
    *p = nullptr;
    if (count == 0) count = 1;
    cudaError_t e = cudaMalloc((void**)p, count * sizeof(T));
    if (e != cudaSuccess) {
        cudaGetLastError();
        set_error(std::string("cudaMalloc(") + what + ", " + std::to_string(count * sizeof(T)) +
                  " bytes): " + cudaGetErrorString(e));
        *p = nullptr;
        return CFPQ_E_NOMEM;
    }
    return CFPQ_OK;
}
template <typename T>
static void dfree(T*& p) {
    if (p) cudaFree((void*)p);
    p = nullptr;
}

// A workspace bank: everything a closure derives into.  A reused result keeps two banks
// and alternates: the next run starts on the clean bank while the previous run's cells are
// cleared from the other bank on a side stream (O(|cells|) scattered stores, overlapped).
struct Bank {
    uint32_t* d_T = nullptr;
    uint32_t* d_snap = nullptr;
    uint64_t* d_K = nullptr;
    NTInfo* d_nt = nullptr;
    uint64_t* d_log = nullptr;
    unsigned long long log_cap = 0;
    unsigned long long n_cells = 0;
    uint32_t* d_rowc = nullptr;
    uint32_t* d_colc = nullptr;
    unsigned long long* d_hset = nullptr;
    unsigned long long hcap = 0;
    std::vector<NTInfo> h_nt;
    std::vector<uint32_t*> Tbase;
    void release() {
        dfree(d_T); dfree(d_snap); dfree(d_K); dfree(d_nt); dfree(d_log); dfree(d_rowc); dfree(d_colc);
        dfree(d_hset);
        log_cap = n_cells = hcap = 0;
    }
};

struct cfpq_result {
    // shape
    int64_t n = 0;
    int32_t n_nt = 0, n_labels = 0;
    int64_t Wp = 0;
    cfpq_options opts{};
    cudaStream_t stream = nullptr;
    int32_t grid = 0;
    std::vector<Rule3> rules;
    std::vector<std::pair<int32_t, int32_t>> term;
    // device buffers
    uint32_t* d_T = nullptr;
    uint32_t* d_snap = nullptr;       // S and ST slots
    uint64_t* d_K = nullptr;
    NTInfo* d_nt = nullptr;
    Expansion* d_exps = nullptr;
    int32_t* d_rules = nullptr;
    int32_t* d_lab_ptr = nullptr;
    int32_t* d_lab_nt = nullptr;
    int32_t max_rules_per_label = 0;
    int32_t* d_slot_row = nullptr;
    int32_t* d_slot_col = nullptr;
    int32_t n_adj_slots = 0;
    int32_t* d_adj_cnt = nullptr;     // counts, then (scanned) pointers
    int32_t* d_adj_ptr = nullptr;
    int32_t* d_adj_cursor = nullptr;
    int32_t* d_adj_idx = nullptr;
    int4* d_adj_ell = nullptr;
    int32_t n_exps = 0;
    int64_t adj_idx_cap = 0;
    uint64_t* d_log = nullptr;
    unsigned long long log_cap = 0;
    // hashed cell set (see engine.cu): replaces the T bit matrices when `hashed`
    bool hashed = false;
    unsigned long long* d_hset = nullptr;
    unsigned long long hcap = 0;              // slots, a power of two >= 2 * log_cap
    EngineState* d_st = nullptr;
    unsigned long long* d_iter_off = nullptr;
    long long iter_off_cap = 0;
    unsigned long long* d_jac = nullptr;
    unsigned long long* d_iter_time = nullptr;
    unsigned long long* d_phase = nullptr;
    uint32_t* d_rowc = nullptr;
    uint32_t* d_colc = nullptr;
    void* d_temp = nullptr;
    size_t temp_bytes = 0;
    // scratch for extraction
    uint64_t* d_keys = nullptr;
    unsigned long long keys_cap = 0;
    unsigned long long* d_small = nullptr;   // [n_nt + 2] counters
    // host-side copies
    std::vector<NTInfo> h_nt;
    int has_snapshots = 0;
    EngineState h_st{};
    int64_t iterations = 0;
    unsigned long long n_cells = 0;
    int64_t regrows = 0;
    int64_t switched = 0;
    int64_t launches = 0;
    std::vector<int64_t> counts;
    bool counts_valid = false;
    bool ran = false;
    // dense (tcgen05) engine state
    bool dense_mode = false;                  // the last (or current) run finished on the dense engine
    unsigned long long switch_cells = 0;      // auto policy: sparse -> dense when |Δ_k| exceeds this
    std::vector<int32_t> is_const;
    DenseEngine* dense = nullptr;
    uint32_t* d_Tn = nullptr;                 // second bit-matrix buffer of the outputs
    std::vector<uint32_t*> Tbase, Tcur, Tnxt;  // per NT
    std::vector<int64_t> dense_new;           // new cells per iteration
    std::vector<int64_t> dense_jac;           // Jacobi AND-true triples per iteration (account_work)
    unsigned long long dense_kb = 0;          // issued 128x256x128 int8 MMA k-blocks
    int32_t n_stages = 0;                     // distinct LHS NTs (Gauss-Seidel stages, schedule 3)
    int32_t grid_r = 0, grid_c = 0;           // 2-D process grid of the tensor engine (0: 1-D)
    // peer-memory exchange of the row-sharded sparse engine (exchange = 1, XrParams)
    bool xr = false;
    std::vector<EngineState*> xr_st;          // [P] state of every rank (own / peer mapped / virtual)
    std::vector<uint64_t*> xr_log;            // [P]
    std::vector<void*> xr_owned;              // emulated: the virtual ranks' buffers (freed here)
    std::vector<void*> xr_opened;             // real GPUs: IPC mappings of peers (closed here)
    EngineState** d_xr_st = nullptr;
    uint64_t** d_xr_log = nullptr;
    uint32_t* d_xr_rows = nullptr;            // [2P] row_lo | row_hi
    uint64_t* xr_log_of = nullptr;            // own log the peers were given (re-exchange on change)
    unsigned long long xr_cap = 0;
    int xr_depth = 0;
    void* comm_row = nullptr;                 // NCCL sub-communicators of the grid row / column
    void* comm_col = nullptr;
    uint32_t* d_stage = nullptr;              // 2-D block exchange staging
    unsigned long long* d_scan_tot = nullptr; // fused seeding: per-CTA totals of the adjacency scan
    size_t stage_cap = 0;
    int32_t n_ranks = 1;                      // row-block shards (NCCL ranks or emulated)
    int32_t my_rank = 0;
    bool emulated = false;
    void* comm = nullptr;                     // ncclComm_t (world_size > 1)
    uint64_t* d_xbuf = nullptr;               // sparse sharding: Δ exchange buffer [ranks * max count]
    size_t xbuf_cap = 0;
    std::vector<int64_t> shard_new;           // sparse sharding: new cells per (iteration, rank), diagnostics
    int64_t rows_alloc = 0;                   // bit-matrix rows allocated (>= n, multiple of blocks)
    int64_t block_rows = 0;                   // rows per shard block (dense engine)
    int32_t* d_rowcnt = nullptr;              // bitmap extraction scratch [n+1]
    int32_t* d_rowoff = nullptr;
    int64_t* d_csr_ptr = nullptr;             // CSR row pointers for a host destination [n+1]
    cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
    cudaEvent_t pipe_ev[2] = {nullptr, nullptr};   // pipelined bit-row iterations
    double seed_ns = 0, loop_ns = 0;

    // second workspace bank (see Bank)
    Bank spare;
    bool have_spare = false, spare_failed = false;
    cudaStream_t side = nullptr;
    cudaEvent_t spare_clean = nullptr, main_done = nullptr;
    // in-kernel clear of the other bank (closure kernel, barrier idle time)
    bool clr_active = false;
    bool t_clean = false;                     // the last run reset its bit words (self_clear)
    const uint64_t* clr_log = nullptr;
    unsigned long long clr_n = 0;
    const NTInfo* clr_nt = nullptr;
    uint32_t *clr_rowc = nullptr, *clr_colc = nullptr;

    ~cfpq_result() {
        if (side) cudaStreamSynchronize(side);
        spare.release();
        if (side) cudaStreamDestroy(side);
        if (spare_clean) cudaEventDestroy(spare_clean);
        if (main_done) cudaEventDestroy(main_done);
        for (auto& e : ev)
            if (e) cudaEventDestroy(e);
        for (auto& e : pipe_ev)
            if (e) cudaEventDestroy(e);
        dfree(d_T); dfree(d_snap); dfree(d_K); dfree(d_nt); dfree(d_exps); dfree(d_rules);
        dfree(d_lab_ptr); dfree(d_lab_nt); dfree(d_slot_row); dfree(d_slot_col); dfree(d_adj_cnt);
        dfree(d_adj_ptr); dfree(d_adj_cursor); dfree(d_adj_idx); dfree(d_adj_ell); dfree(d_log); dfree(d_st);
        dfree(d_iter_off); dfree(d_jac); dfree(d_iter_time); dfree(d_phase); dfree(d_hset); dfree(d_xbuf); dfree(d_rowc); dfree(d_colc); dfree(d_temp); dfree(d_keys);
        dfree(d_small); dfree(d_Tn); dfree(d_rowcnt); dfree(d_rowoff); dfree(d_csr_ptr);
        if (dense) dense_destroy(dense);
        dfree(d_stage);
        dfree(d_scan_tot);
        for (void* q : xr_opened) cudaIpcCloseMemHandle(q);
        for (void* q : xr_owned) cudaFree(q);
        dfree(d_xr_st); dfree(d_xr_log); dfree(d_xr_rows);
        if (comm_row) nccl_comm_destroy(comm_row);
        if (comm_col) nccl_comm_destroy(comm_col);
        if (comm) nccl_comm_destroy(comm);
    }

    // relational sparse runs on one GPU keep their results in the log only, so the closure
    // kernel can reset the bit words at the fixpoint (flags bit 2 disables, diagnostics)
    // Who clears a relational run's bit words for the next run.  One GPU: by default the next
    // run switches to the other workspace bank and its closure kernel clears this bank's
    // cells while its CTAs wait at grid barriers (config 4: 0.532 vs 0.564 ms per step with
    // the reset at the fixpoint), so this run leaves its words; without a second bank (or
    // with diag_flags bit 7) the kernel resets them at the fixpoint instead.  The peer-memory
    // and asynchronous kernels always reset at the end (they have no bank rotation).
    bool self_clear_ok() const {
        if (!(opts.semantics == 0 && !hashed && opts.path_policy < 2 && (opts.diag_flags & 4) == 0)) return false;
        if (xr || opts.schedule == 2) return true;
        if (n_ranks != 1 || comm) return false;
        return spare_failed || (opts.diag_flags & 128) != 0;
    }

    EngineParams params() const {
        EngineParams p{};
        p.n = (int32_t)n;
        p.n_nt = n_nt;
        p.Wp = Wp;
        p.nt = d_nt;
        p.exps = d_exps;
        p.n_exps = n_exps;
        p.adj_idx = d_adj_idx;
        p.adj_cap = adj_idx_cap;
        p.log = d_log;
        p.log_cap = log_cap;
        p.st = d_st;
        p.iter_off = d_iter_off;
        p.iter_off_cap = iter_off_cap;
        p.jac = opts.account_work ? d_jac : nullptr;
        p.iter_time = opts.record_times ? d_iter_time : nullptr;
        p.phase = opts.record_times ? d_phase : nullptr;
        p.rowc = opts.account_work ? d_rowc : nullptr;
        p.colc = opts.account_work ? d_colc : nullptr;
        p.rules = d_rules;
        p.n_rules = (int32_t)rules.size();
        p.lengths = opts.semantics == 1;
        p.max_iter = opts.max_iterations;
        p.solo_max = opts.solo_threshold;
        p.has_snapshots = has_snapshots;
        p.nblocks = grid;
        p.profile = opts.record_times;
        p.gs_stages = opts.schedule == 3 ? n_stages : 0;
        p.switch_cells = opts.schedule == 3 ? 0 : switch_cells;   // Gauss-Seidel stays sparse
        // read a candidate's bit before its atomicOr (skips the RMW on already-set words;
        // config 4: 0.611 vs 0.623 ms per step); flags bit 0 disables (diagnostics)
        p.precheck = (opts.diag_flags & 1) ? 0 : 1;
        p.self_clear = self_clear_ok() ? 1 : 0;
        p.warp_flush = (opts.diag_flags & 8) ? 0 : 1;   // bit 3: the CTA-level flush (round 1 default)
        p.cta_major = (opts.diag_flags & 256) ? 1 : 0;
        p.no_chain = (opts.diag_flags & (1 << 13)) ? 1 : 0;
        p.row_lo = 0;
        p.row_hi = (uint32_t)n;
        p.clr_n = clr_active ? clr_n : 0;
        p.clr_log = clr_log;
        p.clr_nt = clr_nt;
        p.clr_rowc = clr_rowc;
        p.clr_colc = clr_colc;
        p.hset = hashed ? d_hset : nullptr;
        p.hmask = hashed ? hcap - 1 : 0;
        int lg = 0;
        while (hashed && (1ull << lg) < hcap) ++lg;
        p.hshift = 64 - lg;
        return p;
    }
};

// ------------------------------------------------------------------------------------------
// grammar / graph
// ------------------------------------------------------------------------------------------
extern "C" cfpq_status cfpq_grammar_create(int32_t n_nt, int32_t n_labels, const int32_t* bin, int64_t n_bin,
                                           const int32_t* term, int64_t n_term, cfpq_grammar** out) {
    CFPQ_CHECK_ARG(out != nullptr, "cfpq_grammar_create: out is NULL");
    CFPQ_CHECK_ARG(n_nt >= 1 && n_nt <= kMaxNT, "cfpq_grammar_create: n_nt must be in [1, 1024]");
    CFPQ_CHECK_ARG(n_labels >= 0, "cfpq_grammar_create: n_labels < 0");
    CFPQ_CHECK_ARG(n_bin >= 0 && n_term >= 0, "cfpq_grammar_create: negative rule count");
    CFPQ_CHECK_ARG(n_bin == 0 || bin != nullptr, "cfpq_grammar_create: bin is NULL");
    CFPQ_CHECK_ARG(n_term == 0 || term != nullptr, "cfpq_grammar_create: term is NULL");
    std::set<std::tuple<int, int, int>> rs;
    for (int64_t k = 0; k < n_bin; ++k) {
        int A = bin[3 * k], B = bin[3 * k + 1], C = bin[3 * k + 2];
        CFPQ_CHECK_ARG(A >= 0 && A < n_nt && B >= 0 && B < n_nt && C >= 0 && C < n_nt,
                       "cfpq_grammar_create: binary rule id out of range");
        rs.insert(std::make_tuple(A, B, C));
    }
    std::set<std::pair<int, int>> ts;
    for (int64_t k = 0; k < n_term; ++k) {
        int A = term[2 * k], x = term[2 * k + 1];
        CFPQ_CHECK_ARG(A >= 0 && A < n_nt && x >= 0 && x < n_labels,
                       "cfpq_grammar_create: terminal rule id out of range");
        ts.insert(std::make_pair(A, x));
    }
    cfpq_grammar* g = new cfpq_grammar();
    g->n_nt = n_nt;
    g->n_labels = n_labels;
    for (auto& t : rs) g->rules.push_back(Rule3{std::get<0>(t), std::get<1>(t), std::get<2>(t)});
    for (auto& t : ts) g->term.push_back(t);
    g->is_const.assign(n_nt, 1);
    for (auto& r : g->rules) g->is_const[r.A] = 0;
    *out = g;
    return CFPQ_OK;
}

extern "C" void cfpq_grammar_destroy(cfpq_grammar* g) { delete g; }

static cfpq_status upload_edges(cfpq_graph* g, const int32_t* edges, int64_t n_edges, int32_t on_device,
                                cudaStream_t s) {
    CFPQ_CHECK_ARG(n_edges >= 0, "edges: n_edges < 0");
    CFPQ_CHECK_ARG(n_edges == 0 || edges != nullptr, "edges: NULL pointer");
    // ranges are validated on the device by the seed kernel (cfpq_closure -> CFPQ_E_INVAL),
    // for host and device input alike: no O(|E|) host pass on the per-query upload path
    if (n_edges > g->cap_edges) {
        dfree(g->d_edges);
        int64_t cap = std::max<int64_t>(n_edges, 1);
        cfpq_status st = dalloc(&g->d_edges, (size_t)cap * 3, "edges");
        if (st != CFPQ_OK) return st;
        g->cap_edges = cap;
    }
    if (n_edges > 0)
        CFPQ_CUDA_TRY(cudaMemcpyAsync(g->d_edges, edges, (size_t)n_edges * 3 * sizeof(int32_t),
                                      on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, s));
    // asynchronous on `s` for device and page-locked host input (cfpq.h: the caller keeps the
    // buffer until the stream passes the copy; cfpq_closure synchronises it); pageable host
    // memory is staged by the runtime before cudaMemcpyAsync returns
    g->n_edges = n_edges;
    return CFPQ_OK;
}

extern "C" cfpq_status cfpq_graph_create(int64_t n_nodes, const int32_t* edges, int64_t n_edges,
                                         int32_t edges_on_device, void* cuda_stream, cfpq_graph** out) {
    CFPQ_CHECK_ARG(out != nullptr, "cfpq_graph_create: out is NULL");
    CFPQ_CHECK_ARG(n_nodes >= 0 && n_nodes < (int64_t(1) << kNodeBits), "cfpq_graph_create: n_nodes out of range");
    cfpq_graph* g = new cfpq_graph();
    g->n_nodes = n_nodes;
    cfpq_status st = upload_edges(g, edges, n_edges, edges_on_device, (cudaStream_t)cuda_stream);
    if (st != CFPQ_OK) {
        dfree(g->d_edges);
        delete g;
        return st;
    }
    *out = g;
    return CFPQ_OK;
}

extern "C" cfpq_status cfpq_graph_set_edges(cfpq_graph* g, const int32_t* edges, int64_t n_edges,
                                            int32_t edges_on_device, void* cuda_stream) {
    CFPQ_CHECK_ARG(g != nullptr, "cfpq_graph_set_edges: graph is NULL");
    return upload_edges(g, edges, n_edges, edges_on_device, (cudaStream_t)cuda_stream);
}

extern "C" void cfpq_graph_destroy(cfpq_graph* g) {
    if (!g) return;
    dfree(g->d_edges);
    delete g;
}

extern "C" void cfpq_options_default(cfpq_options* o) {
    if (!o) return;
    memset(o, 0, sizeof(*o));
    o->world_size = 1;
    o->solo_threshold = -1;
}

// Create the dense engine and the second bit-matrix buffer of its outputs (at plan time
// for path_policy 2, at the first switch for the auto policy).
static cfpq_status ensure_dense(cfpq_result* r) {
    if (r->dense) return CFPQ_OK;
    std::string err;
    r->dense = dense_create((int32_t)r->n, r->n_nt, r->Wp, r->rules, r->is_const, r->stream, &err,
                            r->opts.path_policy != 3, r->opts.tensor_format != 1, r->opts.rows_list_capacity,
                            r->opts.dense_launch);
    if (!r->dense) {
        set_error(err);
        return CFPQ_E_CUDA;
    }
    dense_set_rgather_variant(r->dense, (r->opts.diag_flags >> 4) & 7);
    const size_t mat_words = (size_t)r->rows_alloc * (size_t)r->Wp;
    int n_out = (int)dense_outputs(r->dense).size();
    cfpq_status st = dalloc(&r->d_Tn, mat_words * std::max(n_out, 1), "dense next bit matrices");
    if (st != CFPQ_OK) return st;
    CFPQ_CUDA_TRY(cudaMemsetAsync(r->d_Tn, 0, mat_words * std::max(n_out, 1) * 4, r->stream));
    return CFPQ_OK;
}

static void swap_with(cfpq_result* r, Bank& b) {
    std::swap(r->d_T, b.d_T);
    std::swap(r->d_snap, b.d_snap);
    std::swap(r->d_K, b.d_K);
    std::swap(r->d_nt, b.d_nt);
    std::swap(r->d_log, b.d_log);
    std::swap(r->log_cap, b.log_cap);
    std::swap(r->n_cells, b.n_cells);
    std::swap(r->d_rowc, b.d_rowc);
    std::swap(r->d_colc, b.d_colc);
    std::swap(r->d_hset, b.d_hset);
    std::swap(r->hcap, b.hcap);
    std::swap(r->h_nt, b.h_nt);
    std::swap(r->Tbase, b.Tbase);
}

// Allocate the second bank with the same shapes as the current one (zeroed bitmaps, EMPTY
// keys).  Returns false (and the result keeps one bank) if the memory is not there.
static bool make_spare(cfpq_result* r) {
    Bank& b = r->spare;
    const size_t mw = (size_t)r->rows_alloc * (size_t)r->Wp;
    int n_snap = 0, n_key = 0;
    for (auto& t : r->h_nt) {
        n_snap += (t.S ? 1 : 0) + (t.ST ? 1 : 0);
        n_key += t.K ? 1 : 0;
    }
    auto ok = [](cudaError_t e) {
        if (e != cudaSuccess) cudaGetLastError();
        return e == cudaSuccess;
    };
    cudaStream_t s = r->stream;
    bool good = true;
    if (r->hashed)
        good = ok(cudaMalloc(&b.d_hset, r->hcap * 8)) && ok(cudaMemsetAsync(b.d_hset, 0xff, r->hcap * 8, s));
    else
        good = ok(cudaMalloc(&b.d_T, mw * r->n_nt * 4)) && ok(cudaMemsetAsync(b.d_T, 0, mw * r->n_nt * 4, s));
    if (good && n_snap) good = ok(cudaMalloc(&b.d_snap, mw * n_snap * 4)) && ok(cudaMemsetAsync(b.d_snap, 0, mw * n_snap * 4, s));
    if (good && n_key)
        good = ok(cudaMalloc(&b.d_K, (size_t)r->n * r->n * n_key * 8)) &&
               ok(cudaMemsetAsync(b.d_K, 0xff, (size_t)r->n * r->n * n_key * 8, s));
    if (good) good = ok(cudaMalloc(&b.d_log, r->log_cap * 8)) && ok(cudaMemsetAsync(b.d_log, 0, r->log_cap * 8, s));
    if (good && r->d_rowc)
        good = ok(cudaMalloc(&b.d_rowc, (size_t)r->n_nt * r->n * 4)) && ok(cudaMalloc(&b.d_colc, (size_t)r->n_nt * r->n * 4)) &&
               ok(cudaMemsetAsync(b.d_rowc, 0, (size_t)r->n_nt * r->n * 4, s)) &&
               ok(cudaMemsetAsync(b.d_colc, 0, (size_t)r->n_nt * r->n * 4, s));
    if (good) good = ok(cudaMalloc(&b.d_nt, r->n_nt * sizeof(NTInfo)));
    if (!good) {
        b.release();
        return false;
    }
    b.log_cap = r->log_cap;
    b.hcap = r->hashed ? r->hcap : 0;
    b.n_cells = 0;
    b.h_nt = r->h_nt;
    b.Tbase.assign(r->n_nt, nullptr);
    int snap_i = 0, key_i = 0;
    for (int A = 0; A < r->n_nt; ++A) {
        NTInfo& t = b.h_nt[A];
        t.T = b.d_T ? b.d_T + (size_t)A * mw : nullptr;
        if (t.S) t.S = b.d_snap + (size_t)(snap_i++) * mw;
        if (t.ST) t.ST = b.d_snap + (size_t)(snap_i++) * mw;
        if (t.K) t.K = b.d_K + (size_t)(key_i++) * r->n * r->n;
        b.Tbase[A] = t.T;
    }
    if (!ok(cudaMemcpyAsync(b.d_nt, b.h_nt.data(), r->n_nt * sizeof(NTInfo), cudaMemcpyHostToDevice, s))) {
        b.release();
        return false;
    }
    if (!r->side && !ok(cudaStreamCreateWithFlags(&r->side, cudaStreamNonBlocking))) return false;
    if (!r->spare_clean && !ok(cudaEventCreateWithFlags(&r->spare_clean, cudaEventDisableTiming))) return false;
    if (!r->main_done && !ok(cudaEventCreateWithFlags(&r->main_done, cudaEventDisableTiming))) return false;
    return true;
}

// ------------------------------------------------------------------------------------------
// planning: per-NT tables, expansions, buffers
// ------------------------------------------------------------------------------------------
// Theorem 3: |V|^2 |N| changes at most -> |V|^2|N| + 1 loop bodies (max_iterations 0)
static long long theorem3_cap(int64_t n, int32_t n_nt) {
    double cap = (double)n * (double)n * (double)n_nt + 1.0;
    return cap > 4e18 ? (long long)4e18 : (long long)cap;
}

// Per-iteration buffers (offsets, timestamps, phases, Jacobi work) sized for the current
// cap (at most 2^22 recorded iterations); grown when a reuse raises the cap.
static cfpq_status size_iteration_buffers(cfpq_result* r) {
    const long long want = std::min<long long>(r->opts.max_iterations + 2, 1ll << 22);
    if (want <= r->iter_off_cap && r->d_iter_off && (!r->opts.account_work || r->d_jac)) return CFPQ_OK;
    const long long cap = std::max(want, r->iter_off_cap);
    dfree(r->d_iter_off);
    dfree(r->d_iter_time);
    dfree(r->d_phase);
    dfree(r->d_jac);
    r->iter_off_cap = 0;
    cfpq_status st;
    if ((st = dalloc(&r->d_iter_off, (size_t)cap, "iteration offsets")) != CFPQ_OK) return st;
    if ((st = dalloc(&r->d_iter_time, (size_t)cap, "iteration timestamps")) != CFPQ_OK) return st;
    if ((st = dalloc(&r->d_phase, (size_t)cap * 4, "iteration phases")) != CFPQ_OK) return st;
    if (r->opts.account_work && (st = dalloc(&r->d_jac, (size_t)cap, "work counts")) != CFPQ_OK) return st;
    r->iter_off_cap = cap;
    return CFPQ_OK;
}

static cfpq_status plan(cfpq_result* r, const cfpq_grammar* g, const cfpq_graph* d, const cfpq_options* o) {
    r->n = d->n_nodes;
    r->n_nt = g->n_nt;
    r->n_labels = g->n_labels;
    r->opts = *o;
    if (r->opts.max_iterations <= 0) r->opts.max_iterations = theorem3_cap(r->n, r->n_nt);
    if (r->opts.solo_threshold < 0) r->opts.solo_threshold = 1024;
    r->stream = (cudaStream_t)o->cuda_stream;
    r->rules = g->rules;
    r->term = g->term;
    const int64_t n = r->n;
    const int64_t wn = (n + 31) / 32;
    r->Wp = std::max<int64_t>(32, (wn + 31) / 32 * 32);

    // expansions per NT (see engine.cu header)
    std::vector<std::vector<Expansion>> ex(g->n_nt);
    std::vector<int> need_csr(g->n_nt, 0), need_csc(g->n_nt, 0), need_S(g->n_nt, 0), need_ST(g->n_nt, 0);
    for (auto& rl : g->rules) {
        bool bc = g->is_const[rl.B], cc = g->is_const[rl.C];
        if (!bc && !cc) {
            ex[rl.B].push_back(Expansion{EXP_L_VAR, rl.A, rl.C, 0});
            ex[rl.C].push_back(Expansion{EXP_R_VAR, rl.A, rl.B, 0});
            need_S[rl.C] = 1;
            need_ST[rl.B] = 1;
        } else if (!bc && cc) {
            ex[rl.B].push_back(Expansion{EXP_L_CONST, rl.A, rl.C, 0});
            need_csr[rl.C] = 1;
        } else if (bc && !cc) {
            // Δ_B = T_B at iteration 1 only, where T_B × Δ_C already equals T_B × T_C
            ex[rl.C].push_back(Expansion{EXP_R_CONST, rl.A, rl.B, 0});
            need_csc[rl.B] = 1;
        } else {
            // both preterminal: only iteration 1 (Δ_0 of B) contributes
            ex[rl.B].push_back(Expansion{EXP_L_CONST, rl.A, rl.C, 0});
            need_csr[rl.C] = 1;
        }
        // the bit-row path gathers rows i of a preterminal left operand from its CSR
        if (o->path_policy == 3 && bc) need_csr[rl.B] = 1;
    }
    // Gauss-Seidel (DESIGN reading c17): the LHS NTs in id order, each reading T as the
    // earlier LHS left it.  Consecutive LHS NTs that do not read each other's results share
    // one barrier step (level): level(s) = max over earlier t of level(t) + 1 if s reads t's
    // cells, and level(t) if t reads s's (so s still sees t's cells of this round and t does
    // not see s's) — the states per round are exactly those of the one-by-one order.
    std::vector<int32_t> stage_of(g->n_nt, -1);
    r->n_stages = 0;
    {
        std::vector<std::vector<char>> reads(g->n_nt, std::vector<char>(g->n_nt, 0));
        for (auto& rl : g->rules) reads[rl.A][rl.B] = reads[rl.A][rl.C] = 1;
        std::vector<int32_t> order;
        for (int A = 0; A < g->n_nt; ++A)
            if (!g->is_const[A]) order.push_back(A);
        for (size_t a = 0; a < order.size(); ++a) {
            const int sA = order[a];
            int lv = 0;
            for (size_t b = 0; b < a; ++b) {
                const int tA = order[b];
                if (reads[sA][tA]) lv = std::max(lv, stage_of[tA] + 1);
                if (reads[tA][sA]) lv = std::max(lv, stage_of[tA]);
            }
            stage_of[sA] = lv;
            r->n_stages = std::max(r->n_stages, lv + 1);
        }
    }
    for (auto& v : ex)
        for (auto& e : v) e.stage = stage_of[e.A];
    std::vector<Expansion> exps;
    r->h_nt.assign(g->n_nt, NTInfo{});
    for (int A = 0; A < g->n_nt; ++A) {
        r->h_nt[A].exp_begin = (int32_t)exps.size();
        for (auto& e : ex[A]) exps.push_back(e);
        r->h_nt[A].exp_end = (int32_t)exps.size();
        r->h_nt[A].is_const = g->is_const[A];
    }
    // terminal rules by label (CSR over labels)
    std::vector<int32_t> lab_ptr(g->n_labels + 1, 0), lab_nt;
    for (auto& t : g->term) lab_ptr[t.second + 1]++;
    for (int x = 0; x < g->n_labels; ++x) lab_ptr[x + 1] += lab_ptr[x];
    lab_nt.resize(g->term.size());
    {
        std::vector<int32_t> cur(lab_ptr.begin(), lab_ptr.end() - 1);
        for (auto& t : g->term) lab_nt[cur[t.second]++] = t.first;
    }
    r->max_rules_per_label = 0;
    for (int x = 0; x < g->n_labels; ++x)
        r->max_rules_per_label = std::max(r->max_rules_per_label, lab_ptr[x + 1] - lab_ptr[x]);

    cfpq_status st;
    // a communicator whenever an id is given (world_size 1 exercises the NCCL exchange path)
    const bool use_nccl = o->nccl_unique_id != nullptr;
    r->n_ranks = o->world_size > 1 ? o->world_size : (o->reserved_emulate > 1 ? o->reserved_emulate : 1);
    r->emulated = !use_nccl && r->n_ranks > 1;
    r->my_rank = o->world_size > 1 ? o->rank : 0;
    r->rows_alloc = n;
    if (o->path_policy == 2) {
        int64_t tlo, thi;
        dense_partition(n, r->n_ranks, 0, &tlo, &thi, &r->block_rows);
        r->rows_alloc = std::max<int64_t>(n, r->block_rows * r->n_ranks);
    }
    if (use_nccl) {
        std::string err;
        r->comm = nccl_comm_create(o->nccl_unique_id, r->n_ranks, r->my_rank, &err);
        (void)cudaGetLastError();   // NCCL's device probing may leave a non-sticky error behind
        if (!r->comm) {
            set_error(err);
            return CFPQ_E_NCCL;
        }
    }
    if (o->path_policy == 2 && o->grid_rows > 0 && o->grid_cols > 0) {
        r->grid_r = o->grid_rows;
        r->grid_c = o->grid_cols;
        if (r->comm) {
            std::string err;
            r->comm_row = nccl_comm_split(r->comm, r->my_rank / r->grid_c, r->my_rank % r->grid_c, &err);
            if (r->comm_row) r->comm_col = nccl_comm_split(r->comm, r->my_rank % r->grid_c, r->my_rank / r->grid_c, &err);
            if (!r->comm_row || !r->comm_col) {
                set_error(err);
                return CFPQ_E_NCCL;
            }
        }
    }
    r->xr = o->exchange == 1 && r->n_ranks > 1 && o->path_policy < 2;
    if (r->xr && r->n_ranks > kMaxXrRanks) {
        set_error("cfpq_closure: the peer-memory exchange supports at most 32 ranks");
        return CFPQ_E_UNSUPPORTED;
    }
    const size_t mat_words = (size_t)r->rows_alloc * (size_t)r->Wp;
    int n_snap = 0;
    for (int A = 0; A < g->n_nt; ++A) n_snap += need_S[A] + need_ST[A];
    // membership structure: the hashed cell set where nothing reads rows of T (relational,
    // sparse engine, no var x var rule), else the bit matrices
    const bool hash_ok = o->semantics == 0 && (o->path_policy == 0 || o->path_policy == 1) && n_snap == 0 &&
                         g->n_nt < kMaxNT;
    if (o->cell_set == 2 && !hash_ok) {
        set_error("cell_set = 2 (hashed) needs relational semantics, the sparse engine, |N| < 1024 and no rule "
                  "whose two operands both change");
        return CFPQ_E_UNSUPPORTED;
    }
    // auto: the bit matrices are faster where they fit (config 4: 0.40 vs 0.52 ms loop; the
    // hashed set halves DRAM traffic but the iteration is barrier/latency-bound), so the
    // hashed set is chosen when the matrices would take more than a quarter of free HBM
    bool want_hash = o->cell_set == 2;
    if (o->cell_set == 0 && hash_ok) {
        size_t free_b = 0, total_b = 0;
        CFPQ_CUDA_TRY(cudaMemGetInfo(&free_b, &total_b));
        want_hash = (double)mat_words * 4.0 * g->n_nt > 0.25 * (double)free_b;
    }
    r->hashed = hash_ok && want_hash && !r->xr;
    if (!r->hashed) {
        if ((st = dalloc(&r->d_T, mat_words * g->n_nt, "T bit matrices")) != CFPQ_OK) return st;
        CFPQ_CUDA_TRY(cudaMemsetAsync(r->d_T, 0, mat_words * g->n_nt * 4, r->stream));
    }
    r->has_snapshots = n_snap > 0;
    if (n_snap) {
        if ((st = dalloc(&r->d_snap, mat_words * n_snap, "snapshots")) != CFPQ_OK) return st;
        CFPQ_CUDA_TRY(cudaMemsetAsync(r->d_snap, 0, mat_words * n_snap * 4, r->stream));
    }
    bool lengths = o->semantics == 1;
    int n_key = 0;
    if (lengths)
        for (int A = 0; A < g->n_nt; ++A) n_key += g->is_const[A] ? 0 : 1;
    if (n_key) {
        if ((st = dalloc(&r->d_K, (size_t)n * n * n_key, "single-path keys")) != CFPQ_OK) return st;
        CFPQ_CUDA_TRY(cudaMemsetAsync(r->d_K, 0xff, (size_t)n * n * n_key * 8, r->stream));
    }
    // adjacency slots
    std::vector<int32_t> slot_row(g->n_nt, -1), slot_col(g->n_nt, -1);
    int slots = 0;
    for (int A = 0; A < g->n_nt; ++A) {
        if (need_csr[A]) slot_row[A] = slots++;
        if (need_csc[A]) slot_col[A] = slots++;
    }
    r->n_adj_slots = slots;
    const size_t adj_len = (size_t)slots * (size_t)(n + 1);
    if ((st = dalloc(&r->d_adj_cnt, adj_len, "adjacency counts")) != CFPQ_OK) return st;
    if ((st = dalloc(&r->d_adj_ptr, adj_len + 1, "adjacency pointers")) != CFPQ_OK) return st;
    if ((st = dalloc(&r->d_adj_ell, (size_t)slots * n, "adjacency ELL heads")) != CFPQ_OK) return st;
    if ((st = dalloc(&r->d_slot_row, g->n_nt, "slots")) != CFPQ_OK) return st;
    if ((st = dalloc(&r->d_slot_col, g->n_nt, "slots")) != CFPQ_OK) return st;
    CFPQ_CUDA_TRY(cudaMemcpyAsync(r->d_slot_row, slot_row.data(), g->n_nt * 4, cudaMemcpyHostToDevice, r->stream));
    CFPQ_CUDA_TRY(cudaMemcpyAsync(r->d_slot_col, slot_col.data(), g->n_nt * 4, cudaMemcpyHostToDevice, r->stream));

    // per-NT pointers
    int snap_i = 0, key_i = 0;
    for (int A = 0; A < g->n_nt; ++A) {
        NTInfo& t = r->h_nt[A];
        t.T = r->d_T ? r->d_T + (size_t)A * mat_words : nullptr;
        t.S = need_S[A] ? r->d_snap + (size_t)(snap_i++) * mat_words : nullptr;
        t.ST = need_ST[A] ? r->d_snap + (size_t)(snap_i++) * mat_words : nullptr;
        t.K = (lengths && !g->is_const[A]) ? r->d_K + (size_t)(key_i++) * n * n : nullptr;
        t.csr_ptr = slot_row[A] >= 0 ? r->d_adj_ptr + (size_t)slot_row[A] * (n + 1) : nullptr;
        t.csc_ptr = slot_col[A] >= 0 ? r->d_adj_ptr + (size_t)slot_col[A] * (n + 1) : nullptr;
        t.csr_ell = slot_row[A] >= 0 ? r->d_adj_ell + (size_t)slot_row[A] * n : nullptr;
        t.csc_ell = slot_col[A] >= 0 ? r->d_adj_ell + (size_t)slot_col[A] * n : nullptr;
        t.needs_snapshot = (t.S || t.ST) ? 1 : 0;
    }
    if ((st = dalloc(&r->d_nt, g->n_nt, "NT table")) != CFPQ_OK) return st;
    CFPQ_CUDA_TRY(cudaMemcpyAsync(r->d_nt, r->h_nt.data(), g->n_nt * sizeof(NTInfo), cudaMemcpyHostToDevice, r->stream));
    r->n_exps = (int32_t)exps.size();
    if ((st = dalloc(&r->d_exps, exps.size(), "expansions")) != CFPQ_OK) return st;
    if (!exps.empty())
        CFPQ_CUDA_TRY(cudaMemcpyAsync(r->d_exps, exps.data(), exps.size() * sizeof(Expansion), cudaMemcpyHostToDevice,
                                      r->stream));
    if ((st = dalloc(&r->d_rules, g->rules.size() * 3, "rules")) != CFPQ_OK) return st;
    if (!g->rules.empty())
        CFPQ_CUDA_TRY(cudaMemcpyAsync(r->d_rules, g->rules.data(), g->rules.size() * sizeof(Rule3),
                                      cudaMemcpyHostToDevice, r->stream));
    if ((st = dalloc(&r->d_lab_ptr, lab_ptr.size(), "label table")) != CFPQ_OK) return st;
    if ((st = dalloc(&r->d_lab_nt, lab_nt.size(), "label table")) != CFPQ_OK) return st;
    CFPQ_CUDA_TRY(cudaMemcpyAsync(r->d_lab_ptr, lab_ptr.data(), lab_ptr.size() * 4, cudaMemcpyHostToDevice, r->stream));
    if (!lab_nt.empty())
        CFPQ_CUDA_TRY(cudaMemcpyAsync(r->d_lab_nt, lab_nt.data(), lab_nt.size() * 4, cudaMemcpyHostToDevice, r->stream));

    if ((st = dalloc(&r->d_st, 1, "state")) != CFPQ_OK) return st;
    if ((st = size_iteration_buffers(r)) != CFPQ_OK) return st;
    if (o->account_work) {
        if ((st = dalloc(&r->d_rowc, (size_t)g->n_nt * n, "row counts")) != CFPQ_OK) return st;
        if ((st = dalloc(&r->d_colc, (size_t)g->n_nt * n, "col counts")) != CFPQ_OK) return st;
        CFPQ_CUDA_TRY(cudaMemsetAsync(r->d_rowc, 0, (size_t)g->n_nt * n * 4, r->stream));
        CFPQ_CUDA_TRY(cudaMemsetAsync(r->d_colc, 0, (size_t)g->n_nt * n * 4, r->stream));
    }
    if ((st = dalloc(&r->d_small, (size_t)g->n_nt + 2, "counters")) != CFPQ_OK) return st;
    // temp storage for the adjacency scan (and later radix sorts)
    size_t tb = 0;
    CFPQ_CUDA_TRY(launch_scan(nullptr, nullptr, (int64_t)adj_len + 1, nullptr, &tb, r->stream));
    r->temp_bytes = std::max<size_t>(tb, 1 << 16);
    if ((st = dalloc((uint8_t**)&r->d_temp, r->temp_bytes, "temp")) != CFPQ_OK) return st;

    r->Tbase.assign(g->n_nt, nullptr);
    for (int A = 0; A < g->n_nt; ++A) r->Tbase[A] = r->h_nt[A].T;
    r->is_const = g->is_const;
    if (o->path_policy == 2 || o->path_policy == 3) {
        if ((st = ensure_dense(r)) != CFPQ_OK) return st;
    } else if (o->path_policy == 0 && o->semantics == 0) {
        // auto: rules whose two operands both change are row scans for the sparse engine;
        // once |Δ| is dense (> n^2/256 cells, at least 4096) the tcgen05 engine takes over
        bool varvar = false;
        for (auto& rl : g->rules) varvar |= !g->is_const[rl.B] && !g->is_const[rl.C];
        if (varvar) r->switch_cells = std::max<unsigned long long>(4096ull, (unsigned long long)n * n / 256);
    }
    if ((st = dalloc(&r->d_rowcnt, (size_t)n + 1, "row counts")) != CFPQ_OK) return st;
    if ((st = dalloc(&r->d_rowoff, (size_t)n + 1, "row offsets")) != CFPQ_OK) return st;
    int dev = 0, sms = 0;
    CFPQ_CUDA_TRY(cudaGetDevice(&dev));
    CFPQ_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    int bps = closure_kernel_blocks_per_sm();
    if (bps <= 0) {
        set_error("closure kernel cannot be resident (occupancy 0)");
        return CFPQ_E_CUDA;
    }
    r->grid = sms * bps;
    if (o->max_ctas > 0 && o->max_ctas < r->grid) r->grid = o->max_ctas;
    return CFPQ_OK;
}

// Hashed cell set capacity: a power of two >= 2 x the log capacity (load <= 1/2 while the
// log does not overflow).  A new table starts empty.
static cfpq_status ensure_hash(cfpq_result* r) {
    unsigned long long want = 1ull << 10;
    while (want < 2 * r->log_cap) want <<= 1;
    if (r->hcap >= want) return CFPQ_OK;
    dfree(r->d_hset);
    r->hcap = 0;
    cfpq_status st = dalloc(&r->d_hset, want, "hashed cell set");
    if (st != CFPQ_OK) return st;
    r->hcap = want;
    CFPQ_CUDA_TRY(cudaMemsetAsync(r->d_hset, 0xff, want * 8, r->stream));
    return CFPQ_OK;
}

// Make sure the log and adjacency arrays can hold this graph's seeds.
static cfpq_status size_for_graph(cfpq_result* r, const cfpq_graph* d) {
    const int64_t seeds_upper = d->n_edges * (int64_t)std::max(r->max_rules_per_label, 0);
    unsigned long long want = r->opts.log_capacity > 0 ? (unsigned long long)r->opts.log_capacity
                                                       : std::max<unsigned long long>(1ull << 22, 4ull * seeds_upper);
    want = std::max<unsigned long long>(want, (unsigned long long)seeds_upper + 64ull);
    if (want > r->log_cap) {
        // keep the old content: a reused result clears its previous cells from the log
        uint64_t* nl = nullptr;
        cfpq_status st = dalloc(&nl, want, "cell log");
        if (st != CFPQ_OK) return st;
        CFPQ_CUDA_TRY(cudaMemsetAsync(nl, 0, want * 8, r->stream));   // no stale async flags
        if (r->d_log && r->n_cells)
            CFPQ_CUDA_TRY(cudaMemcpyAsync(nl, r->d_log, r->n_cells * 8, cudaMemcpyDeviceToDevice, r->stream));
        dfree(r->d_log);
        r->d_log = nl;
        r->log_cap = want;
    }
    if (r->hashed) {
        cfpq_status st = ensure_hash(r);
        if (st != CFPQ_OK) return st;
    }
    int64_t adj_want = std::max<int64_t>(2 * seeds_upper, 1);
    if (adj_want > r->adj_idx_cap) {
        dfree(r->d_adj_idx);
        cfpq_status st = dalloc(&r->d_adj_idx, (size_t)adj_want, "adjacency index");
        if (st != CFPQ_OK) return st;
        r->adj_idx_cap = adj_want;
    }
    return CFPQ_OK;
}

// `valid` = entries of the log that hold cells (default: the prefix below min(reached, cap)).
static cfpq_status grow_log(cfpq_result* r, unsigned long long reached, unsigned long long valid = ~0ull) {
    unsigned long long want = std::max<unsigned long long>(2 * r->log_cap, reached + reached / 4 + 1024);
    uint64_t* nl = nullptr;
    cfpq_status st = dalloc(&nl, want, "cell log (grow)");
    if (st != CFPQ_OK) return st;
    CFPQ_CUDA_TRY(cudaMemcpyAsync(nl, r->d_log, r->log_cap * 8, cudaMemcpyDeviceToDevice, r->stream));
    CFPQ_CUDA_TRY(cudaMemsetAsync(nl + r->log_cap, 0, (want - r->log_cap) * 8, r->stream));
    CFPQ_CUDA_TRY(cudaStreamSynchronize(r->stream));
    const unsigned long long old_cap = r->log_cap;
    dfree(r->d_log);
    r->d_log = nl;
    r->log_cap = want;
    r->regrows++;
    if (r->hashed) {
        // rebuild the table from the log's valid prefix: drops the cells that were inserted
        // but did not fit the log (the re-run of the iteration rediscovers them)
        dfree(r->d_hset);
        r->hcap = 0;
        cfpq_status st2 = ensure_hash(r);
        if (st2 != CFPQ_OK) return st2;
        const bool async = r->opts.schedule == 2;   // async entries carry a valid flag (bit 63)
        valid = std::min<unsigned long long>(valid, std::min<unsigned long long>(reached, old_cap));
        CFPQ_CUDA_TRY(launch_rehash(r->params(), valid, async ? ~(1ull << 63) : ~0ull, async ? 1 : 0, r->stream));
    }
    return CFPQ_OK;
}

// One row-block sharded iteration of the bit-row engine (§8(e); "matrix multiplication
// in the main loop ... may be performed on different GPGPU independently").  Every rank holds
// full replicas of T_{k-1} and T_k and derives the rows it owns (cfpq_shard_rows); the Δ_k
// word lists {A, i, word, bits} of the ranks are exchanged — all-gather of the counts, padded
// all-gather of the words, compaction in rank order — and every rank applies all of them to
// its T_k (the new-cell total, Alg. 1 line 8's "changed", counts the bits they flip).  Emulated
// ranks (one process) run the shards one after another on the shared buffers and pass their
// lists through the same padded buffer and compaction.
static cfpq_status rows_sharded_iteration(cfpq_result* r, bool first, int* launches) {
    cudaStream_t s = r->stream;
    DenseEngine* e = r->dense;
    const int P = r->n_ranks;
    CFPQ_CUDA_TRY(rows_begin(e, r->d_nt, r->d_adj_idx, r->d_log, r->n_cells, first, s, launches));
    const int g_begin = r->emulated ? 0 : r->my_rank, g_end = r->emulated ? P : r->my_rank + 1;
    std::vector<unsigned long long> cnt(P, 0);
    unsigned long long end = 0;
    for (int g = g_begin; g < g_end; ++g) {
        int64_t tlo, thi, br;
        dense_partition(r->n, P, g, &tlo, &thi, &br);
        const int64_t lo = std::min<int64_t>(tlo * 128, r->n), hi = std::min<int64_t>(thi * 128, r->n);
        unsigned long long m = 0;
        for (bool redo = true; redo;) {   // a chunk-list overflow re-runs the shard (grown lists)
            CFPQ_CUDA_TRY(rows_shard(e, lo, hi, s, launches));
            CFPQ_CUDA_TRY(rows_list_settle(e, lo, hi, end, s, &m));
            CFPQ_CUDA_TRY(rows_shard_check(e, s, &redo, false));
        }
        cnt[g] = m - end;
        end = m;
    }
    // exchange buffer: P slots of the largest list (2 uint64 per word)
    auto ensure_x = [&](size_t want) -> cfpq_status {
        if (r->xbuf_cap >= want) return CFPQ_OK;
        dfree(r->d_xbuf);
        r->xbuf_cap = 0;
        cfpq_status st = dalloc(&r->d_xbuf, want, "exchange buffer");
        if (st == CFPQ_OK) r->xbuf_cap = want;
        return st;
    };
    cfpq_status st;
    if (r->comm) {
        if ((st = ensure_x((size_t)P * 64)) != CFPQ_OK) return st;
        uint64_t mine = cnt[r->my_rank];
        CFPQ_CUDA_TRY(cudaMemcpyAsync(r->d_xbuf + r->my_rank, &mine, 8, cudaMemcpyHostToDevice, s));
        std::string err;
        if (!nccl_allgather_u64(r->comm, r->d_xbuf, 1, r->my_rank, s, &err)) {
            set_error(err);
            return CFPQ_E_NCCL;
        }
        std::vector<uint64_t> hc(P);
        CFPQ_CUDA_TRY(cudaMemcpyAsync(hc.data(), r->d_xbuf, 8 * P, cudaMemcpyDeviceToHost, s));
        CFPQ_CUDA_TRY(cudaStreamSynchronize(s));
        for (int g = 0; g < P; ++g) cnt[g] = hc[g];
    }
    unsigned long long tot = 0, mx = 0;
    for (int g = 0; g < P; ++g) {
        tot += cnt[g];
        mx = std::max(mx, cnt[g]);
    }
    void* list = nullptr;
    unsigned long long cap = 0;
    CFPQ_CUDA_TRY(rows_list(e, 0, &list, &cap));
    if ((st = ensure_x((size_t)P * std::max<unsigned long long>(2 * mx, 64))) != CFPQ_OK) return st;
    const size_t slot = (size_t)2 * mx;   // uint64 per rank slot
    {
        unsigned long long off = 0;
        for (int g = g_begin; g < g_end; ++g) {
            if (cnt[g])
                CFPQ_CUDA_TRY(cudaMemcpyAsync(r->d_xbuf + g * slot, (const uint4*)list + off, cnt[g] * 16,
                                              cudaMemcpyDeviceToDevice, s));
            off += cnt[g];
        }
    }
    if (r->comm && mx) {
        std::string err;
        if (!nccl_allgather_u64(r->comm, r->d_xbuf, slot, r->my_rank, s, &err)) {
            set_error(err);
            return CFPQ_E_NCCL;
        }
    }
    CFPQ_CUDA_TRY(cudaStreamSynchronize(s));   // the old list may be replaced below
    CFPQ_CUDA_TRY(rows_list(e, tot, &list, &cap));
    {
        unsigned long long off = 0;
        for (int g = 0; g < P; ++g) {
            if (cnt[g])
                CFPQ_CUDA_TRY(cudaMemcpyAsync((uint4*)list + off, r->d_xbuf + g * slot, cnt[g] * 16,
                                              cudaMemcpyDeviceToDevice, s));
            off += cnt[g];
        }
    }
    CFPQ_CUDA_TRY(rows_apply_all(e, tot, s, launches));
    return CFPQ_OK;
}

// 2-D (SUMMA-style) block sharding of the tensor engine ("|N|^2
// Boolean matrix multiplications", P:572 products "performed on different GPGPU").  The shards
// form a grid_r x grid_c grid; shard (a, b) derives block (I_a, J_b) of every T_A:
//     T_k,A[I_a, J_b] = T_{k-1},A[I_a, J_b] ∪ ⋃_{A->BC} T_{k-1},B[I_a, :] × T_{k-1},C[:, J_b]
// so it reads the row panel I_a of left operands and the column panel J_b of right operands.
// After the products the blocks travel along the grid: the row group (a, *) all-gathers its
// blocks (row panel I_a of T_k), the column group (*, b) all-gathers its blocks (column panel
// J_b), each through a contiguous staging buffer; the new-cell counts are summed over all
// shards (Alg. 1 line 8's "changed").  Per iteration a shard receives n/grid_r x n +
// n x n/grid_c bits per output instead of the 1-D all-gather's n x n.  Emulated shards (one
// process) share the matrices, so their blocks go through the staging buffer as identity
// copies.  At the fixpoint one world all-gather of the blocks makes every T_A whole again.
static cfpq_status grid_exchange(cfpq_result* r, bool final_gather) {
    cudaStream_t s = r->stream;
    const auto& outs = dense_outputs(r->dense);
    const int gr = r->grid_r, gc = r->grid_c, P = gr * gc;
    const int64_t Wp = r->Wp;
    std::vector<int64_t> ti_lo(P), ti_hi(P), tj_lo(P), tj_hi(P);
    int64_t max_rows = 0, max_words = 0;
    for (int g = 0; g < P; ++g) {
        dense_partition2(r->n, gr, gc, g / gc, g % gc, &ti_lo[g], &ti_hi[g], &tj_lo[g], &tj_hi[g]);
        max_rows = std::max(max_rows, (ti_hi[g] - ti_lo[g]) * 128);
        max_words = std::max(max_words, (tj_hi[g] - tj_lo[g]) * 8);
    }
    const int64_t n_out = (int64_t)outs.size();
    auto rows_of = [&](int g, int64_t* lo, int64_t* hi) {
        *lo = std::min<int64_t>(ti_lo[g] * 128, r->n);
        *hi = std::min<int64_t>(ti_hi[g] * 128, r->n);
    };
    auto words_of = [&](int g, int64_t* lo, int64_t* hi) {
        const int64_t wn = (r->n + 31) / 32;
        *lo = std::min<int64_t>(tj_lo[g] * 8, wn);
        *hi = std::min<int64_t>(tj_hi[g] * 8, wn);
    };
    const size_t slot = (size_t)max_rows * max_words * n_out;   // uint32 per shard block (all outputs)
    const size_t want = slot * (size_t)std::max(P, 1);
    if (r->stage_cap < want) {
        dfree(r->d_stage);
        r->stage_cap = 0;
        cfpq_status st = dalloc(&r->d_stage, want, "2-D exchange staging");
        if (st != CFPQ_OK) return st;
        r->stage_cap = want;
    }
    // pack / unpack shard g's block of every output at staging slot `at`
    auto pack = [&](int g, size_t at, int to_buf) -> cudaError_t {
        int64_t rl, rh, wl, wh;
        rows_of(g, &rl, &rh);
        words_of(g, &wl, &wh);
        for (int64_t q = 0; q < n_out; ++q) {
            uint32_t* T = r->Tnxt[outs[q]];
            cudaError_t e = bit_block_copy(T, Wp, rl, rh, wl, wh, r->d_stage + at * slot + (size_t)q * max_rows * max_words,
                                           to_buf, s);
            if (e != cudaSuccess) return e;
        }
        return cudaSuccess;
    };
    if (!r->comm) {
        // emulated: every shard's block through the staging buffer and back (identity)
        for (int g = 0; g < P; ++g) CFPQ_CUDA_TRY(pack(g, (size_t)g, 1));
        for (int g = 0; g < P; ++g) CFPQ_CUDA_TRY(pack(g, (size_t)g, 0));
        return CFPQ_OK;
    }
    const int me = r->my_rank, a = me / gc, b = me % gc;
    std::string err;
    if (final_gather) {
        CFPQ_CUDA_TRY(pack(me, (size_t)me, 1));
        if (!nccl_allgather_u32(r->comm, r->d_stage, slot, me, s, &err)) {
            set_error(err);
            return CFPQ_E_NCCL;
        }
        for (int g = 0; g < P; ++g)
            if (g != me) CFPQ_CUDA_TRY(pack(g, (size_t)g, 0));
        return CFPQ_OK;
    }
    // row group (a, *): slots by b'; column group (*, b): slots by a' (after the row slots)
    CFPQ_CUDA_TRY(pack(me, (size_t)b, 1));
    if (!nccl_allgather_u32(r->comm_row, r->d_stage, slot, b, s, &err)) {
        set_error(err);
        return CFPQ_E_NCCL;
    }
    for (int bb = 0; bb < gc; ++bb)
        if (bb != b) CFPQ_CUDA_TRY(pack(a * gc + bb, (size_t)bb, 0));
    // the column group reuses the staging buffer: the row blocks are unpacked already
    CFPQ_CUDA_TRY(pack(me, (size_t)a, 1));
    if (!nccl_allgather_u32(r->comm_col, r->d_stage, slot, a, s, &err)) {
        set_error(err);
        return CFPQ_E_NCCL;
    }
    for (int aa = 0; aa < gr; ++aa)
        if (aa != a) CFPQ_CUDA_TRY(pack(aa * gc + b, (size_t)aa, 0));
    return CFPQ_OK;
}

static cfpq_status dense_grid_iteration(cfpq_result* r, int* launches) {
    cudaStream_t s = r->stream;
    const int gr = r->grid_r, gc = r->grid_c;
    const int g_begin = r->emulated ? 0 : r->my_rank, g_end = r->emulated ? gr * gc : r->my_rank + 1;
    for (int g = g_begin; g < g_end; ++g) {
        int64_t ilo, ihi, jlo, jhi;
        dense_partition2(r->n, gr, gc, g / gc, g % gc, &ilo, &ihi, &jlo, &jhi);
        CFPQ_CUDA_TRY(dense_product(r->dense, ilo, ihi, s, launches, jlo, jhi));
    }
    cfpq_status st = grid_exchange(r, false);
    if (st != CFPQ_OK) return st;
    if (r->comm) {
        std::string err;
        if (!nccl_allreduce_sum_u64(r->comm, dense_total_counter(r->dense), 1, s, &err)) {
            set_error(err);
            return CFPQ_E_NCCL;
        }
    }
    return CFPQ_OK;
}

// Dense engine loop (path_policy 2): host-driven Jacobi iterations, one tcgen05 product
// launch (+ packs) per iteration; T and Tn swap roles after every iteration.
// Pipelined bit-row iterations (one GPU, compact mode): iteration k+1 is enqueued before the
// host reads iteration k's outcome (rows_pipe_iteration), so the host round trip of every
// iteration overlaps the next one's products; the device stop flag turns the speculative
// iteration after the fixpoint / cap / a list overflow into a no-op.  A list that ran out at
// iteration k is handled exactly as in the unpipelined loop (grow, redo k's products).
static cfpq_status rows_pipelined_loop(cfpq_result* r, int64_t start_k, int64_t* k_out, bool* capped) {
    cudaStream_t s = r->stream;
    DenseEngine* e = r->dense;
    const auto& outs = dense_outputs(e);
    for (auto& ev : r->pipe_ev)
        if (!ev) CFPQ_CUDA_TRY(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    CFPQ_CUDA_TRY(rows_pipe_begin(e, r->Tcur.data(), r->Tnxt.data(), s));
    const long long cap = r->opts.max_iterations;
    int64_t k = start_k + 1;
    int slot = 0;
    int launches = 0;
    auto swap_tk = [&]() {
        for (int A : outs) std::swap(r->Tcur[A], r->Tnxt[A]);
    };
    auto enqueue = [&](int64_t kk, int sl) -> cudaError_t {
        cudaError_t c = rows_pipe_iteration(e, r->d_nt, r->d_adj_idx, r->d_log, r->n_cells, kk == start_k + 1, kk, cap,
                                            sl, r->pipe_ev[sl], s, &launches);
        swap_tk();
        return c;
    };
    cfpq_status result = CFPQ_OK;
    CFPQ_CUDA_TRY(enqueue(k, 0));
    for (;;) {
        CFPQ_CUDA_TRY(enqueue(k + 1, slot ^ 1));   // speculative: a no-op if k ends the loop
        CFPQ_CUDA_TRY(cudaEventSynchronize(r->pipe_ev[slot]));
        unsigned long long nw = 0, lw = 0;
        int st = 0;
        rows_pipe_result(e, slot, &nw, &st, &lw);
        if (st == 2) {
            // a chunk / entry list ran out at k: k+1 did nothing, and the pointers (swapped for k
            // and k+1) are k's again; grow and redo k's products (the counter accumulates)
            CFPQ_CUDA_TRY(cudaStreamSynchronize(s));
            CFPQ_CUDA_TRY(rows_pipe_clear_stop(e, s));
            CFPQ_CUDA_TRY(dense_set_tables(e, r->Tcur.data(), r->Tnxt.data(), s));
            rows_set_first(e, k == start_k + 1);   // the speculative k+1 reset the flag of iteration 1
            for (bool redo = true; redo;) {
                CFPQ_CUDA_TRY(rows_shard_check(e, s, &redo, true));
                if (redo) {
                    CFPQ_CUDA_TRY(rows_shard(e, 0, r->n, s, &launches));
                    CFPQ_CUDA_TRY(dense_finish(e, s, &nw));
                }
            }
            r->dense_new.push_back((int64_t)nw);
            swap_tk();
            if (nw == 0) break;   // T_k = T_{k-1}
            if (k >= cap) {
                *capped = true;
                break;
            }
            // restart the pipeline at k+1 from the host's view (tables, a fresh count)
            CFPQ_CUDA_TRY(rows_pipe_begin(e, r->Tcur.data(), r->Tnxt.data(), s));
            ++k;
            slot = 0;
            CFPQ_CUDA_TRY(enqueue(k, 0));
            continue;
        }
        r->dense_new.push_back((int64_t)nw);
        if (st == 1 || st == 3) {
            // k+1 did nothing: undo its pointer swap (T_k stays where k put it)
            CFPQ_CUDA_TRY(cudaStreamSynchronize(s));
            swap_tk();
            if (st == 3) *capped = true;
            break;
        }
        if (lw > dense_list_capacity(e)) {
            // Δ_k overflowed its list: k+1 copies T_k whole (device-side check); grow the list
            // once k+1 is done with the old one
            CFPQ_CUDA_TRY(cudaStreamSynchronize(s));
            CFPQ_CUDA_TRY(rows_grow_list(e, lw));
        }
        ++k;
        slot ^= 1;
    }
    rows_pipe_end(e);
    r->launches += launches;
    *k_out = k;
    return result;
}

static cfpq_status run_dense(cfpq_result* r, int64_t start_k) {
    cudaStream_t s = r->stream;
    // seeding (and start_k sparse iterations) done; their cells are in the log
    CFPQ_CUDA_TRY(cudaMemcpyAsync(&r->h_st, r->d_st, sizeof(EngineState), cudaMemcpyDeviceToHost, s));
    CFPQ_CUDA_TRY(cudaStreamSynchronize(s));
    if (r->h_st.bad_edge) {
        set_error("graph has an edge with a node id >= n_nodes or a label id >= n_labels");
        return CFPQ_E_INVAL;
    }
    r->dense_mode = true;
    r->n_cells = std::min<unsigned long long>(r->h_st.log_size, r->log_cap);
    std::vector<int64_t> sparse_new;   // new cells of the sparse iterations 1..start_k
    if (start_k > 0) {
        std::vector<unsigned long long> off(start_k + 2);
        CFPQ_CUDA_TRY(cudaMemcpy(off.data(), r->d_iter_off, (start_k + 2) * 8, cudaMemcpyDeviceToHost));
        for (int64_t t = 1; t <= start_k; ++t) sparse_new.push_back((int64_t)(off[t + 1] - off[t]));
    }
    const auto& outs = dense_outputs(r->dense);
    r->Tcur = r->Tbase;
    r->Tnxt.assign(r->n_nt, nullptr);
    const size_t mw = (size_t)r->rows_alloc * (size_t)r->Wp;
    for (size_t q = 0; q < outs.size(); ++q) r->Tnxt[outs[q]] = r->d_Tn + q * mw;
    const int64_t tiles = dense_row_tiles(r->dense);
    std::vector<uint32_t*> out_mats(outs.size());
    r->dense_new = sparse_new;
    int64_t k = start_k;
    bool capped = false;
    r->dense_jac.clear();
    if (r->opts.account_work && start_k > 0) {
        std::vector<unsigned long long> j(start_k + 1);
        CFPQ_CUDA_TRY(cudaMemcpy(j.data(), r->d_jac, (start_k + 1) * 8, cudaMemcpyDeviceToHost));
        for (int64_t t = 1; t <= start_k; ++t) r->dense_jac.push_back((int64_t)j[t]);
    }
    dense_kblocks(r->dense, true);
    cudaEvent_t e0 = r->ev[2], e1 = r->ev[3];
    CFPQ_CUDA_TRY(cudaEventRecord(e0, s));
    const bool pipelined = r->opts.path_policy == 3 && r->n_ranks == 1 && !r->comm && !r->opts.account_work &&
                           (r->opts.diag_flags & (1 << 11)) == 0 && rows_pipe_eligible(r->dense);
    if (pipelined) {
        cfpq_status ps = rows_pipelined_loop(r, start_k, &k, &capped);
        if (ps != CFPQ_OK) return ps;
    }
    for (; !pipelined;) {
        ++k;
        unsigned long long nw = 0;
        int launches = 0;
        if (r->opts.account_work) {
            unsigned long long jt = 0;
            CFPQ_CUDA_TRY(dense_account(r->dense, r->Tcur.data(), r->rules, s, &jt));
            r->dense_jac.push_back((int64_t)jt);
        }
        const bool rows = r->opts.path_policy == 3;
        CFPQ_CUDA_TRY(dense_begin(r->dense, r->Tcur.data(), r->Tnxt.data(), k == start_k + 1, s, &launches, !rows));
        if (rows && r->n_ranks == 1 && !r->comm) {
            CFPQ_CUDA_TRY(rows_product(r->dense, r->Tcur.data(), r->Tnxt.data(), r->d_nt, r->d_adj_idx, r->d_log,
                                       r->n_cells, k == start_k + 1, s, &launches));
        } else if (rows) {
            cfpq_status rs = rows_sharded_iteration(r, k == start_k + 1, &launches);
            if (rs != CFPQ_OK) return rs;
        } else if (r->n_ranks == 1 && !r->comm) {
            CFPQ_CUDA_TRY(dense_product(r->dense, 0, tiles, s, &launches));
        } else if (r->grid_r > 0) {
            cfpq_status gs = dense_grid_iteration(r, &launches);
            if (gs != CFPQ_OK) return gs;
        } else if (r->emulated) {
            // P row-block shards in one process: each writes its rows of the shared T_k
            for (int g = 0; g < r->n_ranks; ++g) {
                int64_t lo, hi, br;
                dense_partition(r->n, r->n_ranks, g, &lo, &hi, &br);
                CFPQ_CUDA_TRY(dense_product(r->dense, lo, hi, s, &launches));
            }
        } else {
            int64_t lo, hi, br;
            dense_partition(r->n, r->n_ranks, r->my_rank, &lo, &hi, &br);
            CFPQ_CUDA_TRY(dense_product(r->dense, lo, hi, s, &launches));
            // all-gather every rank's row block of T_k, sum the new-cell counts (the
            // "changed" flag) — one NCCL group over NVLink per iteration
            for (size_t q = 0; q < outs.size(); ++q) out_mats[q] = r->Tnxt[outs[q]];
            std::string err;
            if (!nccl_exchange_rows(r->comm, out_mats.data(), (int)outs.size(), (size_t)br * r->Wp, r->my_rank,
                                    dense_total_counter(r->dense), s, &err)) {
                set_error(err);
                return CFPQ_E_NCCL;
            }
        }
        CFPQ_CUDA_TRY(dense_finish(r->dense, s, &nw));
        if (rows && r->n_ranks == 1 && !r->comm) {
            // the plan ran without a host round trip: a chunk-list overflow re-runs the
            // products of this iteration with grown lists (the counter keeps accumulating)
            for (bool redo = true; redo;) {
                CFPQ_CUDA_TRY(rows_shard_check(r->dense, s, &redo, true));
                if (redo) {
                    CFPQ_CUDA_TRY(rows_shard(r->dense, 0, r->n, s, &launches));
                    CFPQ_CUDA_TRY(dense_finish(r->dense, s, &nw));
                }
            }
        }
        r->launches += launches;
        r->dense_new.push_back((int64_t)nw);
        for (int A : outs) std::swap(r->Tcur[A], r->Tnxt[A]);
        if (nw == 0) break;   // T_k = T_{k-1}
        if (k >= r->opts.max_iterations) {
            capped = true;
            break;
        }
    }
    if (r->grid_r > 0 && r->comm) {
        // every shard holds its panels only: make T whole for the result queries (T_k was
        // swapped into Tcur; the exchange reads Tnxt, so point it at the final matrices)
        for (int A : outs) std::swap(r->Tcur[A], r->Tnxt[A]);
        cfpq_status gs = grid_exchange(r, true);
        for (int A : outs) std::swap(r->Tcur[A], r->Tnxt[A]);
        if (gs != CFPQ_OK) return gs;
    }
    CFPQ_CUDA_TRY(cudaEventRecord(e1, s));
    CFPQ_CUDA_TRY(cudaEventSynchronize(e1));
    {
        float ms = 0;
        if (start_k == 0) {
            CFPQ_CUDA_TRY(cudaEventElapsedTime(&ms, r->ev[0], r->ev[1]));
            r->seed_ns = ms * 1e6;
            r->loop_ns = 0;
        }
        CFPQ_CUDA_TRY(cudaEventElapsedTime(&ms, e0, e1));
        r->loop_ns += ms * 1e6;
    }
    r->iterations = k;
    r->dense_kb = dense_kblocks(r->dense, false);
    for (int A = 0; A < r->n_nt; ++A) r->h_nt[A].T = r->Tcur[A];
    CFPQ_CUDA_TRY(cudaMemcpyAsync(r->d_nt, r->h_nt.data(), r->n_nt * sizeof(NTInfo), cudaMemcpyHostToDevice, s));
    CFPQ_CUDA_TRY(cudaStreamSynchronize(s));
    r->h_st.iter = k;
    r->h_st.status = capped ? ST_CAP : ST_DONE;
    if (capped) {
        set_error("max_iterations reached before the fixpoint");
        return CFPQ_E_NOT_CONVERGED;
    }
    return CFPQ_OK;
}

// Asynchronous schedule (schedule 2, relational): one barrier-free worklist kernel; on a
// log overflow the host grows the log and the kernel re-expands the whole (still valid,
// flagged) log from slot 0 — idempotent, since re-derived cells are already set.
static cfpq_status run_async(cfpq_result* r, unsigned long long seeds_upper) {
    cudaStream_t s = r->stream;
    bool first = true;
    for (;;) {
        EngineParams p = r->params();
        CFPQ_CUDA_TRY(launch_async(p, r->grid, s, first, seeds_upper));
        CFPQ_CUDA_TRY(cudaEventRecord(r->ev[3], s));
        r->launches += first ? 2 : 1;
        CFPQ_CUDA_TRY(cudaMemcpyAsync(&r->h_st, r->d_st, sizeof(EngineState), cudaMemcpyDeviceToHost, s));
        CFPQ_CUDA_TRY(cudaStreamSynchronize(s));
        first = false;
        if (r->h_st.bad_edge) {
            r->n_cells = std::min<unsigned long long>(r->h_st.log_size, r->log_cap);
            CFPQ_CUDA_TRY(launch_strip_flags(r->d_log, 0, r->n_cells, s));
            set_error("graph has an edge with a node id >= n_nodes or a label id >= n_labels");
            return CFPQ_E_INVAL;
        }
        if (!r->h_st.overflow) break;
        unsigned long long old_cap = r->log_cap;
        cfpq_status st = grow_log(r, r->h_st.log_size);
        if (st != CFPQ_OK) return st;
        CFPQ_CUDA_TRY(cudaMemsetAsync(r->d_log + old_cap, 0, (r->log_cap - old_cap) * 8, s));
        EngineState fix = r->h_st;
        fix.log_size = std::min<unsigned long long>(r->h_st.log_size, old_cap);
        fix.overflow = 0;
        fix.async_head = 0;
        fix.async_done = 0;
        CFPQ_CUDA_TRY(cudaMemcpyAsync(r->d_st, &fix, sizeof(EngineState), cudaMemcpyHostToDevice, s));
    }
    r->n_cells = std::min<unsigned long long>(r->h_st.log_size, r->log_cap);
    if (r->self_clear_ok()) {
        r->t_clean = true;   // the kernel stripped the flags and reset the bit words at quiescence
    } else {
        CFPQ_CUDA_TRY(launch_strip_flags(r->d_log, 0, r->n_cells, s));
    }
    {
        float ms = 0;
        CFPQ_CUDA_TRY(cudaEventElapsedTime(&ms, r->ev[0], r->ev[1]));
        r->seed_ns = ms * 1e6;
        CFPQ_CUDA_TRY(cudaEventElapsedTime(&ms, r->ev[1], r->ev[3]));
        r->loop_ns = ms * 1e6;
    }
    CFPQ_CUDA_TRY(cudaStreamSynchronize(s));
    r->iterations = 0;   // no loop bodies: the asynchronous schedule has no iteration structure
    return CFPQ_OK;
}

// Row-block sharded sparse engine (§8(e)).  Every rank holds the whole Δ list of
// each iteration (identical set on every rank) and derives only the cells of the rows it
// owns: for A -> B C with C preterminal, Δ_B(i,r) gives (A,i,k) in row i; with B preterminal,
// Δ_C(r,j) gives (A,i,j) for the rows i of B's column r (rank-filtered).  Preterminals are
// seeded on every rank (constant after iteration 0), so no row of another rank is read.
// Per iteration: one launch of the closure kernel limited to iteration k and the rank's rows,
// then the exchange: all-gather of the per-rank new-cell counts and of the cells (padded to
// the largest count), appended to every rank's log in rank order = Δ_k; Σ counts == 0 is
// the global no-change test of Alg. 1 line 8.  Emulated ranks (one process) run
// the shards one after another on one shared log and membership set and exchange through
// the same padded buffer and compaction copies.
static cfpq_status run_sharded(cfpq_result* r) {
    cudaStream_t s = r->stream;
    const int P = r->n_ranks;
    CFPQ_CUDA_TRY(cudaMemcpyAsync(&r->h_st, r->d_st, sizeof(EngineState), cudaMemcpyDeviceToHost, s));
    CFPQ_CUDA_TRY(cudaStreamSynchronize(s));
    if (r->h_st.bad_edge) {
        r->n_cells = std::min<unsigned long long>(r->h_st.log_size, r->log_cap);
        set_error("graph has an edge with a node id >= n_nodes or a label id >= n_labels");
        return CFPQ_E_INVAL;
    }
    unsigned long long lo = 0, hi = r->h_st.hi;   // Δ_0 = every seed (seeded on every rank)
    r->shard_new.clear();
    long long k = 0;
    std::vector<int64_t> row_lo(P), row_hi(P);
    for (int g = 0; g < P; ++g) {
        int64_t tlo, thi, br;
        dense_partition(r->n, P, g, &tlo, &thi, &br);
        row_lo[g] = std::min<int64_t>(tlo * 128, r->n);
        row_hi[g] = std::min<int64_t>(thi * 128, r->n);
    }
    std::vector<unsigned long long> cnt(P, 0);
    int status = ST_RUNNING;
    while (status == ST_RUNNING) {
        if (k >= r->opts.max_iterations) {
            status = ST_CAP;
            break;
        }
        ++k;   // iteration k expands Δ_{k-1} = log[lo, hi)
        unsigned long long end = hi;
        const int g_begin = r->emulated ? 0 : r->my_rank, g_end = r->emulated ? P : r->my_rank + 1;
        std::fill(cnt.begin(), cnt.end(), 0ull);
        for (int g = g_begin; g < g_end; ++g) {
            unsigned long long start = end;
            for (;;) {
                EngineState es{};
                es.lo = lo;
                es.hi = hi;
                es.iter = k - 1;
                es.status = ST_RUNNING;
                es.log_size = end;
                CFPQ_CUDA_TRY(cudaMemcpyAsync(r->d_st, &es, sizeof(EngineState), cudaMemcpyHostToDevice, s));
                EngineParams p = r->params();
                p.row_lo = (uint32_t)row_lo[g];
                p.row_hi = (uint32_t)row_hi[g];
                p.max_iter = k;                       // exactly one loop body per launch
                CFPQ_CUDA_TRY(launch_closure(p, r->grid, s));
                r->launches++;
                CFPQ_CUDA_TRY(cudaMemcpyAsync(&r->h_st, r->d_st, sizeof(EngineState), cudaMemcpyDeviceToHost, s));
                CFPQ_CUDA_TRY(cudaStreamSynchronize(s));
                if (r->h_st.status == ST_OVERFLOW || r->h_st.overflow) {
                    const unsigned long long old_cap = r->log_cap;
                    cfpq_status st = grow_log(r, r->h_st.log_size);
                    if (st != CFPQ_OK) return st;
                    end = std::min<unsigned long long>(r->h_st.log_size, old_cap);   // keep the valid prefix
                    continue;
                }
                if (r->h_st.status != ST_DONE && r->h_st.status != ST_CAP) {
                    set_error("closure kernel stopped without finishing the iteration (status " +
                              std::to_string(r->h_st.status) + ")");
                    return CFPQ_E_CUDA;
                }
                break;
            }
            end = r->h_st.log_size;
            cnt[g] = end - start;
        }
        // ---- exchange: counts, then the cells (padded), appended in rank order ----
        if (r->comm) {
            uint64_t* dc = nullptr;
            if (r->xbuf_cap < (size_t)P) {
                dfree(r->d_xbuf);
                cfpq_status st = dalloc(&r->d_xbuf, (size_t)P * 64, "exchange buffer");
                if (st != CFPQ_OK) return st;
                r->xbuf_cap = (size_t)P * 64;
            }
            dc = r->d_xbuf;
            uint64_t mine = cnt[r->my_rank];
            CFPQ_CUDA_TRY(cudaMemcpyAsync(dc + r->my_rank, &mine, 8, cudaMemcpyHostToDevice, s));
            std::string err;
            if (!nccl_allgather_u64(r->comm, dc, 1, r->my_rank, s, &err)) {
                set_error(err);
                return CFPQ_E_NCCL;
            }
            std::vector<uint64_t> hc(P);
            CFPQ_CUDA_TRY(cudaMemcpyAsync(hc.data(), dc, 8 * P, cudaMemcpyDeviceToHost, s));
            CFPQ_CUDA_TRY(cudaStreamSynchronize(s));
            for (int g = 0; g < P; ++g) cnt[g] = hc[g];
        }
        unsigned long long tot = 0, mx = 0;
        for (int g = 0; g < P; ++g) {
            tot += cnt[g];
            mx = std::max<unsigned long long>(mx, cnt[g]);
        }
        for (int g = 0; g < P; ++g) r->shard_new.push_back((int64_t)cnt[g]);
        if ((P > 1 || r->comm) && tot > 0) {
            if (hi + tot + 64 > r->log_cap) {
                cfpq_status st = grow_log(r, hi + tot + 64, end);
                if (st != CFPQ_OK) return st;
            }
            if (r->xbuf_cap < (size_t)P * mx) {
                dfree(r->d_xbuf);
                size_t want = std::max<size_t>((size_t)P * mx, (size_t)P * 64);
                cfpq_status st = dalloc(&r->d_xbuf, want, "exchange buffer");
                if (st != CFPQ_OK) return st;
                r->xbuf_cap = want;
            }
            // each rank's new cells into its slot of the padded buffer
            unsigned long long off = hi;
            for (int g = g_begin; g < g_end; ++g) {
                if (cnt[g])
                    CFPQ_CUDA_TRY(cudaMemcpyAsync(r->d_xbuf + (size_t)g * mx, r->d_log + off, cnt[g] * 8,
                                                  cudaMemcpyDeviceToDevice, s));
                off += cnt[g];
            }
            if (r->comm) {
                std::string err;
                if (!nccl_allgather_u64(r->comm, r->d_xbuf, mx, r->my_rank, s, &err)) {
                    set_error(err);
                    return CFPQ_E_NCCL;
                }
            }
            // compaction: Δ_k = rank 0's cells, rank 1's cells, ... at log[hi, hi + tot)
            off = hi;
            for (int g = 0; g < P; ++g) {
                if (cnt[g])
                    CFPQ_CUDA_TRY(cudaMemcpyAsync(r->d_log + off, r->d_xbuf + (size_t)g * mx, cnt[g] * 8,
                                                  cudaMemcpyDeviceToDevice, s));
                off += cnt[g];
            }
        }
        // iteration offsets of the global log
        unsigned long long offs[2] = {hi, hi + tot};
        if (k + 1 < r->iter_off_cap)
            CFPQ_CUDA_TRY(cudaMemcpyAsync(r->d_iter_off + k, offs, 16, cudaMemcpyHostToDevice, s));
        lo = hi;
        hi = hi + tot;
        if (tot == 0) status = ST_DONE;
    }
    CFPQ_CUDA_TRY(cudaEventRecord(r->ev[3], s));
    CFPQ_CUDA_TRY(cudaStreamSynchronize(s));
    {
        float ms = 0;
        CFPQ_CUDA_TRY(cudaEventElapsedTime(&ms, r->ev[0], r->ev[1]));
        r->seed_ns = ms * 1e6;
        CFPQ_CUDA_TRY(cudaEventElapsedTime(&ms, r->ev[1], r->ev[3]));
        r->loop_ns = ms * 1e6;
    }
    r->h_st.lo = lo;
    r->h_st.hi = hi;
    r->h_st.iter = k;
    r->h_st.status = status;
    r->h_st.log_size = hi;
    r->iterations = k;
    r->n_cells = hi;
    if (status == ST_CAP) {
        set_error("max_iterations reached before the fixpoint");
        return CFPQ_E_NOT_CONVERGED;
    }
    return CFPQ_OK;
}

static cfpq_status run(cfpq_result* r, const cfpq_graph* d);

// Peer pointers of every rank's log and state.  Emulated shards: the virtual ranks 1..P-1 get
// their own logs and states here.  Real GPUs: the own log / state are exported as CUDA IPC
// handles, all-gathered over NCCL, and the peers' mapped (NVLink peer access).
static cfpq_status xr_setup(cfpq_result* r) {
    const int P = r->n_ranks;
    if (r->xr_log.size() == (size_t)P && r->xr_cap == r->log_cap && r->xr_log_of == r->d_log) return CFPQ_OK;
    cudaStream_t s = r->stream;
    CFPQ_CUDA_TRY(cudaStreamSynchronize(s));
    for (void* q : r->xr_opened) cudaIpcCloseMemHandle(q);
    for (void* q : r->xr_owned) cudaFree(q);
    r->xr_opened.clear();
    r->xr_owned.clear();
    r->xr_st.assign(P, nullptr);
    r->xr_log.assign(P, nullptr);
    if (r->emulated) {
        r->xr_st[0] = r->d_st;
        r->xr_log[0] = r->d_log;
        for (int q = 1; q < P; ++q) {
            EngineState* sq = nullptr;
            uint64_t* lq = nullptr;
            cfpq_status st;
            if ((st = dalloc(&sq, 1, "virtual rank state")) != CFPQ_OK) return st;
            r->xr_owned.push_back(sq);
            if ((st = dalloc(&lq, r->log_cap, "virtual rank log")) != CFPQ_OK) return st;
            r->xr_owned.push_back(lq);
            r->xr_st[q] = sq;
            r->xr_log[q] = lq;
        }
    } else {
        const int me = r->my_rank;
        r->xr_st[me] = r->d_st;
        r->xr_log[me] = r->d_log;
        cudaIpcMemHandle_t hl, hs;
        CFPQ_CUDA_TRY(cudaIpcGetMemHandle(&hl, r->d_log));
        CFPQ_CUDA_TRY(cudaIpcGetMemHandle(&hs, r->d_st));
        const size_t per = 2 * sizeof(cudaIpcMemHandle_t);   // 128 bytes = 16 uint64 per rank
        const size_t slot = (per + 7) / 8;
        if (r->xbuf_cap < (size_t)P * slot) {
            dfree(r->d_xbuf);
            r->xbuf_cap = 0;
            cfpq_status st = dalloc(&r->d_xbuf, (size_t)P * slot, "handle exchange");
            if (st != CFPQ_OK) return st;
            r->xbuf_cap = (size_t)P * slot;
        }
        std::vector<unsigned char> mine(slot * 8, 0);
        memcpy(mine.data(), &hl, sizeof(hl));
        memcpy(mine.data() + sizeof(hl), &hs, sizeof(hs));
        CFPQ_CUDA_TRY(cudaMemcpy(r->d_xbuf + (size_t)me * slot, mine.data(), slot * 8, cudaMemcpyHostToDevice));
        std::string err;
        if (!nccl_allgather_u64(r->comm, r->d_xbuf, slot, me, s, &err)) {
            set_error(err);
            return CFPQ_E_NCCL;
        }
        std::vector<unsigned char> all((size_t)P * slot * 8);
        CFPQ_CUDA_TRY(cudaMemcpyAsync(all.data(), r->d_xbuf, all.size(), cudaMemcpyDeviceToHost, s));
        CFPQ_CUDA_TRY(cudaStreamSynchronize(s));
        for (int q = 0; q < P; ++q) {
            if (q == me) continue;
            cudaIpcMemHandle_t ql, qs;
            memcpy(&ql, all.data() + (size_t)q * slot * 8, sizeof(ql));
            memcpy(&qs, all.data() + (size_t)q * slot * 8 + sizeof(ql), sizeof(qs));
            void *pl = nullptr, *ps = nullptr;
            CFPQ_CUDA_TRY(cudaIpcOpenMemHandle(&pl, ql, cudaIpcMemLazyEnablePeerAccess));
            r->xr_opened.push_back(pl);
            CFPQ_CUDA_TRY(cudaIpcOpenMemHandle(&ps, qs, cudaIpcMemLazyEnablePeerAccess));
            r->xr_opened.push_back(ps);
            r->xr_log[q] = (uint64_t*)pl;
            r->xr_st[q] = (EngineState*)ps;
        }
    }
    if (!r->d_xr_st) {
        cfpq_status st;
        if ((st = dalloc(&r->d_xr_st, (size_t)P, "peer states")) != CFPQ_OK) return st;
        if ((st = dalloc(&r->d_xr_log, (size_t)P, "peer logs")) != CFPQ_OK) return st;
        if ((st = dalloc(&r->d_xr_rows, (size_t)2 * P, "rank rows")) != CFPQ_OK) return st;
        std::vector<uint32_t> rows(2 * P);
        for (int g = 0; g < P; ++g) {
            int64_t tlo, thi, br;
            dense_partition(r->n, P, g, &tlo, &thi, &br);
            rows[g] = (uint32_t)std::min<int64_t>(tlo * 128, r->n);
            rows[P + g] = (uint32_t)std::min<int64_t>(thi * 128, r->n);
        }
        CFPQ_CUDA_TRY(cudaMemcpy(r->d_xr_rows, rows.data(), rows.size() * 4, cudaMemcpyHostToDevice));
    }
    CFPQ_CUDA_TRY(cudaMemcpy(r->d_xr_st, r->xr_st.data(), P * sizeof(void*), cudaMemcpyHostToDevice));
    CFPQ_CUDA_TRY(cudaMemcpy(r->d_xr_log, r->xr_log.data(), P * sizeof(void*), cudaMemcpyHostToDevice));
    r->xr_cap = r->log_cap;
    r->xr_log_of = r->d_log;
    return CFPQ_OK;
}

// The row-sharded sparse engine with the device-resident peer-memory exchange (§3.5).
static cfpq_status run_xr(cfpq_result* r, const cfpq_graph* d) {
    cudaStream_t s = r->stream;
    const int P = r->n_ranks;
    CFPQ_CUDA_TRY(cudaMemcpyAsync(&r->h_st, r->d_st, sizeof(EngineState), cudaMemcpyDeviceToHost, s));
    CFPQ_CUDA_TRY(cudaStreamSynchronize(s));
    if (r->h_st.bad_edge) {
        r->n_cells = std::min<unsigned long long>(r->h_st.log_size, r->log_cap);
        set_error("graph has an edge with a node id >= n_nodes or a label id >= n_labels");
        return CFPQ_E_INVAL;
    }
    cfpq_status st = xr_setup(r);
    if (st != CFPQ_OK) return st;
    const unsigned long long n_seed = r->h_st.log_size;
    if (r->emulated) {
        // every virtual rank starts from the same Δ_0 (every rank seeds every cell)
        for (int q = 1; q < P; ++q) {
            CFPQ_CUDA_TRY(cudaMemcpyAsync(r->xr_st[q], r->d_st, sizeof(EngineState), cudaMemcpyDeviceToDevice, s));
            if (n_seed)
                CFPQ_CUDA_TRY(cudaMemcpyAsync(r->xr_log[q], r->d_log, n_seed * 8, cudaMemcpyDeviceToDevice, s));
        }
    } else if (r->comm) {
        // the peers must have seeded (and zeroed their barrier words) before anyone appends
        std::string err;
        if (!nccl_allreduce_sum_u64(r->comm, (unsigned long long*)r->d_xbuf, 1, s, &err)) {
            set_error(err);
            return CFPQ_E_NCCL;
        }
    }
    XrParams x{};
    x.P = P;
    x.my_rank = r->emulated ? -1 : r->my_rank;
    x.cpr = r->emulated ? std::max(1, r->grid / P) : r->grid;
    x.st = r->d_xr_st;
    x.log = r->d_xr_log;
    x.row_lo = r->d_xr_rows;
    x.row_hi = r->d_xr_rows + P;
    EngineParams p = r->params();
    p.self_clear = r->self_clear_ok() ? 1 : 0;
    const int grid = r->emulated ? x.cpr * P : r->grid;
    CFPQ_CUDA_TRY(launch_xr_closure(p, x, grid, s));
    CFPQ_CUDA_TRY(cudaEventRecord(r->ev[3], s));
    r->launches++;
    CFPQ_CUDA_TRY(cudaMemcpyAsync(&r->h_st, r->d_st, sizeof(EngineState), cudaMemcpyDeviceToHost, s));
    CFPQ_CUDA_TRY(cudaStreamSynchronize(s));
    {
        float ms = 0;
        CFPQ_CUDA_TRY(cudaEventElapsedTime(&ms, r->ev[0], r->ev[1]));
        r->seed_ns = ms * 1e6;
        CFPQ_CUDA_TRY(cudaEventElapsedTime(&ms, r->ev[1], r->ev[3]));
        r->loop_ns = ms * 1e6;
    }
    r->n_cells = std::min<unsigned long long>(r->h_st.log_size, r->log_cap);
    if (r->h_st.status == ST_OVERFLOW) {
        // some rank's log ran out: every rank saw it in the same iteration.  Grow every log,
        // clear the matrices and run the closure again from the seeds.
        if (r->xr_depth > 8) {
            set_error("peer-memory exchange: the logs kept overflowing");
            return CFPQ_E_NOMEM;
        }
        const unsigned long long want = std::max<unsigned long long>(2 * r->log_cap, r->h_st.log_size + 1024);
        uint64_t* nl = nullptr;
        if ((st = dalloc(&nl, want, "cell log (grow)")) != CFPQ_OK) return st;
        CFPQ_CUDA_TRY(cudaMemsetAsync(nl, 0, want * 8, s));
        dfree(r->d_log);
        r->d_log = nl;
        r->log_cap = want;
        r->opts.log_capacity = (int64_t)want;
        const size_t mw = (size_t)r->rows_alloc * (size_t)r->Wp;
        CFPQ_CUDA_TRY(cudaMemsetAsync(r->d_T, 0, mw * r->n_nt * 4, s));
        r->n_cells = 0;
        r->t_clean = false;
        r->ran = false;
        r->regrows++;
        ++r->xr_depth;
        st = run(r, d);
        --r->xr_depth;
        return st;
    }
    if (r->h_st.status == ST_TIMEOUT) {
        set_error("peer-memory exchange: a rank did not reach the iteration barrier (watchdog)");
        return CFPQ_E_NCCL;
    }
    r->iterations = r->h_st.iter;
    r->t_clean = r->self_clear_ok() && (r->h_st.status == ST_DONE || r->h_st.status == ST_CAP);
    if (r->h_st.status == ST_CAP) {
        set_error("max_iterations reached before the fixpoint");
        return CFPQ_E_NOT_CONVERGED;
    }
    if (r->h_st.status != ST_DONE) {
        set_error("peer-memory closure stopped without reaching the fixpoint (status " +
                  std::to_string(r->h_st.status) + ")");
        return CFPQ_E_CUDA;
    }
    return CFPQ_OK;
}

// The device-resident fixpoint loop of the one-GPU sparse engine (a2-a5): one persistent
// cooperative launch, re-launched only after a log overflow.  fused_seed: the first launch
// also seeds T_0 and builds the preterminal adjacency (fused_seed_phase).
static cfpq_status run_sparse_loop(cfpq_result* r, const cfpq_graph* d, bool fused_seed) {
    cudaStream_t s = r->stream;
    cfpq_status st;
    EngineParams p;
    bool first = true;
    for (;;) {
        p = r->params();
        if (fused_seed && first) {
            p.fused_seed = 1;
            p.edges = d->d_edges;
            p.n_edges = d->n_edges;
            p.lab_ptr = r->d_lab_ptr;
            p.lab_nt = r->d_lab_nt;
            p.n_labels = r->n_labels;
            p.max_rules = r->max_rules_per_label;
            p.slot_row = r->d_slot_row;
            p.slot_col = r->d_slot_col;
            p.n_slots = r->n_adj_slots;
            p.adj_cursor = r->d_adj_cnt;
            p.adj_idx_w = r->d_adj_idx;
            p.ell = r->d_adj_ell;
            p.scan_tot = r->d_scan_tot;
        }
        if (!first) CFPQ_CUDA_TRY(cudaEventRecord(r->ev[2], s));
        CFPQ_CUDA_TRY(launch_closure(p, r->grid, s));
        CFPQ_CUDA_TRY(cudaEventRecord(r->ev[3], s));
        r->launches++;
        CFPQ_CUDA_TRY(cudaMemcpyAsync(&r->h_st, r->d_st, sizeof(EngineState), cudaMemcpyDeviceToHost, s));
        CFPQ_CUDA_TRY(cudaStreamSynchronize(s));
        if (r->clr_active && r->h_st.clr_cursor >= r->clr_n) {
            r->spare.n_cells = 0;   // the other bank was cleared inside the kernel
            r->clr_active = false;
        }
        {
            float ms = 0;
            if (first) {
                CFPQ_CUDA_TRY(cudaEventElapsedTime(&ms, r->ev[0], r->ev[1]));
                r->seed_ns = ms * 1e6;
                CFPQ_CUDA_TRY(cudaEventElapsedTime(&ms, r->ev[1], r->ev[3]));
            } else {
                CFPQ_CUDA_TRY(cudaEventElapsedTime(&ms, r->ev[2], r->ev[3]));
            }
            r->loop_ns += ms * 1e6;
            first = false;
        }
        if (r->h_st.bad_edge) {
            r->n_cells = std::min<unsigned long long>(r->h_st.log_size, r->log_cap);
            set_error("graph has an edge with a node id >= n_nodes or a label id >= n_labels");
            return CFPQ_E_INVAL;
        }
        if (r->h_st.status == ST_OVERFLOW) {
            // Δ_k did not fit: grow the log keeping its valid prefix (every slot below
            // the old capacity was written) and re-run iteration k.
            unsigned long long old_cap = r->log_cap;
            st = grow_log(r, r->h_st.log_size);
            if (st != CFPQ_OK) return st;
            EngineState fix = r->h_st;
            fix.log_size = std::min<unsigned long long>(r->h_st.log_size, old_cap);
            fix.status = ST_RUNNING;
            fix.overflow = 0;
            fix.bar_count = 0;
            fix.bar_word = 0;
            if (r->opts.account_work && fix.iter + 1 < r->iter_off_cap)
                CFPQ_CUDA_TRY(cudaMemsetAsync(r->d_jac + fix.iter + 1, 0, 8, s));
            CFPQ_CUDA_TRY(cudaMemcpyAsync(r->d_st, &fix, sizeof(EngineState), cudaMemcpyHostToDevice, s));
            continue;
        }
        break;
    }
    // Gauss-Seidel: the kernel counts steps; an iteration is a round of n_stages steps
    r->iterations = r->opts.schedule == 3 && r->n_stages > 0 ? r->h_st.iter / r->n_stages : r->h_st.iter;
    r->n_cells = std::min<unsigned long long>(r->h_st.log_size, r->log_cap);
    r->t_clean = r->self_clear_ok() && (r->h_st.status == ST_DONE || r->h_st.status == ST_CAP);
    if (r->h_st.status == ST_SWITCH) {
        // Δ became dense: continue Alg. 1 from T_k on the tcgen05 engine (same states)
        if ((st = ensure_dense(r)) != CFPQ_OK) return st;
        r->switched++;
        return run_dense(r, r->h_st.iter);
    }
    if (r->h_st.status == ST_CAP) {
        set_error("max_iterations reached before the fixpoint");
        return CFPQ_E_NOT_CONVERGED;
    }
    if (r->h_st.status == ST_LEN_OVERFLOW) {
        set_error("a single-path length exceeded 2^32-1");
        return CFPQ_E_OVERFLOW;
    }
    if (r->h_st.status != ST_DONE) {
        set_error("closure kernel stopped without reaching the fixpoint (status " +
                  std::to_string(r->h_st.status) + ", barrier watchdog?)");
        return CFPQ_E_CUDA;
    }
    return CFPQ_OK;
}

static cfpq_status run(cfpq_result* r, const cfpq_graph* d) {
    cudaStream_t s = r->stream;
    r->clr_active = false;
    r->launches = 0;
    r->counts_valid = false;
    cfpq_status st = size_for_graph(r, d);
    if (st != CFPQ_OK) return st;
    EngineParams p = r->params();
    if (r->dense_mode && r->ran) {
        // the previous run ended on the dense engine, which rewrites whole matrices
        // the dense engine rewrites whole matrices: restore the base buffers and clear them
        for (int A = 0; A < r->n_nt; ++A) r->h_nt[A].T = r->Tbase[A];
        CFPQ_CUDA_TRY(cudaMemcpyAsync(r->d_nt, r->h_nt.data(), r->n_nt * sizeof(NTInfo), cudaMemcpyHostToDevice, s));
        const size_t mw = (size_t)r->rows_alloc * (size_t)r->Wp;
        CFPQ_CUDA_TRY(cudaMemsetAsync(r->d_T, 0, mw * r->n_nt * 4, s));
        CFPQ_CUDA_TRY(cudaMemsetAsync(r->d_Tn, 0, mw * std::max<size_t>(dense_outputs(r->dense).size(), 1) * 4, s));
        if (r->d_snap) {
            int n_snap = 0;
            for (auto& t : r->h_nt) n_snap += (t.S ? 1 : 0) + (t.ST ? 1 : 0);
            CFPQ_CUDA_TRY(cudaMemsetAsync(r->d_snap, 0, mw * n_snap * 4, s));
        }
        if (r->d_rowc) {
            // the sparse iterations before an auto switch counted their cells here
            CFPQ_CUDA_TRY(cudaMemsetAsync(r->d_rowc, 0, (size_t)r->n_nt * r->n * 4, s));
            CFPQ_CUDA_TRY(cudaMemsetAsync(r->d_colc, 0, (size_t)r->n_nt * r->n * 4, s));
        }
        r->n_cells = 0;
        p = r->params();
    }
    r->dense_mode = false;
    // the previous run's cells (bitmaps, snapshots, keys, counters) must go: O(|log|).
    // With two banks, switch to the clean bank and clear the old one on a side stream,
    // overlapped with this run; else clear inline.
    const bool log_clear = !r->hashed || r->opts.account_work;   // hashed: only counters to clear
    if (r->t_clean) {
        r->n_cells = 0;   // the previous run's kernel already reset its words (self_clear)
        r->t_clean = false;
    }
    if (r->ran && (r->n_cells || r->hashed)) {
        if (!r->have_spare && !r->spare_failed && r->opts.path_policy < 2) {
            r->have_spare = make_spare(r);
            r->spare_failed = !r->have_spare;
        }
        // the persistent closure kernel clears the other bank itself (barrier idle time)
        const bool in_kernel = !r->hashed && r->opts.schedule != 2 && r->n_ranks == 1 && !r->comm &&
                               r->opts.path_policy < 2 && (r->opts.diag_flags & 2) == 0;
        if (r->have_spare && in_kernel) {
            swap_with(r, r->spare);                       // current = clean bank
            CFPQ_CUDA_TRY(cudaStreamWaitEvent(s, r->spare_clean, 0));   // a side-stream clear, if any
            r->clr_active = r->spare.n_cells > 0;
            r->clr_log = r->spare.d_log;
            r->clr_n = r->spare.n_cells;
            r->clr_nt = r->spare.d_nt;
            r->clr_rowc = r->spare.d_rowc;
            r->clr_colc = r->spare.d_colc;
            // spare.n_cells is zeroed once the first closure launch has drained the clear
            st = size_for_graph(r, d);
            if (st != CFPQ_OK) return st;
            if (r->log_cap < r->spare.log_cap) {
                uint64_t* nl = nullptr;
                if ((st = dalloc(&nl, r->spare.log_cap, "cell log")) != CFPQ_OK) return st;
                CFPQ_CUDA_TRY(cudaMemsetAsync(nl, 0, r->spare.log_cap * 8, s));
                dfree(r->d_log);
                r->d_log = nl;
                r->log_cap = r->spare.log_cap;
            }
            p = r->params();
        } else if (r->have_spare) {
            swap_with(r, r->spare);                       // current = clean bank
            CFPQ_CUDA_TRY(cudaStreamWaitEvent(s, r->spare_clean, 0));   // its clear has finished
            CFPQ_CUDA_TRY(cudaEventRecord(r->main_done, s));
            CFPQ_CUDA_TRY(cudaStreamWaitEvent(r->side, r->main_done, 0));
            // clear the bank of the previous run (now the spare) on the side stream
            swap_with(r, r->spare);
            EngineParams pc = r->params();                // parameters of the old bank
            const unsigned long long old_cells = r->n_cells;
            swap_with(r, r->spare);
            if (log_clear) CFPQ_CUDA_TRY(launch_clear_log(pc, old_cells, r->side));
            if (r->hashed) CFPQ_CUDA_TRY(cudaMemsetAsync(r->spare.d_hset, 0xff, r->spare.hcap * 8, r->side));
            CFPQ_CUDA_TRY(cudaEventRecord(r->spare_clean, r->side));
            r->spare.n_cells = 0;
            r->launches++;
            st = size_for_graph(r, d);                    // the clean bank's log may be smaller
            if (st != CFPQ_OK) return st;
            if (r->log_cap < r->spare.log_cap) {          // the other bank's log grew last run
                uint64_t* nl = nullptr;
                if ((st = dalloc(&nl, r->spare.log_cap, "cell log")) != CFPQ_OK) return st;
                CFPQ_CUDA_TRY(cudaMemsetAsync(nl, 0, r->spare.log_cap * 8, s));
                dfree(r->d_log);
                r->d_log = nl;
                r->log_cap = r->spare.log_cap;
            }
            if (r->hashed && (st = ensure_hash(r)) != CFPQ_OK) return st;
            p = r->params();
        } else {
            if (log_clear) CFPQ_CUDA_TRY(launch_clear_log(p, r->n_cells, s));
            if (r->hashed) CFPQ_CUDA_TRY(cudaMemsetAsync(r->d_hset, 0xff, r->hcap * 8, s));
            r->launches++;
        }
    }
    r->ran = true;
    r->n_cells = 0;
    const bool fused = r->opts.path_policy < 2 && r->n_ranks == 1 && !r->comm && !r->xr && r->opts.schedule != 2 &&
                       (r->opts.diag_flags & 512) == 0;   // seeding inside the closure kernel
    if (r->n_adj_slots && !fused)
        CFPQ_CUDA_TRY(cudaMemsetAsync(r->d_adj_cnt, 0, (size_t)r->n_adj_slots * (r->n + 1) * 4, s));
    if (r->opts.account_work) CFPQ_CUDA_TRY(cudaMemsetAsync(r->d_jac, 0, r->iter_off_cap * 8, s));
    CFPQ_CUDA_TRY(cudaMemsetAsync(r->d_st, 0, sizeof(EngineState), s));
    const bool async = r->opts.schedule == 2;
    // async valid flags (bit 63): every log buffer is zeroed when allocated, no other schedule
    // sets bit 63 (A < 512), and every async run strips its flags, so no per-run clear
    if (r->opts.record_times) CFPQ_CUDA_TRY(cudaMemsetAsync(r->d_phase, 0, r->iter_off_cap * 32, s));
    if (!r->ev[0])
        for (auto& e : r->ev) CFPQ_CUDA_TRY(cudaEventCreate(&e));
    r->seed_ns = r->loop_ns = 0;
    CFPQ_CUDA_TRY(cudaEventRecord(r->ev[0], s));

    // a1: seed T_0; Δ_0 = the distinct seed cells.  One-GPU sparse runs seed
    // inside the closure kernel (fused_seed_phase); the other engines run the seed kernels.
    const unsigned long long seeds_upper = (unsigned long long)d->n_edges * (unsigned long long)r->max_rules_per_label;
    if (fused) {
        if (!r->d_scan_tot) {
            cfpq_status sa = dalloc(&r->d_scan_tot, (size_t)r->grid + 1, "scan totals");
            if (sa != CFPQ_OK) return sa;
        }
        CFPQ_CUDA_TRY(cudaEventRecord(r->ev[1], s));
        return run_sparse_loop(r, d, true);
    }
    CFPQ_CUDA_TRY(launch_seed(d->d_edges, d->n_edges, (int32_t)r->n, r->d_lab_ptr, r->d_lab_nt, r->n_labels,
                              r->max_rules_per_label, p, s));
    r->launches += 1;
    // preterminal adjacency (CSR rows / CSC columns + ELL heads), built once per closure:
    // count (also opens iteration 1), scan, fill (+ ELL heads; consumes the counts)
    if (r->n_adj_slots) {
        const size_t adj_len = (size_t)r->n_adj_slots * (r->n + 1);
        CFPQ_CUDA_TRY(cudaMemsetAsync(r->d_adj_ell, 0, (size_t)r->n_adj_slots * r->n * sizeof(int4), s));
        CFPQ_CUDA_TRY(launch_adj_count(p, r->d_slot_row, r->d_slot_col, r->d_adj_cnt, seeds_upper, s));
        CFPQ_CUDA_TRY(launch_scan(r->d_adj_cnt, r->d_adj_ptr, (int64_t)adj_len, r->d_temp, &r->temp_bytes, s));
        CFPQ_CUDA_TRY(launch_adj_fill(p, r->d_slot_row, r->d_slot_col, r->d_adj_ptr, r->d_adj_cnt, r->d_adj_idx,
                                      r->d_adj_ell, seeds_upper, s));
        r->launches += 4;   // count, CUB scan (init + scan), fill
    } else {
        CFPQ_CUDA_TRY(launch_begin(p, s));
        r->launches += 1;
    }
    if (r->has_snapshots) {
        CFPQ_CUDA_TRY(launch_seed_snapshots(p, seeds_upper, s));
        r->launches++;
    }
    CFPQ_CUDA_TRY(cudaEventRecord(r->ev[1], s));
    if (r->opts.path_policy == 2 || r->opts.path_policy == 3) return run_dense(r, 0);
    if (async) return run_async(r, seeds_upper);
    if (r->xr) return run_xr(r, d);
    if (r->n_ranks > 1 || r->comm) return run_sharded(r);
    return run_sparse_loop(r, d, false);
}

// ------------------------------------------------------------------------------------------
// closure entry points
// ------------------------------------------------------------------------------------------
static cfpq_status check_inputs(const cfpq_grammar* g, const cfpq_graph* d, const cfpq_options* o) {
    CFPQ_CHECK_ARG(g != nullptr && d != nullptr && o != nullptr, "cfpq_closure: NULL grammar/graph/options");
    CFPQ_CHECK_ARG(o->semantics == 0 || o->semantics == 1, "cfpq_closure: semantics must be 0 or 1");
    CFPQ_CHECK_ARG(o->schedule >= 0 && o->schedule <= 3, "cfpq_closure: schedule must be 0, 1, 2 or 3");
    if (o->schedule == 3) {
        int lhs = 0;
        for (int A = 0; A < g->n_nt; ++A) lhs += g->is_const[A] ? 0 : 1;
        if (o->semantics != 0 || o->path_policy > 1 || o->world_size > 1 || o->reserved_emulate > 1 ||
            o->account_work || lhs > kMaxStages) {
            set_error("cfpq_closure: schedule 3 (Gauss-Seidel) is relational, sparse-engine, one GPU, no work "
                      "accounting, at most 64 LHS nonterminals");
            return CFPQ_E_UNSUPPORTED;
        }
    }
    if (o->schedule == 2 && (o->semantics != 0 || o->path_policy > 1 || g->n_nt > 512)) {
        set_error("cfpq_closure: schedule 2 (asynchronous) is relational, sparse-engine only, |N| <= 512");
        return CFPQ_E_UNSUPPORTED;
    }
    CFPQ_CHECK_ARG(o->world_size >= 0 && o->reserved_emulate >= 0, "cfpq_closure: bad world_size / emulate_ranks");
    if ((o->world_size > 1 || o->reserved_emulate > 1) && (o->path_policy == 0 || o->path_policy == 1)) {
        // sparse-engine sharding: each rank derives the cells of its rows from the whole Δ
        // list, so every rule needs a preterminal operand (no rows of T from other ranks)
        bool varvar = false;
        for (auto& rl : g->rules) varvar |= !g->is_const[rl.B] && !g->is_const[rl.C];
        if (varvar || o->semantics != 0 || o->schedule == 2) {
            set_error("cfpq_closure: row-block sharding of the sparse engine needs relational semantics, "
                      "schedule 0/1 and a preterminal operand in every rule (use path_policy 2 otherwise)");
            return CFPQ_E_UNSUPPORTED;
        }
    }
    if (o->world_size > 1) {
        CFPQ_CHECK_ARG(o->rank >= 0 && o->rank < o->world_size, "cfpq_closure: rank out of range");
        CFPQ_CHECK_ARG(o->nccl_unique_id != nullptr, "cfpq_closure: world_size > 1 needs nccl_unique_id");
    }
    if (o->path_policy == 3 && d->n_nodes > 262144) {
        set_error("cfpq_closure: the bit-row path keeps a row in registers: n_nodes <= 262144");
        return CFPQ_E_UNSUPPORTED;
    }
    if ((o->path_policy == 2 || o->path_policy == 3) && o->semantics == 1) {
        set_error("cfpq_closure: single-path lengths need the sparse engine (min-plus is not a Boolean product)");
        return CFPQ_E_UNSUPPORTED;
    }
    CFPQ_CHECK_ARG(o->path_policy >= 0 && o->path_policy <= 3, "cfpq_closure: bad path_policy");
    CFPQ_CHECK_ARG(o->grid_rows >= 0 && o->grid_cols >= 0, "cfpq_closure: negative grid");
    if (o->grid_rows > 0 || o->grid_cols > 0) {
        const int shards = o->world_size > 1 ? o->world_size : (o->reserved_emulate > 1 ? o->reserved_emulate : 1);
        if (o->path_policy != 2 || o->grid_rows * o->grid_cols != shards) {
            set_error("cfpq_closure: a 2-D grid needs the tensor engine (path_policy 2) and grid_rows * grid_cols "
                      "= world_size (or emulated shards)");
            return CFPQ_E_UNSUPPORTED;
        }
    }
    CFPQ_CHECK_ARG(o->dense_launch >= 0 && o->dense_launch <= 3, "cfpq_closure: dense_launch must be 0..3");
    CFPQ_CHECK_ARG(o->exchange == 0 || o->exchange == 1, "cfpq_closure: exchange must be 0 or 1");
    CFPQ_CHECK_ARG(o->cell_set >= 0 && o->cell_set <= 2, "cfpq_closure: cell_set must be 0, 1 or 2");
    CFPQ_CHECK_ARG(o->tensor_format >= 0 && o->tensor_format <= 2, "cfpq_closure: tensor_format must be 0, 1 or 2");
    return CFPQ_OK;
}

extern "C" cfpq_status cfpq_closure(const cfpq_grammar* g, const cfpq_graph* d, const cfpq_options* o,
                                    cfpq_result** out) {
    CFPQ_CHECK_ARG(out != nullptr, "cfpq_closure: out is NULL");
    cfpq_status st = check_inputs(g, d, o);
    if (st != CFPQ_OK) return st;
    cfpq_result* r = new cfpq_result();
    st = plan(r, g, d, o);
    if (st == CFPQ_OK) st = run(r, d);
    if (st != CFPQ_OK && st != CFPQ_E_NOT_CONVERGED && st != CFPQ_E_OVERFLOW) {
        std::string keep = g_last_error;
        delete r;
        set_error(keep);
        return st;
    }
    *out = r;
    return st;
}

extern "C" cfpq_status cfpq_closure_reuse(const cfpq_grammar* g, const cfpq_graph* d, const cfpq_options* o,
                                          cfpq_result* r) {
    CFPQ_CHECK_ARG(r != nullptr, "cfpq_closure_reuse: result is NULL");
    cfpq_status st = check_inputs(g, d, o);
    if (st != CFPQ_OK) return st;
    CFPQ_CHECK_ARG(d->n_nodes == r->n && g->n_nt == r->n_nt && g->n_labels == r->n_labels &&
                       g->rules.size() == r->rules.size() && o->semantics == r->opts.semantics &&
                       o->account_work == r->opts.account_work && o->path_policy == r->opts.path_policy &&
                       o->cell_set == r->opts.cell_set && o->tensor_format == r->opts.tensor_format &&
                       o->exchange == r->opts.exchange,
                   "cfpq_closure_reuse: grammar/graph/options differ from the result's plan");
    for (size_t k = 0; k < g->rules.size(); ++k)
        CFPQ_CHECK_ARG(g->rules[k].A == r->rules[k].A && g->rules[k].B == r->rules[k].B && g->rules[k].C == r->rules[k].C,
                       "cfpq_closure_reuse: grammar differs from the result's plan");
    CFPQ_CHECK_ARG(g->term == r->term, "cfpq_closure_reuse: terminal rules differ from the result's plan");
    r->stream = (cudaStream_t)o->cuda_stream;
    r->opts.cuda_stream = o->cuda_stream;
    // every option of this call applies to the re-run: max_iterations 0 restores the Theorem 3
    // default, and the per-iteration buffers grow with a larger cap
    r->opts.max_iterations = o->max_iterations > 0 ? o->max_iterations : theorem3_cap(r->n, r->n_nt);
    {
        cfpq_status sb = size_iteration_buffers(r);
        if (sb != CFPQ_OK) return sb;
    }
    r->opts.solo_threshold = o->solo_threshold >= 0 ? o->solo_threshold : 1024;
    r->opts.record_times = o->record_times;
    if (o->schedule == 2 && (r->opts.semantics != 0 || r->n_nt > 512)) {
        set_error("cfpq_closure_reuse: schedule 2 is relational with |N| <= 512");
        return CFPQ_E_UNSUPPORTED;
    }
    r->opts.schedule = o->schedule;
    return run(r, d);
}

extern "C" void cfpq_result_destroy(cfpq_result* r) {
    if (!r) return;
    cudaStreamSynchronize(r->stream);
    delete r;
}

extern "C" cfpq_status cfpq_result_iterations(const cfpq_result* r, int64_t* out) {
    CFPQ_CHECK_ARG(r && out, "cfpq_result_iterations: NULL argument");
    *out = r->iterations;
    return CFPQ_OK;
}

// cells of T_k live in log[0, end_of(k)); k < 0 -> the final T
static unsigned long long log_end(cfpq_result* r, int64_t k, cfpq_status* st) {
    *st = CFPQ_OK;
    if (k < 0 || k >= r->iterations) return r->n_cells;
    if (k + 1 >= r->iter_off_cap) {
        set_error("per-iteration offsets were not recorded for this iteration");
        *st = CFPQ_E_UNSUPPORTED;
        return 0;
    }
    unsigned long long v = 0;
    cudaError_t e = cudaMemcpy(&v, r->d_iter_off + k + 1, 8, cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) {
        set_error(cudaGetErrorString(e));
        *st = CFPQ_E_CUDA;
    }
    return v;
}

static cfpq_status counts_upto(cfpq_result* r, unsigned long long end, std::vector<int64_t>& out) {
    cudaStream_t s = r->stream;
    CFPQ_CUDA_TRY(cudaMemsetAsync(r->d_small, 0, (r->n_nt + 2) * 8, s));
    CFPQ_CUDA_TRY(launch_nt_histogram(r->d_log, end, r->d_small, r->n_nt, s));
    std::vector<unsigned long long> h(r->n_nt);
    CFPQ_CUDA_TRY(cudaMemcpyAsync(h.data(), r->d_small, r->n_nt * 8, cudaMemcpyDeviceToHost, s));
    CFPQ_CUDA_TRY(cudaStreamSynchronize(s));
    out.assign(h.begin(), h.end());
    return CFPQ_OK;
}

// |R_A| from the bit matrix (dense-engine results)
static cfpq_status bitmap_count(cfpq_result* r, int32_t nt, int64_t* out) {
    cudaStream_t s = r->stream;
    CFPQ_CUDA_TRY(cudaMemsetAsync(r->d_small, 0, 8, s));
    CFPQ_CUDA_TRY(launch_bitmap_rowcount(r->h_nt[nt].T, (int32_t)r->n, r->Wp, nullptr, r->d_small, s));
    unsigned long long v = 0;
    CFPQ_CUDA_TRY(cudaMemcpyAsync(&v, r->d_small, 8, cudaMemcpyDeviceToHost, s));
    CFPQ_CUDA_TRY(cudaStreamSynchronize(s));
    *out = (int64_t)v;
    return CFPQ_OK;
}

extern "C" cfpq_status cfpq_result_count(cfpq_result* r, int32_t nt, int64_t* out) {
    CFPQ_CHECK_ARG(r && out, "cfpq_result_count: NULL argument");
    CFPQ_CHECK_ARG(nt >= 0 && nt < r->n_nt, "cfpq_result_count: NT id out of range");
    if (r->dense_mode) return bitmap_count(r, nt, out);
    if (!r->counts_valid) {
        cfpq_status st = counts_upto(r, r->n_cells, r->counts);
        if (st != CFPQ_OK) return st;
        r->counts_valid = true;
    }
    *out = r->counts[nt];
    return CFPQ_OK;
}

extern "C" cfpq_status cfpq_result_count_at(cfpq_result* r, int32_t nt, int64_t k, int64_t* out) {
    CFPQ_CHECK_ARG(r && out, "cfpq_result_count_at: NULL argument");
    CFPQ_CHECK_ARG(nt >= 0 && nt < r->n_nt, "cfpq_result_count_at: NT id out of range");
    CFPQ_CHECK_ARG(k >= 0, "cfpq_result_count_at: k < 0");
    if (r->dense_mode && k < r->iterations) {
        set_error("per-iteration states are kept only by the sparse engine");
        return CFPQ_E_UNSUPPORTED;
    }
    if (r->dense_mode) return bitmap_count(r, nt, out);
    cfpq_status st;
    unsigned long long end = log_end(r, k, &st);
    if (st != CFPQ_OK) return st;
    std::vector<int64_t> c;
    st = counts_upto(r, end, c);
    if (st != CFPQ_OK) return st;
    *out = c[nt];
    return CFPQ_OK;
}

// sorted (i<<27|j) keys of NT `nt` among log[0,end) into r->d_keys; returns the count
// Extraction keys are (i << bits) | j with bits = ceil(log2 n): the radix sort touches only
// 2*bits key bits (4 passes at n = 65,536).
static int key_bits(const cfpq_result* r) {
    int bits = 1;
    while ((1ll << bits) < r->n) ++bits;
    return bits;
}

static bool keys32(const cfpq_result* r) { return 2 * key_bits(r) <= 32; }

// A's cells of log[0, end) as sorted compact keys in d_keys (uint32 if keys32(r)).  The
// filter counts on the device; one read-back sizes the sort.
static cfpq_status sorted_keys(cfpq_result* r, int32_t nt, unsigned long long end, unsigned long long* count) {
    cudaStream_t s = r->stream;
    cfpq_status st;
    if (2 * end + 2 > r->keys_cap) {
        dfree(r->d_keys);
        st = dalloc(&r->d_keys, 2 * end + 2, "extraction keys");
        if (st != CFPQ_OK) return st;
        r->keys_cap = 2 * end + 2;
    }
    const int bits = key_bits(r);
    const bool k32 = keys32(r);
    CFPQ_CUDA_TRY(cudaMemsetAsync(r->d_small + r->n_nt, 0, 8, s));
    CFPQ_CUDA_TRY(launch_filter_nt(r->d_log, end, (uint32_t)nt, r->d_keys, r->d_small + r->n_nt, bits, k32, s));
    unsigned long long m = 0;
    CFPQ_CUDA_TRY(cudaMemcpyAsync(&m, r->d_small + r->n_nt, 8, cudaMemcpyDeviceToHost, s));
    CFPQ_CUDA_TRY(cudaStreamSynchronize(s));
    if (m > 1) {
        const int end_bit = 2 * bits;
        size_t need = 0;
        uint32_t* k4 = reinterpret_cast<uint32_t*>(r->d_keys);
        if (k32) CFPQ_CUDA_TRY(sort_keys32(k4, k4 + m, m, end_bit, nullptr, &need, s));
        else CFPQ_CUDA_TRY(sort_keys(r->d_keys, r->d_keys + m + 1, m, end_bit, nullptr, &need, s));
        if (need > r->temp_bytes) {
            dfree(r->d_temp);
            st = dalloc((uint8_t**)&r->d_temp, need, "sort temp");
            if (st != CFPQ_OK) return st;
            r->temp_bytes = need;
        }
        if (k32) CFPQ_CUDA_TRY(sort_keys32(k4, k4 + m, m, end_bit, r->d_temp, &r->temp_bytes, s));
        else CFPQ_CUDA_TRY(sort_keys(r->d_keys, r->d_keys + m + 1, m, end_bit, r->d_temp, &r->temp_bytes, s));
    }
    *count = m;
    return CFPQ_OK;
}

static cfpq_status bitmap_pairs(cfpq_result* r, int32_t nt, int32_t* dst, int64_t capacity, int32_t on_dev,
                                int64_t* written) {
    cudaStream_t s = r->stream;
    const int64_t n = r->n;
    CFPQ_CUDA_TRY(cudaMemsetAsync(r->d_small, 0, 8, s));
    CFPQ_CUDA_TRY(cudaMemsetAsync(r->d_rowcnt + n, 0, 4, s));
    CFPQ_CUDA_TRY(launch_bitmap_rowcount(r->h_nt[nt].T, (int32_t)n, r->Wp, r->d_rowcnt, r->d_small, s));
    unsigned long long m = 0;
    CFPQ_CUDA_TRY(cudaMemcpyAsync(&m, r->d_small, 8, cudaMemcpyDeviceToHost, s));
    CFPQ_CUDA_TRY(cudaStreamSynchronize(s));
    *written = (int64_t)m;
    CFPQ_CHECK_ARG((int64_t)m <= capacity, "cfpq_result_pairs: capacity < |R_A|");
    CFPQ_CHECK_ARG(m == 0 || dst != nullptr, "cfpq_result_pairs: dst is NULL");
    if (m == 0) return CFPQ_OK;
    size_t need = 0;
    CFPQ_CUDA_TRY(launch_scan(nullptr, nullptr, n + 1, nullptr, &need, s));
    if (need > r->temp_bytes) {
        dfree(r->d_temp);
        cfpq_status st = dalloc((uint8_t**)&r->d_temp, need, "scan temp");
        if (st != CFPQ_OK) return st;
        r->temp_bytes = need;
    }
    CFPQ_CUDA_TRY(launch_scan(r->d_rowcnt, r->d_rowoff, n + 1, r->d_temp, &r->temp_bytes, s));
    int32_t* tmp = dst;
    if (!on_dev) {
        if (m + 1 > r->keys_cap) {
            dfree(r->d_keys);
            cfpq_status st = dalloc(&r->d_keys, m + 1, "extraction scratch");
            if (st != CFPQ_OK) return st;
            r->keys_cap = m + 1;
        }
        tmp = (int32_t*)r->d_keys;
    }
    CFPQ_CUDA_TRY(launch_bitmap_pairs(r->h_nt[nt].T, (int32_t)n, r->Wp, r->d_rowoff, tmp, s));
    if (!on_dev) CFPQ_CUDA_TRY(cudaMemcpyAsync(dst, tmp, m * 2 * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    CFPQ_CUDA_TRY(cudaStreamSynchronize(s));
    return CFPQ_OK;
}

static cfpq_status pairs_impl(cfpq_result* r, int32_t nt, int64_t k, int32_t* dst, int64_t capacity, int32_t on_dev,
                              int64_t* written) {
    CFPQ_CHECK_ARG(r && written, "cfpq_result_pairs: NULL argument");
    CFPQ_CHECK_ARG(nt >= 0 && nt < r->n_nt, "cfpq_result_pairs: NT id out of range");
    if (r->dense_mode) {
        if (k >= 0 && k < r->iterations) {
            set_error("per-iteration states are kept only by the sparse engine");
            return CFPQ_E_UNSUPPORTED;
        }
        return bitmap_pairs(r, nt, dst, capacity, on_dev, written);
    }
    cfpq_status st;
    unsigned long long end = log_end(r, k, &st);
    if (st != CFPQ_OK) return st;
    unsigned long long m = 0;
    st = sorted_keys(r, nt, end, &m);
    if (st != CFPQ_OK) return st;
    *written = (int64_t)m;
    CFPQ_CHECK_ARG((int64_t)m <= capacity, "cfpq_result_pairs: capacity < |R_A|");
    CFPQ_CHECK_ARG(m == 0 || dst != nullptr, "cfpq_result_pairs: dst is NULL");
    if (m == 0) return CFPQ_OK;
    cudaStream_t s = r->stream;
    // unpack into the upper half of the key scratch (2m int32 = m uint64), then copy out
    int32_t* tmp = on_dev ? dst : (int32_t*)(r->d_keys + m + 1);
    CFPQ_CUDA_TRY(launch_unpack_pairs(r->d_keys, m, tmp, key_bits(r), keys32(r), s));
    if (!on_dev) {
        CFPQ_CUDA_TRY(cudaMemcpyAsync(dst, tmp, m * 2 * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    }
    CFPQ_CUDA_TRY(cudaStreamSynchronize(s));
    return CFPQ_OK;
}

extern "C" cfpq_status cfpq_result_pairs(cfpq_result* r, int32_t nt, int32_t* dst_pairs, int64_t capacity,
                                         int32_t dst_is_device, int64_t* written) {
    return pairs_impl(r, nt, -1, dst_pairs, capacity, dst_is_device, written);
}

// R_A in compressed-row form: the same sorted keys as cfpq_result_pairs (sparse engines) or the
// bit-matrix rows (dense engine), written as row pointers + columns.
extern "C" cfpq_status cfpq_result_csr(cfpq_result* r, int32_t nt, int64_t* row_ptr, int32_t* cols, int64_t capacity,
                                       int32_t dst_is_device, int64_t* written) {
    CFPQ_CHECK_ARG(r && written, "cfpq_result_csr: NULL argument");
    CFPQ_CHECK_ARG(nt >= 0 && nt < r->n_nt, "cfpq_result_csr: NT id out of range");
    CFPQ_CHECK_ARG(row_ptr != nullptr, "cfpq_result_csr: row_ptr is NULL");
    cudaStream_t s = r->stream;
    const int64_t n = r->n;
    cfpq_status st;
    int64_t* ptr_dev = row_ptr;
    if (!dst_is_device) {
        if (!r->d_csr_ptr && (st = dalloc(&r->d_csr_ptr, (size_t)n + 1, "CSR row pointers")) != CFPQ_OK) return st;
        ptr_dev = r->d_csr_ptr;
    }
    unsigned long long m = 0;
    int32_t* cols_dev = cols;
    if (r->dense_mode) {
        CFPQ_CUDA_TRY(cudaMemsetAsync(r->d_small, 0, 8, s));
        CFPQ_CUDA_TRY(cudaMemsetAsync(r->d_rowcnt + n, 0, 4, s));
        CFPQ_CUDA_TRY(launch_bitmap_rowcount(r->h_nt[nt].T, (int32_t)n, r->Wp, r->d_rowcnt, r->d_small, s));
        CFPQ_CUDA_TRY(cudaMemcpyAsync(&m, r->d_small, 8, cudaMemcpyDeviceToHost, s));
        CFPQ_CUDA_TRY(cudaStreamSynchronize(s));
        *written = (int64_t)m;
        CFPQ_CHECK_ARG((int64_t)m <= capacity, "cfpq_result_csr: capacity < |R_A|");
        CFPQ_CHECK_ARG(m == 0 || cols != nullptr, "cfpq_result_csr: cols is NULL");
        size_t need = 0;
        CFPQ_CUDA_TRY(launch_scan(nullptr, nullptr, n + 1, nullptr, &need, s));
        if (need > r->temp_bytes) {
            dfree(r->d_temp);
            if ((st = dalloc((uint8_t**)&r->d_temp, need, "scan temp")) != CFPQ_OK) return st;
            r->temp_bytes = need;
        }
        CFPQ_CUDA_TRY(launch_scan(r->d_rowcnt, r->d_rowoff, n + 1, r->d_temp, &r->temp_bytes, s));
        if (!dst_is_device && m) {
            if ((m + 1) / 2 + 1 > r->keys_cap) {
                dfree(r->d_keys);
                if ((st = dalloc(&r->d_keys, (m + 1) / 2 + 1, "extraction scratch")) != CFPQ_OK) return st;
                r->keys_cap = (m + 1) / 2 + 1;
            }
            cols_dev = (int32_t*)r->d_keys;
        }
        if (m) CFPQ_CUDA_TRY(launch_bitmap_pairs(r->h_nt[nt].T, (int32_t)n, r->Wp, r->d_rowoff, cols_dev, s, 1));
        CFPQ_CUDA_TRY(launch_rowoff_to_ptr(r->d_rowoff, n, ptr_dev, s));
    } else {
        unsigned long long end = log_end(r, -1, &st);
        if (st != CFPQ_OK) return st;
        if ((st = sorted_keys(r, nt, end, &m)) != CFPQ_OK) return st;
        *written = (int64_t)m;
        CFPQ_CHECK_ARG((int64_t)m <= capacity, "cfpq_result_csr: capacity < |R_A|");
        CFPQ_CHECK_ARG(m == 0 || cols != nullptr, "cfpq_result_csr: cols is NULL");
        if (!dst_is_device) cols_dev = (int32_t*)(r->d_keys + m + 1);   // upper half of the key scratch
        CFPQ_CUDA_TRY(launch_keys_to_csr(r->d_keys, m, key_bits(r), keys32(r), n, ptr_dev, cols_dev, s));
    }
    if (!dst_is_device) {
        CFPQ_CUDA_TRY(cudaMemcpyAsync(row_ptr, ptr_dev, (size_t)(n + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
        if (m) CFPQ_CUDA_TRY(cudaMemcpyAsync(cols, cols_dev, m * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    }
    CFPQ_CUDA_TRY(cudaStreamSynchronize(s));
    return CFPQ_OK;
}

extern "C" cfpq_status cfpq_result_pairs_at(cfpq_result* r, int32_t nt, int64_t k, int32_t* dst_pairs,
                                            int64_t capacity, int32_t dst_is_device, int64_t* written) {
    CFPQ_CHECK_ARG(k >= 0, "cfpq_result_pairs_at: k < 0");
    return pairs_impl(r, nt, k, dst_pairs, capacity, dst_is_device, written);
}

extern "C" cfpq_status cfpq_result_matrix(cfpq_result* r, int32_t nt, uint32_t* dst, int64_t row_stride_words,
                                          int32_t dst_is_device) {
    CFPQ_CHECK_ARG(r && dst, "cfpq_result_matrix: NULL argument");
    CFPQ_CHECK_ARG(nt >= 0 && nt < r->n_nt, "cfpq_result_matrix: NT id out of range");
    const int64_t wn = (r->n + 31) / 32;
    CFPQ_CHECK_ARG(row_stride_words >= wn, "cfpq_result_matrix: row_stride_words < ceil(n/32)");
    if (r->n == 0) return CFPQ_OK;
    // the log holds every cell when there are no bit matrices (hashed set), when the kernel
    // reset them at the fixpoint (t_clean), or when NCCL row shards derived only their own
    // rows into T (the log has every rank's cells after the exchange)
    const bool sparse_sharded = r->comm != nullptr && !r->dense_mode;
    if (r->hashed || r->t_clean || sparse_sharded) {
        // no (complete) bit matrices: scatter A's cells from the log
        cudaStream_t s = r->stream;
        uint32_t* d = dst;
        int64_t stride = row_stride_words;
        uint32_t* tmp = nullptr;
        if (!dst_is_device) {
            cfpq_status st = dalloc(&tmp, (size_t)wn * r->n, "matrix scratch");
            if (st != CFPQ_OK) return st;
            d = tmp;
            stride = wn;
        }
        CFPQ_CUDA_TRY(cudaMemset2DAsync(d, stride * 4, 0, wn * 4, r->n, s));
        CFPQ_CUDA_TRY(launch_log_to_bitmap(r->d_log, r->n_cells, (uint32_t)nt, d, stride, s));
        if (tmp) {
            cudaError_t e = cudaMemcpy2DAsync(dst, row_stride_words * 4, tmp, wn * 4, wn * 4, r->n,
                                              cudaMemcpyDeviceToHost, s);
            if (e == cudaSuccess) e = cudaStreamSynchronize(s);
            dfree(tmp);
            CFPQ_CUDA_TRY(e);
        }
        CFPQ_CUDA_TRY(cudaStreamSynchronize(s));
        return CFPQ_OK;
    }
    const uint32_t* src = r->h_nt[nt].T;
    CFPQ_CUDA_TRY(cudaMemcpy2DAsync(dst, row_stride_words * 4, src, r->Wp * 4, wn * 4, r->n,
                                    dst_is_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, r->stream));
    CFPQ_CUDA_TRY(cudaStreamSynchronize(r->stream));
    return CFPQ_OK;
}

extern "C" cfpq_status cfpq_result_lengths(cfpq_result* r, int32_t nt, uint32_t* dst_len, int64_t capacity,
                                           int32_t dst_is_device, int64_t* written) {
    CFPQ_CHECK_ARG(r && written, "cfpq_result_lengths: NULL argument");
    CFPQ_CHECK_ARG(nt >= 0 && nt < r->n_nt, "cfpq_result_lengths: NT id out of range");
    if (r->opts.semantics != 1) {
        set_error("cfpq_result_lengths: the closure ran with relational semantics");
        return CFPQ_E_INVAL;
    }
    unsigned long long m = 0;
    cfpq_status st = sorted_keys(r, nt, r->n_cells, &m);
    if (st != CFPQ_OK) return st;
    *written = (int64_t)m;
    CFPQ_CHECK_ARG((int64_t)m <= capacity, "cfpq_result_lengths: capacity < |R_A|");
    CFPQ_CHECK_ARG(m == 0 || dst_len != nullptr, "cfpq_result_lengths: dst is NULL");
    if (m == 0) return CFPQ_OK;
    cudaStream_t s = r->stream;
    uint32_t* tmp = dst_is_device ? dst_len : (uint32_t*)(r->d_keys + m + 1);
    CFPQ_CUDA_TRY(launch_gather_lengths(r->d_keys, m, r->h_nt[nt].K, r->n, tmp, key_bits(r), keys32(r), s));
    if (!dst_is_device) CFPQ_CUDA_TRY(cudaMemcpyAsync(dst_len, tmp, m * 4, cudaMemcpyDeviceToHost, s));
    CFPQ_CUDA_TRY(cudaStreamSynchronize(s));
    return CFPQ_OK;
}

extern "C" cfpq_status cfpq_result_stats(const cfpq_result* r, int64_t* stats, int32_t n_stats) {
    CFPQ_CHECK_ARG(r && stats, "cfpq_result_stats: NULL argument");
    int64_t v[22] = {r->iterations, (int64_t)r->n_cells, (int64_t)r->log_cap, r->regrows, r->launches,
                     r->h_st.solo_iters, (int64_t)r->h_st.candidates, (int64_t)r->h_st.expansions,
                     (int64_t)r->seed_ns, (int64_t)r->loop_ns, (int64_t)r->grid,
                     (int64_t)r->h_st.prof[0], (int64_t)r->h_st.prof[1], (int64_t)r->h_st.prof[2],
                     (int64_t)r->h_st.prof[3], (int64_t)r->h_st.prof[4], (int64_t)r->h_st.prof[5],
                     (int64_t)r->h_st.prof[6], (int64_t)r->dense_kb, (int64_t)r->dense_mode,
                     (int64_t)r->hashed, (int64_t)r->hcap};
    for (int k = 0; k < n_stats && k < 22; ++k) stats[k] = v[k];
    return CFPQ_OK;
}

extern "C" cfpq_status cfpq_result_iteration_stats(cfpq_result* r, int64_t* new_cells, int64_t* jacobi_triples,
                                                   int64_t capacity) {
    return cfpq_result_iteration_stats2(r, new_cells, jacobi_triples, nullptr, capacity);
}

extern "C" cfpq_status cfpq_result_iteration_stats2(cfpq_result* r, int64_t* new_cells, int64_t* jacobi_triples,
                                                    int64_t* end_ns, int64_t capacity) {
    CFPQ_CHECK_ARG(r, "cfpq_result_iteration_stats: NULL result");
    int64_t k = std::min<int64_t>(r->iterations, capacity);
    k = std::min<int64_t>(k, r->iter_off_cap - 2);
    if (k <= 0) return CFPQ_OK;
    if (r->dense_mode) {
        if (new_cells)
            for (int64_t t = 0; t < k; ++t) new_cells[t] = r->dense_new[t];
        if (jacobi_triples) {
            if ((int64_t)r->dense_jac.size() < k) {
                set_error("cfpq_result_iteration_stats: run with account_work = 1 for work counts");
                return CFPQ_E_INVAL;
            }
            for (int64_t t = 0; t < k; ++t) jacobi_triples[t] = r->dense_jac[t];
        }
        if (end_ns) {
            set_error("iteration times are recorded by the sparse engine only");
            return CFPQ_E_UNSUPPORTED;
        }
        return CFPQ_OK;
    }
    std::vector<unsigned long long> off(k + 2);
    CFPQ_CUDA_TRY(cudaMemcpy(off.data(), r->d_iter_off, (k + 2) * 8, cudaMemcpyDeviceToHost));
    if (new_cells)
        for (int64_t t = 1; t <= k; ++t) new_cells[t - 1] = (int64_t)(off[t + 1] - off[t]);
    if (jacobi_triples) {
        if (!r->d_jac) {
            set_error("cfpq_result_iteration_stats: run with account_work = 1 for work counts");
            return CFPQ_E_INVAL;
        }
        std::vector<unsigned long long> j(k + 1);
        CFPQ_CUDA_TRY(cudaMemcpy(j.data(), r->d_jac, (k + 1) * 8, cudaMemcpyDeviceToHost));
        for (int64_t t = 1; t <= k; ++t) jacobi_triples[t - 1] = (int64_t)j[t];
    }
    if (end_ns) {
        std::vector<unsigned long long> t(k + 1);
        CFPQ_CUDA_TRY(cudaMemcpy(t.data(), r->d_iter_time, (k + 1) * 8, cudaMemcpyDeviceToHost));
        for (int64_t q = 1; q <= k; ++q) end_ns[q - 1] = (int64_t)(t[q] - t[0]);
    }
    return CFPQ_OK;
}

// Single-path witness on the GPU (witness.cu): the path of the recorded length of (A,i,j).
extern "C" cfpq_status cfpq_result_witness(cfpq_result* r, const cfpq_graph* d, int32_t nt, int32_t i, int32_t j,
                                           int32_t* out_edges, int64_t capacity, int32_t dst_is_device,
                                           int64_t* written) {
    CFPQ_CHECK_ARG(r && d && written, "cfpq_result_witness: NULL argument");
    CFPQ_CHECK_ARG(r->opts.semantics == 1, "cfpq_result_witness: the closure ran with relational semantics");
    CFPQ_CHECK_ARG(nt >= 0 && nt < r->n_nt, "cfpq_result_witness: NT id out of range");
    CFPQ_CHECK_ARG(i >= 0 && i < r->n && j >= 0 && j < r->n, "cfpq_result_witness: node out of range");
    CFPQ_CHECK_ARG(d->n_nodes == r->n, "cfpq_result_witness: graph differs from the result's");
    cudaStream_t s = r->stream;
    // the recorded length of (A,i,j)
    uint64_t len = 0;
    const NTInfo& t = r->h_nt[nt];
    if (t.K) {
        uint64_t v = 0;
        CFPQ_CUDA_TRY(cudaMemcpyAsync(&v, t.K + (size_t)i * r->n + j, 8, cudaMemcpyDeviceToHost, s));
        CFPQ_CUDA_TRY(cudaStreamSynchronize(s));
        len = v == kEmptyKey ? 0 : (v & 0xffffffffull);
    } else {
        uint32_t w = 0;
        CFPQ_CUDA_TRY(cudaMemcpyAsync(&w, t.T + (size_t)i * r->Wp + (j >> 5), 4, cudaMemcpyDeviceToHost, s));
        CFPQ_CUDA_TRY(cudaStreamSynchronize(s));
        len = (w >> (j & 31)) & 1u;
    }
    *written = (int64_t)len;
    if (len == 0) {
        set_error("cfpq_result_witness: (A, i, j) is not in R_A");
        return CFPQ_E_INVAL;
    }
    CFPQ_CHECK_ARG((int64_t)len <= capacity, "cfpq_result_witness: capacity < path length");
    CFPQ_CHECK_ARG(out_edges != nullptr, "cfpq_result_witness: out_edges is NULL");
    // binary rules grouped by LHS (grammar order inside a group)
    std::vector<int32_t> rule_ptr(r->n_nt + 1, 0), rule_ids(r->rules.size());
    for (auto& rl : r->rules) rule_ptr[rl.A + 1]++;
    for (int A = 0; A < r->n_nt; ++A) rule_ptr[A + 1] += rule_ptr[A];
    {
        std::vector<int32_t> cur(rule_ptr.begin(), rule_ptr.end() - 1);
        for (size_t q = 0; q < r->rules.size(); ++q) rule_ids[cur[r->rules[q].A]++] = (int32_t)q;
    }
    const int64_t n = r->n;
    int32_t *d_rp = nullptr, *d_ri = nullptr, *d_deg = nullptr, *d_ptr = nullptr, *d_cur = nullptr, *d_idx = nullptr;
    int32_t* d_out = nullptr;
    uint8_t* d_stack = nullptr;
    long long* d_res = nullptr;
    void* d_tmp = nullptr;
    size_t tb = 0;
    cfpq_status st = CFPQ_OK;
    auto cleanup = [&]() {
        dfree(d_rp); dfree(d_ri); dfree(d_deg); dfree(d_ptr); dfree(d_cur); dfree(d_idx); dfree(d_stack);
        dfree(d_res);
        if (!dst_is_device) dfree(d_out);
        if (d_tmp) cudaFree(d_tmp);
    };
    const int64_t stack_cap = (int64_t)len + 2;
    if ((st = dalloc(&d_rp, rule_ptr.size(), "witness rules")) != CFPQ_OK ||
        (st = dalloc(&d_ri, std::max<size_t>(rule_ids.size(), 1), "witness rules")) != CFPQ_OK ||
        (st = dalloc(&d_deg, (size_t)n + 1, "witness edge CSR")) != CFPQ_OK ||
        (st = dalloc(&d_ptr, (size_t)n + 1, "witness edge CSR")) != CFPQ_OK ||
        (st = dalloc(&d_cur, (size_t)n + 1, "witness edge CSR")) != CFPQ_OK ||
        (st = dalloc(&d_idx, (size_t)std::max<int64_t>(d->n_edges, 1), "witness edge CSR")) != CFPQ_OK ||
        (st = dalloc(&d_stack, (size_t)stack_cap * witness_frame_bytes(), "witness stack")) != CFPQ_OK ||
        (st = dalloc(&d_res, 1, "witness result")) != CFPQ_OK) {
        cleanup();
        return st;
    }
    if (dst_is_device) d_out = out_edges;
    else if ((st = dalloc(&d_out, (size_t)len * 3, "witness path")) != CFPQ_OK) {
        cleanup();
        return st;
    }
    cudaError_t e = cudaMemcpyAsync(d_rp, rule_ptr.data(), rule_ptr.size() * 4, cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess && !rule_ids.empty())
        e = cudaMemcpyAsync(d_ri, rule_ids.data(), rule_ids.size() * 4, cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess) e = launch_scan(nullptr, nullptr, n + 1, nullptr, &tb, s);
    if (e == cudaSuccess) e = cudaMalloc(&d_tmp, std::max<size_t>(tb, 256));
    if (e == cudaSuccess)
        e = launch_edge_csr(d->d_edges, d->n_edges, (int32_t)n, d_deg, d_ptr, d_cur, d_idx, d_tmp, &tb, s);
    if (e == cudaSuccess)
        e = launch_witness(r->params(), r->d_rules, d_rp, d_ri, d_ptr, d_idx, d->d_edges, r->d_lab_ptr, r->d_lab_nt,
                           r->n_labels, d_stack, stack_cap, (uint32_t)nt, (uint32_t)i, (uint32_t)j, (uint32_t)len, d_out,
                           (int64_t)len, d_res, s);
    long long res = 0;
    if (e == cudaSuccess) e = cudaMemcpyAsync(&res, d_res, 8, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess && !dst_is_device)
        e = cudaMemcpyAsync(out_edges, d_out, (size_t)len * 12, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    cleanup();
    CFPQ_CUDA_TRY(e);
    if (res != (long long)len) {
        set_error("cfpq_result_witness: the recorded lengths do not rebuild a derivation (code " +
                  std::to_string(res) + ")");
        return CFPQ_E_CUDA;
    }
    return CFPQ_OK;
}

extern "C" cfpq_status cfpq_result_iteration_phases(cfpq_result* r, int64_t* cycles, int64_t capacity) {
    CFPQ_CHECK_ARG(r != nullptr && cycles != nullptr, "cfpq_result_iteration_phases: NULL argument");
    CFPQ_CHECK_ARG(r->opts.record_times, "cfpq_result_iteration_phases: run with record_times = 1");
    const int64_t k = std::min<int64_t>(std::min<int64_t>(r->iterations, capacity), r->iter_off_cap - 1);
    CFPQ_CUDA_TRY(cudaStreamSynchronize(r->stream));
    std::vector<unsigned long long> ph((size_t)(k + 1) * 4);
    CFPQ_CUDA_TRY(cudaMemcpy(ph.data(), r->d_phase, ph.size() * 8, cudaMemcpyDeviceToHost));
    for (int64_t t = 1; t <= k; ++t)
        for (int q = 0; q < 4; ++q) {
            unsigned long long v = ph[(size_t)t * 4 + q];
            if (q == 2) v = v ? ~v : 0ull;
            cycles[(t - 1) * 4 + q] = (int64_t)v;
        }
    return CFPQ_OK;
}

extern "C" const char* cfpq_last_error(void) { return g_last_error.c_str(); }

extern "C" cfpq_status cfpq_nccl_unique_id(void* out, int64_t bytes) {
    CFPQ_CHECK_ARG(out != nullptr, "cfpq_nccl_unique_id: out is NULL");
    CFPQ_CHECK_ARG(bytes >= (int64_t)nccl_unique_id_bytes(), "cfpq_nccl_unique_id: buffer smaller than 128 bytes");
    std::string err;
    if (!nccl_unique_id(out, &err)) {
        set_error(err);
        return CFPQ_E_NCCL;
    }
    return CFPQ_OK;
}

extern "C" cfpq_status cfpq_shard_rows(int64_t n_nodes, int32_t world_size, int32_t rank, int64_t* row_lo,
                                       int64_t* row_hi) {
    CFPQ_CHECK_ARG(row_lo && row_hi, "cfpq_shard_rows: NULL argument");
    CFPQ_CHECK_ARG(n_nodes >= 0 && world_size >= 1 && rank >= 0 && rank < world_size, "cfpq_shard_rows: bad argument");
    int64_t lo, hi, br;
    dense_partition(n_nodes, world_size, rank, &lo, &hi, &br);
    *row_lo = std::min<int64_t>(lo * 128, n_nodes);
    *row_hi = std::min<int64_t>(hi * 128, n_nodes);
    return CFPQ_OK;
}

extern "C" cfpq_status cfpq_shard_block(int64_t n_nodes, int32_t grid_rows, int32_t grid_cols, int32_t rank,
                                        int64_t* row_lo, int64_t* row_hi, int64_t* col_lo, int64_t* col_hi) {
    CFPQ_CHECK_ARG(row_lo && row_hi && col_lo && col_hi, "cfpq_shard_block: NULL output");
    CFPQ_CHECK_ARG(n_nodes >= 0 && grid_rows >= 1 && grid_cols >= 1 && rank >= 0 && rank < grid_rows * grid_cols,
                   "cfpq_shard_block: bad grid or rank");
    int64_t ilo, ihi, jlo, jhi;
    dense_partition2(n_nodes, grid_rows, grid_cols, rank / grid_cols, rank % grid_cols, &ilo, &ihi, &jlo, &jhi);
    *row_lo = std::min<int64_t>(ilo * 128, n_nodes);
    *row_hi = std::min<int64_t>(ihi * 128, n_nodes);
    *col_lo = std::min<int64_t>(jlo * 256, n_nodes);
    *col_hi = std::min<int64_t>(jhi * 256, n_nodes);
    return CFPQ_OK;
}

extern "C" const char* cfpq_version(void) {
    return "libcfpq 0.1 sm_100a (sparse semi-naive persistent engine)";
}
