// CPU BITSET BASELINE — a second, independent CPU implementation of the CFPQ closure of
// Azimov & Grigorev, arXiv 1707.01007 (P:n = PAPER.md line n), for the comparison numbers
// of SURVEY §8(d) / BASELINE.md §3: "uint64 bit-packed rows, semi-naive deltas, OpenMP".
//
// It is neither the oracle (oracle/, the root of trust: std::set cells, Jacobi in the
// paper's order) nor the product (paper_1707_01007_b200/, CUDA): it shares no code, header
// or table with either, and is compiled by plain g++ -fopenmp.  Tests check it against the
// oracle (small instances) and against the oracle's committed golden digests (config 4 at
// n = 16,384 and 65,536), which is the parity chain oracle == bitset at the headline size.
//
// What it computes (the same relations as Algorithm 1):
//   seed     T_0 = {(A,i,j) | (i,x,j) ∈ E, A -> x}
//   loop     T_k = T_{k-1} ∪ (T_{k-1} × T_{k-1})
//   stop     T_k = T_{k-1}; loop bodies counted incl. the final pass
// evaluated semi-naively: T only grows, so T_{k-1}×T_{k-1} = T_{k-2}×T_{k-2} ∪ Δ×T ∪ T×Δ
// with Δ = Δ_{k-1} = T_{k-1} \ T_{k-2}, and only the Δ terms can add anything.  Per rule
// A -> B C (one Boolean product per rule):
//   Δ_B entry (i,r) -> (A,i,j) for j ∈ row r of T_C
//   Δ_C entry (r,j) -> (A,i,j) for i ∈ column r of T_B
// NTs that are the LHS of no rule ("preterminals") never change after seeding; their rows
// and columns are sorted adjacency lists.  Rows/columns of changing NTs are read from
// snapshot bitsets of T_{k-1} (updated with Δ between iterations), so every iteration's
// state equals the Jacobi T_k.  Membership of T_A is a uint64 bitset per NT that derives
// cells: a candidate is new iff its __atomic_fetch_or flips the bit.
#include <omp.h>

#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <tuple>
#include <vector>

namespace {

struct Rule { int A, B, C; };

struct Cell { uint32_t X, i, j; };

struct alignas(64) Local {      // per-thread output, padded: no false sharing of the vector headers
    std::vector<Cell> v;
};

struct Adj {                       // adjacency of a preterminal: sorted neighbour lists
    std::vector<int64_t> ptr;      // n + 1
    std::vector<uint32_t> idx;
};

struct Baseline {
    int64_t n = 0;
    int n_nt = 0;
    int64_t W = 0;                 // uint64 words per bit row
    std::vector<Rule> rules;
    std::vector<std::pair<int, int>> term;   // (A, label)
    std::vector<char> is_pre;                // LHS of no rule
    // per NT: membership bitset (derived NTs and preterminals alike: seeds dedupe there too)
    std::vector<uint64_t*> T;
    // snapshots of T_{k-1}: S_X rows (X a changing right operand), ST_X columns (X a
    // changing left operand whose partner also changes)
    std::vector<uint64_t*> S, ST;
    std::vector<Adj> rowadj, coladj;         // preterminals: rows (CSR) / columns (CSC)
    // results of the last run
    std::vector<Cell> cells;                 // Δ_0 | Δ_1 | ... (every cell once)
    std::vector<int64_t> iter_off;           // start of Δ_k in cells
    std::vector<int64_t> candidates;         // per iteration: expanded (entry, neighbour) pairs
    int64_t iterations = 0;
    double seconds = 0;
    int threads_used = 0;
    ~Baseline() {
        for (auto* p : T) free(p);
        for (auto* p : S) free(p);
        for (auto* p : ST) free(p);
    }
};

inline bool set_bit(uint64_t* M, int64_t W, uint32_t i, uint32_t j) {
    uint64_t* w = M + (int64_t)i * W + (j >> 6);
    const uint64_t b = 1ull << (j & 63);
    if (__atomic_load_n(w, __ATOMIC_RELAXED) & b) return false;
    return !(__atomic_fetch_or(w, b, __ATOMIC_RELAXED) & b);
}

uint64_t* zalloc(int64_t words) {
    void* p = nullptr;
    if (posix_memalign(&p, 64, (size_t)std::max<int64_t>(words, 1) * 8) != 0) return nullptr;
    memset(p, 0, (size_t)std::max<int64_t>(words, 1) * 8);   // touched once here, outside timing
    return (uint64_t*)p;
}

// Build the adjacency (rows or columns) of preterminal X from its seed cells.
void build_adj(Adj& a, int64_t n, const std::vector<Cell>& seeds, int X, bool by_row) {
    a.ptr.assign(n + 1, 0);
    for (const Cell& c : seeds)
        if ((int)c.X == X) a.ptr[(by_row ? c.i : c.j) + 1]++;
    for (int64_t v = 0; v < n; ++v) a.ptr[v + 1] += a.ptr[v];
    a.idx.assign(a.ptr[n], 0);
    std::vector<int64_t> cur(a.ptr.begin(), a.ptr.end() - 1);
    for (const Cell& c : seeds)
        if ((int)c.X == X) a.idx[cur[by_row ? c.i : c.j]++] = by_row ? c.j : c.i;
    for (int64_t v = 0; v < n; ++v) std::sort(a.idx.begin() + a.ptr[v], a.idx.begin() + a.ptr[v + 1]);
}

}  // namespace

extern "C" {

// Create a baseline handle for a grammar shape and node count (allocates the bitsets).
void* bitset_create(int64_t n, int32_t n_nt, const int32_t* bin, int64_t n_bin, const int32_t* term, int64_t n_term) {
    if (n < 0 || n_nt <= 0) return nullptr;
    Baseline* B = new Baseline();
    B->n = n;
    B->n_nt = n_nt;
    B->W = (n + 63) / 64;
    std::vector<std::tuple<int, int, int>> rs;
    for (int64_t k = 0; k < n_bin; ++k) rs.emplace_back(bin[3 * k], bin[3 * k + 1], bin[3 * k + 2]);
    std::sort(rs.begin(), rs.end());
    rs.erase(std::unique(rs.begin(), rs.end()), rs.end());
    for (auto& t : rs) B->rules.push_back(Rule{std::get<0>(t), std::get<1>(t), std::get<2>(t)});
    for (int64_t k = 0; k < n_term; ++k) B->term.emplace_back(term[2 * k], term[2 * k + 1]);
    std::sort(B->term.begin(), B->term.end());
    B->term.erase(std::unique(B->term.begin(), B->term.end()), B->term.end());
    B->is_pre.assign(n_nt, 1);
    for (auto& r : B->rules) B->is_pre[r.A] = 0;
    std::vector<char> need_S(n_nt, 0), need_ST(n_nt, 0);
    for (auto& r : B->rules) {
        if (!B->is_pre[r.C]) need_S[r.C] = 1;                          // rows of a changing C
        if (!B->is_pre[r.B] && !B->is_pre[r.C]) need_ST[r.B] = 1;     // columns of a changing B
    }
    B->T.assign(n_nt, nullptr);
    B->S.assign(n_nt, nullptr);
    B->ST.assign(n_nt, nullptr);
    for (int X = 0; X < n_nt; ++X) {
        B->T[X] = zalloc(n * B->W);
        if (need_S[X]) B->S[X] = zalloc(n * B->W);
        if (need_ST[X]) B->ST[X] = zalloc(n * B->W);
        if (!B->T[X] || (need_S[X] && !B->S[X]) || (need_ST[X] && !B->ST[X])) {
            delete B;
            return nullptr;
        }
    }
    B->rowadj.resize(n_nt);
    B->coladj.resize(n_nt);
    return B;
}

void bitset_destroy(void* h) { delete static_cast<Baseline*>(h); }

// Run seed + semi-naive loop to the fixpoint with `threads` OpenMP threads (0 = all).
// Returns iterations (loop bodies incl. the final no-change pass), or -1 on bad input.
// The timed region (bitset_seconds) is seed + adjacency + loop.
int64_t bitset_run(void* h, const int32_t* edges, int64_t n_edges, int32_t threads, int64_t max_iterations) {
    Baseline* B = static_cast<Baseline*>(h);
    const int64_t n = B->n, W = B->W;
    for (int64_t e = 0; e < n_edges; ++e)
        if (edges[3 * e] < 0 || edges[3 * e] >= n || edges[3 * e + 2] < 0 || edges[3 * e + 2] >= n) return -1;
    const int nth = threads > 0 ? threads : omp_get_max_threads();
    B->threads_used = nth;
    // clear the previous run's bits (O(previous cells), outside the timed region)
    {
        const std::vector<Cell>& old = B->cells;
#pragma omp parallel for num_threads(nth) schedule(static)
        for (int64_t e = 0; e < (int64_t)old.size(); ++e) {
            const Cell c = old[e];
            B->T[c.X][(int64_t)c.i * W + (c.j >> 6)] = 0;
            if (B->S[c.X]) B->S[c.X][(int64_t)c.i * W + (c.j >> 6)] = 0;
            if (B->ST[c.X]) B->ST[c.X][(int64_t)c.j * W + (c.i >> 6)] = 0;
        }
    }
    B->cells.clear();
    B->iter_off.clear();
    B->candidates.clear();
    // labels -> NTs with A -> x
    int max_label = -1;
    for (auto& t : B->term) max_label = std::max(max_label, t.second);
    std::vector<std::vector<int>> by_label(max_label + 1);
    for (auto& t : B->term) by_label[t.second].push_back(t.first);
    // expansions of a Δ entry of NT X: (kind, rule)
    //   0: X = B, C preterminal     1: X = C, B preterminal
    //   2: X = B, C changes         3: X = C, B changes (and C changes)
    std::vector<std::vector<std::pair<int, int>>> exps(B->n_nt);
    for (int q = 0; q < (int)B->rules.size(); ++q) {
        const Rule& r = B->rules[q];
        const bool pb = B->is_pre[r.B], pc = B->is_pre[r.C];
        if (!pb && pc) exps[r.B].push_back({0, q});
        else if (pb && !pc) exps[r.C].push_back({1, q});
        else if (!pb && !pc) {
            exps[r.B].push_back({2, q});
            exps[r.C].push_back({3, q});
        } else {
            exps[r.B].push_back({0, q});   // both constant: only iteration 1 contributes
        }
    }

    const auto t0 = std::chrono::steady_clock::now();
    std::vector<Local> local(nth);
    // ---- seed: parallel edges accumulate, duplicates dedupe ----
#pragma omp parallel num_threads(nth)
    {
        std::vector<Cell>& out = local[omp_get_thread_num()].v;
        out.clear();
#pragma omp for schedule(static)
        for (int64_t e = 0; e < n_edges; ++e) {
            const int x = edges[3 * e + 1];
            if (x < 0 || x > max_label) continue;
            const uint32_t i = (uint32_t)edges[3 * e], j = (uint32_t)edges[3 * e + 2];
            for (int A : by_label[x])
                if (set_bit(B->T[A], W, i, j)) out.push_back(Cell{(uint32_t)A, i, j});
        }
    }
    for (auto& l : local) B->cells.insert(B->cells.end(), l.v.begin(), l.v.end());
    B->iter_off.push_back(0);
    B->iter_off.push_back((int64_t)B->cells.size());
    // adjacency of preterminals (constant from here on)
    for (int X = 0; X < B->n_nt; ++X) {
        bool row = false, col = false;
        for (auto& r : B->rules) {
            if (r.C == X && B->is_pre[X]) row = true;
            if (r.B == X && B->is_pre[X]) col = true;
        }
        if (row) build_adj(B->rowadj[X], n, B->cells, X, true);
        if (col) build_adj(B->coladj[X], n, B->cells, X, false);
    }
    auto apply_snapshots = [&](int64_t lo, int64_t hi) {
#pragma omp parallel for num_threads(nth) schedule(static)
        for (int64_t e = lo; e < hi; ++e) {
            const Cell c = B->cells[e];
            if (B->S[c.X]) set_bit(B->S[c.X], W, c.i, c.j);
            if (B->ST[c.X]) set_bit(B->ST[c.X], W, c.j, c.i);
        }
    };
    apply_snapshots(0, (int64_t)B->cells.size());

    // ---- loop ----
    int64_t k = 0;
    const int64_t cap = max_iterations > 0 ? max_iterations : n * n * (int64_t)B->n_nt + 1;
    for (;;) {
        ++k;
        const int64_t lo = B->iter_off[k - 1], hi = B->iter_off[k];
        int64_t cand = 0;
#pragma omp parallel num_threads(nth) reduction(+ : cand)
        {
            std::vector<Cell>& out = local[omp_get_thread_num()].v;
            out.clear();
#pragma omp for schedule(dynamic, 256)
            for (int64_t e = lo; e < hi; ++e) {
                const Cell c = B->cells[e];
                for (auto& ex : exps[c.X]) {
                    const Rule& r = B->rules[ex.second];
                    const uint32_t A = (uint32_t)r.A;
                    if (ex.first == 0) {                  // (i,r) of Δ_B, row r of preterminal C
                        if (B->is_pre[r.B] && k > 1) continue;
                        const Adj& a = B->rowadj[r.C];
                        for (int64_t t = a.ptr[c.j]; t < a.ptr[c.j + 1]; ++t) {
                            ++cand;
                            if (set_bit(B->T[A], W, c.i, a.idx[t])) out.push_back(Cell{A, c.i, a.idx[t]});
                        }
                    } else if (ex.first == 1) {           // (r,j) of Δ_C, column r of preterminal B
                        const Adj& a = B->coladj[r.B];
                        for (int64_t t = a.ptr[c.i]; t < a.ptr[c.i + 1]; ++t) {
                            ++cand;
                            if (set_bit(B->T[A], W, a.idx[t], c.j)) out.push_back(Cell{A, a.idx[t], c.j});
                        }
                    } else {                              // a changing partner: snapshot bit row
                        const bool left = ex.first == 2;
                        const uint64_t* row = left ? B->S[r.C] + (int64_t)c.j * W : B->ST[r.B] + (int64_t)c.i * W;
                        for (int64_t w = 0; w < W; ++w) {
                            uint64_t bits = row[w];
                            while (bits) {
                                const uint32_t v = (uint32_t)(w * 64 + __builtin_ctzll(bits));
                                bits &= bits - 1;
                                ++cand;
                                const uint32_t oi = left ? c.i : v, oj = left ? v : c.j;
                                if (set_bit(B->T[A], W, oi, oj)) out.push_back(Cell{A, oi, oj});
                            }
                        }
                    }
                }
            }
        }
        for (auto& l : local) B->cells.insert(B->cells.end(), l.v.begin(), l.v.end());
        B->iter_off.push_back((int64_t)B->cells.size());
        B->candidates.push_back(cand);
        const int64_t added = (int64_t)B->cells.size() - hi;
        if (added == 0 || k >= cap) break;      // T_k = T_{k-1}: fixpoint
        apply_snapshots(hi, (int64_t)B->cells.size());
    }
    const auto t1 = std::chrono::steady_clock::now();
    B->seconds = std::chrono::duration<double>(t1 - t0).count();
    B->iterations = k;
    return k;
}

double bitset_seconds(void* h) { return static_cast<Baseline*>(h)->seconds; }
int32_t bitset_threads(void* h) { return static_cast<Baseline*>(h)->threads_used; }
int64_t bitset_num_cells(void* h) { return (int64_t)static_cast<Baseline*>(h)->cells.size(); }

// Per iteration k = 1..iterations: new cells |Δ_k| and expanded candidates.
void bitset_iteration_stats(void* h, int64_t* new_cells, int64_t* candidates) {
    Baseline* B = static_cast<Baseline*>(h);
    for (int64_t k = 1; k <= B->iterations; ++k) {
        if (new_cells) new_cells[k - 1] = B->iter_off[k + 1] - B->iter_off[k];
        if (candidates) candidates[k - 1] = B->candidates[k - 1];
    }
}

// Count of R_A, and its pairs (i,j) ascending into out[2*count].
int64_t bitset_count(void* h, int32_t A) {
    Baseline* B = static_cast<Baseline*>(h);
    int64_t c = 0;
    for (const Cell& x : B->cells) c += (int)x.X == A;
    return c;
}

int64_t bitset_pairs(void* h, int32_t A, int32_t* out) {
    Baseline* B = static_cast<Baseline*>(h);
    std::vector<uint64_t> keys;
    for (const Cell& x : B->cells)
        if ((int)x.X == A) keys.push_back(((uint64_t)x.i << 32) | x.j);
    std::sort(keys.begin(), keys.end());
    for (size_t t = 0; t < keys.size(); ++t) {
        out[2 * t] = (int32_t)(keys[t] >> 32);
        out[2 * t + 1] = (int32_t)(keys[t] & 0xffffffffu);
    }
    return (int64_t)keys.size();
}

}  // extern "C"
