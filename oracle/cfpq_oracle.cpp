// ORACLE — TEST INFRASTRUCTURE ONLY.
//
// A plain, slow, obviously-correct CPU implementation of the CFPQ closure of
// Azimov & Grigorev, "Context-Free Path Querying by Matrix Multiplication"
// (arXiv 1707.01007).  PAPER.md line n is cited as P:n.  Only tests/,
// __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may
// load this library.  It shares no code, header or table with the CUDA path in
// paper_1707_01007_b200/ and is compiled by plain g++.
//
// Representation: the |V|x|V| matrix T whose cells are
// subsets of N.  Stored sparsely: row i -> (column j -> std::set of NT ids);
// an absent cell is the empty set.
//
// Everything is single threaded and written in the paper's order:
//   seed    (Alg. 1 lines 6-7 = P:216-219; parallel edges accumulate P:230)
//   loop    (Alg. 1 lines 8-9 = P:220-222):  T <- T ∪ (T × T), Jacobi/snapshot
//           (reading c4), stop when T no longer changes; the loop-body count
//           includes the final no-change pass ("k = 6 since T6 = T5", c3).
//   product: (T×T)_ij = ∪_k T_ik · T_kj,
//           N1·N2 = {A | ∃B∈N1, ∃C∈N2, (A->BC) ∈ P}.
//   lengths: seed (A,1); a cell first added in iteration p through
//           A->BC with (B,lB) ∈ T(p-1)_ir, (C,lC) ∈ T(p-1)_rj gets lA = lB + lC;
//           never overwritten afterwards.  Within one iteration the paper is
//           silent on which candidate wins: reading c7 takes the minimum.
//   cap     Theorem 3: at most |V|^2|N| changes, so the loop is
//           capped at |V|^2|N|+1 bodies.
// The oracle also counts, per iteration, the AND-true triples (i,r,j,rule) of
// the full Jacobi product (the work Alg. 1 line 9 does on sparse operands) and
// of the semi-naive split Δ_B×T_C + T_B×Δ_C; those counts are the
// numerators of the bench's effective boolean Gop/s.
//
// Path reconstruction ("found by a simple search") is exposed as
// oracle_witness(); it works from any supplied length table.

#include <cstdint>
#include <cstring>
#include <map>
#include <set>
#include <vector>
#include <utility>
#include <tuple>
#include <algorithm>

namespace {

typedef std::set<int> NTSet;                    // a cell: subset of N
typedef std::map<int, NTSet> Row;               // column -> cell
typedef std::vector<Row> Matrix;                // row -> Row
typedef std::map<int, uint64_t> LCell;          // NT -> length   (single-path cells)
typedef std::vector<std::map<int, LCell>> LMatrix;

struct Rule { int A, B, C; };

struct Result {
    int64_t n = 0;
    int n_nt = 0;
    int status = 0;                 // 0 ok, -5 not converged, -6 length overflow (> 2^32-1)
    int64_t iterations = 0;
    Matrix T;                        // the fixpoint T^cf
    LMatrix L;                       // lengths (if requested)
    bool have_lengths = false;
    std::vector<Matrix> snapshots;   // T_0, T_1, ... (if requested)
    std::vector<int64_t> new_bits;   // |T_k \ T_{k-1}| per iteration k = 1..iterations
    std::vector<int64_t> jacobi_triples;    // per iteration: #(i,r,j,rule) with B∈T_ir, C∈T_rj
    std::vector<int64_t> seminaive_triples; // per iteration: #Δ_B×T_C + #T_B×Δ_C
};

// Set product N1 · N2, restricted to one rule: true iff B∈N1 and C∈N2.
inline bool rule_applies(const Rule& r, const NTSet& n1, const NTSet& n2) {
    return n1.count(r.B) && n2.count(r.C);
}

bool cell_has(const Matrix& M, int i, int j, int A) {
    auto it = M[i].find(j);
    return it != M[i].end() && it->second.count(A);
}

}  // namespace

extern "C" {

// Runs Algorithm 1.  Inputs are plain arrays:
//   bin  [n_bin][3]  = (A,B,C) for A->BC;   term [n_term][2] = (A,label) for A->x;
//   edges[n_edges][3] = (src,label,dst).    P is a set: duplicate rules collapse.
// Returns an opaque handle (free with oracle_free) or nullptr on invalid input.
void* oracle_run(int64_t n, int32_t n_nt, const int32_t* bin, int64_t n_bin,
                 const int32_t* term, int64_t n_term, const int32_t* edges, int64_t n_edges,
                 int32_t with_lengths, int32_t keep_snapshots, int64_t max_iterations) {
    if (n < 0 || n_nt <= 0) return nullptr;
    std::set<std::tuple<int, int, int>> rule_set;
    for (int64_t k = 0; k < n_bin; ++k) {
        int A = bin[3 * k], B = bin[3 * k + 1], C = bin[3 * k + 2];
        if (A < 0 || A >= n_nt || B < 0 || B >= n_nt || C < 0 || C >= n_nt) return nullptr;
        rule_set.insert(std::make_tuple(A, B, C));
    }
    std::vector<Rule> P;
    for (auto& t : rule_set) P.push_back(Rule{std::get<0>(t), std::get<1>(t), std::get<2>(t)});
    for (int64_t k = 0; k < n_term; ++k)
        if (term[2 * k] < 0 || term[2 * k] >= n_nt) return nullptr;
    for (int64_t e = 0; e < n_edges; ++e)
        if (edges[3 * e] < 0 || edges[3 * e] >= n || edges[3 * e + 2] < 0 || edges[3 * e + 2] >= n)
            return nullptr;

    Result* R = new Result();
    R->n = n;
    R->n_nt = n_nt;
    R->have_lengths = with_lengths != 0;
    Matrix T(n);
    LMatrix L(with_lengths ? n : 0);

    // Matrix initialisation, Alg. 1 lines 6-7:
    //   T_ij <- T_ij ∪ {A | (A -> x) ∈ P} for every (i,x,j) ∈ E.
    // With lengths every seeded pair is (A,1).
    for (int64_t e = 0; e < n_edges; ++e) {
        int i = edges[3 * e], x = edges[3 * e + 1], j = edges[3 * e + 2];
        for (int64_t k = 0; k < n_term; ++k) {
            if (term[2 * k + 1] == x) {
                int A = term[2 * k];
                T[i][j].insert(A);
                if (with_lengths) L[i][j][A] = 1;
            }
        }
    }
    if (keep_snapshots) R->snapshots.push_back(T);

    // Theorem 3: at most |V|^2 |N| changes -> at most |V|^2|N|+1 loop bodies.
    int64_t cap = max_iterations > 0 ? max_iterations : n * n * (int64_t)n_nt + 1;
    Matrix Dprev = T;   // Δ_0 = T_0, used only to count the semi-naive split
    int64_t k = 0;
    while (true) {
        ++k;   // loop body k computes T_k = T_{k-1} ∪ (T_{k-1} × T_{k-1})
        Matrix Prod(n);
        std::vector<std::map<int, std::map<int, uint64_t>>> cand(with_lengths ? n : 0);
        int64_t jac = 0, sn = 0;
        // (T×T)_ij = ∪_r T_ir · T_rj: only non-empty T_ir, T_rj contribute.
        for (int64_t i = 0; i < n; ++i) {
            for (auto& ir : T[i]) {
                int r = ir.first;
                const NTSet& N1 = ir.second;
                for (auto& rj : T[r]) {
                    int j = rj.first;
                    const NTSet& N2 = rj.second;
                    for (const Rule& p : P) {
                        if (!rule_applies(p, N1, N2)) continue;
                        ++jac;
                        sn += cell_has(Dprev, (int)i, r, p.B) ? 1 : 0;
                        sn += cell_has(Dprev, r, j, p.C) ? 1 : 0;
                        Prod[i][j].insert(p.A);
                        if (with_lengths && !cell_has(T, (int)i, j, p.A)) {
                            // candidate for a cell absent from T_{k-1}: l_A = l_B + l_C
                            uint64_t l = L[i].at(r).at(p.B) + L[r].at(j).at(p.C);
                            auto& c = cand[i][j];
                            auto it = c.find(p.A);
                            if (it == c.end() || l < it->second) c[p.A] = l;   // reading c7: min
                        }
                    }
                }
            }
        }
        // T_k = T_{k-1} ∪ Prod; changed iff some NT is new in some cell.
        Matrix D(n);
        int64_t added = 0;
        for (int64_t i = 0; i < n; ++i) {
            for (auto& jc : Prod[i]) {
                for (int A : jc.second) {
                    if (!cell_has(T, (int)i, jc.first, A)) {
                        D[i][jc.first].insert(A);
                        ++added;
                    }
                }
            }
        }
        for (int64_t i = 0; i < n; ++i)
            for (auto& jc : D[i])
                for (int A : jc.second) {
                    T[i][jc.first].insert(A);
                    if (with_lengths) {
                        uint64_t l = cand[i].at(jc.first).at(A);
                        if (l > 0xFFFFFFFFull) R->status = -6;
                        L[i][jc.first][A] = l;   // first write wins: never overwritten later
                    }
                }
        R->new_bits.push_back(added);
        R->jacobi_triples.push_back(jac);
        R->seminaive_triples.push_back(sn);
        if (keep_snapshots) R->snapshots.push_back(T);
        Dprev.swap(D);
        if (added == 0) break;                 // fixpoint: T_k = T_{k-1}
        if (k >= cap) { R->status = -5; break; }
    }
    R->iterations = k;
    R->T.swap(T);
    R->L.swap(L);
    return R;
}

void oracle_free(void* h) { delete static_cast<Result*>(h); }
int32_t oracle_status(void* h) { return static_cast<Result*>(h)->status; }
int64_t oracle_iterations(void* h) { return static_cast<Result*>(h)->iterations; }

static const Matrix& pick(Result* R, int64_t snap) {
    return snap < 0 ? R->T : R->snapshots.at((size_t)snap);
}

// |R_A| (Theorem 2: (i,j) ∈ R_A iff A ∈ T^cf_ij), or |{(i,j): A ∈ T_snap_ij}|.
int64_t oracle_count(void* h, int32_t A, int64_t snap) {
    Result* R = static_cast<Result*>(h);
    if (snap >= (int64_t)R->snapshots.size()) return -1;
    const Matrix& M = pick(R, snap);
    int64_t c = 0;
    for (auto& row : M)
        for (auto& jc : row) c += jc.second.count(A);
    return c;
}

// Writes the pairs (i,j) of R_A in ascending (i,j) order into out[2*count].
int64_t oracle_pairs(void* h, int32_t A, int64_t snap, int32_t* out) {
    Result* R = static_cast<Result*>(h);
    if (snap >= (int64_t)R->snapshots.size()) return -1;
    const Matrix& M = pick(R, snap);
    int64_t c = 0;
    for (int64_t i = 0; i < (int64_t)M.size(); ++i)
        for (auto& jc : M[i])
            if (jc.second.count(A)) { out[2 * c] = (int32_t)i; out[2 * c + 1] = jc.first; ++c; }
    return c;
}

int64_t oracle_num_snapshots(void* h) { return (int64_t)static_cast<Result*>(h)->snapshots.size(); }

// Per-iteration statistics, arrays of length oracle_iterations().
void oracle_stats(void* h, int64_t* new_bits, int64_t* jacobi_triples, int64_t* seminaive_triples) {
    Result* R = static_cast<Result*>(h);
    for (size_t k = 0; k < R->new_bits.size(); ++k) {
        if (new_bits) new_bits[k] = R->new_bits[k];
        if (jacobi_triples) jacobi_triples[k] = R->jacobi_triples[k];
        if (seminaive_triples) seminaive_triples[k] = R->seminaive_triples[k];
    }
}

// Lengths of NT A as triples (i, j, l) ascending in (i,j): out[3*count] (int64).
int64_t oracle_lengths(void* h, int32_t A, int64_t* out) {
    Result* R = static_cast<Result*>(h);
    if (!R->have_lengths) return -1;
    int64_t c = 0;
    for (int64_t i = 0; i < (int64_t)R->L.size(); ++i)
        for (auto& jc : R->L[i]) {
            auto it = jc.second.find(A);
            if (it != jc.second.end()) {
                out[3 * c] = i; out[3 * c + 1] = jc.first; out[3 * c + 2] = (int64_t)it->second; ++c;
            }
        }
    return c;
}

// Path reconstruction for single-path semantics (Lemma 4).
// Input: a length table given as n_cells rows (A, i, j, l) (from any source), the
// grammar and the graph.  Finds a path of exactly l edges from i to j whose label
// word A derives, by the recursion of Lemma 4: l = 1 -> an edge (i,x,j) with A->x;
// l > 1 -> a rule A->BC and a node r with l_B(i,r) + l_C(r,j) = l, then recurse.
// Writes the path's edges (src,label,dst) into path_out[3*l] and, for every
// internal node of the derivation, nothing else.  Returns the path length, or
// -1 if (A,i,j) has no recorded length, -2 if the recursion gets stuck (the
// table is not realisable), -3 if path_cap is too small.
int64_t oracle_witness(int64_t n, int32_t n_nt, const int32_t* bin, int64_t n_bin,
                       const int32_t* term, int64_t n_term, const int32_t* edges, int64_t n_edges,
                       const int64_t* cells, int64_t n_cells,
                       int32_t A, int64_t i, int64_t j, int32_t* path_out, int64_t path_cap) {
    (void)n;
    // length lookup (A,i,j) -> l, and per (B,i) the list of (r, l) for the split search
    std::map<std::tuple<int, int64_t, int64_t>, uint64_t> len;
    std::map<std::pair<int, int64_t>, std::vector<std::pair<int64_t, uint64_t>>> rows;
    for (int64_t c = 0; c < n_cells; ++c) {
        int a = (int)cells[4 * c];
        int64_t ci = cells[4 * c + 1], cj = cells[4 * c + 2];
        uint64_t l = (uint64_t)cells[4 * c + 3];
        len[std::make_tuple(a, ci, cj)] = l;
        rows[std::make_pair(a, ci)].push_back(std::make_pair(cj, l));
    }
    auto it0 = len.find(std::make_tuple((int)A, i, j));
    if (it0 == len.end()) return -1;
    if ((int64_t)it0->second > path_cap) return -3;
    // explicit stack of goals (A, i, j, l); leaves are emitted left to right
    struct Goal { int A; int64_t i, j; uint64_t l; };
    std::vector<Goal> stack;
    stack.push_back(Goal{(int)A, i, j, it0->second});
    int64_t m = 0;
    while (!stack.empty()) {
        Goal g = stack.back();
        stack.pop_back();
        if (g.l == 1) {
            bool found = false;
            for (int64_t e = 0; e < n_edges && !found; ++e) {
                if (edges[3 * e] != g.i || edges[3 * e + 2] != g.j) continue;
                for (int64_t t = 0; t < n_term; ++t)
                    if (term[2 * t] == g.A && term[2 * t + 1] == edges[3 * e + 1]) {
                        path_out[3 * m] = (int32_t)g.i; path_out[3 * m + 1] = edges[3 * e + 1];
                        path_out[3 * m + 2] = (int32_t)g.j; ++m; found = true; break;
                    }
            }
            if (!found) return -2;
            continue;
        }
        bool found = false;
        for (int64_t k = 0; k < n_bin && !found; ++k) {
            if (bin[3 * k] != g.A) continue;
            int B = bin[3 * k + 1], C = bin[3 * k + 2];
            auto rit = rows.find(std::make_pair(B, g.i));
            if (rit == rows.end()) continue;
            for (auto& rl : rit->second) {
                if (rl.second >= g.l) continue;
                auto cit = len.find(std::make_tuple(C, rl.first, g.j));
                if (cit == len.end() || rl.second + cit->second != g.l) continue;
                // push right part first so the left part is expanded (and emitted) first
                stack.push_back(Goal{C, rl.first, g.j, cit->second});
                stack.push_back(Goal{B, g.i, rl.first, rl.second});
                found = true;
                break;
            }
        }
        if (!found) return -2;
    }
    return m;
}

// CYK membership (P:139 cites CYK): does A derive the word w[0..len)?  Plain
// O(len^3 |P|) table over spans; used to check reconstructed witness words.
int32_t oracle_cyk(int32_t n_nt, const int32_t* bin, int64_t n_bin, const int32_t* term,
                   int64_t n_term, const int32_t* word, int64_t len, int32_t A) {
    if (len <= 0) return 0;
    // tab[s][l-1] = set of NTs deriving word[s .. s+l)
    std::vector<std::vector<std::vector<char>>> tab(
        len, std::vector<std::vector<char>>(len, std::vector<char>(n_nt, 0)));
    for (int64_t s = 0; s < len; ++s)
        for (int64_t t = 0; t < n_term; ++t)
            if (term[2 * t + 1] == word[s]) tab[s][0][term[2 * t]] = 1;
    for (int64_t l = 2; l <= len; ++l)
        for (int64_t s = 0; s + l <= len; ++s)
            for (int64_t split = 1; split < l; ++split)
                for (int64_t k = 0; k < n_bin; ++k) {
                    int a = bin[3 * k], b = bin[3 * k + 1], c = bin[3 * k + 2];
                    if (tab[s][split - 1][b] && tab[s + split][l - split - 1][c]) tab[s][l - 1][a] = 1;
                }
    return tab[0][len - 1][A];
}

}  // extern "C"
