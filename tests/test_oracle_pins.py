"""Pins for the CPU oracle (tests/ -m "not gpu").

The oracle (oracle/) is checked against things other than itself:
  * the paper's printed worked example (tests/golden/);
  * closed forms derived from Lemma 3 + the Chinese remainder theorem
    for a^n b^n on two coprime cycles (SURVEY V-2), including per-iteration bit and
    work counts and the single-path lengths;
  * the textbook BFS transitive closure for S -> S S | a (SURVEY V-5);
  * brute-force CYK over every path (the definition of R_A);
  * Valiant's closure a⁺ — Theorem 1 says a⁺ = a^cf;
  * realisability of every single-path length (Lemma 4 / Theorem 5);
  * invariants: monotone T_k, fixpoint idempotence, rule-order and node-relabel
    independence, disjoint-union additivity, the Theorem 3 bound.
"""
from collections import deque
from math import gcd

import numpy as np
import pytest

import inputs as I
import oracle as O


def _cells(res, snap, names):
    out = set()
    for A, name in enumerate(names):
        for i, j in res.pairs(A, snap).tolist():
            out.add((i, j, name))
    return out


# ------------------------------------------------------------------------------------------
# Worked example
# ------------------------------------------------------------------------------------------

def test_golden_example_per_iteration(example_golden):
    g = example_golden
    w = I.bind("example", I.same_generation_grammar(), 3, g["edges"], "S")
    res = O.run(w, snapshots=True)
    names = w.nt_names
    assert res.status == 0
    # "k = 6 since T6 = T5"
    assert res.iterations == g["K"] == 6
    for k in range(0, 6):
        assert _cells(res, k, names) == g["T"][k], f"T{k} differs from the printed matrix"
    assert _cells(res, 6, names) == g["T"][5]
    # T1 = T0 ∪ (T0 × T0) with T0 × T0 = {(1,2): {S}}
    assert _cells(res, 1, names) - _cells(res, 0, names) == g["P0"]
    # R_A
    for A, name in enumerate(names):
        assert set(map(tuple, res.pairs(A).tolist())) == g["R"][name], name


def test_golden_example_single_path(example_golden):
    g = example_golden
    w = I.bind("example", I.same_generation_grammar(), 3, g["edges"], "S")
    res = O.run(w, lengths=True)
    for name, i, j, l in g["L"]:
        A = w.nt(name)
        L = {(a, b): c for a, b, c in res.lengths(A).tolist()}
        assert L[(i, j)] == l        # type^-1 type, two edges
    # the witness of S(1,2) is exactly the path the text names
    cells = _all_length_cells(res, w)
    path = O.witness(w, cells, w.nt("S"), 1, 2)
    lab = [w.labels[x] for x in path[:, 1]]
    assert lab == ["type_r", "type"] and path[0, 0] == 1 and path[-1, 2] == 2


def _all_length_cells(res, w):
    rows = []
    for A in range(w.n_nt):
        for i, j, l in res.lengths(A).tolist():
            rows.append((A, i, j, l))
    return np.array(rows, dtype=np.int64).reshape(-1, 4)


# ------------------------------------------------------------------------------------------
# a^n b^n on two coprime cycles: closed forms (Lemma 3 + CRT)
# ------------------------------------------------------------------------------------------

def _crt(p, q, a, b):
    """The unique m in [1, pq] with m ≡ a (mod p), m ≡ b (mod q)."""
    for m in range(1, p * q + 1):
        if (m - a) % p == 0 and (m - b) % q == 0:
            return m
    raise AssertionError


ANBN_PAIRS = [(3, 2), (2, 3), (2, 5), (5, 3), (4, 7), (7, 4), (3, 8), (9, 5), (2, 31)]


@pytest.mark.parametrize("p,q", ANBN_PAIRS)
def test_anbn_closed_form(p, q):
    """a-node i reaches b-node b_r by a^m b^m iff (i+m) ≡ 0 (mod p) (node 0 is the only
    node with a b out-edge) and m ≡ r (mod q): by CRT every (i, b_r) has exactly one
    m in [1,pq], so R_S = R_S1 = Va × Vb.  A derivation of a^m b^m has height 2m and of
    a^m b^(m+1) (S1) height 2m+1, so by Lemma 3 the Jacobi loop adds exactly one cell
    per iteration and runs max height = 2pq+1 bodies (with the final no-change pass)."""
    assert gcd(p, q) == 1
    w = I.anbn_workload(p, q)
    res = O.run(w, lengths=True)
    va = list(range(p))
    vb = [0] + list(range(p, p + q - 1))
    full = {(i, j) for i in va for j in vb}
    S, S1, A, B = (w.nt(x) for x in ("S", "S1", "A", "B"))
    assert set(map(tuple, res.pairs(S).tolist())) == full
    assert set(map(tuple, res.pairs(S1).tolist())) == full
    assert set(map(tuple, res.pairs(A).tolist())) == {(k, (k + 1) % p) for k in range(p)}
    assert set(map(tuple, res.pairs(B).tolist())) == {(vb[k], vb[(k + 1) % q]) for k in range(q)}
    assert res.iterations == 2 * p * q + 1
    st = res.stats()
    assert st["new_bits"].tolist() == [1] * (2 * p * q) + [0]
    # work: at iteration k the AND-true triples are 1 (S->AB at r=0) + |S1_{k-1}| (S->A S1:
    # one a-edge into each a-node) + |S_{k-1}| (S1->S B: one b-edge out of each b-node) = k.
    assert st["jacobi_triples"].tolist() == list(range(1, 2 * p * q + 2))
    # semi-naive: iteration 1 has Δ0 = T0 and only S->AB fires, counted for both operands;
    # afterwards Δ is the single newest cell, in exactly one AND-true triple.
    assert st["seminaive_triples"].tolist() == [2] + [1] * (2 * p * q)
    # lengths: the unique minimal m gives l_S = 2m, l_S1 = 2m'+1 (m' + 1 ≡ r mod q)
    LS = {(i, j): l for i, j, l in res.lengths(S).tolist()}
    LS1 = {(i, j): l for i, j, l in res.lengths(S1).tolist()}
    for i in va:
        for r, j in enumerate(vb):
            assert LS[(i, j)] == 2 * _crt(p, q, (-i) % p, r % q)
            assert LS1[(i, j)] == 2 * _crt(p, q, (-i) % p, (r - 1) % q) + 1


# ------------------------------------------------------------------------------------------
# S -> S S | a  ==  strict transitive closure (BFS)
# ------------------------------------------------------------------------------------------

def _bfs_closure(n, edges):
    adj = [[] for _ in range(n)]
    for s, _, d in edges:
        adj[s].append(d)
    out = set()
    for s in range(n):
        seen = set()
        dq = deque(adj[s])
        for v in adj[s]:
            seen.add(v)
        while dq:
            u = dq.popleft()
            for v in adj[u]:
                if v not in seen:
                    seen.add(v)
                    dq.append(v)
        out |= {(s, v) for v in seen}
    return out


@pytest.mark.parametrize("n,d,seed", [(30, 1, 0), (60, 2, 1), (80, 1, 2), (40, 3, 3)])
def test_dense_stress_is_transitive_closure(n, d, seed):
    """S ⇒* a^m for every m ≥ 1, so R_S = pairs joined by a path of ≥ 1 edges."""
    w = I.dense_stress_workload(n, d, seed)
    res = O.run(w)
    assert set(map(tuple, res.pairs(0).tolist())) == _bfs_closure(n, w.edges.tolist())


# ------------------------------------------------------------------------------------------
# Brute-force CYK over all paths (definition) and Valiant's a⁺ (Theorem 1)
# ------------------------------------------------------------------------------------------

def _tiny_instances(count, seed0, max_nodes=4, max_edges=8):
    out = []
    s = seed0
    while len(out) < count:
        w = I.random_workload(s, max_nodes=max_nodes, max_edges=max_edges, max_nt=3, max_bin=6,
                              max_term=3, n_labels=2)
        s += 1
        out.append(w)
    return out


def test_bruteforce_paths_equal_closure():
    """Every triple has a witness of its recorded length (Lemma 4), so enumerating all
    paths up to the max recorded length is exact in both directions."""
    checked = 0
    for w in _tiny_instances(60, 1000):
        res = O.run(w, lengths=True)
        lmax = max([int(res.lengths(A)[:, 2].max()) for A in range(w.n_nt) if res.count(A)] + [1])
        if lmax > 9:
            continue
        brute = O.paths_relations(w, lmax)
        assert res.relation_sets() == brute, w.name
        checked += 1
    assert checked >= 40


def test_theorem1_valiant_equals_cf():
    """a⁺ = a^cf (Theorem 1).  Lemma 1 gives a⁽ᵏ⁾₊ ⊆ a^cf for all k; every cell of a^cf
    is in a⁽ˡ⁾₊ for its witness length l, so ∪_{i ≤ lmax} a⁽ⁱ⁾₊ must equal a^cf."""
    rng = np.random.default_rng(7)
    checked = 0
    for t in range(40):
        dim = int(rng.integers(1, 5))
        n_nt = int(rng.integers(1, 4))
        rules = sorted({tuple(int(x) for x in rng.integers(0, n_nt, 3)) for _ in range(int(rng.integers(1, 6)))})
        a = [[frozenset(int(x) for x in np.nonzero(rng.random(n_nt) < 0.3)[0]) for _ in range(dim)]
             for _ in range(dim)]
        # the set-valued matrix a as a graph: A ∈ a_ij <=> edge (i, x_A, j) and rule A -> x_A
        edges = np.array([(i, A, j) for i in range(dim) for j in range(dim) for A in a[i][j]],
                         dtype=np.int32).reshape(-1, 3)
        w = I.Workload("thm1", dim, [f"N{k}" for k in range(n_nt)], [f"x{k}" for k in range(n_nt)],
                       np.array(rules, dtype=np.int32).reshape(-1, 3),
                       np.array([(k, k) for k in range(n_nt)], dtype=np.int32), edges)
        res = O.run(w, lengths=True)
        lmax = max([int(res.lengths(A)[:, 2].max()) for A in range(n_nt) if res.count(A)] + [1])
        if lmax > 12:
            continue
        vp = O.valiant_closure(a, rules, lmax)
        got = {(i, j, A) for i in range(dim) for j in range(dim) for A in vp[i][j]}
        cf = {(i, j, A) for A in range(n_nt) for i, j in res.pairs(A).tolist()}
        assert got == cf
        checked += 1
    assert checked >= 25


# ------------------------------------------------------------------------------------------
# Single-path realisability (Lemma 4 / Theorem 5)
# ------------------------------------------------------------------------------------------

def test_lengths_realisable_random():
    checked = 0
    for w in _tiny_instances(50, 5000, max_nodes=6, max_edges=12):
        res = O.run(w, lengths=True)
        cells = _all_length_cells(res, w)
        for A, i, j, l in cells.tolist():
            path = O.witness(w, cells, A, i, j)
            assert path is not None and len(path) == l
            assert path[0, 0] == i and path[-1, 2] == j
            assert all(path[k, 2] == path[k + 1, 0] for k in range(l - 1))
            edge_set = set(map(tuple, w.edges.tolist()))
            assert all(tuple(e) in edge_set for e in path.tolist())
            if l <= 24:
                assert O.cyk(w, path[:, 1].tolist(), A)
            checked += 1
        # occupancy agreement: lengths exist exactly for the relational cells
        for A in range(w.n_nt):
            assert set(map(tuple, res.lengths(A)[:, :2].tolist())) == set(map(tuple, res.pairs(A).tolist()))
    assert checked > 100


def test_min_tiebreak_counterexample():
    """SURVEY V-3: A -> A A | x with two x-paths 0->5 of lengths 3 and 4 discovered in the
    same iteration: the recorded length is the minimum (reading c7), 3."""
    g = I.Grammar(["A"], [("A", "A", "A")], [("A", "x")])
    # path 0-1-2-5 (3 edges) and 0-3-4-6-5 (4 edges)
    e = [(0, "x", 1), (1, "x", 2), (2, "x", 5), (0, "x", 3), (3, "x", 4), (4, "x", 6), (6, "x", 5)]
    w = I.bind("tie", g, 7, e, "A")
    res = O.run(w, lengths=True)
    L = {(i, j): l for i, j, l in res.lengths(0).tolist()}
    assert L[(0, 5)] == 3


# ------------------------------------------------------------------------------------------
# Invariants
# ------------------------------------------------------------------------------------------

@pytest.mark.parametrize("seed", range(8))
def test_invariants_random(seed):
    w = I.random_workload(300 + seed, max_nodes=10, max_edges=30)
    res = O.run(w, snapshots=True)
    n, nn = w.n_nodes, w.n_nt
    # monotone ascent T_k ⪰ T_{k-1}
    prev = None
    for k in range(res.num_snapshots):
        cur = {(A, i, j) for A in range(nn) for i, j in res.pairs(A, k).tolist()}
        if prev is not None:
            assert prev <= cur
        prev = cur
    # Theorem 3 bound
    assert sum(res.stats()["new_bits"]) <= n * n * nn
    assert res.iterations <= n * n * nn + 1
    final = {(A, i, j) for A in range(nn) for i, j in res.pairs(A).tolist()}
    # fixpoint idempotence: seeding with T^cf itself adds nothing in one pass
    lab = [f"x{A}" for A in range(nn)]
    w2 = I.Workload("idem", n, w.nt_names, lab, w.bin, np.array([(A, A) for A in range(nn)], np.int32),
                    np.array([(i, A, j) for A, i, j in sorted(final)], np.int32).reshape(-1, 3))
    r2 = O.run(w2)
    assert r2.iterations == 1
    assert {(A, i, j) for A in range(nn) for i, j in r2.pairs(A).tolist()} == final
    # rule order and NT renaming independence
    rng = np.random.default_rng(seed)
    perm = rng.permutation(nn)
    inv = np.argsort(perm)
    b3 = perm[w.bin][rng.permutation(len(w.bin))] if len(w.bin) else w.bin
    t3 = w.term.copy()
    if len(t3):
        t3[:, 0] = perm[t3[:, 0]]
    w3 = I.Workload("perm", n, w.nt_names, w.labels, b3.astype(np.int32), t3, w.edges)
    r3 = O.run(w3)
    got = {(int(inv[A]), i, j) for A in range(nn) for i, j in r3.pairs(A).tolist()}
    assert got == final
    # node relabel equivariance
    pn = rng.permutation(n)
    e4 = w.edges.copy()
    if len(e4):
        e4[:, 0] = pn[e4[:, 0]]
        e4[:, 2] = pn[e4[:, 2]]
    r4 = O.run(I.Workload("relabel", n, w.nt_names, w.labels, w.bin, w.term, e4))
    got = {(A, int(np.where(pn == i)[0][0]), int(np.where(pn == j)[0][0]))
           for A in range(nn) for i, j in r4.pairs(A).tolist()}
    assert got == final


def test_disjoint_union_additivity():
    """g1..g3 are 8 disjoint copies: relations of the union = union of relations."""
    base = I.ontology_workload("q1", 60, depth=4, seed=3, relabel=False)
    named = [(s, base.labels[x], d) for s, x, d in base.edges.tolist()]
    n8, e8 = I.disjoint_copies(base.n_nodes, named, 8)
    w8 = I.bind("g8", I.same_generation_grammar(), n8, e8, "S", extra_labels=base.labels)
    r1 = O.run(base)
    r8 = O.run(w8)
    assert r8.iterations == r1.iterations
    for A in range(base.n_nt):
        p1 = set(map(tuple, r1.pairs(A).tolist()))
        exp = {(i + c * base.n_nodes, j + c * base.n_nodes) for c in range(8) for i, j in p1}
        assert set(map(tuple, r8.pairs(A).tolist())) == exp


def test_union_grammar_restricts_to_q1_and_q2():
    """Under the config-4 union grammar, S_Q1 derives exactly what S derives under Q1 alone
    and S_Q2 what S derives under Q2 alone (the rule sets only share preterminals)."""
    w = I.ontology_workload("union", 120, depth=5, seed=1)
    w1 = I.ontology_workload("q1", 120, depth=5, seed=1)
    w2 = I.ontology_workload("q2", 120, depth=5, seed=1)
    ru, r1, r2 = O.run(w), O.run(w1), O.run(w2)
    assert set(map(tuple, ru.pairs(w.nt("S_Q1")).tolist())) == set(map(tuple, r1.pairs(w1.nt("S")).tolist()))
    assert set(map(tuple, ru.pairs(w.nt("S_Q2")).tolist())) == set(map(tuple, r2.pairs(w2.nt("S")).tolist()))


def test_seed_semantics():
    g = I.Grammar(["A", "B"], [], [("A", "a"), ("B", "b")])
    # duplicates collapse (set E); parallel labels accumulate; unknown label ignored
    w = I.bind("seed", g, 3, [(0, "a", 1), (0, "a", 1), (0, "b", 1), (1, "c", 2)], "A")
    res = O.run(w)
    assert res.pairs(0).tolist() == [[0, 1]] and res.pairs(1).tolist() == [[0, 1]]
    assert res.iterations == 1
    # empty graph: empty relations, one (no-change) iteration
    w0 = I.bind("empty", g, 4, [], "A")
    r0 = O.run(w0)
    assert r0.iterations == 1 and r0.count(0) == 0
