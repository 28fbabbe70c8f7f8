"""GPU parity: libcfpq (through its C-ABI / Python binding) against the oracle,
element by element, bit-exact (integer work, so exact equality)."""
import dataclasses
from math import gcd

import numpy as np
import pytest

import inputs as I
import oracle as O
from tests.gpu_util import assert_parity, cuda_ok, gpu_closure

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_ok(), reason="needs a CUDA device")]


# ------------------------------------------------------------------------------------------
# Worked example: per-iteration states, k = 6, R_A, lengths
# ------------------------------------------------------------------------------------------

@pytest.mark.parametrize("cell_set", [1, 2])
@pytest.mark.parametrize("solo", [-1, 0, 1 << 30])
def test_example_per_iteration(example_golden, solo, cell_set):
    g = example_golden
    w = I.bind("example", I.same_generation_grammar(), 3, g["edges"], "S")
    r, _, _ = gpu_closure(w, solo_threshold=solo, cell_set=cell_set)
    assert r.stats()["hashed"] == (cell_set == 2)
    assert r.iterations == g["K"] == 6
    for k in range(0, 6):
        cells = {(i, j, w.nt_names[A]) for A in range(w.n_nt) for i, j in r.pairs_at(A, k).tolist()}
        assert cells == g["T"][k], f"T{k}"
    for A, name in enumerate(w.nt_names):
        assert set(map(tuple, r.pairs(A).tolist())) == g["R"][name]


def test_example_lengths(example_golden):
    g = example_golden
    w = I.bind("example", I.same_generation_grammar(), 3, g["edges"], "S")
    r, _, _ = gpu_closure(w, semantics=1)
    assert_parity(w, r, lengths=True)
    for name, i, j, l in g["L"]:
        A = w.nt(name)
        L = dict(zip(map(tuple, r.pairs(A).tolist()), r.lengths(A).tolist()))
        assert L[(i, j)] == l


# ------------------------------------------------------------------------------------------
# a^n b^n (configs 1a, 3, 5)
# ------------------------------------------------------------------------------------------

def _crt(p, q, a, b):
    m = a % p
    while (m - b) % q:
        m += p
    return m if m > 0 else p * q


@pytest.mark.parametrize("p,q", [(3, 2), (2, 5), (5, 3), (4, 7), (9, 5), (2, 31)])
def test_anbn_small_parity(p, q):
    w = I.anbn_workload(p, q)
    r, _, _ = gpu_closure(w, semantics=1)
    ores = assert_parity(w, r, lengths=True)
    nc, _ = r.iteration_stats()
    assert nc.tolist() == ores.stats()["new_bits"].tolist()


@pytest.mark.parametrize("p,q,lengths", [(2, 4095, False), (3, 1366, False), (2, 16383, False), (2, 16383, True)])
def test_anbn_full_size_closed_form(p, q, lengths):
    """Configs 3 and 5 at n = p+q-1 (4096 / 16384) in the bench's launch configuration:
    R_S = R_S1 = Va x Vb, 2pq+1 iterations, one new cell per iteration, and the CRT
    closed form of every length (tests/test_oracle_pins.py derives it)."""
    assert gcd(p, q) == 1
    w = I.anbn_workload(p, q)
    r, _, _ = gpu_closure(w, semantics=int(lengths))
    assert r.iterations == 2 * p * q + 1
    va = np.arange(p)
    vb = np.array([0] + list(range(p, p + q - 1)))
    exp = np.array(sorted((int(i), int(j)) for i in va for j in vb), dtype=np.int32)
    for name in ("S", "S1"):
        got = r.pairs(w.nt(name))
        assert np.array_equal(got, exp), name
    nc, _ = r.iteration_stats()
    assert (nc[:-1] == 1).all() and nc[-1] == 0
    if lengths:
        bidx = {int(b): k for k, b in enumerate(vb)}
        for name, shift, extra in (("S", 0, 0), ("S1", 1, 1)):
            A = w.nt(name)
            pr = r.pairs(A)
            L = r.lengths(A).astype(np.int64)
            for (i, j), l in zip(pr.tolist(), L.tolist()):
                m = _crt(p, q, (-i) % p, (bidx[j] - shift) % q)
                assert l == 2 * m + extra, (name, i, j, l)
        # realisability of sampled cells through the oracle's path reconstruction
        cells = []
        for A in range(w.n_nt):
            pr = r.pairs(A)
            L = r.lengths(A)
            cells += [(A, i, j, int(l)) for (i, j), l in zip(pr.tolist(), L.tolist())]
        cells = np.array(cells, dtype=np.int64)
        rng = np.random.default_rng(0)
        S = w.nt("S")
        sel = cells[cells[:, 0] == S]
        for row in sel[rng.choice(len(sel), 5, replace=False)]:
            path = O.witness(w, cells, int(row[0]), int(row[1]), int(row[2]))
            assert path is not None and len(path) == row[3]
            labs = [w.labels[x] for x in path[:, 1]]
            m = len(labs) // 2
            assert labs == ["a"] * m + ["b"] * m
            assert path[0, 0] == row[1] and path[-1, 2] == row[2]


# ------------------------------------------------------------------------------------------
# Random instances (SPEC S:456 sizes) — relations, iterations, per-iteration counts, lengths
# ------------------------------------------------------------------------------------------

def test_random_parity_200():
    for s in range(200):
        w = I.random_workload(10_000 + s)
        lengths = s % 2 == 1
        # even seeds: auto cell set (hashed where allowed) and forced bit matrices alternate
        r, _, _ = gpu_closure(w, semantics=int(lengths), account_work=True, cell_set=1 if s % 4 == 2 else 0)
        ores = assert_parity(w, r, lengths=lengths)
        nc, jt = r.iteration_stats(work=True)
        st = ores.stats()
        assert nc.tolist() == st["new_bits"].tolist(), w.name
        assert jt.tolist() == st["jacobi_triples"].tolist(), w.name


def test_random_larger_parity():
    for s in range(30):
        w = I.random_workload(20_000 + s, max_nodes=300, max_edges=900, max_nt=6, max_bin=12, max_term=6,
                              n_labels=4)
        r, _, _ = gpu_closure(w, semantics=s % 2)
        assert_parity(w, r, lengths=bool(s % 2))


# ------------------------------------------------------------------------------------------
# Ontology-shaped graphs (config 2, Table 1 #triples) with Q1 / Q2 / union grammar
# ------------------------------------------------------------------------------------------

@pytest.mark.parametrize("name", ["skos", "travel", "foaf", "funding", "pizza"])
@pytest.mark.parametrize("query", ["q1", "q2"])
def test_ontology_parity(name, query):
    tr = I.TABLE1_TRIPLES[name]
    for seed in range(3):
        w = I.ontology_workload(query, int(tr / 2.28), depth=8, seed=seed, n_triples=tr)
        r, _, _ = gpu_closure(w, account_work=True)
        ores = assert_parity(w, r)
        _, jt = r.iteration_stats(work=True)
        assert jt.tolist() == ores.stats()["jacobi_triples"].tolist()


def test_g_style_copies():
    """g1-style: 8 disjoint copies: parity and exactly 8x the base counts."""
    base = I.ontology_workload("q1", int(1086 / 2.28), depth=8, seed=0, n_triples=1086)
    w8 = I.ontology_workload("q1", int(1086 / 2.28), depth=8, seed=0, n_triples=1086, copies=8)
    r1, _, _ = gpu_closure(base)
    r8, _, _ = gpu_closure(w8)
    assert_parity(w8, r8)
    for A in range(base.n_nt):
        assert r8.count(A) == 8 * r1.count(A)


@pytest.mark.parametrize("n", [1024, 2048])
def test_union_grammar_parity(n):
    w = I.config4_workload(n=n)
    r, _, _ = gpu_closure(w)
    assert_parity(w, r)


# ------------------------------------------------------------------------------------------
# S -> S S | a (var x var rules: snapshots)
# ------------------------------------------------------------------------------------------

@pytest.mark.parametrize("n,d", [(64, 1), (150, 2)])
def test_dense_stress_parity(n, d):
    w = I.dense_stress_workload(n, d, seed=n)
    r, _, _ = gpu_closure(w, semantics=1)
    assert_parity(w, r, lengths=True)


# ------------------------------------------------------------------------------------------
# Engine mechanics: log overflow + regrow, solo/grid equivalence, reuse, device edges, caps
# ------------------------------------------------------------------------------------------

def test_log_overflow_regrow():
    w = I.ontology_workload("union", 700, depth=6, seed=5)
    ores = O.run(w)
    for solo in (0, 1 << 30):
        r, _, _ = gpu_closure(w, log_capacity=64, solo_threshold=solo)
        assert r.stats()["regrows"] > 0
        assert_parity(w, r, ores)
    wl = I.anbn_workload(5, 7)
    r, _, _ = gpu_closure(wl, semantics=1, log_capacity=8)
    assert_parity(wl, r, lengths=True)


def test_reuse_and_set_edges():
    from paper_1707_01007_b200 import cfpq as C
    w1 = I.ontology_workload("q1", 300, depth=6, seed=1)
    w2 = I.ontology_workload("q1", 300, depth=6, seed=2)
    g = C.Grammar.from_workload(w1)
    d = C.Graph(w1.n_nodes, w1.edges)
    r = C.closure(g, d)
    assert_parity(w1, r)
    C.closure_reuse(g, d, r)
    assert_parity(w1, r)
    d.set_edges(w2.edges)
    C.closure_reuse(g, d, r)
    assert_parity(w2, r)


def test_reuse_bank_rotation():
    """Reused results alternate two workspace banks (the old one is cleared on a side
    stream): many reuses over graphs of different sizes, a log that regrows in one bank
    only, lengths semantics and the auto switch to the dense engine keep exact parity."""
    from paper_1707_01007_b200 import cfpq as C
    ws = [I.ontology_workload("union", 500, depth=6, seed=s) for s in range(3)]
    ws.append(dataclasses.replace(ws[0], name="small", edges=ws[0].edges[: len(ws[0].edges) // 6].copy()))
    ores = [O.run(w) for w in ws]
    g = C.Grammar.from_workload(ws[0])
    d = C.Graph(ws[0].n_nodes, ws[0].edges)
    r = C.closure(g, d, log_capacity=64)
    for rep in range(9):
        k = [0, 1, 3, 2, 0, 0, 3, 1, 2][rep]
        d.set_edges(ws[k].edges)
        C.closure_reuse(g, d, r, log_capacity=64)
        assert_parity(ws[k], r, ores[k])
    wl = [I.anbn_workload(4, 6), I.anbn_workload(6, 4)]
    gl = C.Grammar.from_workload(wl[0])
    dl = C.Graph(wl[0].n_nodes, wl[0].edges)
    rl = C.closure(gl, dl, semantics=1)
    for rep in range(4):
        w = wl[rep % 2]
        dl.set_edges(w.edges)
        C.closure_reuse(gl, dl, rl, semantics=1)
        assert_parity(w, rl, lengths=True)
    # auto policy: a sparse run, then one that switches to the dense engine, then sparse
    wd = I.dense_stress_workload(300, 2, seed=11)
    ws2 = I.dense_stress_workload(300, 1, seed=4)
    gd = C.Grammar.from_workload(wd)
    dd = C.Graph(wd.n_nodes, ws2.edges)
    rd = C.closure(gd, dd)
    for w in (ws2, wd, ws2, ws2, wd):
        dd.set_edges(w.edges)
        C.closure_reuse(gd, dd, rd)
        assert_parity(w, rd)


def test_device_edges():
    import torch
    from paper_1707_01007_b200 import cfpq as C
    w = I.ontology_workload("q2", 400, depth=7, seed=3)
    g = C.Grammar.from_workload(w)
    d = C.Graph(w.n_nodes, torch.from_numpy(w.edges).cuda())
    r = C.closure(g, d, stream=torch.cuda.current_stream())
    assert_parity(w, r)


def test_bad_device_edge_rejected():
    import torch
    from paper_1707_01007_b200 import cfpq as C
    w = I.example_workload()
    e = torch.tensor([[0, 0, 1], [0, 99, 1]], dtype=torch.int32, device="cuda")
    g = C.Grammar.from_workload(w)
    d = C.Graph(3, e)
    with pytest.raises(C.CfpqError) as ei:
        C.closure(g, d)
    assert ei.value.status == C.CFPQ_E_INVAL


def test_bad_host_edge_rejected():
    """Host edges are validated by the seed kernel too (no host pass on the upload path)."""
    from paper_1707_01007_b200 import cfpq as C
    w = I.example_workload()
    g = C.Grammar.from_workload(w)
    for bad in ([[0, 0, 1], [0, 0, 7]], [[0, 0, 1], [-1, 0, 1]], [[0, 9, 1]]):
        d = C.Graph(3, np.array(bad, dtype=np.int32))
        with pytest.raises(C.CfpqError) as ei:
            C.closure(g, d)
        assert ei.value.status == C.CFPQ_E_INVAL
    d = C.Graph(3, w.edges)
    r = C.closure(g, d)
    d.set_edges(np.array([[0, 0, 1], [3, 0, 1]], dtype=np.int32))
    with pytest.raises(C.CfpqError):
        C.closure_reuse(g, d, r)
    d.set_edges(w.edges)
    C.closure_reuse(g, d, r)
    assert_parity(w, r)


def test_max_iterations_partial_state():
    w = I.anbn_workload(3, 5)
    ores = O.run(w, max_iterations=7)
    assert ores.status == -5
    r, _, _ = gpu_closure(w, max_iterations=7)
    from paper_1707_01007_b200 import cfpq as C
    assert r.status == C.CFPQ_E_NOT_CONVERGED and r.iterations == 7
    assert_parity(w, r, ores)


def test_empty_graph_and_no_rules():
    w = I.bind("empty", I.anbn_grammar(), 5, [], "S")
    r, _, _ = gpu_closure(w)
    assert r.iterations == 1 and all(r.count(A) == 0 for A in range(w.n_nt))
    w2 = I.bind("nolab", I.anbn_grammar(), 3, [(0, "c", 1)], "S", extra_labels=["c"])
    r2, _, _ = gpu_closure(w2)
    assert r2.iterations == 1 and r2.count(0) == 0


def test_matrix_export_matches_pairs():
    w = I.ontology_workload("q1", 250, depth=6, seed=4)
    r, _, _ = gpu_closure(w)
    A = w.start
    M = r.matrix(A)
    bits = np.unpackbits(M.view(np.uint8), axis=1, bitorder="little")[:, : w.n_nodes]
    got = np.argwhere(bits).astype(np.int32)
    assert np.array_equal(got, r.pairs(A))
