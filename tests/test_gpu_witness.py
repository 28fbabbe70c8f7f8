"""GPU single-path witness extraction (cfpq_result_witness; P:391,
P:417) against the oracle's reconstruction (oracle_witness) on the same length table.
Both take the first rule of A in grammar order, the smallest split node r and the
lowest-index seed edge, so the paths are compared element by element; every path is
also checked directly: consecutive edges of the graph from i to j, exactly l edges,
and a word that A derives (CYK)."""
import dataclasses

import numpy as np
import pytest

import inputs as I
import oracle as O
from tests.gpu_util import cuda_ok

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_ok(), reason="needs a CUDA device")]


def _closure(w):
    from paper_1707_01007_b200 import cfpq as C
    g = C.Grammar.from_workload(w)
    d = C.Graph(w.n_nodes, w.edges)
    r = C.closure(g, d, semantics=1)
    return r, d


def _table(ores, n_nt):
    rows = []
    for A in range(n_nt):
        L = ores.lengths(A)
        if len(L):
            rows.append(np.column_stack([np.full(len(L), A, dtype=np.int64), L]))
    t = np.concatenate(rows) if rows else np.zeros((0, 4), dtype=np.int64)
    return t[np.lexsort((t[:, 2], t[:, 1], t[:, 0]))]


def _check_path(w, A, i, j, l, path):
    assert path.shape == (l, 3)
    E = set(map(tuple, w.edges.tolist()))
    assert all(tuple(e) in E for e in path.tolist())
    assert path[0, 0] == i and path[-1, 2] == j
    assert np.array_equal(path[1:, 0], path[:-1, 2])


def _compare_all(w, max_cells=None, cyk_max=40):
    r, d = _closure(w)
    ores = O.run(w, lengths=True)
    # the library keeps the rules deduplicated in (A, B, C) order (P is a set): hand
    # the oracle's reconstruction the same rule order
    ws = dataclasses.replace(w, bin=np.unique(w.bin.reshape(-1, 3), axis=0).astype(np.int32))
    table = _table(ores, w.n_nt)
    cells = table if max_cells is None else table[:: max(1, len(table) // max_cells)]
    for A, i, j, l in cells.tolist():
        got = r.witness(d, A, i, j)
        exp = O.witness(ws, table, A, i, j)
        assert exp is not None
        assert np.array_equal(got, exp), (w.name, A, i, j, l)
        _check_path(w, A, i, j, l, got)
        if l <= cyk_max:
            assert O.cyk(w, got[:, 1].tolist(), A)
    return len(cells)


def test_witness_example(example_golden):
    g = example_golden
    w = I.bind("example", I.same_generation_grammar(), 3, g["edges"], "S")
    assert _compare_all(w) > 0
    # S(1,2) has length 2 (type_r then type)
    r, d = _closure(w)
    p = r.witness(d, w.nt_names.index("S"), 1, 2)
    assert [w.labels[x] for x in p[:, 1]] == ["type_r", "type"]


@pytest.mark.parametrize("p,q", [(3, 2), (2, 5), (5, 3), (4, 7)])
def test_witness_anbn(p, q):
    _compare_all(I.anbn_workload(p, q))


def test_witness_random():
    n = 0
    for s in range(40):
        w = I.random_workload(90_000 + s, max_nodes=30, max_edges=80, max_nt=5, max_bin=8, max_term=5)
        n += _compare_all(w, max_cells=60)
    assert n > 100


def test_witness_ontology():
    w = I.ontology_workload("q1", 300, depth=6, seed=3)
    _compare_all(w, max_cells=80)


def test_witness_config5_long_paths():
    """Config 5 (a^n b^n, p=2, q=16383, lengths): the longest paths (65,533 edges) are a^m b^m
    words (S) / a^m b^(m+1) (S1) by the grammar; lengths follow the CRT closed form."""
    p, q = 2, 16383
    w = I.anbn_workload(p, q)
    r, d = _closure(w)
    S, S1 = w.nt_names.index("S"), w.nt_names.index("S1")
    a, b = w.labels.index("a"), w.labels.index("b")
    for A, i, j in [(S, 0, 0), (S, 1, p + 5), (S1, 0, p + q - 2), (S1, 1, 0), (S, 1, p + q - 2)]:
        path = r.witness(d, A, i, j)
        l = len(path)
        _check_path(w, A, i, j, l, path)
        m = l // 2
        labs = path[:, 1]
        assert (labs[:m] == a).all()
        assert (labs[m:] == b).all()
        assert (l % 2 == 0) if A == S else (l % 2 == 1)
    assert max(len(r.witness(d, S1, i, j)) for i, j in [(0, p + q - 2), (1, 0), (1, p)]) > 1000


def test_witness_rejections():
    from paper_1707_01007_b200 import cfpq as C
    w = I.anbn_workload(3, 2)
    r, d = _closure(w)
    with pytest.raises(C.CfpqError):
        r.witness(d, w.nt_names.index("S"), 3, 1)     # not in R_S
    g = C.Grammar.from_workload(w)
    r2 = C.closure(g, d)                              # relational run: no lengths
    with pytest.raises(C.CfpqError):
        r2.witness(d, 0, 0, 0)
