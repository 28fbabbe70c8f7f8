"""GPU parity of the Gauss-Seidel schedule (schedule 3; DESIGN reading c17):
the fixpoint equals the oracle's T^cf (monotone operator), and the per-round states
equal the pinned test-only model (tests/gs_model.py: stages = LHS NTs in id order, each
reading T as it stands) round by round; a^n b^n needs pq + 1 rounds instead of 2pq + 1
Jacobi bodies, including config 3 at full size (n = 16,384: 32,767 rounds)."""
import numpy as np
import pytest

import inputs as I
import oracle as O
from tests.gpu_util import cuda_ok
from tests.gs_model import gs_model

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_ok(), reason="needs a CUDA device")]


def _gs(w, **kw):
    from paper_1707_01007_b200 import cfpq as C
    g, d = C.Grammar.from_workload(w), C.Graph(w.n_nodes, w.edges)
    r = C.closure(g, d, schedule=3, **kw)
    return r, g, d


def _check_model(w, r):
    rel, rounds, per = gs_model(w)
    for A in range(w.n_nt):
        assert set(map(tuple, r.pairs(A).tolist())) == rel[A], (w.name, A)
    assert r.iterations == rounds, (w.name, r.iterations, rounds)
    nc, _ = r.iteration_stats()
    assert nc.tolist() == per, w.name


def test_example():
    w = I.example_workload()
    r, _, _ = _gs(w)
    _check_model(w, r)
    o = O.run(w)
    assert r.iterations < o.iterations   # 6 Jacobi bodies


@pytest.mark.parametrize("seed", range(0, 80, 2))
def test_random_grammars(seed):
    w = I.random_workload(50_000 + seed, max_nodes=40, max_edges=120, max_nt=5, max_bin=10, max_term=5)
    r, _, _ = _gs(w)
    _check_model(w, r)


@pytest.mark.parametrize("solo", [-1, 0])
def test_union_grammar_grid_and_solo(solo):
    """solo_threshold 0 forces every step through the grid-wide path."""
    w = I.config4_workload(n=1500, seed=2)
    r, _, _ = _gs(w, solo_threshold=solo)
    _check_model(w, r)


def test_dense_var_var_rules():
    w = I.dense_stress_workload(200, 2, seed=4)
    r, _, _ = _gs(w)
    o = O.run(w)
    assert np.array_equal(r.pairs(0), o.pairs(0))


@pytest.mark.parametrize("p,q", [(3, 2), (2, 31), (5, 7), (2, 255)])
def test_anbn_rounds(p, q):
    w = I.anbn_workload(p, q)
    r, _, _ = _gs(w)
    assert r.iterations == p * q + 1
    nc, _ = r.iteration_stats()
    assert nc.tolist() == [2] * (p * q) + [0]
    o = O.run(w)
    for A in range(w.n_nt):
        assert np.array_equal(r.pairs(A), o.pairs(A))


def test_config3_full_size_closed_form():
    """Config 3 (p = 2, q = 16,383): R_S = R_S1 = a-nodes x b-nodes (Lemma 3 + CRT), in
    pq + 1 = 32,767 rounds (Jacobi: 65,533 bodies)."""
    import torch

    from paper_1707_01007_b200 import cfpq as C
    w = I.anbn_workload(2, 16383)
    g = C.Grammar.from_workload(w)
    d = C.Graph(w.n_nodes, torch.from_numpy(w.edges).cuda(), stream=torch.cuda.current_stream())
    s = torch.cuda.current_stream()
    r = C.closure(g, d, schedule=3, stream=s)
    C.closure_reuse(g, d, r, schedule=3, stream=s)
    assert r.iterations == 2 * 16383 + 1
    S = w.nt_names.index("S")
    got = r.pairs(S)
    assert len(got) == 2 * 16383
    va = np.array([0, 1])
    vb = np.array([0] + list(range(2, 2 + 16382)))
    exp = np.array([(i, j) for i in va for j in sorted(vb)], dtype=np.int32)
    assert np.array_equal(got, exp)


def test_hashed_cell_set_and_reuse():
    from paper_1707_01007_b200 import cfpq as C
    w = I.ontology_workload("q2", 600, depth=7, seed=3)
    r, g, d = _gs(w, cell_set=2)
    _check_model(w, r)
    C.closure_reuse(g, d, r, schedule=3, cell_set=2)
    _check_model(w, r)
    # a reuse may switch back to the Jacobi states
    C.closure_reuse(g, d, r, schedule=0, cell_set=2)
    o = O.run(w)
    assert r.iterations == o.iterations and np.array_equal(r.pairs(w.start), o.pairs(w.start))


def test_rejects_unsupported_combinations():
    from paper_1707_01007_b200 import cfpq as C
    w = I.example_workload()
    g, d = C.Grammar.from_workload(w), C.Graph(w.n_nodes, w.edges)
    for kw in (dict(semantics=1), dict(path_policy=2), dict(path_policy=3), dict(account_work=True),
               dict(emulate_ranks=2)):
        with pytest.raises(C.CfpqError):
            C.closure(g, d, schedule=3, **kw)
