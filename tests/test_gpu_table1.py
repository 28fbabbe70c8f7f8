"""Config 2: Q1 and Q2 on synthetic ontology-shaped graphs with the #triples of
the paper's Tables 1-2 and a g-style 8-copy graph, every engine against the
oracle element by element, with its per-iteration new-cell counts (Jacobi states)."""
import numpy as np
import pytest

import inputs as I
from tests.gpu_util import cuda_ok, gpu_closure, oracle_run

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_ok(), reason="needs a CUDA device")]

ENGINES = {
    "sparse": dict(path_policy=1),
    "rows": dict(path_policy=3),
    "tensor_fp4": dict(path_policy=2, tensor_format=2),
    "hashed": dict(path_policy=1, cell_set=2),
}


def _workload(query, triples, copies=1, seed=0):
    return I.ontology_workload(query, max(14, int(triples / 2.28)), depth=8, seed=seed, n_triples=triples,
                               copies=copies)


@pytest.mark.parametrize("engine", list(ENGINES))
@pytest.mark.parametrize("query", ["q1", "q2"])
@pytest.mark.parametrize("triples", [252, 640, 1980])
def test_table1_sizes(triples, query, engine):
    w = _workload(query, triples)
    o = oracle_run(w)
    r, _, _ = gpu_closure(w, **ENGINES[engine])
    for A in range(w.n_nt):
        assert np.array_equal(r.pairs(A), o.pairs(A)), (w.name, engine, w.nt_names[A])
    assert r.iterations == o.iterations
    nc, _ = r.iteration_stats()
    assert nc.tolist() == o.stats()["new_bits"].tolist()


@pytest.mark.parametrize("query", ["q1", "q2"])
def test_gstyle_is_eight_copies(query):
    """g-style graphs (8 disjoint copies): #results exactly 8 x the base graph's."""
    base, g8 = _workload(query, 1086), _workload(query, 1086, copies=8)
    rb, _, _ = gpu_closure(base)
    r8, _, _ = gpu_closure(g8)
    assert r8.count(g8.start) == 8 * rb.count(base.start)
    assert r8.iterations == rb.iterations
