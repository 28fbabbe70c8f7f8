"""GPU parity of the asynchronous schedule (schedule = 2): same fixpoint T^cf as the
oracle's Jacobi closure (the operator T -> T ∪ T×T is monotone), relations
compared element by element; no per-iteration states."""
import numpy as np
import pytest

import inputs as I
import oracle as O
from tests.gpu_util import assert_parity, cuda_ok, gpu_closure

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_ok(), reason="needs a CUDA device")]


def test_async_example_and_random():
    w = I.example_workload()
    r, _, _ = gpu_closure(w, schedule=2)
    assert r.iterations == 0
    assert_parity(w, r, check_iterations=False)
    for s in range(100):
        w = I.random_workload(70_000 + s, max_nodes=40, max_edges=150, max_nt=5, max_bin=10, max_term=5)
        r, _, _ = gpu_closure(w, schedule=2)
        assert_parity(w, r, check_iterations=False)


@pytest.mark.parametrize("query", ["q1", "q2", "union"])
def test_async_ontology(query):
    for seed in range(2):
        w = I.ontology_workload(query, 900, depth=7, seed=seed)
        r, _, _ = gpu_closure(w, schedule=2)
        assert_parity(w, r, check_iterations=False)


def test_async_anbn_and_dense():
    w = I.anbn_workload(5, 7)
    r, _, _ = gpu_closure(w, schedule=2)
    assert_parity(w, r, check_iterations=False)
    w = I.dense_stress_workload(150, 2, seed=5)       # var x var rule: live snapshots
    r, _, _ = gpu_closure(w, schedule=2)
    assert_parity(w, r, check_iterations=False)


def test_async_log_overflow_and_reuse():
    from paper_1707_01007_b200 import cfpq as C
    w = I.ontology_workload("union", 700, depth=6, seed=5)
    ores = O.run(w)
    r, g, d = gpu_closure(w, schedule=2, log_capacity=64)
    assert r.stats()["regrows"] > 0
    assert_parity(w, r, ores, check_iterations=False)
    # the same result object, back and forth between the schedules
    C.closure_reuse(g, d, r, schedule=0)
    assert_parity(w, r, ores)
    C.closure_reuse(g, d, r, schedule=2)
    assert_parity(w, r, ores, check_iterations=False)


def test_async_full_size_config4_equals_jacobi():
    """At the bench's size the asynchronous closure equals the Jacobi closure bit for bit."""
    w = I.config4_workload()
    ra, _, _ = gpu_closure(w, schedule=2)
    rj, _, _ = gpu_closure(w, schedule=0)
    for A in range(w.n_nt):
        assert np.array_equal(ra.pairs(A), rj.pairs(A)), w.nt_names[A]


def test_async_rejects_lengths():
    from paper_1707_01007_b200 import cfpq as C
    with pytest.raises(C.CfpqError) as e:
        gpu_closure(I.example_workload(), schedule=2, semantics=1)
    assert e.value.status == C.CFPQ_E_UNSUPPORTED
