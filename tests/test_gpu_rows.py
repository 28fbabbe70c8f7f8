"""GPU parity of the bit-row CUDA-core path (path_policy = 3): the paper-faithful
full-operand Jacobi products over packed rows (Alg. 1 line 9)."""
import pytest

import inputs as I
from tests.gpu_util import assert_parity, cuda_ok, gpu_closure

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_ok(), reason="needs a CUDA device")]


def test_rows_example(example_golden):
    g = example_golden
    w = I.bind("example", I.same_generation_grammar(), 3, g["edges"], "S")
    r, _, _ = gpu_closure(w, path_policy=3)
    assert r.iterations == 6
    ores = assert_parity(w, r)
    nc, _ = r.iteration_stats()
    assert nc.tolist() == ores.stats()["new_bits"].tolist()


def test_rows_random_and_dense():
    for s in range(40):
        w = I.random_workload(60_000 + s, max_nodes=60, max_edges=200, max_nt=5, max_bin=10, max_term=5)
        r, _, _ = gpu_closure(w, path_policy=3)
        assert_parity(w, r)
    for n, d in ((100, 2), (257, 1), (300, 3)):
        w = I.dense_stress_workload(n, d, seed=n)
        r, _, _ = gpu_closure(w, path_policy=3)
        ores = assert_parity(w, r)
        nc, _ = r.iteration_stats()
        assert nc.tolist() == ores.stats()["new_bits"].tolist()


@pytest.mark.parametrize("n", [700, 2048])
def test_rows_union_grammar(n):
    w = I.config4_workload(n=n)
    r, _, _ = gpu_closure(w, path_policy=3)
    assert_parity(w, r)


def test_rows_wide_rows_agree_with_sparse():
    """n = 9000 spans several 256-word slices per row: the row path equals the sparse engine."""
    import numpy as np
    w = I.ontology_workload("q1", 9000, depth=7, seed=4)
    r3, _, _ = gpu_closure(w, path_policy=3)
    r1, _, _ = gpu_closure(w, path_policy=1)
    assert r3.iterations == r1.iterations
    for A in range(w.n_nt):
        assert np.array_equal(r3.pairs(A), r1.pairs(A))
