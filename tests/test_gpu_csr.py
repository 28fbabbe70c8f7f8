"""cfpq_result_csr: R_A (Theorem 2) in compressed-row form, checked against the oracle's
relation (row pointers from its row counts, columns in ascending order) for every engine, with
host and device destinations, an empty relation and a too-small capacity."""
import numpy as np
import pytest

import inputs as I
from tests.gpu_util import cuda_ok, gpu_closure, oracle_run

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_ok(), reason="needs a CUDA device")]

ENGINES = {
    "sparse": dict(path_policy=1, cell_set=1),
    "hashed": dict(path_policy=1, cell_set=2),
    "rows": dict(path_policy=3),
    "tensor_fp4": dict(path_policy=2, tensor_format=2),
    "peer_exchange3": dict(emulate_ranks=3, exchange=1),
}


def _expected(w, A, ores):
    p = ores.pairs(A)
    p = p[np.lexsort((p[:, 1], p[:, 0]))] if len(p) else np.zeros((0, 2), np.int64)
    counts = np.bincount(p[:, 0], minlength=w.n_nodes) if len(p) else np.zeros(w.n_nodes, np.int64)
    row_ptr = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    return row_ptr, p[:, 1].astype(np.int32)


@pytest.mark.parametrize("engine", list(ENGINES))
@pytest.mark.parametrize("n", [129, 1025])
def test_csr_matches_oracle(engine, n):
    w = I.config4_workload(n=n, seed=5)
    ores = oracle_run(w)
    r, _, _ = gpu_closure(w, **ENGINES[engine])
    for A in range(w.n_nt):
        rp, cols = r.csr(A)
        erp, ecols = _expected(w, A, ores)
        assert np.array_equal(rp, erp), (engine, w.nt_names[A])
        assert np.array_equal(cols, ecols), (engine, w.nt_names[A])


def test_csr_device_and_pinned_destinations():
    import torch
    w = I.config4_workload(n=1025, seed=6)
    ores = oracle_run(w)
    r, _, _ = gpu_closure(w)
    A = w.nt_names.index("S_Q1")
    erp, ecols = _expected(w, A, ores)
    m = len(ecols)
    rp_d = torch.full((w.n_nodes + 1,), -1, dtype=torch.int64, device="cuda")
    cols_d = torch.full((m + 7,), -1, dtype=torch.int32, device="cuda")
    rp, cols = r.csr(A, rp_d, cols_d)
    assert np.array_equal(rp.cpu().numpy(), erp) and np.array_equal(cols.cpu().numpy(), ecols)
    assert int(cols_d[m:].min()) == -1   # nothing past |R_A|
    rp_h = torch.empty((w.n_nodes + 1,), dtype=torch.int64).pin_memory()
    cols_h = torch.empty((m,), dtype=torch.int32).pin_memory()
    rp, cols = r.csr(A, rp_h, cols_h)
    assert np.array_equal(rp.numpy(), erp) and np.array_equal(cols.numpy(), ecols)
    # the pair form, row by row
    pairs = r.pairs(A)
    assert np.array_equal(pairs[:, 1], ecols)
    assert np.array_equal(np.repeat(np.arange(w.n_nodes), np.diff(erp)), pairs[:, 0])


def test_csr_empty_relation_and_small_capacity():
    from paper_1707_01007_b200 import cfpq as C
    w = I.bind("zero_csr", I.union_grammar(), 300, [], "S_Q1")
    r, _, _ = gpu_closure(w)
    rp, cols = r.csr(0)
    assert len(cols) == 0 and not rp.any() and len(rp) == 301
    w = I.config4_workload(n=1025, seed=7)
    r, _, _ = gpu_closure(w)
    A = w.nt_names.index("S_Q1")
    m = r.count(A)
    assert m > 1
    import torch
    rp = torch.zeros((w.n_nodes + 1,), dtype=torch.int64)
    cols = torch.zeros((m - 1,), dtype=torch.int32)
    with pytest.raises(C.CfpqError) as e:
        r.csr(A, rp, cols)
    assert e.value.status == C.CFPQ_E_INVAL


def test_csr_long_rows():
    """S -> S S | a on a random digraph: rows of up to 288 entries."""
    w = I.dense_stress_workload(300, 3, seed=3)
    ores = oracle_run(w)
    erp, ecols = _expected(w, w.start, ores)
    assert np.diff(erp).max() > 256
    # the sparse engine (the hashed set and row shards do not take S -> S S); device destination too
    import torch
    r, _, _ = gpu_closure(w, **ENGINES["sparse"])
    rp, cols = r.csr(w.start)
    assert np.array_equal(rp, erp) and np.array_equal(cols, ecols)
    rp_d = torch.empty((w.n_nodes + 1,), dtype=torch.int64, device="cuda")
    cols_d = torch.empty((len(ecols),), dtype=torch.int32, device="cuda")
    rp, cols = r.csr(w.start, rp_d, cols_d)
    assert np.array_equal(rp.cpu().numpy(), erp) and np.array_equal(cols.cpu().numpy(), ecols)


def test_csr_large_n_hashed():
    """n = 2^18 + 3 (row pointers past 2^18, 64-bit sort keys) on the hashed cell set."""
    n = (1 << 18) + 3
    g = I.union_grammar()
    edges = [(0, "subClassOf_r", 5), (5, "subClassOf", n - 1), (n - 1, "subClassOf_r", 7), (7, "subClassOf", n - 2),
             (n - 2, "type_r", 9), (9, "type", 11)]
    w = I.bind("large_n_csr", g, n, edges, "S_Q1")
    ores = oracle_run(w)
    r, _, _ = gpu_closure(w, cell_set=2)
    for A in range(w.n_nt):
        rp, cols = r.csr(A)
        erp, ecols = _expected(w, A, ores)
        assert np.array_equal(rp, erp) and np.array_equal(cols, ecols), w.nt_names[A]
