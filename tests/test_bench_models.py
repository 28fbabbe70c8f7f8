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


def test_tensor_roofline_accounting():
    """bench.tensor_roofline: issued MMA work is counted in 128 x 32 x 128 units (an M=128 x
    N=256 x K=128 int8 k-block = 8 units, a 256-deep fp4 k-block = 16), the fp4 peak is twice
    the int8 one (nominal fp4 / int8 = 9 / 4.5), both derived from the same bf16 figure."""
    stats = {"mma_kblocks": 8 * 1000, "loop_ns": 1e6}
    r8 = bench.tensor_roofline(stats, 1.0, fmt=1)
    r4 = bench.tensor_roofline(stats, 1.0, fmt=2)
    ops = 1000 * 2 * 128 * 256 * 128
    assert r8["issued_ops"] == ops and r4["issued_ops"] == ops
    assert abs(r8["achieved"] - ops / 1e-3 / 1e12) < 1e-6
    assert abs(r4["peak"] - 2 * r8["peak"]) < 1e-6
    assert abs(r4["frac_of_nominal"] * 9000.0 - r8["frac_of_nominal"] * 4500.0) < 1e-6


def _rows_bytes_by_definition(w, snaps):
    """DESIGN §5's bit-row byte model written out with plain loops over the oracle's T_k
    (an independent count of what bench.rows_alg_bytes computes with scipy)."""
    n = w.n_nodes
    W = (n + 31) // 32
    rules = sorted(set(map(tuple, np.asarray(w.bin).reshape(-1, 3).tolist())))
    lhs = {a for a, _, _ in rules}
    K = len(snaps) - 1
    total = 8 * sum(len(snaps[0][A]) for A in range(w.n_nt))
    for k in range(1, K + 1):
        T = snaps[k - 1]
        scanned = set()
        for A, B, C in rules:
            tb, tc = T[B], T[C]
            pb, pc = B not in lhs, C not in lhs
            rows_b = {i for i, _ in tb}
            scan = 4 * W * len(rows_b)
            if not pb and pc:           # L rules sharing B scan each row of T_B once
                if B in scanned:
                    scan = 0
                scanned.add(B)
            if not tb or not tc:
                if not pb and tb:
                    total += scan
                continue
            row_c = {}
            for r, j in tc:
                row_c.setdefault(r, set()).add(j)
            if not pb and pc:
                total += scan + 8 * len(tb) + 4 * sum(len(row_c.get(r, ())) for _, r in tb)
            elif pb and not pc:
                refs = {r for _, r in tb}
                total += 8 * len(rows_b) + 4 * len(tb) + 4 * W * sum(1 for r in refs if r in row_c)
            elif not pb and not pc:
                refs = {r for _, r in tb}
                total += 4 * W * len(rows_b) + 4 * W * sum(1 for r in refs if r in row_c)
            else:
                if k > 1:
                    continue
                total += 8 * len(rows_b) + 12 * len(tb) + 4 * sum(len(row_c.get(r, ())) for _, r in tb)
            words = {(i, j // 32) for i, r in tb for j in row_c.get(r, ())}
            total += 8 * len(words)
        for A in lhs:
            new = snaps[k][A] - snaps[k - 1][A]
            total += 32 * len({(i, j // 32) for i, j in new})
    return total


def test_rows_alg_bytes_equals_the_definition_counted_by_hand():
    """bench.rows_alg_bytes (scipy) == the same model counted cell by cell, on the paper's
    example (n = 3: W = 1 word per row) and on small union-grammar / random instances."""
    for w in (I.example_workload(), I.config4_workload(n=300, seed=2), I.random_workload(31),
              I.ontology_workload("q2", 200, depth=5, seed=1)):
        s = _Snapshots(w)
        snaps = [{A: set(map(tuple, s.pairs_at(A, k).tolist())) for A in range(w.n_nt)}
                 for k in range(s.iterations + 1)]
        assert bench.rows_alg_bytes(w, s) == _rows_bytes_by_definition(w, snaps), w.name
