"""CPU tests of the independent OpenMP bitset baseline (cpu_baseline/):

* equal to the oracle (relations, loop bodies, per-iteration |Δ_k|) on random instances, the
  paper's example, a^n b^n and S->SS|a;
* equal to the oracle's committed full-size digests of config 4 (n = 16,384 and the benched
  n = 65,536): the parity chain oracle == bitset at the headline size;
* its candidate count (the unit of bench.py's `value`) equal to a brute-force count of the
  expanded semi-naive pairs from the oracle's per-iteration states T_k.
"""
import hashlib
import json
import os

import numpy as np
import pytest

import cpu_baseline as CB
import inputs as I
import oracle as O

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _same_as_oracle(w, threads=0):
    b = CB.BitsetBaseline(w)
    k = b.run(w.edges, threads=threads)
    o = O.run(w)
    assert k == o.iterations, (w.name, k, o.iterations)
    nc, _ = b.iteration_stats(k)
    assert nc.tolist() == o.stats()["new_bits"].tolist(), w.name
    for A in range(w.n_nt):
        assert np.array_equal(b.pairs(A), o.pairs(A)), (w.name, A)
    return b, o


@pytest.mark.parametrize("seed", range(0, 120, 3))
def test_random_instances(seed):
    _same_as_oracle(I.random_workload(seed), threads=2)


def test_example_and_anbn_closed_form():
    _same_as_oracle(I.example_workload())
    for p, q in [(3, 2), (2, 5), (4, 7)]:
        w = I.anbn_workload(p, q)
        b, _ = _same_as_oracle(w)
        S = w.nt_names.index("S")
        # Lemma 3 + CRT (SURVEY V-2): R_S = a-cycle nodes x b-cycle nodes, 2pq+1 bodies
        va = set(range(p))
        vb = {0} | set(range(p, p + q - 1))
        assert set(map(tuple, b.pairs(S).tolist())) == {(i, j) for i in va for j in vb}


def test_dense_stress_and_ontology():
    _same_as_oracle(I.dense_stress_workload(150, 2, seed=3))
    _same_as_oracle(I.ontology_workload("q1", 300, depth=6, seed=1))
    _same_as_oracle(I.ontology_workload("q2", 300, depth=6, seed=2))
    _same_as_oracle(I.config4_workload(n=500, seed=4))


def _brute_candidates(w):
    """Expanded semi-naive pairs per iteration, by definition, from the oracle's T_k:
    rule A->BC, Δ = T_{k-1} minus T_{k-2} (Δ_0 = T_0), T = T_{k-1}:
      B changes, C preterminal: Σ_{(i,r) ∈ Δ_B} |row r of T_C|
      B preterminal, C changes: Σ_{(r,j) ∈ Δ_C} |column r of T_B|
      both change             : both sums
      both preterminal        : iteration 1 only, the first sum."""
    o = O.run(w, snapshots=True)
    rules = sorted(set(map(tuple, np.asarray(w.bin).reshape(-1, 3).tolist())))
    lhs = {a for a, _, _ in rules}
    K = o.iterations
    snap = [{A: set(map(tuple, o.pairs(A, snap=k).tolist())) for A in range(w.n_nt)} for k in range(K + 1)]
    out = []
    for k in range(1, K + 1):
        T = snap[k - 1]
        D = {A: T[A] - (snap[k - 2][A] if k >= 2 else set()) for A in range(w.n_nt)}
        c = 0
        for A, B, C in rules:
            pb, pc = B not in lhs, C not in lhs
            row_c = lambda r: sum(1 for (x, _) in T[C] if x == r)     # noqa: E731
            col_b = lambda r: sum(1 for (_, y) in T[B] if y == r)     # noqa: E731
            if (not pb) or (pb and pc and k == 1):
                if not (pb and not pc):
                    c += sum(row_c(r) for (_, r) in D[B])
            if not pc and not (pb and pc):
                c += sum(col_b(r) for (r, _) in D[C])
        out.append(c)
    return out


@pytest.mark.parametrize("seed", [1, 4, 7, 10, 13, 16])
def test_candidate_count_is_the_semi_naive_pairs(seed):
    w = I.random_workload(seed, max_nodes=8, max_edges=20)
    b = CB.BitsetBaseline(w)
    k = b.run(w.edges)
    _, cand = b.iteration_stats(k)
    assert cand.tolist() == _brute_candidates(w), w.name


def test_candidate_count_example():
    w = I.example_workload()
    b = CB.BitsetBaseline(w)
    k = b.run(w.edges)
    _, cand = b.iteration_stats(k)
    assert cand.tolist() == _brute_candidates(w)


def _digest_check(path):
    with open(path) as f:
        gd = json.load(f)
    seed = int(gd["workload"].rsplit("_s", 1)[1])
    w = I.config4_workload(seed=seed, n=gd["n_nodes"])
    assert w.name == gd["workload"] and len(w.edges) == gd["n_edges"]
    b = CB.BitsetBaseline(w)
    k = b.run(w.edges)
    assert k == gd["iterations"]
    nc, _ = b.iteration_stats(k)
    assert nc.tolist() == gd["new_cells"]
    for A in range(w.n_nt):
        p = np.ascontiguousarray(b.pairs(A).astype("<i4"))
        assert len(p) == gd["count"][A], (w.nt_names[A], len(p), gd["count"][A])
        assert hashlib.sha256(p.tobytes()).hexdigest() == gd["sha256"][A], w.nt_names[A]


@pytest.mark.parametrize("name", ["config4_n16384_s0.json", "config4_n65536_s0.json"])
def test_full_size_digests_of_the_oracle(name):
    """oracle == bitset at the benched size: the committed digest was written by
    scripts/golden_oracle_digest.py from oracle/ alone."""
    path = os.path.join(GOLDEN, name)
    if not os.path.exists(path):
        pytest.skip(f"{name} not generated yet (scripts/golden_oracle_digest.py)")
    _digest_check(path)
