"""CPU pins of the test-only Gauss-Seidel model (tests/gs_model.py) before it judges the GPU
schedule 3: its fixpoint equals the oracle's T^cf (Alg. 1; the least fixpoint of
a monotone operator does not depend on the update order), and on a^n b^n over coprime
cycles it needs exactly pq + 1 rounds with two new cells per round (Jacobi: 2pq + 1
bodies with one cell each, SURVEY V-2)."""
import pytest

import inputs as I
import oracle as O
from tests.gs_model import gs_model


@pytest.mark.parametrize("seed", range(0, 60, 2))
def test_model_fixpoint_is_the_oracles(seed):
    w = I.random_workload(seed)
    rel, rounds, per = gs_model(w)
    o = O.run(w)
    assert rel == o.relation_sets()
    assert rounds <= o.iterations          # in-place never needs more rounds than Jacobi
    assert sum(per) == sum(o.stats()["new_bits"])


def test_model_example_and_ontology():
    for w in (I.example_workload(), I.ontology_workload("q1", 120, depth=5, seed=2), I.config4_workload(n=300)):
        rel, rounds, _ = gs_model(w)
        o = O.run(w)
        assert rel == o.relation_sets() and rounds <= o.iterations


@pytest.mark.parametrize("p,q", [(2, 3), (3, 2), (2, 5), (3, 4), (4, 5), (5, 7), (2, 9)])
def test_model_anbn_rounds(p, q):
    w = I.anbn_workload(p, q)
    rel, rounds, per = gs_model(w)
    assert rounds == p * q + 1 and per == [2] * (p * q) + [0]
    o = O.run(w)
    assert rel == o.relation_sets() and o.iterations == 2 * p * q + 1
