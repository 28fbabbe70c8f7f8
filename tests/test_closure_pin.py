"""CPU pin of tests/closure_pin.py (the strict transitive closure used to judge config S at
full size) against the oracle's S -> S S | a closure and a brute-force BFS."""
import numpy as np
import pytest

import inputs as I
import oracle as O
from tests.closure_pin import strict_closure_bits


def _bits_to_pairs(bits, n):
    out = set()
    for i in range(n):
        for w in np.nonzero(bits[i])[0].tolist():
            v = int(bits[i, w])
            while v:
                b = (v & -v).bit_length() - 1
                out.add((i, 32 * w + b))
                v &= v - 1
    return out


@pytest.mark.parametrize("n,d,seed", [(60, 1, 0), (90, 2, 1), (130, 1, 2), (200, 3, 3), (33, 1, 4)])
def test_pin_equals_oracle(n, d, seed):
    w = I.dense_stress_workload(n, d, seed)
    e = np.asarray(w.edges)
    bits = strict_closure_bits(n, e[:, 0], e[:, 2])
    assert _bits_to_pairs(bits, n) == set(map(tuple, O.run(w).pairs(0).tolist()))


def test_pin_self_loops_and_paths():
    n = 70
    src = [i for i in range(n - 1)] + [5, 40]
    dst = [i + 1 for i in range(n - 1)] + [5, 40]
    bits = strict_closure_bits(n, src, dst)
    exp = {(i, j) for i in range(n) for j in range(i + 1, n)} | {(5, 5), (40, 40)}
    assert _bits_to_pairs(bits, n) == exp
