"""Test-only model of the Gauss-Seidel schedule (schedule 3, DESIGN reading c17), small
inputs only: one iteration (round) applies the rules stage by stage, the LHS nonterminals
in id order; the product of stage A reads T as it stands when the stage starts (every cell
derived by earlier stages of the same round included), T <- T ∪ {A-cells of T x T}.
The fixpoint is Alg. 1's (monotone operator); per-round counts are this order's."""
import numpy as np


def gs_model(w):
    rules = sorted(set(map(tuple, np.asarray(w.bin).reshape(-1, 3).tolist())))
    stages = sorted({a for a, _, _ in rules})
    term = np.asarray(w.term).reshape(-1, 2).tolist()
    T = set()
    for s, x, d in np.asarray(w.edges).reshape(-1, 3).tolist():
        for A, lab in term:
            if lab == x:
                T.add((A, s, d))
    per_round = []
    while True:
        added = 0
        for A in stages:
            rows = {}
            for (X, i, j) in T:
                rows.setdefault((X, i), []).append(j)
            new = set()
            for (a, B, C) in rules:
                if a != A:
                    continue
                for (X, i, r) in T:
                    if X == B:
                        for j in rows.get((C, r), ()):
                            if (A, i, j) not in T:
                                new.add((A, i, j))
            T |= new
            added += len(new)
        per_round.append(added)
        if added == 0:
            break
    rel = {A: set() for A in range(w.n_nt)}
    for (A, i, j) in T:
        rel[A].add((i, j))
    return rel, len(per_round), per_round
