"""Repro: bit-row engine on the all-one 1025-node S->SS|a input (chunk-list overflow + redo)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import inputs as I
from paper_1707_01007_b200 import cfpq as C

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1025
w = I.bind(f"allone_n{n}", I.dense_stress_grammar(), n, [(i, "a", j) for i in range(n) for j in range(n)], "S",
           extra_labels=["a"])
r = C.closure(C.Grammar.from_workload(w), C.Graph(w.n_nodes, w.edges), path_policy=3)
print("iterations", r.iterations, "count", r.count(0), "expected", n * n)
