"""Jacobi (schedule 0) vs asynchronous (schedule 2) closure time."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import inputs as I
from paper_1707_01007_b200 import cfpq as C
for name, w in (("config4", I.config4_workload()), ("config3", I.anbn_workload(2, 16383)),
                ("config2-g", I.ontology_workload("q1", int(1980 / 2.28), depth=8, seed=0, n_triples=1980, copies=8)),
                ("dense-2048", I.dense_stress_workload(2048, 2, 0))):
    g = C.Grammar.from_workload(w)
    d = C.Graph(w.n_nodes, torch.from_numpy(w.edges).cuda())
    for sch in (0, 2):
        if name == "dense-2048" and sch == 0:
            continue
        r = C.closure(g, d, schedule=sch)
        ts = []
        for _ in range(3):
            C.closure_reuse(g, d, r, schedule=sch)
            st = r.stats()
            ts.append((st["loop_ns"] + st["seed_ns"]) / 1e6)
        print(f"{name} schedule={sch}: closure {min(ts):.3f} ms (loop {st['loop_ns']/1e6:.3f}) cells={st['cells']} "
              f"regrows={st['regrows']}")
