"""Config 2: Q1 and Q2 on synthetic ontology-shaped graphs with the #triples of
the paper's Tables 1 and 2, plus the g-style graphs (8 disjoint copies of the
funding / wine / pizza sizes).  Closure time on the B200 (device events, median of 10 reuses)
beside the paper's sGPU column (GTX 1070, CUSPARSE; context only: other hardware, the real RDF
graphs, unstated timing scope — BASELINE.md §1).  Each base graph's relation is checked against
the oracle; each g-style graph's #results against 8x its base graph's.

usage: python scripts/table1.py [> profiles/r02/table1.md]
"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import inputs as I
import oracle as O
from paper_1707_01007_b200 import cfpq as C

# name, #triples, paper Q1 sGPU ms, paper Q2 sGPU ms
TABLE = [("skos", 252, 12, 1), ("generations", 273, 13, 0), ("travel", 277, 30, 10), ("univ-bench", 293, 15, 9),
         ("atom-primitive", 425, 22, 2), ("biomedical-measure-primitive", 459, 20, 24), ("foaf", 631, 9, 3),
         ("people-pets", 640, 32, 6), ("funding", 1086, 36, 27), ("wine", 1839, 54, 6), ("pizza", 1980, 24, 23)]
GSTYLE = [("g1 (8 x funding)", 1086, 82, 38), ("g2 (8 x wine)", 1839, 185, 21), ("g3 (8 x pizza)", 1980, 127, 40)]


def workload(query, triples, copies, seed):
    return I.ontology_workload(query, max(14, int(triples / 2.28)), depth=8, seed=seed, n_triples=triples,
                               copies=copies)


def timed(w, reps=10):
    g = C.Grammar.from_workload(w)
    s = torch.cuda.current_stream()
    d = C.Graph(w.n_nodes, torch.from_numpy(w.edges).cuda(), stream=s)
    r = C.closure(g, d, stream=s)
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        C.closure_reuse(g, d, r, stream=s)
        e1.record(s)
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    return r, statistics.median(ts)


def main():
    seed = 0
    print("| graph | #triples | query | #results (start NT) | iterations | B200 closure ms | paper sGPU ms (GTX 1070, context) | check |")
    print("|---|---|---|---|---|---|---|---|")
    base = {}
    for name, tri, q1, q2 in TABLE:
        for query, paper in (("q1", q1), ("q2", q2)):
            w = workload(query, tri, 1, seed)
            r, ms = timed(w)
            o = O.run(w)
            ok = all(np.array_equal(r.pairs(A), o.pairs(A)) for A in range(w.n_nt))
            cnt = r.count(w.start)
            base[(tri, query)] = cnt
            print(f"| {name} | {tri} | {query.upper()} | {cnt} | {r.iterations} | {ms:.3f} | {paper} | "
                  f"{'= oracle' if ok else 'MISMATCH'} |", flush=True)
            assert ok, (name, query)
    for name, tri, q1, q2 in GSTYLE:
        for query, paper in (("q1", q1), ("q2", q2)):
            w = workload(query, tri, 8, seed)
            r, ms = timed(w)
            cnt = r.count(w.start)
            ok = cnt == 8 * base[(tri, query)]
            print(f"| {name} | {8 * tri} | {query.upper()} | {cnt} | {r.iterations} | {ms:.3f} | {paper} | "
                  f"{'= 8 x base' if ok else 'MISMATCH'} |", flush=True)
            assert ok, (name, query)


if __name__ == "__main__":
    main()
