"""Node-order probe for config 4: the closure is invariant under a relabelling of the nodes
(R_A of the relabelled graph = the relabelled R_A), but the bit-matrix words a candidate touches
depend on it.  Times the unchanged closure (CUDA events, L2 flushed, interleaved) on the seeded
ids and on host-computed locality orders (BFS over the undirected graph, reverse Cuthill-McKee,
degree-sorted), and checks |R_A| is the same for every order.  Timing only — the relabelling is
done on the host outside the timed region.

usage: python scripts/reorder_probe.py
"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import scipy.sparse as sp
import scipy.sparse.csgraph as cg
import torch

import inputs as I
from paper_1707_01007_b200 import cfpq as C


def orders(w):
    n = w.n_nodes
    e = w.edges
    a = sp.coo_matrix((np.ones(len(e)), (e[:, 0], e[:, 2])), shape=(n, n)).tocsr()
    u = (a + a.T).tocsr()
    out = {"seeded": np.arange(n)}
    # BFS from every unvisited node, in order of decreasing degree (one tree per component)
    deg = np.diff(u.indptr)
    seen = np.zeros(n, bool)
    seq = []
    for r in np.argsort(-deg, kind="stable"):
        if seen[r]:
            continue
        o = cg.breadth_first_order(u, r, directed=False, return_predecessors=False)
        o = o[~seen[o]]
        seen[o] = True
        seq.append(o)
    out["bfs"] = np.concatenate(seq)
    out["rcm"] = cg.reverse_cuthill_mckee(u, symmetric_mode=True).astype(np.int64)
    out["degree"] = np.argsort(-deg, kind="stable")
    return out


def relabel(w, order):
    new_id = np.empty(w.n_nodes, np.int64)
    new_id[order] = np.arange(w.n_nodes)
    e = w.edges.copy()
    e[:, 0] = new_id[e[:, 0]]
    e[:, 2] = new_id[e[:, 2]]
    return e


def main():
    w = I.config4_workload()
    s = torch.cuda.current_stream()
    g = C.Grammar.from_workload(w)
    ords = orders(w)
    graphs = {k: C.Graph(w.n_nodes, torch.from_numpy(relabel(w, o)).cuda(), stream=s) for k, o in ords.items()}
    res = {k: C.closure(g, d, stream=s) for k, d in graphs.items()}
    counts = {k: [r.count(A) for A in range(w.n_nt)] for k, r in res.items()}
    assert all(c == counts["seeded"] for c in counts.values()), counts
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    t = {k: [] for k in graphs}
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for rep in range(30):
        for k, d in graphs.items():
            flush.fill_(1)
            e0.record(s)
            C.closure_reuse(g, d, res[k], stream=s)
            e1.record(s)
            e1.synchronize()
            if rep >= 5:
                t[k].append(e0.elapsed_time(e1))
    for k in graphs:
        st = res[k].stats()
        print(f"{k:8s} step {statistics.median(t[k]):.4f} ms (min {min(t[k]):.4f})  loop {st['loop_ns'] / 1e6:.3f}"
              f"  iterations {res[k].iterations}  cells {st['cells']}")


if __name__ == "__main__":
    main()
