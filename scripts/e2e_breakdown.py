"""Wall-clock breakdown of the end-to-end config-4 step (set_edges from pinned host memory,
closure, sorted pairs of the start NT into pinned host memory)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import inputs as I
from paper_1707_01007_b200 import cfpq as C

w = I.config4_workload()
stream = torch.cuda.current_stream()
g = C.Grammar.from_workload(w)
pinned = torch.from_numpy(w.edges.copy()).pin_memory()
d = C.Graph(w.n_nodes, pinned, stream=stream)
r = C.closure(g, d, stream=stream)
m = r.count(w.start)
out = torch.empty((m, 2), dtype=torch.int32).pin_memory()
outd = torch.empty((m, 2), dtype=torch.int32, device="cuda")
T = {k: [] for k in ["set_edges", "closure", "pairs_host", "pairs_dev", "count", "total"]}
for it in range(25):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    d.set_edges(pinned, stream=stream)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    C.closure_reuse(g, d, r, stream=stream)
    t2 = time.perf_counter()
    r.pairs(w.start, out=out)
    t3 = time.perf_counter()
    if it >= 5:
        T["set_edges"].append(t1 - t0)
        T["closure"].append(t2 - t1)
        T["pairs_host"].append(t3 - t2)
        T["total"].append(t3 - t0)
    torch.cuda.synchronize()
    t4 = time.perf_counter()
    r.pairs(w.start, out=outd)
    torch.cuda.synchronize()
    t5 = time.perf_counter()
    r.count(w.start)
    t6 = time.perf_counter()
    if it >= 5:
        T["pairs_dev"].append(t5 - t4)
        T["count"].append(t6 - t5)
# the same step reading R_start back as CSR (cfpq_result_csr) instead of pairs
rp = torch.empty((w.n_nodes + 1,), dtype=torch.int64).pin_memory()
cols = torch.empty((m,), dtype=torch.int32).pin_memory()
T["csr_host"], T["total_csr"] = [], []
for it in range(25):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    d.set_edges(pinned, stream=stream)
    C.closure_reuse(g, d, r, stream=stream)
    t2 = time.perf_counter()
    r.csr(w.start, rp, cols)
    t3 = time.perf_counter()
    if it >= 5:
        T["csr_host"].append(t3 - t2)
        T["total_csr"].append(t3 - t0)
for k, v in T.items():
    print(f"{k:12s} {1e3 * np.median(v):8.3f} ms (median)  min {1e3 * min(v):8.3f}")
st = r.stats()
print("device: seed", st["seed_ns"] / 1e6, "loop", st["loop_ns"] / 1e6, "launches", st["launches"])
