"""Where the result read of the config-4 e2e step goes: wall time of r.csr(S) into pinned host
memory and into device buffers, r.count(S), and (run under ncu) the kernels one csr call
launches.  usage: python scripts/csr_probe.py [reps]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import inputs as I
from paper_1707_01007_b200 import cfpq as C

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 30
w = I.config4_workload()
s = torch.cuda.current_stream()
g = C.Grammar.from_workload(w)
d = C.Graph(w.n_nodes, torch.from_numpy(w.edges).cuda(), stream=s)
r = C.closure(g, d, stream=s)
m = r.count(w.start)
rp = torch.empty((w.n_nodes + 1,), dtype=torch.int64).pin_memory()
cols = torch.empty((m,), dtype=torch.int32).pin_memory()
rpd = torch.empty((w.n_nodes + 1,), dtype=torch.int64, device="cuda")
colsd = torch.empty((m,), dtype=torch.int32, device="cuda")
T = {k: [] for k in ("csr_host", "csr_dev", "d2h_only")}
for it in range(reps):
    C.closure_reuse(g, d, r, stream=s)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r.csr(w.start, rp, cols)
    t1 = time.perf_counter()
    r.csr(w.start, rpd, colsd)
    t2 = time.perf_counter()
    rp.copy_(rpd, non_blocking=True)
    cols.copy_(colsd, non_blocking=True)
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    if it >= 3:
        T["csr_host"].append(t1 - t0)
        T["csr_dev"].append(t2 - t1)
        T["d2h_only"].append(t3 - t2)
for k, v in T.items():
    print(f"{k:10s} {1e3 * np.median(v):7.3f} ms (median)  min {1e3 * min(v):7.3f}")
print("m", m)
