# in-process e2e probe: the bench's e2e loop run at several points of a bench-like process
import os, sys, time, statistics
sys.path.insert(0, '.')
import torch
import inputs as I
from paper_1707_01007_b200 import cfpq as C
w = I.config4_workload()
stream = torch.cuda.current_stream()
g = C.Grammar.from_workload(w)
d = C.Graph(w.n_nodes, torch.from_numpy(w.edges).cuda(), stream=stream)
kw = dict(stream=stream, semantics=0, solo_threshold=-1, path_policy=0, tensor_format=0, schedule=0)
pinned = torch.from_numpy(w.edges.copy()).pin_memory()
def e2e(r, tag, n=20):
    m = r.count(w.start)
    rp = torch.empty((w.n_nodes + 1,), dtype=torch.int64).pin_memory()
    cols = torch.empty((m,), dtype=torch.int32).pin_memory()
    tr, tt = [], []
    for it in range(n + 5):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        d.set_edges(pinned, stream=stream)
        C.closure_reuse(g, d, r, **kw)
        ta = time.perf_counter()
        r.csr(w.start, rp, cols)
        t1 = time.perf_counter()
        if it >= 5:
            tr.append(ta - t0); tt.append(t1 - t0)
    print(f"{tag:28s} run {1e3*statistics.median(tr):.3f} total {1e3*statistics.median(tt):.3f}", flush=True)
r = C.closure(g, d, **kw)
e2e(r, "fresh")
ra = C.closure(g, d, account_work=True, stream=stream, path_policy=0)
e2e(r, "after account_work closure")
del ra
e2e(r, "after del account result")
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
for _ in range(50):
    flush.fill_(1)
    C.closure_reuse(g, d, r, **kw)
    r.stats()
torch.cuda.synchronize()
e2e(r, "after 50 flushed steps")
import pynvml
pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)
e2e(r, "after nvmlInit")
