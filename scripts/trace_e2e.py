"""CUPTI timeline (torch.profiler) of one end-to-end config-4 step: every kernel, memcpy and
memset of libcfpq with its start/duration, to find idle gaps and host overhead."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import ProfilerActivity, profile

import inputs as I
from paper_1707_01007_b200 import cfpq as C

w = I.config4_workload()
stream = torch.cuda.current_stream()
g = C.Grammar.from_workload(w)
pinned = torch.from_numpy(w.edges.copy()).pin_memory()
d = C.Graph(w.n_nodes, pinned, stream=stream)
r = C.closure(g, d, stream=stream)
out = torch.empty((r.count(w.start), 2), dtype=torch.int32).pin_memory()
for _ in range(5):
    d.set_edges(pinned, stream=stream)
    C.closure_reuse(g, d, r, stream=stream)
    r.pairs(w.start, out=out)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    for _ in range(2):
        d.set_edges(pinned, stream=stream)
        C.closure_reuse(g, d, r, stream=stream)
        r.pairs(w.start, out=out)
    torch.cuda.synchronize()
evs = [e for e in prof.events() if e.device_type.name == "CUDA"]
evs.sort(key=lambda e: e.time_range.start)
t0 = evs[len(evs) // 2].time_range.start if False else evs[0].time_range.start
prev_end = None
for e in evs:
    s, en = e.time_range.start, e.time_range.end
    gap = (s - prev_end) if prev_end is not None else 0
    print(f"{(s - t0):9.1f} us  dur {en - s:8.1f}  gap {gap:7.1f}  {e.name[:90]}")
    prev_end = en
