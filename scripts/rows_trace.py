"""CUPTI timeline (torch.profiler) of one config-4 bit-row closure: kernels, copies, gaps."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import ProfilerActivity, profile
import inputs as I
from paper_1707_01007_b200 import cfpq as C
w = I.config4_workload()
s = torch.cuda.current_stream()
g = C.Grammar.from_workload(w)
d = C.Graph(w.n_nodes, torch.from_numpy(w.edges).cuda(), stream=s)
r = C.closure(g, d, stream=s, path_policy=3)
for _ in range(2):
    C.closure_reuse(g, d, r, stream=s, path_policy=3)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    C.closure_reuse(g, d, r, stream=s, path_policy=3)
    torch.cuda.synchronize()
evs = sorted([e for e in prof.events() if e.device_type.name == "CUDA"], key=lambda e: e.time_range.start)
t0 = evs[0].time_range.start
busy = 0.0
last_end = t0
idle = 0.0
for e in evs:
    st, en = e.time_range.start, e.time_range.end
    if st > last_end:
        idle += st - last_end
    last_end = max(last_end, en)
    print(f"{st - t0:9.1f} us dur {en - st:8.1f}  {e.name[:70]}")
print(f"span {last_end - t0:.1f} us, idle {idle:.1f} us")
