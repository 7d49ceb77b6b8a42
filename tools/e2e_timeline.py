"""CUPTI timeline (torch.profiler) of one GF_HOST_IO energies call on C3: kernels and copies per stream."""
import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile

import paper_2306_11686_b200 as gf

n = 17_000_000
g = gf.Grid(gf.Params.xsbench(355, 11303, gf.UNIONIZED))
rng = np.random.default_rng(1)
Eh = torch.from_numpy(rng.random(n)).pin_memory()
mh = torch.from_numpy(rng.integers(0, 12, n).astype(np.uint8)).pin_memory()
for _ in range(2):
    g.lookup_energies(Eh, mh, want_macro=False)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    g.lookup_energies(Eh, mh, want_macro=False)
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
t0 = min(e.time_range.start for e in ev)
for e in sorted(ev, key=lambda e: e.time_range.start):
    print(f"{(e.time_range.start - t0) / 1e3:8.3f} {(e.time_range.end - t0) / 1e3:8.3f} ms  "
          f"stream {getattr(e, 'device_resource_id', '?'):>4}  {e.name[:60]}")
