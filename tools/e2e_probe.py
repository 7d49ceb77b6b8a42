import time, torch, numpy as np, sys
sys.path.insert(0, '.')
import paper_2306_11686_b200 as gf
g = gf.Grid(gf.Params.xsbench(355, 11303, gf.UNIONIZED))
n = 17_000_000
rng = np.random.default_rng(1)
Eh = torch.from_numpy(rng.random(n)).pin_memory()
mh = torch.from_numpy(rng.integers(0, 12, n).astype(np.uint8)).pin_memory()
out = torch.empty((n, 5), dtype=torch.float64, pin_memory=True)
for i in range(4):
    t = time.perf_counter(); g.lookup_energies(Eh, mh, out=out); print('host-io call', time.perf_counter() - t)
d = torch.empty(n * 5, dtype=torch.float64, device='cuda')
torch.cuda.synchronize()
t = time.perf_counter(); out.view(-1).copy_(d, non_blocking=True); torch.cuda.synchronize(); dt = time.perf_counter() - t
print('D2H 680 MB pinned', dt, 680e6 / dt / 1e9, 'GB/s')
t = time.perf_counter(); d[:n].copy_(Eh, non_blocking=True); torch.cuda.synchronize(); dt = time.perf_counter() - t
print('H2D 136 MB pinned', dt, 136e6 / dt / 1e9, 'GB/s')
