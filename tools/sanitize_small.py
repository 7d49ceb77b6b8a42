"""Small end-to-end workload for compute-sanitizer (memcheck / racecheck / synccheck): every kernel family
of libgfxs.so on C1-sized grids with small batches (the sanitizers slow kernels 10-100x).
    compute-sanitizer --tool memcheck python tools/sanitize_small.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2306_11686_b200 as gf  # noqa: E402

n = int(os.environ.get("GF_SAN_N", "40000"))
rng = np.random.default_rng(1)
E = torch.from_numpy(rng.random(20000))
M = torch.from_numpy(rng.integers(0, 12, 20000).astype(np.uint8))
out = []
for gt in (gf.NUCLIDE, gf.UNIONIZED, gf.HASH):
    g = gf.Grid(gf.Params.xsbench(68, 11303, gt))
    kernels = ["auto", "warp"] if gt == gf.NUCLIDE else ["tile", "group", "thread", "tilenb"][: 4 if gt == gf.UNIONIZED else 3]
    for k in kernels:
        g.set_kernel(k)
        out.append((gt, k, g.lookup_batch(0, n, want_macro=True)[0]))
    if gt == gf.UNIONIZED:  # per-tile union indices from the sort's scan (TixSpec) + the tile kernel's PREP path
        g.set_kernel("tile")
        g.set_prep_min(0)
        out.append((gt, "tile-prep", g.lookup_batch(0, n, want_macro=True)[0]))
        g.set_prep_min(8 << 20)
    g.set_kernel("auto")
    out.append((gt, "unsorted", g.lookup_batch(0, n, sort=False)))
    out.append((gt, "energies", g.lookup_energies(E.cuda(), M.cuda())[0]))
    out.append((gt, "host-io", g.lookup_energies(E.pin_memory(), M.pin_memory())[0]))
    out.append((gt, "host-io-whole", g.lookup_energies(E.pin_memory(), M.pin_memory(), want_macro=False)))
    out.append((gt, "history", g.history_batch(0, 300, 8)))
    out.append((gt, "history-direct", g.history_batch(0, 300, 8, mode="direct")))
    del g
    torch.cuda.empty_cache()
for band in (0, 3):
    gb = gf.Grid(gf.Params.xsbench(68, 11303, gf.UNIONIZED, n_bands=4, band=band))
    out.append(("band", band, gb.lookup_batch(0, n)))
    gb.set_kernel("tile")
    gb.set_prep_min(0)
    out.append(("band-tile", band, gb.lookup_batch(0, n, want_macro=True)[0]))
    del gb
r = gf.Grid(gf.Params.rsbench(68))
out.append(("rs", "sorted", r.lookup_batch(0, 20000)))
out.append(("rs", "unsorted", r.lookup_batch(0, 5000, sort=False)))
out.append(("rs", "history", r.history_batch(0, 100, 4)))
torch.cuda.synchronize()
for o in out:
    print(*o)
print("sanitize workload done")
