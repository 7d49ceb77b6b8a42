"""A/B of the sorted lookup kernels against batch size: device time of one sorted
lookup_batch (sort + lookup; CUDA events, median of 5 after a warm-up) for n in a list, per kernel
forced with gf_xs_debug_set_kernel.  Also checks that every kernel gives the same raw sum.
    python tools/ab_batch_n.py [C3|C2|C4] [kernel,kernel,...] [n,n,...] > gpurun_out/ab_batch_n.txt"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2306_11686_b200 as gf  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
kernels = sys.argv[2].split(",") if len(sys.argv) > 2 else ["tile", "group", "thread"]
ns = [int(x) for x in sys.argv[3].split(",")] if len(sys.argv) > 3 else \
    [500_000, 1 << 20, 2_125_000, 4_250_000, 8_500_000, 17_000_000]
n_iso, gt = {"C2": (68, 1), "C3": (355, 1), "C4": (355, 2)}[cfg]
g = gf.Grid(gf.Params.xsbench(n_iso, 11303, gt))
vs = torch.zeros(1, dtype=torch.int64, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for n in ns:
    row, raws = [f"{n:>9d}"], set()
    for k in kernels:
        g.set_kernel(k)
        ts = []
        for r in range(6):
            flush.fill_(r)
            vs.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            g.lookup_batch_async(0, n, vs)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
            raws.add(int(vs.item()))
        t = statistics.median(ts[1:])
        row.append(f"{k} {t:7.3f} ms {n / t / 1e6:6.3f} G/s")
    print(cfg, "  ".join(row), "raw-agree" if len(raws) == 1 else f"RAW MISMATCH {raws}", flush=True)
g.set_kernel("auto")
