"""A/B of the sorted lookup kernels against batch size: device time of one sorted
lookup_batch (sort + lookup) for n in a list, with GF_XS_KERNEL=group and =thread.
    python tools/ab_batch_n.py [C3|C2|C4] > gpurun_out/ab_batch_n.txt"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2306_11686_b200 as gf  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
n_iso, gt = {"C2": (68, 1), "C3": (355, 1), "C4": (355, 2)}[cfg]
g = gf.Grid(gf.Params.xsbench(n_iso, 11303, gt))
vs = torch.zeros(1, dtype=torch.int64, device="cuda")
for n in [250_000, 500_000, 1 << 20, 2 << 20, 4 << 20, 8 << 20, 17_000_000]:
    row = [f"{n:>9d}"]
    for k in ("group", "thread"):
        os.environ["GF_XS_KERNEL"] = k
        ts = []
        for r in range(6):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            g.lookup_batch_async(r * n, n, vs)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        t = statistics.median(ts[1:])
        row.append(f"{k} {t:8.3f} ms {n / t / 1e6:6.3f} G/s")
    print(cfg, "  ".join(row), flush=True)
