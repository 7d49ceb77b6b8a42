"""Per-shard device time (sort + lookup; median of 5 after a warm-up, L2 flushed) of the W-way strong split
of a config on this one GPU -- the strong-scaling proxy of bench.py, per shard, with the kernel used.
    python tools/shard_times.py [C3|C4|C2] [W]"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2306_11686_b200 as gf  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
W = int(sys.argv[2]) if len(sys.argv) > 2 else 8
n_iso, gt, n = {"C2": (68, 1, 17_000_000), "C3": (355, 1, 17_000_000), "C4": (355, 2, 170_000_000)}[cfg]
g = gf.Grid(gf.Params.xsbench(n_iso, 11303, gt))
vs = torch.zeros(1, dtype=torch.int64, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
raw = 0
for r in range(W):
    lo, cnt = gf.shard_range(n, r, W)
    ts = []
    for k in range(6):
        flush.fill_(k)
        vs.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.lookup_batch_async(lo, cnt, vs)
        e1.record()
        torch.cuda.synchronize()
        if k:
            ts.append(e0.elapsed_time(e1))
    raw += int(vs.item())
    print(f"{cfg} W={W} shard {r} [{lo}, {lo + cnt}) {g.kernel_for(cnt)} {statistics.median(ts):.3f} ms "
          f"(min {min(ts):.3f} max {max(ts):.3f})", flush=True)
print(f"{cfg} W={W} hash {gf.verify(raw)}")
