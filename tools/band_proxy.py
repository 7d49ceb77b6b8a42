"""Energy-band strong split of C3 (SURVEY.md Sec. 8(e) "Alternative ... energy-band sharding"), timed on one
GPU: for W in a list, every band replica r of W (E in [r/W, (r+1)/W)) is built in turn and runs the whole
17 M-lookup batch (the sort samples all of it and keeps the band's lookups); per band the median of 5 device
times (sort + lookup, L2 flushed before each) and the stage split.  The bands' raw sums add up to the
whole grid's.
    python tools/band_proxy.py [W,W,...] [n] > gpurun_out/band_proxy.txt"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes as C  # noqa: E402

import torch  # noqa: E402

import paper_2306_11686_b200 as gf  # noqa: E402

Ws = [int(x) for x in sys.argv[1].split(",")] if len(sys.argv) > 1 else [1, 2, 4, 8]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 17_000_000
vs = torch.zeros(1, dtype=torch.int64, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
L = gf.lib()
st = torch.cuda.current_stream()
T1 = None
for W in Ws:
    per, raw = [], 0
    for b in range(W):
        g = gf.Grid(gf.Params.xsbench(355, 11303, gf.UNIONIZED, n_bands=W, band=b))
        scratch = torch.empty(g.scratch_bytes(n, gf.SORT_LOCALITY), dtype=torch.uint8, device="cuda")
        ts, ss = [], []
        for r in range(6):
            flush.fill_(r)
            vs.zero_()
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
            for e in ev:  # (created lazily: record once before the library records them)
                e.record()
            se = (C.c_void_p * 3)(ev[0].cuda_event, ev[1].cuda_event, ev[2].cuda_event)
            gf._check(L.gf_xs_lookup_batch_ev(g.h, 0, n, gf.STARTING_SEED, gf.SORT_LOCALITY, None,
                                              C.c_void_p(vs.data_ptr()), C.c_void_p(scratch.data_ptr()),
                                              scratch.numel(), C.c_void_p(st.cuda_stream), se))
            torch.cuda.synchronize()
            if r:
                ts.append(ev[0].elapsed_time(ev[2]))
                ss.append(ev[0].elapsed_time(ev[1]))
        raw += int(vs.item())
        per.append((statistics.median(ts), statistics.median(ss)))
        del g, scratch
        torch.cuda.empty_cache()
    mx = max(t for t, _ in per)
    if W == 1:
        T1 = mx
    print(f"W={W} max_band_ms {mx:.4f} speedup {T1 / mx if T1 else float('nan'):.2f} hash {gf.verify(raw)} raw {raw} "
          f"bands " + " ".join(f"{t:.4f}(sort {s:.4f})" for t, s in per), flush=True)
