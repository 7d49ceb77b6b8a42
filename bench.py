#!/usr/bin/env python
"""bench.py -- lookups/s of the B200-native XSBench / RSBench lookup (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C3|C2|C4|C5|C1] [--impl ours|reference]
    torchrun --nproc-per-node N --master-addr 127.0.0.1 bench.py --gpus N ...

A step is one pass of the whole hot path (or B1-B4 for C5) over
the rank's shard of the config's event lookups: sample -> locality sort -> search / interpolate /
accumulate -> hash reduction, then the cross-rank int64 all-reduce of the raw hash (NCCL) when
N > 1.  The grid build (A0) runs once before timing and is reported separately (grid_build_ms),
like the paper's kernel-only timing.  Default workload: C3 = XSBench large,
unionized grid, 17 M lookups (BASELINE.json configs[2], the north_star's target), strong-scaled
over N ranks by default (rank r runs the global indices [floor(r n / N), floor((r+1) n / N)) of the
config's n lookups; --scaling weak gives every rank its own n-lookup range
instead).  At N = 1 the line also carries strong_proxy: the per-rank step of the 2 / 4 / 8-way
split timed on this one GPU (every shard, the slowest counts).  Every step is timed with CUDA events
on the launching stream; L2 is flushed by a 256 MiB write between steps (outside the events).  Rank
0 prints one JSON line.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (bench, n_iso, grid_type, n_lookups, description)
    "C1": ("xs", 68, 0, 100_000, "XSBench small 68x11303, nuclide-grid search, 100k event lookups"),
    "C2": ("xs", 68, 1, 17_000_000, "XSBench small 68x11303, unionized grid, 17M event lookups"),
    "C3": ("xs", 355, 1, 17_000_000, "XSBench large 355x11303, unionized grid, 17M event lookups"),
    "C4": ("xs", 355, 2, 170_000_000, "XSBench large 355x11303, hash grid 10000 bins, 170M event lookups"),
    "C5": ("rs", 355, None, 10_200_000, "RSBench large 355 nuclides, windowed multipole + Faddeeva, 10.2M lookups"),
    # NEXT-3: the nuclide grid at scale -- not a BASELINE.json config
    "C5D0": ("rs", 355, None, 10_200_000, "RSBench large 355 nuclides, 0 K multipole kernel (doppler off, NEXT-3), 10.2M lookups"),
    "C3N": ("xs", 355, 0, 17_000_000, "XSBench large 355x11303, nuclide-grid search, 17M event lookups (NEXT-3)"),
    # NEXT-2 point counts: XSBench XL, 238,847 gridpoints per nuclide (the hash grid: the unionized
    # grid's index grid would be 355 x 84.8 M entries)
    "C6": ("xs", 355, 2, 17_000_000, "XSBench XL 355x238847, hash grid 10000 bins, 17M event lookups (NEXT-2)"),
    # NEXT-2 energy-band sharding: XSBench XL on the unionized grid, whose index grid (355 x 84.8 M
    # entries) fits no GPU whole; 8 energy bands, rank r of N serves bands r, r + N, ...
    "C7": ("xs", 355, 1, 17_000_000, "XSBench XL 355x238847, unionized grid in 8 energy bands, 17M event lookups (NEXT-2)"),
    # NEXT-2 XXL (R-XXL: 2.1 x XL = 501,579 gridpoints per nuclide): the unionized grid in 16 bands (a band's
    # index grid needs < 65,536 points per nuclide); one GPU runs them in turn
    "C8": ("xs", 355, 1, 17_000_000, "XSBench XXL 355x501579, unionized grid in 16 energy bands, 17M event lookups (NEXT-2)"),
    # NEXT-4: page-rank propagation step (HeCBench page-rank), 2^24 nodes, out-degree 16
    "P1": ("pr", 1 << 24, 16, 0, "page-rank propagation step, 2^24 nodes, average out-degree 16 (NEXT-4)"),
    # NEXT-4: AMGmk relax kernel: one Jacobi sweep, 27-point Laplacian on 256^3
    "A1": ("amg", 256, 256, 256, "AMGmk relax: Jacobi sweep, 27-point Laplacian on a 256^3 grid (NEXT-4)"),
    # NEXT-1 history-based mode: particles x 34 dependent lookups (gf_xs_history_batch)
    "H2": ("xs", 68, 1, 17_000_000, "XSBench small 68x11303, unionized, HISTORY mode 500k particles x 34 lookups"),
    "H3": ("xs", 355, 1, 17_000_000, "XSBench large 355x11303, unionized, HISTORY mode 500k particles x 34 lookups"),
    "H5": ("rs", 355, None, 10_200_000, "RSBench large 355 nuclides, HISTORY mode 300k particles x 34 lookups"),
}
HIST_L = {"H2": 34, "H3": 34, "H5": 34}  # lookups per particle (history configs)
# The paper's own numbers for the same benchmark and mode (context only): kernel speedup
# of GPU First / manual offload over the CPU OpenMP parallel region, A100-40GB vs AMD EPYC 7532.
PAPER = {
    "xs_event_small": {"gpu_first": 11.772, "manual_offload": 9.757, "cite": "PAPER.md:1185,1193 (Fig. 8a)"},
    "xs_event_large": {"gpu_first": 11.434, "manual_offload": 11.503, "cite": "PAPER.md:1223,1231 (Fig. 8a)"},
    "xs_history_small": {"gpu_first": 14.360, "cite": "PAPER.md:1210 (Fig. 8a)"},
    "xs_history_large": {"gpu_first": 10.64, "cite": "PAPER.md:1247 (Fig. 8a)"},
    "rs_event_large": {"gpu_first": 4.6102, "manual_offload": 4.5159, "cite": "PAPER.md:1342,1350 (Fig. 8b)"},
    "rs_history_large": {"gpu_first": 4.6277, "cite": "PAPER.md:1366 (Fig. 8b)"},
}
PAPER_KEY = {"C1": "xs_event_small", "C2": "xs_event_small", "C3": "xs_event_large", "C4": "xs_event_large",
             "C3N": "xs_event_large", "C5": "rs_event_large", "C5D0": "rs_event_large", "H2": "xs_history_small",
             "H3": "xs_history_large", "H5": "rs_history_large"}
# Per-lookup algorithmic work of the dominant kernel:
#   sector bytes of the random-order gather model, and fp64 flops (division counted as 1).
#   C5: RSBench flops counted from the oracle's arithmetic: 55.4 nuclides x (51 per
#   nuclide + 9.09 poles x 85 per pole) + 0.5% Abrarov evaluations ~ 49,000 (transcendental = 1 flop);
#   C5D0 (0 K): 55.4 x (51 + 9.09 x 43 per pole: sqrt, two textbook complex divisions, 3 products) ~ 24,500.
GRIDPOINTS = {"C6": 238847, "C7": 238847, "C8": 501579}  # (else 11,303)
BANDS = {"C7": 8, "C8": 16}
ALG = {"C8": (6517, 1551), "C1": (7187, 434), "C2": (1887, 434), "C3": (6517, 1551), "C4": (6203, 1551), "C5": (0, 49000),
       "C3N": (0, 1551), "C5D0": (0, 24500), "C6": (6203, 1551), "C7": (6517, 1551), "H2": (1887, 434), "H3": (6517, 1551), "H5": (0, 49000)}


def oracle_run(o, cfg, first, n, threads):
    """The oracle on lookups [first, first + n) of a config (history configs: whole particles)."""
    L = HIST_L.get(cfg)
    if L:
        return o.history_batch(first // L, max(1, n // L), L, threads=threads), max(1, n // L) * L
    return o.lookup_batch(first, n, threads=threads), n


def launches_per_step(bench, gt, sorted_, kern="", n=0, slices=1):
    """Our kernels per step: the sort's count, scan_local, scan_add and `slices` scatter launches (A1-A2;
    band grids: sort_count_band, the scans, sort_scatter_band), then the lookup kernel.  idx_prep (A3)
    precedes the hash-grid tile / group kernels and the unionized ones below 8 M lookups; sampled
    unionized tile batches from 8 M lookups get their per-tile union indices from scan_add."""
    if not sorted_:
        return 1
    prep = bench == "xs" and ((gt == 2 and kern in ("tile", "group", "")) or
                              (gt == 1 and (kern == "group" or (kern in ("tile", "") and n < (8 << 20)))))
    return 3 + slices + 1 + (1 if prep else 0)


def load_profile(cfg, sorted_):
    """ncu numbers of the dominant kernel, committed under profiles/ (per-launch DRAM bytes)."""
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if not os.path.exists(p):
        return None
    d = json.load(open(p))
    return d.get(f"{cfg}{'' if sorted_ else '_nosort'}")


def env_int(k, d):
    try:
        return int(os.environ.get(k, d))
    except ValueError:
        return d


class ClockSampler:
    """SM clock and clock-event (throttle) reasons polled through NVML every ~2 ms during the timed
    region (the timed region of a C3 step is a few ms, shorter than nvidia-smi's sampling period).
    Same fields as B200_PROFILING.md's nvidia-smi clocks line."""

    REASONS = {"hw_slowdown": "nvmlClocksEventReasonHwSlowdown",
               "hw_thermal_slowdown": "nvmlClocksEventReasonHwThermalSlowdown",
               "sw_thermal_slowdown": "nvmlClocksEventReasonSwThermalSlowdown",
               "sw_power_cap": "nvmlClocksEventReasonSwPowerCap"}

    def __init__(self, index):
        self.index, self.rows, self.stop, self.t = index, [], threading.Event(), None

    def __enter__(self):
        try:
            import pynvml as N
            N.nvmlInit()
            self.N, self.h = N, N.nvmlDeviceGetHandleByIndex(self.index)
            self.mx = N.nvmlDeviceGetMaxClockInfo(self.h, N.NVML_CLOCK_SM)
            self.t = threading.Thread(target=self._poll, daemon=True)
            self.t.start()
        except Exception:  # no NVML: report unsampled
            self.t = None
        return self

    def _poll(self):
        N = self.N
        while not self.stop.is_set():
            try:
                self.rows.append((N.nvmlDeviceGetClockInfo(self.h, N.NVML_CLOCK_SM),
                                  N.nvmlDeviceGetCurrentClocksEventReasons(self.h)))
            except Exception:
                pass
            time.sleep(0.002)

    def __exit__(self, *a):
        self.stop.set()
        if self.t:
            self.t.join(timeout=2)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [r[0] for r in self.rows]
        reasons = set()
        for _, bits in self.rows:
            for nm, attr in self.REASONS.items():
                if bits & getattr(self.N, attr, 0):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": self.mx, "reasons": sorted(reasons),
                "samples": len(sm), "source": "NVML every 2 ms"}


def load_peaks():
    peaks = {"hbm_gbs": 6650.0, "src": "fallback B200_PROFILING.md"}
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        peaks.update(hbm_gbs=d.get("hbm_gbs", peaks["hbm_gbs"]), sm_max_mhz=d.get("sm_max_mhz", 1965.0),
                     src="MEASURED_PEAKS.json")
    probe = os.path.join(ROOT, "profiles", "roofline_probe.json")
    if os.path.exists(probe):
        d = json.load(open(probe))
        peaks["fp64_dadd_ops_per_s"] = d.get("fp64_dadd_ops_per_s")
        peaks["gather96_GBps"] = d.get("gather96_best_useful_GBps")
        peaks["probe_src"] = "profiles/roofline_probe.json"
    if not peaks.get("fp64_dadd_ops_per_s"):
        # guide unit counts: 148 SMs x 64 FP64 lanes x 1.965 GHz (non-FMA op rate)
        peaks["fp64_dadd_ops_per_s"] = 148 * 64 * 1.965e9
        peaks["probe_src"] = "derived 148 SM x 64 lanes x 1965 MHz"
    return peaks


def cpu_baseline(cfg_name, seconds=12.0):
    """The oracle as it stands, timed on this host's cores on a bounded sample of the workload."""
    import oracle as O
    bench, n_iso, gt, n, _ = CONFIGS[cfg_name]
    threads = len(os.sched_getaffinity(0))
    if bench == "xs":
        o = O.XSOracle(n_iso, GRIDPOINTS.get(cfg_name, 11303), O.NUCLIDE if cfg_name in BANDS else gt,
                       bins=10000)  # (C7 / C8: the nuclide grid gives the unionized grid's results; its IG is 120 GB+)
    else:
        o = O.RSOracle(n_iso, 1000, 100, 4, doppler=0 if cfg_name == "C5D0" else 1)
    k = 20_000
    t = time.perf_counter()
    _, k = oracle_run(o, cfg_name, 0, k, threads)
    dt = time.perf_counter() - t
    k2 = int(min(n, max(k, k * seconds / max(dt, 1e-6))))
    t = time.perf_counter()
    _, k2 = oracle_run(o, cfg_name, 0, k2, threads)
    dt = time.perf_counter() - t
    res = {"value": k2 / dt, "unit": "lookups/s", "cores": threads, "kind": "oracle",
           "sample": f"global lookup indices [0, {k2}) of {cfg_name} ({k2 / n:.2%} of the workload), "
                     f"plain C oracle -O2 -ffp-contract=off, OpenMP {threads} threads, {dt:.1f} s"}
    if cfg_name in ("C1", "C2"):  # also a 1-thread run for the small configs
        k1 = max(1000, int(k2 / threads / 4))
        t = time.perf_counter()
        _, k1 = oracle_run(o, cfg_name, 0, k1, 1)
        d1 = time.perf_counter() - t
        res["single_thread"] = {"value": k1 / d1, "unit": "lookups/s", "cores": 1,
                                "sample": f"global lookup indices [0, {k1}), 1 thread, {d1:.1f} s"}
    return res


def run_reference(args, rank, world):
    """--impl reference: the oracle (the reference arm for this tier), on this host's cores."""
    if rank != 0:
        return
    import oracle as O
    cfg_name = args.config
    bench, n_iso, gt, n, desc = CONFIGS[cfg_name]
    threads = len(os.sched_getaffinity(0))
    if bench == "amg":  # AMGmk relax: whole sweeps of the same matrix
        import numpy as np
        rp, col, val = O.amg_matrix(n_iso, gt, n)
        rows = len(rp) - 1
        rng = np.random.default_rng(7)
        f, u = rng.random(rows), rng.random(rows)
        for _ in range(args.warmup):
            u = O.amg_relax(rp, col, val, f, u, threads=threads)
        times = []
        for _ in range(args.steps):
            t = time.perf_counter()
            u = O.amg_relax(rp, col, val, f, u, threads=threads)
            times.append(time.perf_counter() - t)
        v = len(col) * args.steps / sum(times)
        line = {"impl": "reference", "metric": "nonzeros/sec", "value": v, "unit": "nonzeros/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * sum(times) / args.steps,
                "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "f64",
                "data": "synthetic (27-point Laplacian; seeded uniform f and u)",
                "config": {"workload": f"{cfg_name}: {desc}", "rows": rows, "nonzeros": len(col)},
                "cpu_baseline": {"value": v, "unit": "nonzeros/s", "cores": threads, "kind": "oracle",
                                 "sample": "whole relaxation sweeps"},
                "e2e": {"value": v, "unit": "nonzeros/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return
    if bench == "pr":  # page-rank: whole propagation steps of the same graph
        import numpy as np
        o = O.PROracle(n_iso, gt)
        r = np.full(n_iso, 1.0 / n_iso)
        for _ in range(args.warmup):
            r = o.propagate(r, threads=threads)
        times = []
        for _ in range(args.steps):
            t = time.perf_counter()
            r = o.propagate(r, threads=threads)
            times.append(time.perf_counter() - t)
        v = o.nnz * args.steps / sum(times)
        line = {"impl": "reference", "metric": "edges/sec", "value": v, "unit": "edges/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * sum(times) / args.steps,
                "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "f64",
                "data": "synthetic (LCG-generated graph, seed 42; uniform initial ranks)",
                "config": {"workload": f"{cfg_name}: {desc}", "nodes": n_iso, "edges": o.nnz},
                "cpu_baseline": {"value": v, "unit": "edges/s", "cores": threads, "kind": "oracle",
                                 "sample": "whole propagation steps"},
                "e2e": {"value": v, "unit": "edges/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return
    o = (O.XSOracle(n_iso, GRIDPOINTS.get(cfg_name, 11303), O.NUCLIDE if cfg_name in BANDS else gt,
                    bins=10000) if bench == "xs"
         else O.RSOracle(n_iso, 1000, 100, 4, doppler=0 if cfg_name == "C5D0" else 1))
    t = time.perf_counter()
    _, k0 = oracle_run(o, cfg_name, 0, 20_000, threads)
    per = (time.perf_counter() - t) / k0
    step_n = int(max(20_000, min(n, 2.0 / max(per, 1e-9))))  # ~2 s of CPU per step
    first = 0
    HLr = HIST_L.get(cfg_name, 1)
    step_n = HLr * max(1, step_n // HLr)  # history configs: whole particles
    for _ in range(args.warmup):
        oracle_run(o, cfg_name, first, step_n, threads)
        first = (first + step_n) % max(1, n - step_n)
    times = []
    for _ in range(args.steps):
        t = time.perf_counter()
        oracle_run(o, cfg_name, first, step_n, threads)
        times.append(time.perf_counter() - t)
        first = (first + step_n) % max(1, n - step_n)
    tot = sum(times)
    v = step_n * args.steps / tot
    line = {"impl": "reference", "metric": "lookups/sec", "value": v, "unit": "lookups/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps,
            "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (LCG-generated grids and lookups, seeds 42 / 1070)",
            "config": {"workload": f"{cfg_name}: {desc}", "n_lookups": n, "step_sample": step_n},
            "cpu_baseline": {"value": v, "unit": "lookups/s", "cores": threads, "kind": "oracle",
                             "sample": f"{step_n} consecutive lookups per step out of {n}"},
            "e2e": {"value": v, "unit": "lookups/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def bench_bands(args, rank, world, dev, gf, torch, dist, C):
    """C7 / C8: every rank builds, in turn, the band replicas of its bands (r, r + N, ... of W = 8 / 16;
    grid build untimed), and runs the full event batch through each -- the sort keeps the band's lookups.
    A step is one batch through all of the rank's bands; value = 17 M / max-over-ranks step time."""
    from paper_2306_11686_b200 import dist as gdist
    cfg = args.config
    W, n, n_gp = BANDS[cfg], CONFIGS[cfg][3], GRIDPOINTS[cfg]
    mine = list(range(rank, W, world))
    st = torch.cuda.current_stream()
    vsum = torch.zeros(1, dtype=torch.int64, device=dev)
    per_band, raws, builds = [], 0, 0.0
    for b in mine:
        t0 = time.perf_counter()
        grid = gf.Grid(gf.Params.xsbench(355, n_gp, gf.UNIONIZED, n_bands=W, band=b), device=dev)
        builds += time.perf_counter() - t0
        sc = torch.empty(grid.scratch_bytes(n, gf.SORT_LOCALITY), dtype=torch.uint8, device=dev)
        ts = []
        for k in range(args.warmup + args.steps):
            vsum.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            gf._check(gf.lib().gf_xs_lookup_batch(grid.h, 0, n, gf.STARTING_SEED, gf.SORT_LOCALITY, None,
                                                  C.c_void_p(vsum.data_ptr()), C.c_void_p(sc.data_ptr()),
                                                  sc.numel(), C.c_void_p(st.cuda_stream)))
            e1.record()
            torch.cuda.synchronize()
            if k >= args.warmup:
                ts.append(e0.elapsed_time(e1))
        raws += int(vsum.item())
        per_band.append(statistics.median(ts))
        del grid, sc
        torch.cuda.empty_cache()
    step_ms = sum(per_band)
    rv = torch.tensor([raws], dtype=torch.int64, device=dev)
    if dist is not None:
        gdist.reduce_raw(rv)
        step_ms = gdist.max_over_ranks([step_ms], dev)[0]
    if rank == 0:
        peaks = load_peaks()
        look_s = step_ms * 1e-3
        roof = {"bound": "alu", "kernel": "band sort + xs_lookup_tile<unionized> per band",
                "achieved": 1551 * n / look_s / 1e12, "peak": peaks["fp64_dadd_ops_per_s"] / 1e12,
                "unit": "TFLOP/s", "traffic": None,
                "note": "1551 fp64 flops/lookup x 17 M lookups / summed band step time (each band re-samples and "
                        "sorts all 17 M lookups, keeping its own)"}
        roof["frac"] = roof["achieved"] / roof["peak"]
        line = {"metric": "lookups/sec", "value": n / look_s, "unit": "lookups/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": step_ms, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic (LCG-generated grids and lookups, seeds 42 / 1070)",
                "config": {"workload": f"{cfg}: {CONFIGS[cfg][4]}", "n_lookups": n, "bands": W,
                           "bands_per_rank": len(mine), "band_ms": per_band,
                           "parallelism": f"energy bands over {world} rank(s), 1 int64 all-reduce"},
                "roofline": roof, "cpu_baseline": None, "e2e": None,
                "gpu_launches": args.steps * len(mine) * 5, "hash": gf.verify(int(rv.item())),
                "raw": int(rv.item()), "grid_build_s": builds}
        print(json.dumps(line), flush=True)


def bench_pagerank(args, rank, world, dev, gf, torch, dist):
    """P1 (NEXT-4): one step = contributions + in-edge gather over the whole graph (include/gf_pr.h).
    Every rank runs its own replica (weak scaling; independent problems, no exchange)."""
    from paper_2306_11686_b200 import dist as gdist
    import numpy as np
    n, D = CONFIGS["P1"][1], CONFIGS["P1"][2]
    t0 = time.perf_counter()
    g = gf.PRGraph(n, D, device=dev.index)
    build_s = time.perf_counter() - t0
    nnz = g.n_edges
    a = torch.full((n,), 1.0 / n, dtype=torch.float64, device=dev)
    b = torch.empty_like(a)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.warmup + args.steps)]
    clocks = ClockSampler(dev.index)
    ts = []
    with clocks:
        if dist is not None:
            dist.barrier()
        for k, (e0, e1) in enumerate(evs):
            flush.fill_(k & 0xFF)
            e0.record()
            g.propagate(a, b)
            e1.record()
            a, b = b, a
        torch.cuda.synchronize()
    ts = [e0.elapsed_time(e1) for e0, e1 in evs[args.warmup:]]
    step_ms = sum(ts) / len(ts)
    if dist is not None:
        step_ms = gdist.max_over_ranks([step_ms], dev)[0]
    # end to end through the public API: ranks in from pinned host memory, result back
    e2e = None
    if not args.no_e2e:
        rh = torch.full((n,), 1.0 / n, dtype=torch.float64).pin_memory()
        oh = torch.empty((n,), dtype=torch.float64).pin_memory()
        reps = 3
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(reps):
            a.copy_(rh, non_blocking=True)
            g.propagate(a, b)
            oh.copy_(b, non_blocking=True)
            torch.cuda.synchronize()
        el = (time.perf_counter() - t0) / reps
        e2e = {"value": world * nnz / el, "unit": "edges/s", "h2d_bytes_per_step": 8 * n, "d2h_bytes_per_step": 8 * n,
               "path": "PRGraph.propagate: rank vector H2D, step, result D2H; host-timed"}
    if rank == 0:
        peaks = load_peaks()
        alg = 12 * nnz + 32 * n  # col (4 B) + contribution gather (8 B useful) per edge; 32 B per node
        gbs = alg / (step_ms * 1e-3) / 1e9
        prof = load_profile("P1", True)
        roof = {"bound": "hbm", "kernel": "pr_contrib + pr_gather", "achieved": gbs, "peak": peaks["hbm_gbs"],
                "unit": "GB/s", "frac": gbs / peaks["hbm_gbs"], "traffic": prof.get("dram_bytes") if prof else None,
                "note": f"algorithmic bytes per step = 12 x {nnz} edges + 32 x {n} nodes / mean step time "
                        f"(CUDA events on the launch stream); the random gathers move whole DRAM sectors for 8 "
                        f"useful bytes, so traffic (ncu dram read+write of pr_gather, "
                        f"{prof.get('src') if prof else 'no capture'}) / step time is the physical bandwidth; "
                        f"peak {peaks['src']}"}
        if prof:
            roof["traffic_frac"] = prof["dram_bytes"] / (step_ms * 1e-3) / 1e9 / peaks["hbm_gbs"]
        cb = None
        if not args.no_cpu_baseline and world == 1:
            import oracle as O
            threads = len(os.sched_getaffinity(0))
            o = O.PROracle(n, D)
            r = np.full(n, 1.0 / n)
            o.propagate(r, threads=threads)
            t0 = time.perf_counter()
            o.propagate(r, threads=threads)
            dt = time.perf_counter() - t0
            cb = {"value": o.nnz / dt, "unit": "edges/s", "cores": threads, "kind": "oracle",
                  "sample": f"one full propagation step of the same graph ({o.nnz} edges), plain C oracle, "
                            f"OpenMP {threads} threads, {dt:.2f} s"}
        line = {"metric": "edges/sec", "value": world * nnz / (step_ms * 1e-3), "unit": "edges/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": step_ms, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic (LCG-generated graph, seed 42; uniform initial ranks)",
                "config": {"workload": f"P1: {CONFIGS['P1'][4]}", "nodes": n, "edges": nnz,
                           "l2": "flushed between steps by a 256 MiB write (outside events)",
                           "parallelism": f"independent replicas x{world}"},
                "roofline": roof, "cpu_baseline": cb, "e2e": e2e, "gpu_launches": 2 * args.steps,
                "clocks": clocks.summary(), "graph_build_s": build_s}
        print(json.dumps(line), flush=True)


def bench_amg(args, rank, world, dev, gf, torch, dist):
    """A1 (NEXT-4): one relaxation sweep over the whole matrix (include/gf_amg.h); replicas per rank."""
    from paper_2306_11686_b200 import dist as gdist
    import numpy as np
    nx, ny, nz = CONFIGS["A1"][1:4]
    A = gf.AMGMatrix(nx, ny, nz, device=dev.index)
    n, nnz = A.n, A.nnz
    rng = np.random.default_rng(7)
    f = torch.from_numpy(rng.random(n)).to(dev)
    a = torch.from_numpy(rng.random(n)).to(dev)
    b = torch.empty_like(a)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.warmup + args.steps)]
    clocks = ClockSampler(dev.index)
    with clocks:
        if dist is not None:
            dist.barrier()
        for k, (e0, e1) in enumerate(evs):
            flush.fill_(k & 0xFF)
            e0.record()
            A.relax(f, a, b)
            e1.record()
            a, b = b, a
        torch.cuda.synchronize()
    step_ms = sum(e0.elapsed_time(e1) for e0, e1 in evs[args.warmup:]) / args.steps
    if dist is not None:
        step_ms = gdist.max_over_ranks([step_ms], dev)[0]
    e2e = None
    if not args.no_e2e:
        uh = torch.from_numpy(rng.random(n)).pin_memory()
        oh = torch.empty((n,), dtype=torch.float64).pin_memory()
        reps = 3
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(reps):
            a.copy_(uh, non_blocking=True)
            A.relax(f, a, b)
            oh.copy_(b, non_blocking=True)
            torch.cuda.synchronize()
        el = (time.perf_counter() - t0) / reps
        e2e = {"value": world * nnz / el, "unit": "nonzeros/s", "h2d_bytes_per_step": 8 * n,
               "d2h_bytes_per_step": 8 * n, "path": "AMGMatrix.relax: iterate H2D, sweep, result D2H; host-timed"}
    if rank == 0:
        peaks = load_peaks()
        alg = 12 * nnz + 28 * n  # col (4 B) + value (8 B) per nonzero; rowptr, f, u (diagonal row) and out per row
        gbs = alg / (step_ms * 1e-3) / 1e9
        prof = load_profile("A1", True)
        roof = {"bound": "hbm", "kernel": "amg_relax", "achieved": gbs, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                "frac": gbs / peaks["hbm_gbs"], "traffic": prof.get("dram_bytes") if prof else None,
                "note": f"algorithmic bytes per sweep = 12 x {nnz} nonzeros + 28 x {n} rows / mean sweep time "
                        f"(CUDA events); the stencil's u gathers hit in cache; traffic = ncu dram read+write "
                        f"({prof.get('src') if prof else 'no capture'}); peak {peaks['src']}"}
        cb = None
        if not args.no_cpu_baseline and world == 1:
            import oracle as O
            threads = len(os.sched_getaffinity(0))
            rp, col, val = O.amg_matrix(nx, ny, nz)
            fh, uh2 = f.cpu().numpy(), rng.random(n)
            O.amg_relax(rp, col, val, fh, uh2, threads=threads)
            sweeps, t0 = 0, time.perf_counter()
            while sweeps == 0 or time.perf_counter() - t0 < 10.0:
                uh2 = O.amg_relax(rp, col, val, fh, uh2, threads=threads)
                sweeps += 1
            dt = time.perf_counter() - t0
            cb = {"value": sweeps * nnz / dt, "unit": "nonzeros/s", "cores": threads, "kind": "oracle",
                  "sample": f"{sweeps} full sweeps of the same matrix ({nnz} nonzeros each), plain C oracle, "
                            f"OpenMP {threads} threads, {dt:.1f} s"}
        line = {"metric": "nonzeros/sec", "value": world * nnz / (step_ms * 1e-3), "unit": "nonzeros/s",
                "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": step_ms,
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic (27-point Laplacian; seeded uniform f and u)",
                "config": {"workload": f"A1: {CONFIGS['A1'][4]}", "rows": n, "nonzeros": nnz,
                           "l2": "flushed between sweeps by a 256 MiB write (outside events)",
                           "parallelism": f"independent replicas x{world}"},
                "roofline": roof, "cpu_baseline": cb, "e2e": e2e, "gpu_launches": args.steps,
                "clocks": clocks.summary()}
        print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C3", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--scaling", default="strong", choices=["weak", "strong"],
                    help="strong (default): the config's lookups are split over the ranks (SURVEY.md 8(e)); "
                         "weak: every rank runs the config's lookups (global indices [r n, (r+1) n))")
    ap.add_argument("--split", default="auto", choices=["auto", "index", "band"],
                    help="strong split: index = rank r takes global lookups [r n / N, (r+1) n / N) on a replicated "
                         "grid; band = rank r holds energy band r of N of the unionized grid and takes the batch's "
                         "lookups in it (SURVEY.md 8(e) 'Alternative: energy-band sharding'); auto = band for "
                         "unionized event configs, index otherwise")
    ap.add_argument("--no-proxy", action="store_true", help="skip the N=1 strong-scaling proxies (W = 2, 4, 8)")
    ap.add_argument("--no-sort", action="store_true", help="skip the A2 locality sort (unsorted gather kernel)")
    ap.add_argument("--hist-mode", default="sorted", choices=["sorted", "waves", "direct"],
                    help="history configs: sorted step waves (default), unsorted waves, or one thread per particle")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-graph", dest="graph", action="store_false",
                    help="history configs: launch the step's waves directly instead of replaying them as one "
                         "captured CUDA graph (H2 4.12 -> 3.72 ms with the graph)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    rank, world, local = env_int("RANK", 0), env_int("WORLD_SIZE", 1), env_int("LOCAL_RANK", 0)
    if args.impl == "reference":
        return run_reference(args, rank, world)

    import ctypes as C

    import torch
    import paper_2306_11686_b200 as gf
    from paper_2306_11686_b200 import build as gfbuild
    from paper_2306_11686_b200 import dist as gdist
    if rank == 0 and gfbuild.needs_build():
        gfbuild.build()
    # one process per GPU; GF_DIST_BACKEND=gloo lets several ranks share one GPU (path tests only)
    backend = os.environ.get("GF_DIST_BACKEND", "nccl")
    local = local % max(torch.cuda.device_count(), 1) if backend != "nccl" else local
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
        dist.barrier()
    dev = torch.device("cuda", local)
    if args.config in ("C7", "C8", "P1", "A1"):
        if args.config in BANDS:
            bench_bands(args, rank, world, dev, gf, torch, dist, C)
        elif args.config == "P1":
            bench_pagerank(args, rank, world, dev, gf, torch, dist)
        else:
            bench_amg(args, rank, world, dev, gf, torch, dist)
        if dist is not None:
            dist.barrier()
            dist.destroy_process_group()
        return
    bench, n_iso, gt, n_total, desc = CONFIGS[args.config]
    HL = HIST_L.get(args.config)
    if HL:  # history mode: the unit of work is a particle (HL dependent lookups); shard whole particles
        p_total = n_total // HL
        if args.scaling == "weak":
            np_first, n_part = gf.weak_range(p_total, rank)
            p_total *= world
        else:
            np_first, n_part = gf.shard_range(p_total, rank, world)
        n_total, first, n = p_total * HL, np_first * HL, n_part * HL
    elif args.scaling == "weak":
        first, n = gf.weak_range(n_total, rank)
        n_total = n * world
    else:
        first, n = gf.shard_range(n_total, rank, world)
    band_ok = bench == "xs" and gt == gf.UNIONIZED and not HL and not args.no_sort
    split = ("band" if band_ok else "index") if args.split == "auto" else args.split
    if split == "band" and not band_ok:
        raise SystemExit(f"--split band needs a sorted unionized event config, not {args.config}")
    banded = split == "band" and args.scaling == "strong" and world > 1
    if banded:  # every rank samples the whole batch; its band grid keeps the lookups in its band
        first, n = 0, n_total
    st = torch.cuda.current_stream()

    # ---------------------------------------------------------------- A0: grid build (untimed)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    n_gp = 238847 if args.config == "C6" else 11303
    params = (gf.Params.xsbench(n_iso, n_gp, gt, 10000, n_bands=world if banded else 1, band=rank if banded else 0)
              if bench == "xs" else gf.Params.rsbench(n_iso, doppler=0 if args.config == "C5D0" else 1))
    grid = gf.Grid(params, device=dev)
    e1.record()
    torch.cuda.synchronize()
    grid_ms = e0.elapsed_time(e1)

    flags = 0 if args.no_sort else gf.SORT_LOCALITY
    if HL:
        flags = gf.Grid.HIST_MODES[args.hist_mode]
        hb = C.c_size_t()
        gf._check(gf.lib().gf_xs_history_bytes(grid.h, n_part, flags, C.byref(hb)))
        scratch = torch.empty(max(hb.value, 256), dtype=torch.uint8, device=dev)
    else:
        scratch = torch.empty(grid.scratch_bytes(n, flags), dtype=torch.uint8, device=dev)
    vsum = torch.zeros(1, dtype=torch.int64, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    L = gf.lib()

    K = args.steps
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(K + args.warmup)]

    graph = None
    if HL and args.graph:  # the HL waves (~8 launches each) captured once and replayed per step
        graph = torch.cuda.CUDAGraph()
        gs = torch.cuda.Stream()
        gs.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(gs):
            gf._check(L.gf_xs_history_batch(grid.h, np_first, n_part, HL, gf.STARTING_SEED, flags, None,
                                            C.c_void_p(vsum.data_ptr()), C.c_void_p(scratch.data_ptr()),
                                            scratch.numel(), C.c_void_p(gs.cuda_stream)))
        torch.cuda.current_stream().wait_stream(gs)
        torch.cuda.synchronize()
        with torch.cuda.graph(graph, stream=gs):
            gf._check(L.gf_xs_history_batch(grid.h, np_first, n_part, HL, gf.STARTING_SEED, flags, None,
                                            C.c_void_p(vsum.data_ptr()), C.c_void_p(scratch.data_ptr()),
                                            scratch.numel(), C.c_void_p(gs.cuda_stream)))
        torch.cuda.synchronize()

    def step(k):
        ev = evs[k]
        vsum.zero_()
        if HL:  # one gf_xs_history_batch call: HL waves (or one direct kernel)
            ev[0].record()
            ev[1].record()
            if graph is not None:
                graph.replay()
            else:
                gf._check(L.gf_xs_history_batch(grid.h, np_first, n_part, HL, gf.STARTING_SEED, flags, None,
                                                C.c_void_p(vsum.data_ptr()), C.c_void_p(scratch.data_ptr()),
                                                scratch.numel(), C.c_void_p(st.cuda_stream)))
            ev[2].record()
            if dist is not None:
                gdist.reduce_raw(vsum)
            ev[3].record()
            return
        se = (C.c_void_p * 3)(ev[0].cuda_event, ev[1].cuda_event, ev[2].cuda_event)
        gf._check(L.gf_xs_lookup_batch_ev(grid.h, first, n, gf.STARTING_SEED, flags, None,
                                          C.c_void_p(vsum.data_ptr()), C.c_void_p(scratch.data_ptr()),
                                          scratch.numel(), C.c_void_p(st.cuda_stream), se))
        if dist is not None:
            gdist.reduce_raw(vsum)
        ev[3].record()

    # events must be created before use: touch them
    for ev in evs:
        for e in ev:
            e.record()
    torch.cuda.synchronize()
    for k in range(args.warmup):
        flush.fill_(k & 0xFF)
        step(k)
    torch.cuda.synchronize()
    raws = []
    clocks = ClockSampler(local)
    with clocks:
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()
        wall0 = time.perf_counter()
        for k in range(args.warmup, args.warmup + K):
            flush.fill_(k & 0xFF)           # L2 flush between timed steps (outside the events)
            step(k)
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
        wall = time.perf_counter() - wall0
    raw = int(vsum.item())
    step_ms = [evs[k][0].elapsed_time(evs[k][3]) for k in range(args.warmup, args.warmup + K)]
    sort_ms = [evs[k][0].elapsed_time(evs[k][1]) for k in range(args.warmup, args.warmup + K)]
    look_ms = [evs[k][1].elapsed_time(evs[k][2]) for k in range(args.warmup, args.warmup + K)]
    tot_ms = sum(step_ms)
    if dist is not None:
        tot_ms, look_tot = gdist.max_over_ranks([tot_ms, sum(look_ms)], dev)
    else:
        look_tot = sum(look_ms)
    value = n_total * K / (tot_ms * 1e-3)

    # ---------------------------------------------------------------- strong-scaling proxies (N = 1)
    # The per-rank step of the W-way split of this config (rank r takes
    # [floor(r n / W), floor((r+1) n / W))), every shard timed on this one GPU exactly as a rank runs it
    # (same call, same flags; L2 flushed before each rep).  The slowest shard bounds a W-GPU step, so
    # speedup = T_1 / max shard; the W-GPU step adds one 8-B all-reduce (~10-30 us over NVLink).
    proxy = None
    if (world == 1 and not args.no_proxy and not HL and args.scaling == "strong" and bench in ("xs", "rs")
            and n_total >= 1_000_000):
        T1 = tot_ms / K
        proxy = {"T1_ms": T1}
        for W in (2, 4, 8):
            shard_ms, raw_w = [], 0
            for r in range(W):
                lo, cnt = gf.shard_range(n_total, r, W)
                ts = []
                for k in range(4):  # 1 warm-up + 3 timed
                    flush.fill_(k & 0xFF)
                    vsum.zero_()
                    p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    p0.record()
                    gf._check(L.gf_xs_lookup_batch(grid.h, lo, cnt, gf.STARTING_SEED, flags, None,
                                                   C.c_void_p(vsum.data_ptr()), C.c_void_p(scratch.data_ptr()),
                                                   scratch.numel(), C.c_void_p(st.cuda_stream)))
                    p1.record()
                    torch.cuda.synchronize()
                    if k:
                        ts.append(p0.elapsed_time(p1))
                raw_w += int(vsum.item())
                shard_ms.append(statistics.median(ts))
            mx = max(shard_ms)
            proxy[str(W)] = {"lookups_per_rank": n_total // W, "max_shard_ms": mx, "speedup": T1 / mx,
                             "kernel": grid.kernel_for(n_total // W, flags) if bench == "xs" else "rs_lookup_sorted",
                             "shard_ms": [round(x, 4) for x in shard_ms], "hash": gf.verify(raw_w)}
        proxy["note"] = ("per-rank step (sort + lookup) of the W-way strong split, each shard timed on this GPU; "
                         "speedup = T1 / slowest shard (excludes the 8-B all-reduce)")
    # The energy-band split (--split band, the default for unionized event configs at N > 1): every band
    # replica r of W is built in turn on this GPU (build untimed) and runs the whole batch, its sort keeping
    # the lookups in band r; the slowest band bounds a W-GPU step.
    proxy_band = None
    if proxy is not None and band_ok:
        T1 = tot_ms / K
        proxy_band = {"T1_ms": T1}
        for W in (2, 4, 8):
            band_ms, raw_w = [], 0
            for r in range(W):
                gb = gf.Grid(gf.Params.xsbench(n_iso, n_gp, gt, 10000, n_bands=W, band=r), device=dev)
                need = gb.scratch_bytes(n_total, flags)  # (band grids add the compacted in-band list)
                bscratch = scratch if scratch.numel() >= need else torch.empty(need, dtype=torch.uint8, device=dev)
                ts = []
                for k in range(4):  # 1 warm-up + 3 timed
                    flush.fill_(k & 0xFF)
                    vsum.zero_()
                    p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    p0.record()
                    gf._check(L.gf_xs_lookup_batch(gb.h, 0, n_total, gf.STARTING_SEED, flags, None,
                                                   C.c_void_p(vsum.data_ptr()), C.c_void_p(bscratch.data_ptr()),
                                                   bscratch.numel(), C.c_void_p(st.cuda_stream)))
                    p1.record()
                    torch.cuda.synchronize()
                    if k:
                        ts.append(p0.elapsed_time(p1))
                raw_w += int(vsum.item())
                del bscratch
                band_ms.append(statistics.median(ts))
                gb.close()
            mx = max(band_ms)
            proxy_band[str(W)] = {"lookups_per_rank": n_total // W, "max_band_ms": mx, "speedup": T1 / mx,
                                  "band_ms": [round(x, 4) for x in band_ms], "hash": gf.verify(raw_w)}
        proxy_band["note"] = ("per-rank step (sort of the whole batch keeping band r, lookup of its ~n/W lookups on "
                              "the band-r grid replica) of the W-way energy-band split, each band timed on this GPU; "
                              "speedup = T1 / slowest band (excludes the 8-B all-reduce)")

    # ---------------------------------------------------------------- end-to-end through the public API
    e2e = None
    if not args.no_e2e and HL:  # history: no per-step inputs (indices + seed); the raw sum comes back
        reps = 3
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(reps):
            r_e2e = grid.history_batch(np_first, n_part, HL, mode=args.hist_mode)
            if dist is not None:
                rt = torch.tensor([r_e2e], dtype=torch.int64, device=dev)
                gdist.reduce_raw(rt)
        el = time.perf_counter() - t0
        if dist is not None:
            el = gdist.max_over_ranks([el], dev)[0]
        e2e = {"value": n_total * reps / el, "unit": "lookups/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 8,
               "path": "Grid.history_batch (gf_xs_history_batch): particle indices + seed in, raw sum (8 B) out; "
                       "host-timed incl. launch and sync"}
    elif not args.no_e2e and banded:  # band grids take sampled lookups only: indices + seed in, raw sum out
        reps = 3
        torch.cuda.synchronize()
        dist.barrier()
        t0 = time.perf_counter()
        for _ in range(reps):
            r_e2e = grid.lookup_batch(first, n)
            rt = torch.tensor([r_e2e], dtype=torch.int64, device=dev)
            gdist.reduce_raw(rt)
        el = gdist.max_over_ranks([time.perf_counter() - t0], dev)[0]
        e2e = {"value": n_total * reps / el, "unit": "lookups/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 8,
               "path": "Grid.lookup_batch (gf_xs_lookup_batch) on the rank's band grid: batch indices + seed in, "
                       "raw sum (8 B) out; host-timed incl. launch and sync (band grids take no caller energies)"}
    elif not args.no_e2e:
        import numpy as np
        rng = np.random.default_rng(1234 + rank)
        P = np.array([0.139, 0.052, 0.275, 0.134, 0.154, 0.064, 0.066, 0.055, 0.008, 0.015, 0.025, 0.013])
        Eh = torch.from_numpy(rng.random(n)).pin_memory()
        mh = torch.from_numpy(rng.choice(12, size=n, p=P / P.sum()).astype(np.uint8)).pin_memory()
        mout = torch.empty((n, grid.channels), dtype=torch.float64, pin_memory=True)  # reused host output

        def e2e_leg(want_macro):
            for _ in range(2):
                grid.lookup_energies(Eh, mh, want_macro=want_macro, out=mout if want_macro else None)
            reps = 3
            torch.cuda.synchronize()
            if dist is not None:
                dist.barrier()
            t0 = time.perf_counter()
            for _ in range(reps):
                r_e2e = grid.lookup_energies(Eh, mh, want_macro=want_macro, out=mout if want_macro else None)
                r_e2e = r_e2e[0] if want_macro else r_e2e
                if dist is not None:
                    rt = torch.tensor([r_e2e], dtype=torch.int64, device=dev)
                    gdist.reduce_raw(rt)
            el = time.perf_counter() - t0
            if dist is not None:
                el = gdist.max_over_ranks([el], dev)[0]
            return n_total * reps / el

        def e2e_streamed(steps=8):
            """Back-to-back batches through gf_xs_lookup_energies_async: every step copies its inputs from
            pinned host memory and reads its raw sum back (8 B), on one of two streams with its own scratch,
            so that batch k+1's copy overlaps batch k's sort and lookup."""
            sts = [torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)]
            need = grid.scratch_bytes(n, gf.SORT_LOCALITY | gf.HOST_IO, whole=True)
            scr = [torch.empty(need, dtype=torch.uint8, device=dev) for _ in range(2)]
            dv = torch.zeros(2, dtype=torch.int64, device=dev)
            res = torch.zeros(steps + 2, dtype=torch.int64).pin_memory()

            def step(k, slot):
                with torch.cuda.stream(sts[k % 2]):
                    dv[k % 2].zero_()
                    grid.lookup_energies_async(Eh, mh, dv[k % 2:k % 2 + 1], scr[k % 2], stream=sts[k % 2])
                    res[slot].copy_(dv[k % 2], non_blocking=True)
            step(0, steps)
            step(1, steps + 1)  # (warm-up, both buffers)
            torch.cuda.synchronize()
            if dist is not None:
                dist.barrier()
            t0 = time.perf_counter()
            for k in range(steps):
                step(k, k)
            torch.cuda.synchronize()
            el = time.perf_counter() - t0
            raws = set(int(x) for x in res.tolist())
            if len(raws) != 1:
                raise SystemExit(f"streamed e2e: the steps' raw sums differ: {sorted(raws)}")
            if dist is not None:
                el = gdist.max_over_ranks([el], dev)[0]
            return n_total * steps / el

        # the step's result is the verification value (XSBench's output); the macro variant also returns
        # every lookup's macro xs vector (5 x 8 B per lookup, which makes the leg PCIe-bound)
        sync_v = e2e_leg(False)
        e2e = {"value": e2e_streamed(), "unit": "lookups/s", "h2d_bytes_per_step": 9 * n, "d2h_bytes_per_step": 8,
               "path": "gf_xs_lookup_energies_async, back-to-back batches: each step copies pinned host E[n] (f64) + "
                       "mat[n] (u8) in and its raw verification sum (8 B) out, two streams with one scratch each "
                       "(step k+1's H2D overlaps step k's sort and lookups); host-timed over the steps, per rank",
               "sync": {"value": sync_v, "unit": "lookups/s",
                        "path": "gf_xs_lookup_energies with GF_HOST_IO, one call per step (returns after its D2H): "
                                "the whole-batch mode, chunk H2D overlapped with the sort's counting pass only"}}
        e2e["with_macro"] = {"value": e2e_leg(True), "unit": "lookups/s", "h2d_bytes_per_step": 9 * n,
                             "d2h_bytes_per_step": 8 * grid.channels * n + 8,
                             "path": f"as above, plus macro[n][{grid.channels}] (f64) copied to pinned host memory"}
        del Eh, mh

    if rank == 0:
        peaks = load_peaks()
        alg_bytes, alg_flops = ALG[args.config]
        # one lookup-kernel launch per step per rank (a band rank's launch covers its band's lookups, n / N expected)
        per_launch_lookups = n_total // world if banded else n
        look_avg_s = look_tot / K * 1e-3
        gname = {0: "nuclide", 1: "unionized", 2: "hash"}.get(gt, "")
        kern = grid.kernel_for(n, flags) if (bench == "xs" and not HL) else ""
        if bench == "rs":
            kname = "rs_lookup_sorted" if flags else "rs_lookup_direct"
        elif not flags:
            kname = f"xs_lookup_direct<{gname}>"
        elif gt == 0:
            kname = {"thread": "xs_lookup_sorted<kGridNB> (per-nuclide bin brackets)",
                     "tilenb": "xs_lookup_tile<nuclide grid> (warp tiles, runs from the per-nuclide bin brackets)"}.get(
                kern, "xs_lookup_warp_nuclide (warp-cooperative search)")
        else:
            kname = {"tile": f"xs_lookup_tile<{gname}> (warp tiles, SMEM-staged interval runs; + idx_prep where used)",
                     "group": f"xs_lookup_group<{gname}> (+ idx_prep)",
                     "thread": "xs_lookup_sorted<kGridNB> (one lookup per thread)"}.get(kern, kern)
        if HL:
            kname = ({"direct": f"{bench}_history_direct (one thread per particle, {HL} dependent lookups)"}.get(
                args.hist_mode, f"{HL} waves of hist_sample + " + ("sort + " if flags & gf.SORT_LOCALITY else "")
                + kname) + "; stage = the whole history call")
        flops = alg_flops * per_launch_lookups
        prof = load_profile(args.config, not args.no_sort)
        roof = {"bound": "alu", "kernel": kname,
                "achieved": flops / look_avg_s / 1e12, "peak": peaks["fp64_dadd_ops_per_s"] / 1e12,
                "unit": "TFLOP/s", "traffic": prof.get("dram_bytes") if prof else None,
                "note": f"{alg_flops} fp64 flops/lookup (DESIGN.md Sec. 5; division counted once) x "
                        f"{per_launch_lookups} lookups per launch / mean lookup-stage time (CUDA events on the "
                        f"launch stream); peak = measured non-FMA FP64 op rate ({peaks['probe_src']}); traffic = "
                        f"ncu dram read+write bytes per launch ({prof.get('src') if prof else 'no capture'})"}
        roof["frac"] = roof["achieved"] / roof["peak"]
        # SURVEY.md 8(d) R-ROOF: the four numbers per run.  rho_thru divides the random-order sector bytes
        # per lookup by the measured random-gather bandwidth (K6, tools/roofline_probe.cu) -- it can exceed
        # 1 because the locality sort removes those bytes, so it is never a DRAM fraction; rho_dram /
        # rho_L2 / l2_hit come from the committed ncu capture of the dominant kernel (src, kernel).
        rho = None
        if bench == "xs" or prof:
            rho = {"rho_fp64_live": roof["frac"]}
            if alg_bytes and peaks.get("gather96_GBps"):
                gb = value / world * alg_bytes / 1e9
                rho.update(rho_thru=gb / peaks["gather96_GBps"], gather_GBps=peaks["gather96_GBps"],
                           alg_sector_bytes_per_lookup=alg_bytes)
            if prof:
                dur = prof.get("duration_s") or 0
                rho.update(rho_dram=(prof["dram_bytes"] / dur / 1e9 / peaks["hbm_gbs"]) if dur else None,
                           dram_GBps=(prof["dram_bytes"] / dur / 1e9) if dur else None,
                           rho_L2=(prof["lts_pct"] / 100) if prof.get("lts_pct") is not None else None,
                           l2_hit_pct=prof.get("l2_hit_pct"),
                           rho_fp64_ncu=(prof["fp64_pipe_pct"] / 100) if prof.get("fp64_pipe_pct") else None,
                           capture=prof.get("src"), capture_kernel=prof.get("kernel", "")[:60])
        paper = None
        if args.config in PAPER_KEY:
            paper = dict(PAPER[PAPER_KEY[args.config]], hardware="NVIDIA A100 40GB vs AMD EPYC 7532 (PAPER.md:812)",
                         metric="kernel speedup over the CPU OpenMP parallel region (PAPER.md:1069)",
                         note="context only: other hardware, and the paper's CPU baseline is the original program")
        cb = None
        if not args.no_cpu_baseline and world == 1:
            cb = cpu_baseline(args.config)
        clk = clocks.summary()
        line = {
            "metric": "lookups/sec", "value": value, "unit": "lookups/s", "n_gpus": world, "steps": K,
            "warmup": args.warmup, "ms_per_step": tot_ms / K, "higher_is_better": True, "scaling": args.scaling,
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (LCG-generated grids and lookups, seeds 42 / 1070)",
            "config": {"workload": f"{args.config}: {desc}", "n_lookups": n_total, "lookups_per_rank": n_total // world if banded else n,
                       **({"mode": f"history ({args.hist_mode})", "particles_per_rank": n_part,
                           "launch": "one CUDA graph of the gf_xs_history_batch call, replayed per step"
                           if graph is not None else "direct",
                           "lookups_per_particle": HL} if HL else {}),
                       "sort": not args.no_sort, "l2": "flushed between steps by a 256 MiB write (outside events)",
                       "split": split if world > 1 else None,
                       "parallelism": (f"strong-scaled energy bands x{world} (rank 0: band [0, 1/{world}) of the "
                                       f"unionized grid, all {n_total} lookups sampled, its band's kept), 1 int64 "
                                       if banded else
                                       f"{args.scaling}-scaled lookup shards x{world} (global indices [{first}, "
                                       f"{first + n}) on rank 0), grid replicated, 1 int64 ")
                                      + f"{os.environ.get('GF_DIST_BACKEND', 'nccl').upper()} all-reduce/step"},
            "roofline": roof, "rho": rho, "strong_proxy": proxy, "strong_proxy_band": proxy_band,
            "paper_context": paper,
            "cpu_baseline": cb, "e2e": e2e,
            "gpu_launches": K * (launches_per_step(bench, gt, flags & gf.SORT_LOCALITY, kern, per_launch_lookups,
                                                   1 if banded else int(os.environ.get("GF_SCATTER_SLICES", "2")))
                                 if not HL else
                                 (1 if args.hist_mode == "direct" else
                                  HL * (1 + launches_per_step(bench, gt, flags & gf.SORT_LOCALITY)))),
            "clocks": clk,
            "stage_ms": {"sort": statistics.median(sort_ms), "lookup": statistics.median(look_ms),
                         "step": statistics.median(step_ms), "grid_build": grid_ms},
            "hash": gf.verify(raw), "raw": raw, "wall_s": wall,
        }
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
