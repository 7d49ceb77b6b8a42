"""Where does the host-IO (e2e) time of C3 go?  Prints: pinned H2D bandwidth, the energies API on
device-resident inputs (sorted, 17 M), and the GF_HOST_IO call (hash only) -- each host-timed."""
import time

import numpy as np
import torch

import paper_2306_11686_b200 as gf


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / reps


n = 17_000_000
g = gf.Grid(gf.Params.xsbench(355, 11303, gf.UNIONIZED))
rng = np.random.default_rng(1)
P = np.array([0.139, 0.052, 0.275, 0.134, 0.154, 0.064, 0.066, 0.055, 0.008, 0.015, 0.025, 0.013])
Eh = torch.from_numpy(rng.random(n)).pin_memory()
mh = torch.from_numpy(rng.choice(12, size=n, p=P / P.sum()).astype(np.uint8)).pin_memory()
Ed, md = Eh.cuda(), mh.cuda()
t_h2d = timed(lambda: (Ed.copy_(Eh, non_blocking=True), md.copy_(mh, non_blocking=True)))
print(f"H2D {9 * n / 1e6:.0f} MB: {t_h2d * 1e3:.2f} ms = {9 * n / t_h2d / 1e9:.1f} GB/s")
t_dev = timed(lambda: g.lookup_energies(Ed, md, want_macro=False))
print(f"energies, device inputs: {t_dev * 1e3:.2f} ms")
t_host = timed(lambda: g.lookup_energies(Eh, mh, want_macro=False))
print(f"energies, GF_HOST_IO: {t_host * 1e3:.2f} ms")
t_ev = timed(lambda: g.lookup_batch(0, n))
print(f"event batch (sampled on device): {t_ev * 1e3:.2f} ms")
import os
os.environ["GF_XS_KERNEL"] = "thread"
t_host_t = timed(lambda: g.lookup_energies(Eh, mh, want_macro=False))
t_dev_t = timed(lambda: g.lookup_energies(Ed, md, want_macro=False))
print(f"thread kernel: device inputs {t_dev_t * 1e3:.2f} ms, GF_HOST_IO {t_host_t * 1e3:.2f} ms")
os.environ.pop("GF_XS_KERNEL")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
E2, m2 = torch.empty_like(Ed), torch.empty_like(md)


def both():  # the copy is enqueued first (lookup_batch returns the hash, i.e. synchronises)
    with torch.cuda.stream(s2):
        E2.copy_(Eh, non_blocking=True)
        m2.copy_(mh, non_blocking=True)
    with torch.cuda.stream(s1):
        g.lookup_batch(0, n)
    torch.cuda.synchronize()


print(f"event batch on one stream + 153 MB H2D on another: {timed(both) * 1e3:.2f} ms")
os.environ["GF_XS_KERNEL"] = "thread"
print(f"  same with the thread kernel: {timed(both) * 1e3:.2f} ms")
