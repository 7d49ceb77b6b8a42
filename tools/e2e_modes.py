"""Host-I/O (GF_HOST_IO) modes of gf_xs_lookup_energies on C3, hash only, host-timed: the whole-batch mode
(one sort + lookup over the batch; the chunk copies overlap the counting pass) against the chunked
pipeline (each 2^22-lookup chunk sorted and looked up on its own while the next one is copied), chosen
by the scratch size the caller passes.
    python tools/e2e_modes.py > gpurun_out/e2e_modes.txt"""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2306_11686_b200 as gf  # noqa: E402

n = 17_000_000
g = gf.Grid(gf.Params.xsbench(355, 11303, gf.UNIONIZED))
rng = np.random.default_rng(1)
P = np.array([0.139, 0.052, 0.275, 0.134, 0.154, 0.064, 0.066, 0.055, 0.008, 0.015, 0.025, 0.013])
Eh = torch.from_numpy(rng.random(n)).pin_memory()
mh = torch.from_numpy(rng.choice(12, size=n, p=P / P.sum()).astype(np.uint8)).pin_memory()
flags = gf.SORT_LOCALITY | gf.HOST_IO
st = torch.cuda.current_stream().cuda_stream
for name, whole in (("whole", True), ("chunked", False), ("whole", True), ("chunked", False)):
    sc = torch.empty(g.scratch_bytes(n, flags, whole=whole), dtype=torch.uint8, device="cuda")
    vs = C.c_uint64(0)

    def call():
        vs.value = 0
        gf._check(gf.lib().gf_xs_lookup_energies(g.h, C.c_void_p(Eh.data_ptr()), C.c_void_p(mh.data_ptr()), n, flags,
                                                 None, C.byref(vs), C.c_void_p(sc.data_ptr()), sc.numel(), C.c_void_p(st)))
    call()
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        t = time.perf_counter()
        call()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t)
    ts.sort()
    print(f"{name:8s} scratch {sc.numel() / 1e6:.0f} MB: {ts[2] * 1e3:.2f} ms = {n / ts[2]:.3e} lookups/s raw {vs.value}",
          flush=True)
    del sc
    torch.cuda.empty_cache()
