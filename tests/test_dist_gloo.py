"""N > 1 host path on CPU: world_size-2 gloo process group.  Each rank computes its contiguous shard
of the lookups (here with the oracle, since there is no GPU), the raw sums are all-reduced with the
package's reduce_raw, and the finished hash equals the single-process hash."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle as O
    import paper_2306_11686_b200 as gf
    from paper_2306_11686_b200 import dist as gdist
    o = O.XSOracle(68, 11303, O.NUCLIDE)
    first, cnt = gf.shard_range(n, rank, world)
    raw = o.lookup_batch(first, cnt, threads=1)
    vsum = torch.tensor([raw], dtype=torch.int64)
    gdist.reduce_raw(vsum)
    t = gdist.max_over_ranks([float(rank + 1), 10.0 - rank], "cpu")
    if rank == 0:
        q.put((int(vsum.item()), gdist.finish_hash(int(vsum.item())), t))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_gloo_sharded_hash_equals_single_process(world):
    import oracle as O
    import paper_2306_11686_b200 as gf
    n = 30_011  # not a multiple of the world size
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    import queue
    import time
    deadline = time.time() + 300
    while True:  # fail fast if a worker dies instead of waiting for the queue
        try:
            raw, h, t = q.get(timeout=2)
            break
        except queue.Empty:
            dead = [p.exitcode for p in procs if p.exitcode not in (None, 0)]
            assert not dead and time.time() < deadline, f"gloo workers failed: exit codes {dead}"
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    full = O.XSOracle(68, 11303, O.NUCLIDE).lookup_batch(0, n)
    assert raw == full
    assert h == gf.verify(full)
    assert t == [2.0, 10.0]


def test_weak_ranges_tile_the_batch():
    """Weak scaling (bench --scaling weak): rank r of W runs [r n, (r+1) n); the ranges tile [0, W n), so the
    all-reduced raw sum of W ranks is the raw sum of one W n batch (hash additivity)."""
    import oracle as O
    import paper_2306_11686_b200 as gf
    n, world = 997, 3
    rs = [gf.weak_range(n, r) for r in range(world)]
    assert [f for f, _ in rs] == [0, n, 2 * n] and all(c == n for _, c in rs)
    o = O.XSOracle(68, 11303, O.NUCLIDE)
    assert sum(o.lookup_batch(f, c, threads=1) for f, c in rs) == o.lookup_batch(0, world * n, threads=1)


def _band_worker(rank, world, port, W, n, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import numpy as np
    import oracle as O
    from paper_2306_11686_b200 import dist as gdist
    o = O.XSOracle(68, 11303, O.NUCLIDE)
    E = np.array([O.sample(i)[0] for i in range(n)])
    band = np.clip(np.floor(E * W).astype(np.int64), 0, W - 1)
    raw = 0
    for b in range(rank, W, world):  # bench.py C7: rank r serves bands r, r + N, ...
        idx = np.flatnonzero(band == b).astype(np.uint64)
        if len(idx):
            raw += o.lookup_indices(idx)[0]
    vsum = torch.tensor([raw], dtype=torch.int64)
    gdist.reduce_raw(vsum)
    if rank == 0:
        q.put(int(vsum.item()))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_energy_bands_partition_the_batch():
    """NEXT-2 band sharding over ranks (bench.py C7): every lookup belongs to exactly one of W energy
    bands, ranks serve bands r, r + N, ...; the all-reduced raw sum equals the whole batch's."""
    import oracle as O
    W, n, world = 8, 20_000, 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_band_worker, args=(r, world, port, W, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    raw = q.get(timeout=300)
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    assert raw == O.XSOracle(68, 11303, O.NUCLIDE).lookup_batch(0, n)
