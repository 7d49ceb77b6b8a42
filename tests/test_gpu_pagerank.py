"""GPU parity of the page-rank propagation step (NEXT-4, include/gf_pr.h) against the oracle
(tests/test_oracle_pr.py pins it): the device-built graph equals the oracle's CSR exactly, and one or
several propagation steps are bit-identical (both follow R-PR-STEP's left-to-right row sums)."""
import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gf():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("no CUDA device: the gpu tests must run on a B200 (no CPU fallback exists)")
    import paper_2306_11686_b200 as G
    from paper_2306_11686_b200 import build
    build.build()
    return G


@pytest.mark.parametrize("n,D", [(1, 1), (7, 1), (1000, 4), (4099, 16), (1 << 20, 16), (100_003, 32)])
def test_graph_and_steps_bit_exact(gf, n, D):
    import torch
    o = O.PROracle(n, D)
    g = gf.PRGraph(n, D)
    rp, col, od = g.arrays()
    orp, ocol, ood = o.arrays()
    assert g.n_edges == o.nnz
    assert np.array_equal(rp, orp) and np.array_equal(col, ocol) and np.array_equal(od, ood)
    r = np.random.default_rng(n).random(n)
    r /= r.sum()
    a = torch.from_numpy(r).cuda()
    b = torch.empty_like(a)
    want = r
    for _ in range(3):  # a few steps: the iterate stays bit-identical
        g.propagate(a, b)
        want = o.propagate(want)
        assert np.array_equal(b.cpu().numpy(), want)
        a, b = b, a


def test_full_size_sampled(gf):
    """The bench configuration (2^24 nodes, 16 average out-degree): full step bit-exact."""
    import torch
    n, D = 1 << 24, 16
    o = O.PROracle(n, D)
    g = gf.PRGraph(n, D)
    assert g.n_edges == o.nnz
    r = np.full(n, 1.0 / n)
    out = g.propagate(torch.from_numpy(r).cuda()).cpu().numpy()
    assert np.array_equal(out, o.propagate(r))
