"""GPU parity of the AMGmk relax kernel (NEXT-4, include/gf_amg.h) against the oracle
(tests/test_oracle_amg.py pins it): the device-built CSR equals the oracle's, and relaxation sweeps
are bit-identical (both follow R-AMG-RELAX's left-to-right row sums)."""
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


@pytest.mark.parametrize("dims", [(1, 1, 1), (2, 1, 1), (5, 4, 3), (1, 7, 2), (33, 17, 9), (128, 128, 64)])
def test_matrix_and_sweeps_bit_exact(gf, dims):
    import torch
    A = gf.AMGMatrix(*dims)
    rp, col, val = A.arrays()
    orp, ocol, oval = O.amg_matrix(*dims)
    assert A.nnz == len(ocol)
    assert np.array_equal(rp, orp) and np.array_equal(col, ocol) and np.array_equal(val, oval)
    rng = np.random.default_rng(sum(dims))
    f, u = rng.random(A.n), rng.random(A.n)
    df, du = torch.from_numpy(f).cuda(), torch.from_numpy(u).cuda()
    dv = torch.empty_like(du)
    want = u
    for _ in range(3):
        A.relax(df, du, dv)
        want = O.amg_relax(orp, ocol, oval, f, want)
        assert np.array_equal(dv.cpu().numpy(), want)
        du, dv = dv, du


def test_bench_size_sweep_bit_exact(gf):
    """A1's full size (256^3, 449 M nonzeros) in the launch configuration bench.py times: the whole
    device matrix and one sweep compared element by element with the oracle (needs ~12 GB host RAM)."""
    import psutil
    import torch
    if psutil.virtual_memory().available < 24 << 30:
        pytest.skip("needs ~24 GB free host memory for the oracle's 256^3 matrix")
    A = gf.AMGMatrix(256, 256, 256)
    orp, ocol, oval = O.amg_matrix(256, 256, 256)
    rp, col, val = A.arrays()
    assert np.array_equal(rp, orp)
    assert np.array_equal(col, ocol)
    assert np.array_equal(val, oval)
    del col, val
    rng = np.random.default_rng(7)
    f, u = rng.random(A.n), rng.random(A.n)
    out = torch.empty(A.n, dtype=torch.float64, device="cuda")
    A.relax(torch.from_numpy(f).cuda(), torch.from_numpy(u).cuda(), out)
    assert np.array_equal(out.cpu().numpy(), O.amg_relax(orp, ocol, oval, f, u))
