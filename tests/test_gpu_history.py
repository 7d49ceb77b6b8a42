"""GPU parity of the history-based mode (NEXT-1; readings R-HIST / R-HIST-RS) through
gf_xs_history_batch against the oracle's xso_history_batch / rso_history_batch (pinned in
tests/test_oracle_history.py).  XSBench: every macro xs of every step bit-identical and the raw
sum equal, in all three device mappings (one thread per particle; step waves; sorted step waves).
RSBench: macro xs within 1e-10 * S (R-UNIQ) and raw sums equal; the smallest |macro_c| / S is
reported because the chain branches on the sign of macro_c.
"""
import json
import os

import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu
MODES = ["direct", "waves", "sorted"]


@pytest.fixture(scope="module")
def gf():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("no CUDA device: the gpu tests must run on a B200 (no CPU fallback exists)")
    import paper_2306_11686_b200 as G
    from paper_2306_11686_b200 import build
    build.build()
    return G


@pytest.mark.parametrize("grid_type", [0, 1, 2])
def test_xs_small_history_all_modes(gf, grid_type):
    o = O.XSOracle(68, 11303, grid_type)
    g = gf.Grid(gf.Params.xsbench(68, 11303, grid_type))
    first, n_p, L = 1234, 3001, 34  # several CTAs and a ragged tail, global particle offset
    raw_o, m_o = o.history_batch(first, n_p, L, want_macro=True)
    for mode in MODES:
        raw_g, m_g = g.history_batch(first, n_p, L, mode=mode, want_macro=True)
        assert raw_g == raw_o, mode
        m_g = m_g.cpu().numpy()
        bad = np.argwhere(m_g != m_o)
        assert bad.size == 0, f"{mode}: {len(bad)} mismatches, first {bad[:3]}"
        assert g.history_batch(first, n_p, L, mode=mode) == raw_o  # no-output path


@pytest.mark.parametrize("L", [1, 2, 7])
def test_xs_history_short_chains_and_tiny_batches(gf, L):
    o = O.XSOracle(68, 11303, O.UNIONIZED)
    g = gf.Grid(gf.Params.xsbench(68, 11303, gf.UNIONIZED))
    for first, n_p in ((0, 1), (5, 31), (100_000, 333)):
        raw_o, m_o = o.history_batch(first, n_p, L, want_macro=True)
        for mode in MODES:
            raw_g, m_g = g.history_batch(first, n_p, L, mode=mode, want_macro=True)
            assert raw_g == raw_o and np.array_equal(m_g.cpu().numpy(), m_o), (mode, first, n_p)
    assert g.history_batch(0, 0, L) == 0


def test_xs_large_history_full_size(gf):
    """C3 shapes in history mode: 500,000 particles x 34 lookups on the large unionized grid, the
    launch configuration bench.py times; raw equals the oracle's over all 17 M dependent lookups,
    and sampled particles' full chains are bit-identical."""
    import torch
    o = O.XSOracle(355, 11303, O.UNIONIZED)
    g = gf.Grid(gf.Params.xsbench(355, 11303, gf.UNIONIZED))
    n_p, L = 500_000, 34
    raw_g = g.history_batch(0, n_p, L, mode="sorted")
    raw_o = o.history_batch(0, n_p, L)
    assert raw_g == raw_o
    assert g.history_batch(0, n_p, L, mode="direct") == raw_o
    raw_s, m_g = g.history_batch(0, n_p, L, mode="sorted", want_macro=True)
    assert raw_s == raw_o
    rng = np.random.default_rng(9)
    for p in list(rng.integers(0, n_p, 40)) + [0, n_p - 1]:
        _, m_o = o.history_batch(int(p), 1, L, want_macro=True)
        assert np.array_equal(m_g[int(p)].cpu().numpy(), m_o[0]), p
    del m_g
    torch.cuda.empty_cache()


@pytest.mark.parametrize("n_iso,n_p", [(68, 600), (355, 150)])
def test_rs_history_all_modes(gf, n_iso, n_p):
    o = O.RSOracle(n_iso)
    g = gf.Grid(gf.Params.rsbench(n_iso))
    L = 34
    raw_o, m_o, S = o.history_batch(77, n_p, L, want_macro=True)
    print(f"RS history n_iso={n_iso}: min |macro_c| / S = {np.min(np.abs(m_o) / S[..., None]):.3e}")
    for mode in MODES:
        raw_g, m_g = g.history_batch(77, n_p, L, mode=mode, want_macro=True)
        assert raw_g == raw_o, mode
        err = np.abs(m_g.cpu().numpy() - m_o) / S[..., None]
        assert err.max() <= 1e-10, (mode, err.max())


def test_history_full_size_goldens(gf):
    """H2 / H3 (XSBench small / large, 500 k particles x 34) and H5 (RSBench large, 300 k x 34): whole-run
    raw sums against the oracle's (tests/golden/make_golden.py --extra)."""
    gold = json.load(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "oracle_hashes.json")))
    for name, n_iso in (("H2", 68), ("H3", 355)):
        g = gf.Grid(gf.Params.xsbench(n_iso, 11303, gf.UNIONIZED))
        assert g.history_batch(0, 500_000, 34) == gold[name]["raw"], name
        del g
    r = gf.Grid(gf.Params.rsbench(355))
    assert r.history_batch(0, 300_000, 34) == gold["H5"]["raw"]
