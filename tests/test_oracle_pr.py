"""Pins for the page-rank propagation oracle (NEXT-4; readings R-PR-GRAPH / R-PR-STEP, DESIGN.md
Sec. 3).  CPU only.  The generator is checked against an independent Python transcription (exact
integer LCG, correctly rounded rationals); the step against exact rational arithmetic, closed forms
on special graphs (a directed cycle, a circulant regular graph) and rank-mass conservation.
"""
import math
from fractions import Fraction

import numpy as np
import pytest

import oracle as O

A_LCG = 2806196910506780709
M63 = 1 << 63
M64 = 1 << 64


def _step(s):
    return (A_LCG * s + 1) % M64 % M63


def _ff(s, n):
    an = pow(A_LCG, n, M63 * (A_LCG - 1))
    return (pow(A_LCG, n, M63) * s + (an - 1) // (A_LCG - 1)) % M63


def _draw(st):
    st[0] = _step(st[0])
    return float(Fraction(st[0], M63))


def py_graph(n, D, seed=42):
    rows = [[] for _ in range(n)]
    outdeg = []
    for u in range(n):
        st = [_ff(seed, 2 * D * u)]
        d = min(1 + int(_draw(st) * (2 * D - 1)), 2 * D - 1)
        outdeg.append(d)
        for _ in range(d):
            v = min(int(_draw(st) * n), n - 1)
            rows[v].append(u)
    rowptr = np.cumsum([0] + [len(r) for r in rows])
    return rowptr, np.array([u for r in rows for u in r], dtype=np.int32), np.array(outdeg, dtype=np.int32)


def test_generator_matches_python_transcription():
    for n, D in ((257, 4), (1000, 16)):
        o = O.PROracle(n, D)
        rp, col, od = o.arrays()
        prp, pcol, pod = py_graph(n, D)
        assert np.array_equal(od, pod) and np.array_equal(rp, prp) and np.array_equal(col, pcol)


def test_step_matches_exact_rationals():
    n, D = 300, 6
    o = O.PROracle(n, D)
    rp, col, od = o.arrays()
    rng = np.random.default_rng(3)
    r = rng.random(n)
    r /= r.sum()
    got = o.propagate(r)
    d = Fraction(85, 100)
    base = (1 - d) / n
    for v in range(n):
        exact = base + d * sum(Fraction(r[u]) / int(od[u]) for u in col[rp[v]:rp[v + 1]])
        deg = rp[v + 1] - rp[v]
        bound = (deg + 4) * 2.0 ** -52 * max(float(exact), 1e-300)
        assert abs(Fraction(got[v]) - exact) <= Fraction(bound), v


def test_directed_cycle_and_regular_graph():
    n = 1000
    rng = np.random.default_rng(4)
    # directed cycle u -> u + 1: one in-edge per node, out-degree 1: r'[v] = base + 0.85 r[v - 1] exactly
    rowptr = np.arange(n + 1, dtype=np.int64)
    col = ((np.arange(n) - 1) % n).astype(np.int32)
    r = rng.random(n)
    out = O.pr_propagate_csr(rowptr, col, np.ones(n, dtype=np.int32), r)
    assert np.array_equal(out, (1.0 - 0.85) / n + 0.85 * r[col])
    # circulant graph with 8 offsets: in = out = 8 everywhere, so the uniform vector is a fixed point
    offs = np.array([1, 2, 3, 5, 8, 13, 21, 34])
    col = np.stack([(np.arange(n) - o) % n for o in offs], axis=1).reshape(-1).astype(np.int32)
    rowptr = np.arange(0, 8 * n + 1, 8, dtype=np.int64)
    u = np.full(n, 1.0 / n)
    out = O.pr_propagate_csr(rowptr, col, np.full(n, 8, dtype=np.int32), u)
    assert np.max(np.abs(out - 1.0 / n)) <= 8 * np.spacing(1.0 / n)


def test_mass_conservation_and_degree_statistics():
    n, D = 1 << 18, 16
    o = O.PROracle(n, D)
    rp, col, od = o.arrays()
    assert od.min() >= 1 and od.max() <= 2 * D - 1
    assert abs(od.mean() - D) < 5 * math.sqrt((4 * D * D - 1) / 12 / n) + 1e-9  # uniform on 1..2D-1
    assert o.nnz == od.sum() == rp[-1]
    indeg = np.diff(rp)
    assert abs(indeg.mean() - od.mean()) < 1e-12
    r = np.random.default_rng(5).random(n)
    out = o.propagate(r)
    want = (1 - 0.85) + 0.85 * math.fsum(r)  # no dangling nodes: all rank mass flows
    assert abs(math.fsum(out) - want) <= 1e-10 * want
