"""Pins for the AMGmk relax oracle (NEXT-4; readings R-AMG-MAT / R-AMG-RELAX).  CPU."""
from fractions import Fraction

import numpy as np

import oracle as O


def test_matrix_structure():
    nx, ny, nz = 5, 4, 3
    rp, col, val = O.amg_matrix(nx, ny, nz)
    n = nx * ny * nz
    # entries per row = product over axes of the neighbour counts (2 at a face, 3 inside)
    cnt = lambda k, m: 2 if (k == 0 or k == m - 1) and m > 1 else (1 if m == 1 else 3)
    for i in range(n):
        x, y, z = i % nx, (i // nx) % ny, i // (nx * ny)
        row = slice(rp[i], rp[i + 1])
        assert rp[i + 1] - rp[i] == cnt(x, nx) * cnt(y, ny) * cnt(z, nz)
        assert col[rp[i]] == i and val[rp[i]] == 26.0  # diagonal first
        nb = col[rp[i] + 1:rp[i + 1]]
        assert np.all(np.diff(nb) > 0) and i not in nb and np.all(val[rp[i] + 1:rp[i + 1]] == -1.0)
        for j in nb:  # every off-diagonal is a true 27-point neighbour
            X, Y, Z = j % nx, (j // nx) % ny, j // (nx * ny)
            assert max(abs(X - x), abs(Y - y), abs(Z - z)) == 1
    assert np.array_equal(rp[-1], len(col))


def test_relax_special_cases():
    nx = ny = nz = 6
    rp, col, val = O.amg_matrix(nx, ny, nz)
    n = nx * ny * nz
    c = 0.375
    u = np.full(n, c)
    deg = np.diff(rp) - 1  # off-diagonal count
    # f = A u for a constant u: one sweep returns u exactly (all values are small dyadics, exact in fp64)
    f = 26 * c - deg * c
    assert np.array_equal(O.amg_relax(rp, col, val, f, u), u)
    # u = 0: u' = f / 26 exactly
    f = np.random.default_rng(1).random(n)
    assert np.array_equal(O.amg_relax(rp, col, val, f, np.zeros(n)), f / 26.0)


def test_relax_matches_exact_rationals():
    nx, ny, nz = 4, 5, 3
    rp, col, val = O.amg_matrix(nx, ny, nz)
    n = nx * ny * nz
    rng = np.random.default_rng(2)
    f, u = rng.random(n), rng.random(n)
    got = O.amg_relax(rp, col, val, f, u)
    for i in range(n):
        s = Fraction(f[i]) - sum(Fraction(val[jj]) * Fraction(u[col[jj]]) for jj in range(rp[i] + 1, rp[i + 1]))
        exact = s / 26
        bound = (rp[i + 1] - rp[i] + 2) * 2.0 ** -52 * (abs(float(Fraction(f[i]))) + 26)
        assert abs(Fraction(got[i]) - exact) <= Fraction(bound) / 26, i
