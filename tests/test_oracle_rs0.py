"""Pins for the RSBench 0 K pole kernel (doppler = 0; NEXT-3; reading R-RS0 in
DESIGN.md Sec. 3).  CPU only.

The oracle's fp64 macro xs are checked against a 50-digit mpmath evaluation of the same data (the
exact value of the reading's formula; the fp64 result must lie within a rounding bound of it), and
against the structural facts the kernel must keep: sigma_E = sigma_T - sigma_A, a window without
poles gives E (T, A, F, T - A), the background does not depend on the kernel, the flag is live,
and hash bounds / additivity.
"""
import mpmath
import numpy as np
import pytest

import oracle as O


@pytest.fixture(scope="module")
def rs0():
    return O.RSOracle(68, doppler=0)


def _macro_mp(o, d, E, mat):
    """50-digit macro xs of R-RS0: sigma = E (T, A, F) + sum_p Re(R * i / ((EA - sqrt E) E) [* fac_l])."""
    mpmath.mp.dps = 50
    npo, nwi = o.counts()
    nn, mats = O.builtin_tables(o.n_nuc)
    poff = np.concatenate([[0], np.cumsum(npo)])
    woff = np.concatenate([[0], np.cumsum(nwi)])
    Em = mpmath.mpf(E)
    sq = mpmath.sqrt(Em)
    macro = [mpmath.mpf(0)] * 4
    scale = mpmath.mpf(0)
    for j in range(nn[mat]):
        nuc = mats[mat, j]
        w = int(E / (1.0 / nwi[nuc]))  # the window index is an fp64 decision: same as the oracle
        w = min(w, nwi[nuc] - 1)
        q = woff[nuc] + w
        fac = []
        for l in range(4):
            phi = mpmath.mpf(d["K0RS"][nuc, l]) * sq
            if l == 1:
                phi = phi + mpmath.atan(phi)
            elif l == 2:
                phi = phi - mpmath.atan(3 * phi / (3 - phi * phi))
            elif l == 3:
                phi = phi - mpmath.atan(phi * (15 - phi * phi) / (15 - 6 * phi * phi))
            phi = 2 * phi
            fac.append(mpmath.mpc(mpmath.cos(phi), -mpmath.sin(phi)))
        T, A, F = (mpmath.mpf(x) for x in d["win"][q])
        sT, sA, sF = Em * T, Em * A, Em * F
        S = abs(sT) + abs(sA) + abs(sF)
        for p in range(d["win_start"][q], d["win_end"][q]):
            P = d["pole"][poff[nuc] + p]
            EA = mpmath.mpc(P[0], P[1])
            cdum = mpmath.mpc(0, 1) / (EA - sq) / Em
            t = (mpmath.mpc(P[2], P[3]) * cdum * fac[d["pole_l"][poff[nuc] + p]]).real
            a = (mpmath.mpc(P[4], P[5]) * cdum).real
            f = (mpmath.mpc(P[6], P[7]) * cdum).real
            sT, sA, sF = sT + t, sA + a, sF + f
            S += abs(t) + abs(a) + abs(f)
        conc = mpmath.mpf(d["concs"][mat, j])
        for c, v in enumerate((sT, sA, sF, sT - sA)):
            macro[c] += v * conc
        scale += S * abs(conc)
    return np.array([float(x) for x in macro]), float(scale)


def test_rs0_matches_50_digit_evaluation(rs0):
    d = rs0.data()
    for i in list(range(6)) + [1000, 77_777]:
        E, mat = O.sample(i)
        m, S = rs0.macro(E, mat)
        m_mp, S_mp = _macro_mp(rs0, d, E, mat)
        assert np.all(np.abs(m - m_mp) <= 1e-13 * S_mp), (i, m, m_mp)
        assert abs(S - S_mp) <= 1e-12 * S_mp


def test_rs0_identities_and_flag(rs0):
    rs1 = O.RSOracle(68)
    raw, m, S = rs0.lookup_batch(0, 2000, want_macro=True)
    assert np.all(np.abs(m[:, 3] - (m[:, 0] - m[:, 1])) <= 1e-12 * S)
    assert 2000 <= raw <= 4 * 2000
    assert raw == rs0.lookup_batch(0, 700) + rs0.lookup_batch(700, 1300)
    _, m1, _ = rs1.lookup_batch(0, 2000, want_macro=True)
    assert np.mean(np.abs(m - m1) > 1e-6 * S[:, None]) > 0.5  # the 0 K kernel is a different function
    # the data (and so the window background) do not depend on the kernel
    d0, d1 = rs0.data(), rs1.data()
    assert all(np.array_equal(d0[k], d1[k]) for k in d0)


def test_rs0_empty_window_is_background():
    """avg_poles = avg_windows: some windows hold one pole, whose loop [start, end) is empty (R-RSEND)
    -- their micro xs is exactly E (T, A, F, T - A) whatever the kernel."""
    o = O.RSOracle(68, avg_poles=2, avg_windows=2, doppler=0)
    d = o.data()
    npo, nwi = o.counts()
    nn, mats = O.builtin_tables(68)
    woff = np.concatenate([[0], np.cumsum(nwi)])
    hit = 0
    for i in range(300):
        E, mat = O.sample(i)
        exp = np.zeros(4)
        ok = True
        for j in range(nn[mat]):
            nuc = mats[mat, j]
            w = min(int(E / (1.0 / nwi[nuc])), nwi[nuc] - 1)
            q = woff[nuc] + w
            if d["win_end"][q] > d["win_start"][q]:
                ok = False
                break
            T, A, F = d["win"][q]
            micro = np.array([E * T, E * A, E * F, E * T - E * A])
            exp = exp + micro * d["concs"][mat, j]
        if ok:
            m, _ = o.macro(E, mat)
            assert np.array_equal(m, exp)
            hit += 1
    assert hit > 0
