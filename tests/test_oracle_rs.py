"""Pins for the RSBench oracle (RS rows; Appendix A.1, A.7).  CPU only."""
import json
import math
import os

import mpmath
import numpy as np
import pytest
import scipy.special

import oracle as O

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "survey_a8.json")))


@pytest.fixture(scope="module")
def rs():
    return O.RSOracle(355, 1000, 100, 4)


def test_faddeeva_asymptotic_matches_wofz_upper_half_plane():
    """|z| >= 6: the 4-point Gauss-Hermite form approximates w(z) (A.1: max rel. err 1.1e-6).  A wrong
    constant a..d (closed forms (3+-sqrt6)/(6 sqrt(pi)), (3-+sqrt6)/2) would fail this."""
    rng = np.random.default_rng(7)
    worst = 0.0
    for _ in range(3000):
        r = 6 + 60 * rng.random()
        th = math.pi * rng.random()
        z = complex(r * math.cos(th), r * math.sin(th))
        ref = complex(scipy.special.wofz(z))
        worst = max(worst, abs(O.faddeeva_W(z) - ref) / abs(ref))
    assert worst < 2e-6


def test_faddeeva_abrarov_matches_wofz_upper_half_plane():
    """|z| < 6: Abrarov-Quine with tau_m = 12, N = 10 and 7-digit constants (A.1: max rel. err 5.5e-4)."""
    rng = np.random.default_rng(8)
    worst = 0.0
    for _ in range(3000):
        r = 0.05 + 5.9 * rng.random()
        th = math.pi * (0.02 + 0.96 * rng.random())
        z = complex(r * math.cos(th), r * math.sin(th))
        ref = complex(scipy.special.wofz(z))
        worst = max(worst, abs(O.faddeeva_W(z) - ref) / abs(ref))
    assert worst < 1e-3


def test_faddeeva_constants_closed_forms():
    """The printed 7-digit Abrarov coefficients equal (2 sqrt(pi)/12) exp(-(n pi/12)^2) and (n pi)^2,
    and 81.24330 = 144/sqrt(pi) (A.1).  The oracle's W is affine in each constant, so perturbing one
    by its printed precision moves W by < 1e-6 relative: check W against a high-precision evaluation
    of the same formula with exact constants."""
    mpmath.mp.dps = 40
    an = [2 * mpmath.sqrt(mpmath.pi) / 12 * mpmath.e ** (-(n * mpmath.pi / 12) ** 2) for n in range(1, 11)]
    den = [(n * mpmath.pi) ** 2 for n in range(1, 11)]
    pref = 144 / mpmath.sqrt(mpmath.pi)

    def W_exact(z):
        z = mpmath.mpc(z)
        e = mpmath.exp(12j * z)  # fast_exp/fast_cexp approximate exp; difference ~ x^2/8192
        W = 1j * (1 - e) / (12 * z)
        s = sum(an[n] * ((-1) ** (n + 1) * e - 1) / (den[n] - 144 * z * z) for n in range(10))
        return complex(W + 1j * pref * z * s)

    rng = np.random.default_rng(9)
    for _ in range(200):
        z = complex(rng.uniform(-4, 4), rng.uniform(0.1, 4))
        if abs(z) >= 6:
            continue
        got, ref = O.faddeeva_W(z), W_exact(z)
        assert abs(got - ref) <= 2e-4 * max(abs(ref), 1e-3)


def test_fast_exp_closed_form():
    mpmath.mp.dps = 50
    for x in (-3.0, -0.5, 0.0, 0.25, 1.0, 2.5):
        ref = (1 + mpmath.mpf(x) / 4096) ** 4096
        assert abs(O.fast_exp(x) - float(ref)) <= 1e-11 * float(ref)


def test_pole_and_window_counts(rs):
    npo, nwi = rs.counts()
    assert npo.sum() == 1000 * 355 and nwi.sum() == 100 * 355
    assert npo.min() >= 1 and nwi.min() >= 1
    d = rs.data()
    off = 0
    for i in range(355):
        ws, we = d["win_start"][off:off + nwi[i]], d["win_end"][off:off + nwi[i]]
        assert ws[0] == 0 and we[-1] == npo[i] - 1                  # windows tile [0, n_poles)
        assert np.all(ws[1:] == we[:-1] + 1)                        # contiguously
        assert int((we - ws + 1).sum()) == npo[i]
        off += nwi[i]
    assert np.all((d["pole_l"] >= 0) & (d["pole_l"] < 4))
    assert np.all((d["pole"] >= 0) & (d["pole"] < 152.5))


def test_abrarov_branch_share(rs):
    """Share of pole evaluations with |Z| < 6 is ~0.5% (A.1 measured 0.52%)."""
    npo, nwi = rs.counts()
    d = rs.data()
    nn, mats = O.builtin_tables(355)
    poff = np.concatenate([[0], np.cumsum(npo)])
    woff = np.concatenate([[0], np.cumsum(nwi)])
    small = total = 0
    for i in range(400):
        E, mat = O.sample(i)
        for j in range(nn[mat]):
            nuc = mats[mat, j]
            w = min(int(E / (1.0 / nwi[nuc])), nwi[nuc] - 1)
            q = woff[nuc] + w
            ps = d["pole"][poff[nuc] + d["win_start"][q]: poff[nuc] + d["win_end"][q]]
            Z = (E - (ps[:, 0] + 1j * ps[:, 1])) * 0.5
            small += int((np.abs(Z) < 6).sum())
            total += len(Z)
    share = small / total
    assert 0.002 < share < 0.01, share


def test_rs_golden(rs):
    m, S = rs.macro(*O.sample(0))
    want = np.array(GOLD["RS_lookup0_macro"])
    assert np.all(np.abs(m - want) <= 1e-10 * S)
    assert rs.lookup_batch(0, 2000) == GOLD["RS_raw_0_2000"]


def test_rs_identities_and_additivity(rs):
    raw, m, S = rs.lookup_batch(0, 3000, want_macro=True)
    # sigma_E = sigma_T - sigma_A per nuclide; summed with concentrations the identity holds to rounding
    assert np.all(np.abs(m[:, 3] - (m[:, 0] - m[:, 1])) <= 1e-12 * S)
    assert 3000 <= raw <= 4 * 3000
    assert raw == rs.lookup_batch(0, 1234) + rs.lookup_batch(1234, 3000 - 1234)
    r2, m2, _ = rs.lookup_indices(np.arange(3000))
    assert r2 == raw and np.array_equal(m, m2)
    # hash robustness: top-2 gap far above the 1e-10 tolerance (A.7: >= 1.7e-3)
    s = np.sort(m, axis=1)
    assert ((s[:, -1] - s[:, -2]) / S).min() > 1e-8
