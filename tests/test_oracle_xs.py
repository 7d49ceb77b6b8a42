"""Pins for the XSBench oracle.  CPU only.

Every test here checks oracle/ against something other than itself: exact integer / rational
arithmetic, brute force on tiny inputs, closed forms, invariants, a library routine, or the
survey's independently computed golden values (tests/golden/survey_a8.json).
"""
import json
import math
import os
from fractions import Fraction

import numpy as np
import pytest

import oracle as O

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "survey_a8.json")))
A_LCG = 2806196910506780709
M63 = 1 << 63


# ----------------------------------------------------------------------------- LCG (SURVEY.md:540-547)
def _py_step(s):  # exact big-integer arithmetic: (a*s + 1) mod 2^63
    return (A_LCG * s + 1) % M63


def test_lcg_step_matches_exact_integer_arithmetic():
    rng = np.random.default_rng(1)
    for s in [0, 1, 42, 1070, M63 - 1] + [int(x) for x in rng.integers(0, 2**62, 200)]:
        assert O.lcg_step(s) == _py_step(s)


def test_fast_forward_equals_stepping_brute_force():
    rng = np.random.default_rng(2)
    for seed in (42, 1070, 12345):
        for n in [0, 1, 2, 3, 5, 63, 64, 1000] + [int(x) for x in rng.integers(0, 20000, 5)]:
            s = seed
            for _ in range(n):
                s = _py_step(s)
            assert O.fast_forward(seed, n) == s


def test_fast_forward_composition_law_and_range():
    rng = np.random.default_rng(3)
    for _ in range(200):
        s = int(rng.integers(0, 2**62))
        a, b = int(rng.integers(0, 2**40)), int(rng.integers(0, 2**40))
        x = O.fast_forward(O.fast_forward(s, a), b)
        assert x == O.fast_forward(s, a + b)
        assert 0 <= x < M63
    # closed form of an affine LCG: ff(s, n) = a^n s + c (a^n - 1)/(a - 1)  (mod 2^63), via pow()
    for n in (7, 1000, 2**33 + 17):
        an = pow(A_LCG, n, M63 * (A_LCG - 1))
        geo = (an - 1) // (A_LCG - 1)  # exact: sum_{k<n} a^k
        assert O.fast_forward(42, n) == (pow(A_LCG, n, M63) * 42 + geo) % M63


def test_lcg_double_is_correctly_rounded_rational():
    s = 42
    got = O.lcg_doubles(42, 50)
    for g in got:
        s = _py_step(s)
        assert g == float(Fraction(s, M63))  # Fraction -> float rounds to nearest
        assert 0.0 <= g <= 1.0


# ----------------------------------------------------------------------------- pick_mat (R-PICK)
DIST = [Fraction(x) for x in ("0.140", "0.052", "0.275", "0.134", "0.154", "0.064", "0.066", "0.055", "0.008",
                              "0.015", "0.025", "0.013")]


def test_thresholds_match_golden_and_exact_sums():
    T = O.thresholds()
    assert T[0] == 0.0
    assert [float.hex(float(x)) for x in T[1:]] == GOLD["thresholds_hex_1_to_11"]
    for m in range(1, 12):
        exact = sum(DIST[1:m + 1])
        assert abs(Fraction(T[m]) - exact) <= m * Fraction(2) ** -52  # m roundings of <= 1/2 ulp
    assert abs(1.0 - T[11] - 0.139) < 1e-12  # fuel interval [T[11], 1)


def test_pick_mat_boundaries():
    T = O.thresholds()
    assert O.pick_mat(0.0) == 1
    for m in range(1, 12):
        below = math.nextafter(T[m], 0.0)
        assert O.pick_mat(below) == (m if m == 1 or below >= T[m - 1] else m - 1)
        at = T[m]
        assert O.pick_mat(at) == (m + 1 if m < 11 else 0)
    assert O.pick_mat(math.nextafter(1.0, 0.0)) == 0
    assert O.pick_mat(1.0) == 0


def test_material_frequencies_statistics():
    n = 200_000
    mats = np.array([O.sample(i)[1] for i in range(0, n * 7, 7)])
    p = np.array([0.139, 0.052, 0.275, 0.134, 0.154, 0.064, 0.066, 0.055, 0.008, 0.015, 0.025, 0.013])
    cnt = np.bincount(mats, minlength=12)
    sigma = np.sqrt(n * p * (1 - p))
    assert np.all(np.abs(cnt - n * p) < 5 * sigma), (cnt, n * p)


def test_sample_golden():
    for i, E, mat in GOLD["samples"]:
        assert O.sample(i) == (E, mat)
    assert O.lcg_doubles(42, 6) == GOLD["first6_lcg_doubles_seed42"]


def test_sample_is_stream_position_2i():
    # lookup i uses draws 2i+1 (E) and 2i+2 (material roll) of the stream from 1070 (SURVEY.md:573)
    for i in (0, 1, 17, 1000):
        s = 1070
        for _ in range(2 * i):
            s = _py_step(s)
        s1 = _py_step(s)
        s2 = _py_step(s1)
        E, mat = O.sample(i)
        assert E == float(Fraction(s1, M63))
        assert mat == O.pick_mat(float(Fraction(s2, M63)))


# ----------------------------------------------------------------------------- tables (SURVEY.md:552-558)
def test_builtin_tables_shapes():
    for n_iso, fuel in ((68, 34), (355, 321)):
        nn, mats = O.builtin_tables(n_iso)
        assert list(nn) == [fuel, 5, 4, 4, 27, 21, 21, 21, 21, 21, 9, 9]
        for m in range(12):
            row = mats[m, :nn[m]]
            assert len(set(row.tolist())) == nn[m]  # no duplicate nuclide within a material
            assert row.min() >= 0 and row.max() < n_iso
        if n_iso == 355:
            assert list(mats[0, 34:321]) == list(range(68, 355))
    with pytest.raises(ValueError):
        O.builtin_tables(70)


# ----------------------------------------------------------------------------- tiny custom grids
def tiny(grid_type, n_iso=5, n_gp=40, bins=16, seed=42):
    nn = np.array([3, 1, 2, 1, 1, 1, 5, 2, 1, 1, 1, 1], dtype=np.int32)
    mats = np.zeros((12, 5), dtype=np.int32)
    rows = [[0, 2, 4], [1], [3, 0], [2], [4], [0], [4, 3, 2, 1, 0], [1, 3], [0], [1], [2], [3]]
    for m, r in enumerate(rows):
        r = list(dict.fromkeys(x % n_iso for x in r))
        nn[m] = len(r)
        mats[m, :len(r)] = r
    return O.XSOracle(n_iso, n_gp, grid_type, bins=bins, seed=seed, num_nucs=nn, mats=mats)


def _stream(seed, n):
    s, out = seed, []
    for _ in range(n):
        s = _py_step(s)
        out.append(float(Fraction(s, M63)))
    return out


def test_nuclide_grid_is_sorted_permutation_of_the_stream():
    o = tiny(O.NUCLIDE)
    G = o.nuclide_grid()
    raw = np.array(_stream(42, 5 * 40 * 6)).reshape(5, 40, 6)
    for i in range(5):
        assert np.all(np.diff(G[i, :, 0]) >= 0)
        assert sorted(map(tuple, G[i])) == sorted(map(tuple, raw[i]))  # rows move whole
    # concentrations continue the same stream (R-CONC)
    nn, mats, concs = o.tables()
    rest = _stream(42, 5 * 40 * 6 + int(nn.sum()))[5 * 40 * 6:]
    flat = [concs[m, j] for m in range(12) for j in range(nn[m])]
    assert flat == rest


def test_golden_grid_and_concs():
    o = O.XSOracle(68, 11303, O.NUCLIDE)
    G = o.nuclide_grid()
    assert [float.hex(float(x)) for x in G[0, 0]] == GOLD["nuclide0_first_point_hex"]
    _, _, c = o.tables()
    assert c[0, 0] == GOLD["concs_small"]["0_0"] and c[11, 8] == GOLD["concs_small"]["11_8"]


def _brute_count(A, q):
    return int(sum(1 for a in A if a <= q))


def test_grid_search_equals_brute_force_clamped_count():
    rng = np.random.default_rng(5)
    for trial in range(40):
        n = int(rng.integers(2, 30))
        A = np.sort(np.round(rng.random(n) * 8) / 8)  # quantised: duplicates and exact hits
        lo = int(rng.integers(0, n - 1))
        hi = int(rng.integers(lo + 1, n))
        for q in list(A) + [-1.0, 2.0, 0.0, 1.0] + list(rng.random(10)):
            k = O.grid_search(A, q, lo, hi)
            sub = A[lo:hi + 1]
            want = min(max(lo + _brute_count(sub, q) - 1, lo), hi - 1)
            assert k == want, (A, q, lo, hi)


def test_unionized_and_index_grid_brute_force():
    o = tiny(O.UNIONIZED)
    G = o.nuclide_grid()
    U = o.unionized()
    assert np.all(np.diff(U) >= 0)
    assert sorted(U.tolist()) == sorted(G[:, :, 0].ravel().tolist())
    IG = o.ig_rows(0, len(U))
    n_gp = 40
    for e in range(len(U)):
        for i in range(5):
            want = min(max(_brute_count(G[i, :, 0], U[e]) - 1, 0), n_gp - 2)
            assert IG[e, i] == want


def test_index_grid_equals_xsbench_sweep_without_duplicates():
    """The recalled XSBench v20 sweep (SURVEY.md:649 R-IG) agrees with the closed form when U has no
    duplicate values (A.2).  The sweep below is written from that description, independently."""
    o = tiny(O.UNIONIZED, n_iso=4, n_gp=30)
    G = o.nuclide_grid()
    U = o.unionized()
    assert len(np.unique(U)) == len(U)
    n_iso, n_gp = 4, 30
    idx_low = [0] * n_iso
    e_high = [G[i, 1, 0] for i in range(n_iso)]
    sweep = np.zeros((len(U), n_iso), dtype=np.int64)
    for e, ue in enumerate(U):
        for i in range(n_iso):
            if ue < e_high[i]:
                sweep[e, i] = idx_low[i]
            elif idx_low[i] == n_gp - 2:
                sweep[e, i] = idx_low[i]
            else:
                idx_low[i] += 1
                sweep[e, i] = idx_low[i]
                e_high[i] = G[i, idx_low[i] + 1, 0]
    assert np.array_equal(sweep, o.ig_rows(0, len(U)))


def test_hash_grid_brute_force():
    o = tiny(O.HASH, bins=16)
    G = o.nuclide_grid()
    HG = o.hash_grid()
    du = 1.0 / 16
    for b in range(16):
        for i in range(5):
            want = min(max(_brute_count(G[i, :, 0], b * du) - 1, 0), 40 - 2)
            assert HG[b, i] == want


def _plain_interval(A, E):
    return min(max(_brute_count(A, E) - 1, 0), len(A) - 2)


def _exact_macro(G, nn, mats, concs, E, mat):
    """The plain definition (SURVEY.md:520-526) evaluated in exact rational arithmetic from the fp64
    inputs, plus the magnitude sum used by the rounding-error bound."""
    out = [Fraction(0)] * 5
    mag = [Fraction(0)] * 5
    Ef = Fraction(E)
    for j in range(nn[mat]):
        nuc = mats[mat, j]
        A = G[nuc]
        k = _plain_interval(A[:, 0], E)
        lo, hi = A[k], A[k + 1]
        f = (Fraction(hi[0]) - Ef) / (Fraction(hi[0]) - Fraction(lo[0]))
        for c in range(5):
            x = Fraction(hi[c + 1]) - f * (Fraction(hi[c + 1]) - Fraction(lo[c + 1]))
            out[c] += x * Fraction(concs[mat, j])
            mag[c] += (abs(Fraction(hi[c + 1])) + abs(f) * (abs(Fraction(hi[c + 1])) + abs(Fraction(lo[c + 1])))) \
                * abs(Fraction(concs[mat, j]))
    return out, mag


@pytest.mark.parametrize("grid_type", [O.NUCLIDE, O.UNIONIZED, O.HASH])
def test_macro_within_rounding_bound_of_exact_plain_definition(grid_type):
    o = tiny(grid_type)
    G = o.nuclide_grid()
    nn, mats, concs = o.tables()
    eps = 2.0 ** -53
    for i in range(300):
        E, mat = O.sample(i)
        got = o.macro(E, mat)
        ex, mag = _exact_macro(G, nn, mats, concs, E, mat)
        for c in range(5):
            # f carries 3 roundings, x 3 more, the product and the running sum <= nn+1 more
            bound = (8 + nn[mat]) * 4 * eps * float(mag[c]) + 1e-300
            assert abs(float(Fraction(got[c]) - ex[c])) <= bound, (i, c)


def test_interpolation_endpoint_and_betweenness():
    """1-nuclide materials: macro = RN(x * conc).  E at the last gridpoint -> f == 0 -> x == hi exactly;
    E inside an interval -> x between the endpoints (+-1 ulp); x monotone in E (A.5)."""
    o = tiny(O.NUCLIDE)
    G = o.nuclide_grid()
    nn, mats, concs = o.tables()
    for mat in (1, 3, 4, 5):  # one nuclide each
        nuc, conc = mats[mat, 0], concs[mat, 0]
        A = G[nuc]
        top = A[-1]
        got = o.macro(float(top[0]), mat)
        assert np.array_equal(got, np.float64(top[1:]) * np.float64(conc))  # numpy multiply is RN
        for k in (0, 7, 20, 38):
            lo, hi = A[k], A[k + 1]
            Es = np.linspace(lo[0], hi[0], 9)[1:-1]
            vals = np.array([o.macro(float(E), mat) for E in Es])
            for c in range(5):
                a, b = sorted((lo[c + 1] * conc, hi[c + 1] * conc))
                tol = 4 * np.spacing(max(abs(a), abs(b)))
                assert np.all(vals[:, c] >= a - tol) and np.all(vals[:, c] <= b + tol)
                d = np.diff(vals[:, c])
                assert np.all(d >= 0) or np.all(d <= 0)  # monotone
            # 1-ulp steps stay monotone too
            E0 = float((lo[0] + hi[0]) / 2)
            seq = [E0]
            for _ in range(30):
                seq.append(math.nextafter(seq[-1], 2.0))
            v = np.array([o.macro(E, mat) for E in seq])
            for c in range(5):
                d = np.diff(v[:, c])
                assert np.all(d >= 0) or np.all(d <= 0)


def test_extrapolation_below_and_above_grid():
    o = tiny(O.NUCLIDE)
    G = o.nuclide_grid()
    nn, mats, concs = o.tables()
    mat = 1
    nuc, conc = mats[mat, 0], concs[mat, 0]
    A = G[nuc]
    for E, k in ((A[0, 0] / 2, 0), (0.0, 0), (min(1.0, A[-1, 0] + (1 - A[-1, 0]) / 2), 38)):
        lo, hi = A[k], A[k + 1]
        f = (Fraction(hi[0]) - Fraction(E)) / (Fraction(hi[0]) - Fraction(lo[0]))
        want = [float((Fraction(hi[c + 1]) - f * (Fraction(hi[c + 1]) - Fraction(lo[c + 1]))) * Fraction(conc))
                for c in range(5)]
        got = o.macro(float(E), mat)
        assert np.allclose(got, want, rtol=1e-11, atol=1e-12)


@pytest.mark.parametrize("n_iso", [68])
def test_cross_grid_identity_bitwise(n_iso, xs_small_nuclide, xs_small_unionized, xs_small_hash):
    """NUCLIDE == UNIONIZED == HASH per lookup, bitwise (A.2; ties have measure zero)."""
    r0, m0 = xs_small_nuclide.lookup_batch(0, 20000, want_macro=True)
    r1, m1 = xs_small_unionized.lookup_batch(0, 20000, want_macro=True)
    r2, m2 = xs_small_hash.lookup_batch(0, 20000, want_macro=True)
    assert r0 == r1 == r2
    assert np.array_equal(m0, m1) and np.array_equal(m0, m2)


def test_hash_raw_bounds_additivity_threads(xs_small_nuclide):
    o = xs_small_nuclide
    n = 30000
    raw = o.lookup_batch(0, n)
    assert n <= raw <= 5 * n
    a = 12345
    assert raw == o.lookup_batch(0, a) + o.lookup_batch(a, n - a)
    assert raw == o.lookup_batch(0, n, threads=1)
    raw_i, _ = o.lookup_indices(np.arange(n))
    assert raw_i == raw


def test_argmax_first_strict_maximum():
    assert O.argmax5_plus1([1, 1, 1, 1, 1]) == 1
    assert O.argmax5_plus1([0, 2, 2, 1, 0]) == 2
    assert O.argmax5_plus1([-5, -4, -3, -2, -1.5]) == 1  # nothing above -1.0 -> index 0
    assert O.argmax5_plus1([-5, -4, -3, -2, -0.5]) == 5


def test_argmax_robustness_small(xs_small_nuclide):
    """min top-2 relative gap over C1 is far above the 1e-12 tolerance, so the hash is decided by
    values that agree to 1e-12 (SURVEY.md:682)."""
    _, m = xs_small_nuclide.lookup_batch(0, 100000, want_macro=True)
    s = np.sort(m, axis=1)
    gap = (s[:, -1] - s[:, -2]) / np.abs(s[:, -1])
    assert gap.min() > 1e-9


def test_golden_small(xs_small_nuclide):
    E, mat = O.sample(0)
    got = xs_small_nuclide.macro(E, mat)
    assert [float.hex(float(x)) for x in got] == GOLD["macro_small_lookup0_hex"]
    r = xs_small_nuclide.lookup_batch(0, 100000)
    assert r == GOLD["C1"]["raw"] and r % O.HASH_MOD == GOLD["C1"]["hash"]


def test_golden_large_macros():
    o = O.XSOracle(355, 11303, O.NUCLIDE)
    _, _, c = o.tables()
    assert c[0, 0] == GOLD["concs_large"]["0_0"] and c[11, 8] == GOLD["concs_large"]["11_8"]
    for i, key in ((0, "macro_large_lookup0_hex"), (2, "macro_large_lookup2_hex")):
        assert [float.hex(float(x)) for x in o.macro(*O.sample(i))] == GOLD[key]


@pytest.mark.full
def test_golden_C2_full(xs_small_unionized):
    r = xs_small_unionized.lookup_batch(0, 17_000_000)
    assert r == GOLD["C2"]["raw"] and r % O.HASH_MOD == GOLD["C2"]["hash"]


@pytest.mark.full
def test_golden_C3_full():
    o = O.XSOracle(355, 11303, O.UNIONIZED)
    raws = [o.lookup_batch(k * 4_250_000, 4_250_000) for k in range(4)]
    assert raws == GOLD["C3"]["chunk_raws_4x4250000"]
    assert sum(raws) % O.HASH_MOD == GOLD["C3"]["hash"]


@pytest.mark.full
def test_golden_C4_full():
    o = O.XSOracle(355, 11303, O.HASH, bins=10000)
    r = sum(o.lookup_batch(k * 10_625_000, 10_625_000) for k in range(16))
    assert r == GOLD["C4"]["raw"] and r % O.HASH_MOD == GOLD["C4"]["hash"]


def test_problem_sizes_closed_form():
    """The paper's stated shapes (via BASELINE.json configs): gridpoint counts and nuclide-grid bytes."""
    o = O.XSOracle(68, 11303, O.NUCLIDE)
    assert o.npts == 768_604 and o.npts * 48 == 36_892_992
    assert 355 * 11303 == 4_012_565


def test_energies_input_domain(xs_small_nuclide):
    """Caller states must be finite energies with material ids 0..11 (caller energies;
    the same rule as the product, include/gf_xs.h): anything else is rejected before any lookup runs.
    Finite energies outside [0, 1) are in the domain (the literal algorithm clamps)."""
    o = xs_small_nuclide
    E = np.array([0.1, 0.2, 0.3])
    for bad_e, bad_m in ((np.nan, 0), (np.inf, 1), (-np.inf, 2), (0.5, 12), (0.5, -1)):
        E2, m2 = E.copy(), np.array([0, 1, 2], dtype=np.int32)
        E2[1], m2[1] = bad_e, bad_m
        with pytest.raises(ValueError):
            o.lookup_energies(E2, m2)
    raw, m = o.lookup_energies(np.array([-0.5, 0.5, 1.5]), np.array([0, 11, 4], dtype=np.int32))
    assert 3 <= raw <= 15 and np.isfinite(m).all()
