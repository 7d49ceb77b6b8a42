"""Pins for the oracle's history-based mode (NEXT-1; readings
R-HIST / R-HIST-RS).  CPU only.

The particle chain is checked against an independent Python transcription that uses exact integer
LCG arithmetic, correctly rounded rationals for the doubles and the golden pick_mat thresholds
(tests/golden/survey_a8.json); only the per-step macro xs comes from the oracle's xso_macro /
rso_macro, which tests/test_oracle_xs.py and tests/test_oracle_rs.py pin on their own.  Plus the
L = 1 reduction to event-based lookups, hash bounds, additivity and thread invariance.
"""
import json
import os
from fractions import Fraction

import numpy as np
import pytest

import oracle as O

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "survey_a8.json")))
A_LCG = 2806196910506780709
M63 = 1 << 63
M64 = 1 << 64
T_GOLD = [0.0] + [float.fromhex(h) for h in GOLD["thresholds_hex_1_to_11"]]


def _step(s):
    return (A_LCG * s + 1) % M64 % M63  # u64 wraparound, then mod 2^63


def _ff(s, n):  # closed form of n steps: a^n s + (a^n - 1)/(a - 1)  (mod 2^63)
    an = pow(A_LCG, n, M63 * (A_LCG - 1))
    return (pow(A_LCG, n, M63) * s + (an - 1) // (A_LCG - 1)) % M63


def _draw(st):
    st[0] = _step(st[0])
    return float(Fraction(st[0], M63))


def _pick(roll):
    for m in range(1, 12):
        if roll < T_GOLD[m]:
            return m
    return 0


def py_xs_history(o, p, L, seed=O.STARTING_SEED):
    st = [_ff(seed, p * L * 2 * 4)]
    E = _draw(st)
    mat = _pick(_draw(st))
    raw, macros, fwd = 0, [], []
    for _ in range(L):
        m = o.macro(E, mat)
        macros.append(m)
        raw += 1 + _argmax(m, -1.0)
        nf = int(np.sum(m > 1.0))
        fwd.append(nf)
        for _ in range(nf):
            st[0] = _step(st[0])
        E = _draw(st)
        mat = _pick(_draw(st))
    return raw, np.array(macros), fwd


def _argmax(m, start):
    mx, idx = start, 0
    for c, x in enumerate(m):
        if x > mx:
            mx, idx = x, c
    return idx


def py_rs_history(o, p, L, seed=O.STARTING_SEED):
    st = [_ff(seed, p * L * 2)]
    E = _draw(st)
    mat = _pick(_draw(st))
    raw, macros = 0, []
    for _ in range(L):
        m, _S = o.macro(E, mat)
        macros.append(m)
        raw += 1 + _argmax(m, -1.7976931348623157e308)
        for x in range(4):
            st[0] = (st[0] + (1337 * p if m[x] > 0.0 else 42)) % M64
        E = _draw(st)
        mat = _pick(_draw(st))
    return raw, np.array(macros)


@pytest.fixture(scope="module")
def xs_small():
    return O.XSOracle(68, 11303, O.UNIONIZED)


def test_thresholds_golden_match_oracle():
    assert list(O.thresholds()) == T_GOLD


@pytest.mark.parametrize("particles", [[0, 1, 2, 3, 17], [499_999, 123_456, 250_000]])
def test_xs_history_chain_matches_python_transcription(xs_small, particles):
    L = 34
    fwd_all = []
    for p in particles:
        raw, m, fwd = py_xs_history(xs_small, p, L)
        raw_o, m_o = xs_small.history_batch(p, 1, L, want_macro=True)
        assert raw_o == raw
        assert np.array_equal(m_o[0], m)
        fwd_all += fwd
    # the coupling is exercised: the skip-ahead varies from step to step (mostly 5 at this size)
    assert len(set(fwd_all)) >= 2 and max(fwd_all) == 5


def test_xs_history_large_chain():
    o = O.XSOracle(355, 11303, O.HASH, bins=10000)
    for p in (7, 400_000):
        raw, m, _ = py_xs_history(o, p, 34)
        raw_o, m_o = o.history_batch(p, 1, 34, want_macro=True)
        assert raw_o == raw and np.array_equal(m_o[0], m)


@pytest.mark.parametrize("grid", [O.NUCLIDE, O.UNIONIZED, O.HASH])
def test_xs_history_L1_is_event_lookup_4p(grid):
    """L = 1: particle p starts at fast_forward(1070, 8p) = event lookup 4p's stream and does exactly
    that lookup."""
    o = O.XSOracle(68, 11303, grid)
    n = 3000
    raw, m = o.history_batch(0, n, 1, want_macro=True)
    raw_e, m_e = o.lookup_indices(4 * np.arange(n, dtype=np.uint64))
    assert raw == raw_e and np.array_equal(m[:, 0, :], m_e)


def test_xs_history_bounds_additivity_threads(xs_small):
    L, n = 34, 600
    raw = xs_small.history_batch(0, n, L, threads=1)
    assert n * L <= raw <= 5 * n * L
    assert xs_small.history_batch(0, 250, L) + xs_small.history_batch(250, n - 250, L) == raw
    assert xs_small.history_batch(0, n, L, threads=max(2, O.max_threads())) == raw
    # grid types agree (NUCLIDE == UNIONIZED == HASH): the chain sees the same macro bits
    assert O.XSOracle(68, 11303, O.NUCLIDE).history_batch(0, 200, L) == xs_small.history_batch(0, 200, L)


@pytest.fixture(scope="module")
def rs_small():
    return O.RSOracle(68)


def test_rs_history_chain_matches_python_transcription(rs_small):
    for p in (0, 1, 5, 299_999):
        raw, m = py_rs_history(rs_small, p, 34)
        raw_o, m_o, _S = rs_small.history_batch(p, 1, 34, want_macro=True)
        assert raw_o == raw and np.array_equal(m_o[0], m)


def test_rs_history_L1_is_event_batch(rs_small):
    """L = 1: particle p starts at fast_forward(1070, 2p), event lookup p's stream."""
    raw, m, S = rs_small.history_batch(0, 400, 1, want_macro=True)
    raw_e, m_e, S_e = rs_small.lookup_batch(0, 400, want_macro=True)
    assert raw == raw_e and np.array_equal(m[:, 0, :], m_e) and np.array_equal(S[:, 0], S_e)


def test_rs_history_bounds_additivity(rs_small):
    L, n = 34, 60
    raw = rs_small.history_batch(0, n, L)
    assert n * L <= raw <= 4 * n * L
    assert rs_small.history_batch(0, 25, L) + rs_small.history_batch(25, n - 25, L) == raw
