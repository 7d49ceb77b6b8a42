"""Plain CPU oracle for the XSBench / RSBench lookup -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` / ``--impl reference``
legs may import this package.  The product (``paper_2306_11686_b200``) never imports it and shares
no code with it (see the header of ``gf_oracle.c``).  This module is argument marshalling over
``libgforacle.so`` (plain C, ``-O2 -ffp-contract=off``) plus a build helper.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "gf_oracle.c")
LIB = os.path.join(HERE, "libgforacle.so")

NUCLIDE, UNIONIZED, HASH = 0, 1, 2
GRID_SEED = 42          # SURVEY.md:548 (R-SEED)
STARTING_SEED = 1070    # SURVEY.md:548 (R-SEED)
HASH_MOD = 999983       # BASELINE.json north_star


def build(force: bool = False) -> str:
    """Compile the oracle (gcc, no FMA contraction: R-FP, SURVEY.md:655)."""
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        cmd = ["gcc", "-O2", "-std=c11", "-fopenmp", "-ffp-contract=off", "-fno-fast-math",
               "-fPIC", "-shared", SRC, "-o", LIB, "-lm"]
        subprocess.check_call(cmd)
    return LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(LIB)
        u64, i32, dbl, vp = C.c_uint64, C.c_int, C.c_double, C.c_void_p
        P = C.POINTER
        L.o_lcg_step.restype = u64; L.o_lcg_step.argtypes = [u64]
        L.o_lcg_double.restype = dbl; L.o_lcg_double.argtypes = [P(u64)]
        L.o_lcg_int.restype = u64; L.o_lcg_int.argtypes = [P(u64)]
        L.o_fast_forward.restype = u64; L.o_fast_forward.argtypes = [u64, u64]
        L.o_thresholds.restype = None; L.o_thresholds.argtypes = [vp]
        L.o_pick_mat.restype = i32; L.o_pick_mat.argtypes = [dbl]
        L.o_builtin_tables.restype = i32; L.o_builtin_tables.argtypes = [i32, vp, vp]
        L.o_sample.restype = None; L.o_sample.argtypes = [u64, u64, P(dbl), P(i32)]
        L.o_grid_search.restype = C.c_long
        L.o_grid_search.argtypes = [vp, C.c_long, dbl, C.c_long, C.c_long]
        L.o_argmax5_plus1.restype = i32; L.o_argmax5_plus1.argtypes = [vp]
        L.o_argmax4_plus1.restype = i32; L.o_argmax4_plus1.argtypes = [vp]
        L.o_fast_exp.restype = dbl; L.o_fast_exp.argtypes = [dbl]
        L.o_max_threads.restype = i32; L.o_max_threads.argtypes = []
        L.xso_create.restype = vp
        L.xso_create.argtypes = [i32, C.c_long, i32, i32, u64, vp, vp, i32]
        L.xso_free.restype = None; L.xso_free.argtypes = [vp]
        L.xso_nuclide_grid.restype = vp; L.xso_nuclide_grid.argtypes = [vp]
        L.xso_unionized.restype = vp; L.xso_unionized.argtypes = [vp]
        L.xso_hash_grid.restype = vp; L.xso_hash_grid.argtypes = [vp]
        L.xso_max_num_nucs.restype = i32; L.xso_max_num_nucs.argtypes = [vp]
        L.xso_tables.restype = None; L.xso_tables.argtypes = [vp, vp, vp, vp]
        L.xso_ig_entry.restype = C.c_int32; L.xso_ig_entry.argtypes = [vp, C.c_long, i32]
        L.xso_ig_rows.restype = None; L.xso_ig_rows.argtypes = [vp, C.c_long, C.c_long, vp]
        L.xso_macro.restype = None; L.xso_macro.argtypes = [vp, dbl, i32, vp]
        L.xso_lookup_batch.restype = u64; L.xso_lookup_batch.argtypes = [vp, u64, u64, u64, vp, i32]
        L.xso_lookup_indices.restype = u64; L.xso_lookup_indices.argtypes = [vp, vp, u64, u64, vp]
        L.xso_lookup_energies.restype = u64; L.xso_lookup_energies.argtypes = [vp, vp, vp, u64, vp]
        L.rso_fast_nuclear_W.restype = None; L.rso_fast_nuclear_W.argtypes = [dbl, dbl, P(dbl), P(dbl)]
        L.rso_create.restype = vp; L.rso_create.argtypes = [i32, i32, i32, i32, u64]
        L.rso_free.restype = None; L.rso_free.argtypes = [vp]
        L.rso_total_poles.restype = C.c_long; L.rso_total_poles.argtypes = [vp]
        L.rso_total_windows.restype = C.c_long; L.rso_total_windows.argtypes = [vp]
        L.rso_counts.restype = None; L.rso_counts.argtypes = [vp, vp, vp]
        L.rso_data.restype = None; L.rso_data.argtypes = [vp] * 8
        L.rso_macro.restype = None; L.rso_macro.argtypes = [vp, dbl, i32, vp, P(dbl)]
        L.rso_lookup_batch.restype = u64; L.rso_lookup_batch.argtypes = [vp, u64, u64, u64, vp, vp, i32]
        L.rso_lookup_indices.restype = u64; L.rso_lookup_indices.argtypes = [vp, vp, u64, u64, vp, vp]
        L.rso_set_doppler.restype = None; L.rso_set_doppler.argtypes = [vp, i32]
        L.amo_nnz.restype = C.c_long; L.amo_nnz.argtypes = [i32, i32, i32]
        L.amo_matrix.restype = None; L.amo_matrix.argtypes = [i32, i32, i32, vp, vp, vp]
        L.amo_relax.restype = None; L.amo_relax.argtypes = [C.c_long, vp, vp, vp, vp, vp, vp, i32]
        L.pro_create.restype = vp; L.pro_create.argtypes = [C.c_long, i32, u64]
        L.pro_free.restype = None; L.pro_free.argtypes = [vp]
        L.pro_nnz.restype = C.c_long; L.pro_nnz.argtypes = [vp]
        L.pro_arrays.restype = None; L.pro_arrays.argtypes = [vp, vp, vp, vp]
        L.pro_propagate_csr.restype = None; L.pro_propagate_csr.argtypes = [C.c_long, vp, vp, vp, vp, vp, i32]
        L.pro_propagate.restype = None; L.pro_propagate.argtypes = [vp, vp, vp, i32]
        L.xso_history_batch.restype = u64; L.xso_history_batch.argtypes = [vp, u64, u64, i32, u64, vp, i32]
        L.rso_history_batch.restype = u64; L.rso_history_batch.argtypes = [vp, u64, u64, i32, u64, vp, vp, i32]
        _lib = L
    return _lib


def _ptr(a: np.ndarray | None):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


# ------------------------------------------------------------------ scalar helpers
def lcg_step(s: int) -> int:
    return lib().o_lcg_step(s)


def lcg_doubles(seed: int, n: int) -> list[float]:
    s = C.c_uint64(seed)
    return [lib().o_lcg_double(C.byref(s)) for _ in range(n)]


def fast_forward(seed: int, n: int) -> int:
    return lib().o_fast_forward(seed, n)


def thresholds() -> np.ndarray:
    T = np.zeros(12, dtype=np.float64)
    lib().o_thresholds(_ptr(T))
    return T


def pick_mat(roll: float) -> int:
    return lib().o_pick_mat(roll)


def sample(i: int, seed: int = STARTING_SEED) -> tuple[float, int]:
    E, m = C.c_double(), C.c_int()
    lib().o_sample(i, seed, C.byref(E), C.byref(m))
    return E.value, m.value


def grid_search(A: np.ndarray, q: float, lo: int, hi: int, stride: int = 1) -> int:
    A = np.ascontiguousarray(A, dtype=np.float64)
    return lib().o_grid_search(_ptr(A), stride, q, lo, hi)


def builtin_tables(n_iso: int):
    nn = np.zeros(12, dtype=np.int32)
    mx = lib().o_builtin_tables(n_iso, _ptr(nn), None)
    if mx < 0:
        raise ValueError("built-in tables exist for n_iso = 68 or 355 only")
    mats = np.zeros((12, mx), dtype=np.int32)
    lib().o_builtin_tables(n_iso, _ptr(nn), _ptr(mats))
    return nn, mats


def argmax5_plus1(macro) -> int:
    m = np.ascontiguousarray(macro, dtype=np.float64)
    return lib().o_argmax5_plus1(_ptr(m))


def argmax4_plus1(macro) -> int:
    m = np.ascontiguousarray(macro, dtype=np.float64)
    return lib().o_argmax4_plus1(_ptr(m))


def fast_exp(x: float) -> float:
    return lib().o_fast_exp(x)


def max_threads() -> int:
    return lib().o_max_threads()


def faddeeva_W(z: complex) -> complex:
    wr, wi = C.c_double(), C.c_double()
    lib().rso_fast_nuclear_W(z.real, z.imag, C.byref(wr), C.byref(wi))
    return complex(wr.value, wi.value)


# ------------------------------------------------------------------ XSBench oracle
class XSOracle:
    """Grids built on the host exactly as SURVEY.md Sec. 8(c) c.2 reads them."""

    def __init__(self, n_iso=68, n_gp=11303, grid_type=NUCLIDE, bins=10000, seed=GRID_SEED,
                 num_nucs=None, mats=None):
        self.n_iso, self.n_gp, self.grid_type, self.bins = n_iso, n_gp, grid_type, bins
        nn_p = mats_p = None
        mx = 0
        if num_nucs is not None:
            nn = np.ascontiguousarray(num_nucs, dtype=np.int32)
            mt = np.ascontiguousarray(mats, dtype=np.int32)
            mx = mt.shape[1]
            nn_p, mats_p = _ptr(nn), _ptr(mt)
            self._keep = (nn, mt)
        h = lib().xso_create(n_iso, n_gp, grid_type, bins, seed, nn_p, mats_p, mx)
        if not h:
            raise ValueError("xso_create rejected the parameters")
        self.h = h

    def __del__(self):
        h = getattr(self, "h", None)
        if h:
            lib().xso_free(h)
            self.h = None

    @property
    def npts(self) -> int:
        return self.n_iso * self.n_gp

    def nuclide_grid(self) -> np.ndarray:
        p = lib().xso_nuclide_grid(self.h)
        buf = (C.c_double * (self.npts * 6)).from_address(p)
        return np.ctypeslib.as_array(buf).reshape(self.n_iso, self.n_gp, 6).copy()

    def unionized(self) -> np.ndarray:
        p = lib().xso_unionized(self.h)
        if not p:
            raise ValueError("not a unionized grid")
        return np.ctypeslib.as_array((C.c_double * self.npts).from_address(p)).copy()

    def hash_grid(self) -> np.ndarray:
        p = lib().xso_hash_grid(self.h)
        if not p:
            raise ValueError("not a hash grid")
        return np.ctypeslib.as_array((C.c_int32 * (self.bins * self.n_iso)).from_address(p)).reshape(
            self.bins, self.n_iso).copy()

    def tables(self):
        mx = lib().xso_max_num_nucs(self.h)
        nn = np.zeros(12, dtype=np.int32)
        mats = np.zeros((12, mx), dtype=np.int32)
        concs = np.zeros((12, mx), dtype=np.float64)
        lib().xso_tables(self.h, _ptr(nn), _ptr(mats), _ptr(concs))
        return nn, mats, concs

    def ig_entry(self, e: int, i: int) -> int:
        return lib().xso_ig_entry(self.h, e, i)

    def ig_rows(self, e0: int, e1: int) -> np.ndarray:
        out = np.zeros((e1 - e0, self.n_iso), dtype=np.int32)
        lib().xso_ig_rows(self.h, e0, e1, _ptr(out))
        return out

    def macro(self, E: float, mat: int) -> np.ndarray:
        out = np.zeros(5, dtype=np.float64)
        lib().xso_macro(self.h, E, mat, _ptr(out))
        return out

    def lookup_batch(self, first: int, n: int, seed: int = STARTING_SEED, want_macro=False, threads=0):
        out = np.zeros((n, 5), dtype=np.float64) if want_macro else None
        raw = lib().xso_lookup_batch(self.h, first, n, seed, _ptr(out), threads)
        return (raw, out) if want_macro else raw

    def lookup_indices(self, idx, seed: int = STARTING_SEED):
        idx = np.ascontiguousarray(idx, dtype=np.uint64)
        out = np.zeros((len(idx), 5), dtype=np.float64)
        raw = lib().xso_lookup_indices(self.h, _ptr(idx), len(idx), seed, _ptr(out))
        return raw, out

    def history_batch(self, first_p: int, n_p: int, L: int = 34, seed: int = STARTING_SEED, want_macro=False,
                      threads=0):
        """History-based mode (NEXT-1, reading R-HIST): particles [first_p, first_p + n_p), L lookups each.
        Returns raw (and macro [n_p][L][5])."""
        out = np.zeros((n_p, L, 5), dtype=np.float64) if want_macro else None
        raw = lib().xso_history_batch(self.h, first_p, n_p, L, seed, _ptr(out), threads)
        return (raw, out) if want_macro else raw

    def lookup_energies(self, E, mat):
        E = np.ascontiguousarray(E, dtype=np.float64)
        mat = np.ascontiguousarray(mat, dtype=np.int32)
        out = np.zeros((len(E), 5), dtype=np.float64)
        raw = lib().xso_lookup_energies(self.h, _ptr(E), _ptr(mat), len(E), _ptr(out))
        if raw == (1 << 64) - 1:
            raise ValueError("invalid caller inputs: material ids must be 0..11 and energies finite")
        return raw, out


# ------------------------------------------------------------------ RSBench oracle
class RSOracle:
    def __init__(self, n_nuc=355, avg_poles=1000, avg_windows=100, numL=4, seed=GRID_SEED, doppler=1):
        h = lib().rso_create(n_nuc, avg_poles, avg_windows, numL, seed)
        if not h:
            raise ValueError("rso_create rejected the parameters")
        self.h, self.n_nuc, self.numL, self.doppler = h, n_nuc, numL, doppler
        lib().rso_set_doppler(h, doppler)

    def __del__(self):
        h = getattr(self, "h", None)
        if h:
            lib().rso_free(h)
            self.h = None

    def counts(self):
        npo = np.zeros(self.n_nuc, dtype=np.int32)
        nwi = np.zeros(self.n_nuc, dtype=np.int32)
        lib().rso_counts(self.h, _ptr(npo), _ptr(nwi))
        return npo, nwi

    def data(self):
        tp, tw = lib().rso_total_poles(self.h), lib().rso_total_windows(self.h)
        nn, mats = builtin_tables(self.n_nuc)
        d = dict(pole=np.zeros((tp, 8)), pole_l=np.zeros(tp, dtype=np.int32), win=np.zeros((tw, 3)),
                 win_start=np.zeros(tw, dtype=np.int32), win_end=np.zeros(tw, dtype=np.int32),
                 K0RS=np.zeros((self.n_nuc, self.numL)), concs=np.zeros((12, mats.shape[1])))
        lib().rso_data(self.h, *[_ptr(d[k]) for k in ("pole", "pole_l", "win", "win_start", "win_end",
                                                       "K0RS", "concs")])
        return d

    def macro(self, E: float, mat: int):
        out = np.zeros(4)
        S = C.c_double()
        lib().rso_macro(self.h, E, mat, _ptr(out), C.byref(S))
        return out, S.value

    def lookup_batch(self, first: int, n: int, seed: int = STARTING_SEED, want_macro=False, threads=0):
        out = np.zeros((n, 4)) if want_macro else None
        sc = np.zeros(n) if want_macro else None
        raw = lib().rso_lookup_batch(self.h, first, n, seed, _ptr(out), _ptr(sc), threads)
        return (raw, out, sc) if want_macro else raw

    def lookup_indices(self, idx, seed: int = STARTING_SEED):
        idx = np.ascontiguousarray(idx, dtype=np.uint64)
        out = np.zeros((len(idx), 4))
        sc = np.zeros(len(idx))
        raw = lib().rso_lookup_indices(self.h, _ptr(idx), len(idx), seed, _ptr(out), _ptr(sc))
        return raw, out, sc

    def history_batch(self, first_p: int, n_p: int, L: int = 34, seed: int = STARTING_SEED, want_macro=False,
                      threads=0):
        """History-based mode (NEXT-1, reading R-HIST-RS).  Returns raw (and macro [n_p][L][4], S [n_p][L])."""
        out = np.zeros((n_p, L, 4)) if want_macro else None
        sc = np.zeros((n_p, L)) if want_macro else None
        raw = lib().rso_history_batch(self.h, first_p, n_p, L, seed, _ptr(out), _ptr(sc), threads)
        return (raw, out, sc) if want_macro else raw


# ------------------------------------------------------------------ page-rank oracle (NEXT-4)
class PROracle:
    """In-edge CSR page-rank graph and propagation step (readings R-PR-GRAPH / R-PR-STEP)."""

    def __init__(self, n, D=16, seed=GRID_SEED):
        h = lib().pro_create(n, D, seed)
        if not h:
            raise ValueError("pro_create rejected the parameters")
        self.h, self.n, self.D = h, n, D
        self.nnz = lib().pro_nnz(h)

    def __del__(self):
        h = getattr(self, "h", None)
        if h:
            lib().pro_free(h)
            self.h = None

    def arrays(self):
        rowptr = np.zeros(self.n + 1, dtype=np.int64)
        col = np.zeros(max(self.nnz, 1), dtype=np.int32)
        outdeg = np.zeros(self.n, dtype=np.int32)
        lib().pro_arrays(self.h, _ptr(rowptr), _ptr(col), _ptr(outdeg))
        return rowptr, col[:self.nnz], outdeg

    def propagate(self, r, threads=0):
        r = np.ascontiguousarray(r, dtype=np.float64)
        out = np.zeros(self.n, dtype=np.float64)
        lib().pro_propagate(self.h, _ptr(r), _ptr(out), threads)
        return out


def pr_propagate_csr(rowptr, col, outdeg, r, threads=1):
    rowptr = np.ascontiguousarray(rowptr, dtype=np.int64)
    col = np.ascontiguousarray(col, dtype=np.int32)
    outdeg = np.ascontiguousarray(outdeg, dtype=np.int32)
    r = np.ascontiguousarray(r, dtype=np.float64)
    out = np.zeros(len(rowptr) - 1, dtype=np.float64)
    lib().pro_propagate_csr(len(rowptr) - 1, _ptr(rowptr), _ptr(col), _ptr(outdeg), _ptr(r), _ptr(out), threads)
    return out


# ------------------------------------------------------------------ AMGmk relax oracle (NEXT-4)
def amg_matrix(nx, ny, nz):
    """27-point Laplacian CSR (R-AMG-MAT): (rowptr int64, col int32, val float64)."""
    nnz = lib().amo_nnz(nx, ny, nz)
    n = nx * ny * nz
    rowptr = np.zeros(n + 1, dtype=np.int64)
    col = np.zeros(nnz, dtype=np.int32)
    val = np.zeros(nnz, dtype=np.float64)
    lib().amo_matrix(nx, ny, nz, _ptr(rowptr), _ptr(col), _ptr(val))
    return rowptr, col, val


def amg_relax(rowptr, col, val, f, u, threads=0):
    """One Jacobi sweep (R-AMG-RELAX)."""
    rowptr = np.ascontiguousarray(rowptr, dtype=np.int64)
    col = np.ascontiguousarray(col, dtype=np.int32)
    val = np.ascontiguousarray(val, dtype=np.float64)
    f = np.ascontiguousarray(f, dtype=np.float64)
    u = np.ascontiguousarray(u, dtype=np.float64)
    out = np.zeros(len(rowptr) - 1)
    lib().amo_relax(len(rowptr) - 1, _ptr(rowptr), _ptr(col), _ptr(val), _ptr(f), _ptr(u), _ptr(out), threads)
    return out
