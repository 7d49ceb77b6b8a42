"""Host-side checks of the C ABI (no GPU): the library loads, exports every symbol include/gf_xs.h
declares, validates arguments, sizes buffers by closed form, and fails loudly without a device."""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

import paper_2306_11686_b200 as gf
from paper_2306_11686_b200 import build as gfbuild

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "gf_xs.h")


@pytest.fixture(scope="module", autouse=True)
def built():
    gfbuild.build()


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(gf_xs_\w+)\s*\(", src)))


def test_exports_every_declared_symbol():
    names = declared_functions()
    assert len(names) >= 10
    L = gf.lib()
    for n in names:
        assert hasattr(L, n), n
    out = subprocess.run(["nm", "-D", "--defined-only", gfbuild.LIB], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (gf_xs_\w+)", out))
    assert set(names) <= exported


def test_built_for_sm100a_only():
    out = subprocess.run(["cuobjdump", "--list-elf", gfbuild.LIB], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out)


def test_no_fma_contraction_in_xs_lookup_sass():
    """R-FP: in every XS lookup kernel the 5 interpolation products and 5 accumulation products stay
    separate DMULs and the subtractions / additions separate DADDs (a contracted a*b+c would turn a
    DMUL+DADD pair into one DFMA).  DFMA remains only inside the IEEE division sequence."""
    out = subprocess.run(["cuobjdump", "-sass", gfbuild.LIB], capture_output=True, text=True).stdout
    funcs = re.split(r"\n\s+Function : ", out)
    checked = 0
    for f in funcs:
        name = f.split("\n", 1)[0]
        if "xs_lookup" in name:
            body = f.split("\n", 1)[1]
            assert len(re.findall(r"\bDMUL\b", body)) >= 10, name
            assert len(re.findall(r"\bDADD\b", body)) >= 17, name
            checked += 1
    assert checked >= 6


def test_verify_rejects_invalid_input_flag():
    """Bit 63 of a raw sum is the device-side invalid-input flag of gf_xs_lookup_energies (include/gf_xs.h):
    gf_xs_verify returns GF_E_INVAL for it; a valid raw sum (< 2^63) is untouched."""
    import ctypes as C
    h = C.c_uint64(7)
    assert gf.lib().gf_xs_verify((1 << 63) | 51112661, (1 << 64) - 1, C.byref(h)) == 1
    assert h.value == 7  # not written
    assert "invalid-input" in gf.lib().gf_xs_last_error().decode()
    with pytest.raises(gf.GFError) as e:
        gf.verify((1 << 63) | 5)
    assert e.value.status == 1
    assert gf.verify((1 << 63) - 1) == ((1 << 63) - 1) % 999983


def test_version_and_verify():
    assert b"sm_100a" in gf.lib().gf_xs_version()
    assert gf.verify(51112661) == 113528
    assert gf.verify(51112661, 113528) == 113528
    with pytest.raises(gf.GFError) as e:
        gf.verify(51112661, 1)
    assert e.value.status == 5


def test_default_params():
    p = gf.Params.xsbench()
    assert (p.abi_version, p.n_isotopes, p.n_gridpoints, p.grid_type, p.hash_bins, p.init_seed) == (
        1, 355, 11303, gf.UNIONIZED, 10000, 42)
    r = gf.Params.rsbench()
    assert (r.bench, r.avg_n_poles, r.avg_n_windows, r.numL, r.doppler) == (gf.RSBENCH, 1000, 100, 4, 1)


def _bytes(p):
    gb, sb = C.c_size_t(), C.c_size_t()
    st = gf.lib().gf_xs_grid_bytes(C.byref(p), C.byref(gb), C.byref(sb))
    return st, gb.value, sb.value


def test_grid_bytes_closed_form():
    """Byte sizes of the paper's shapes (BASELINE.json configs) follow from the layout."""
    al = lambda x: (x + 255) // 256 * 256
    for n_iso, gt in ((68, gf.NUCLIDE), (68, gf.UNIONIZED), (355, gf.UNIONIZED), (355, gf.HASH)):
        p = gf.Params.xsbench(n_iso, 11303, gt)
        st, gb, sb = _bytes(p)
        assert st == 0
        npts = n_iso * 11303
        total = (34 if n_iso == 68 else 321) + 5 + 4 + 4 + 27 + 5 * 21 + 2 * 9
        want = al(npts * 48) + al(npts * 8) + al(npts * 8) + al(16)  # G, Ed, reciprocal widths, flags
        if gt == gf.UNIONIZED:
            pitch = (npts + 63) // 64 * 64
            want += al(npts * 8) + al(n_iso * pitch * 2) + al((2 ** 20 + 1) * 4)
            want += al(n_iso * ((2 ** 14 + 1 + 63) // 64 * 64) * 2)  # per-nuclide bin counts (sparse batches)
        want += al(npts * 128 + 256)  # interval records of the sorted kernels (+ 2 records of tile-slot overrun)
        if gt == gf.NUCLIDE:
            want += al(n_iso * ((2 ** 14 + 1 + 63) // 64 * 64) * 2)  # per-nuclide bin counts
        if gt == gf.HASH:
            want += al(n_iso * 10048 * 2)
        # thresholds T, S + the samplers' material-bucket table (4 KB) and offset maps (4 KB); material tables
        want += al(256 + 4096 + 4096) + al(64) + al(total * 4) + al(total * 8)
        assert gb == want, (n_iso, gt)
    # C3: the 355 x 4,012,565 u16 index grid (2.85 GB) dominates the 3.67 GB total (incl. 11.6 MB of per-nuclide bin counts)
    st, gb, _ = _bytes(gf.Params.xsbench(355, 11303, gf.UNIONIZED))
    assert 3.66e9 < gb < 3.67e9


@pytest.mark.parametrize("field,value,status", [
    ("abi_version", 2, 1), ("n_isotopes", 0, 1), ("n_gridpoints", 1, 1), ("n_gridpoints", 70000, 4), ("n_gridpoints", 2 ** 20 + 1, 4),
    ("grid_type", 3, 1), ("n_isotopes", 70, 1)])
def test_invalid_params(field, value, status):
    p = gf.Params.xsbench()
    setattr(p, field, value)
    st, _, _ = _bytes(p)
    assert st == status
    assert gf.lib().gf_xs_last_error()


def test_invalid_rs_params():
    p = gf.Params.rsbench()
    p.numL = 3
    assert _bytes(p)[0] == 1
    p = gf.Params.rsbench(doppler=0)  # the 0 K kernel (NEXT-3) is built
    assert _bytes(p)[0] == 0
    p.doppler = 2
    assert _bytes(p)[0] == 1


def test_custom_tables_validation():
    p = gf.Params.xsbench(5, 40, gf.NUCLIDE)
    nn = np.array([1] * 12, dtype=np.int32)
    mats = np.array([[7]] * 12, dtype=np.int32)  # nuclide 7 does not exist
    p.num_nucs, p.mats, p.max_num_nucs = nn.ctypes.data, mats.ctypes.data, 1
    assert _bytes(p)[0] == 1
    mats[:] = 3
    assert _bytes(p)[0] == 0


def test_grid_init_without_device_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    p = gf.Params.xsbench(68, 11303, gf.NUCLIDE)
    buf = (C.c_ubyte * 512)()
    h = C.c_void_p()
    st = gf.lib().gf_xs_grid_init(C.byref(p), 0, C.addressof(buf) // 256 * 256 + 256, 1 << 40, None, 0, None,
                                  C.byref(h))
    assert st != 0 and not h.value


def test_lookup_argument_checks():
    # NULL grid
    assert gf.lib().gf_xs_lookup_batch(None, 0, 10, 1070, 0, None, None, None, 0, None) == 1
    h = C.c_uint64()
    assert gf.lib().gf_xs_verify(5, (1 << 64) - 1, None) == 1


def test_shard_range_exact_cover():
    """Rank shards cover [0, N) exactly once, contiguously (cf. SPEC.md:425-433 partition checks)."""
    for n in (0, 1, 7, 100, 17_000_000, 170_000_000):
        for w in (1, 2, 3, 4, 8):
            seen, nxt = 0, 0
            for r in range(w):
                lo, cnt = gf.shard_range(n, r, w)
                assert lo == nxt and cnt >= 0
                nxt = lo + cnt
                seen += cnt
            assert seen == n and nxt == n


def test_history_argument_checks():
    """gf_xs_history_batch validates synchronously, before any CUDA call (no GPU here)."""
    L = gf.lib()
    assert L.gf_xs_history_batch(None, 0, 10, 34, 1070, 0, None, None, None, 0, None) == 1
    b = C.c_size_t()
    assert L.gf_xs_history_bytes(None, 10, 0, C.byref(b)) == 1


def test_large_gridpoint_counts_accepted():
    """NEXT-2: XL point counts (238,847 per nuclide) are accepted for the hash and nuclide grids, with
    u32 hash-grid entries; the unionized grid stays limited to 65,536 (u16 index grid)."""
    for gt in (gf.NUCLIDE, gf.HASH):
        st, gb, sb = _bytes(gf.Params.xsbench(355, 238847, gt))
        assert st == 0
        assert sb >= 355 * 238847 * 24  # chunked grid sort scratch
    st, gb, _ = _bytes(gf.Params.xsbench(355, 238847, gf.HASH))
    npts = 355 * 238847
    assert gb > npts * (48 + 8 + 8 + 128) + 355 * 10048 * 4
    assert _bytes(gf.Params.xsbench(68, 65536, gf.UNIONIZED))[0] == 0


def test_energy_band_params():
    """NEXT-2: unionized grids shard by energy band; the XL unionized grid needs >= 4 bands (u16 index
    grid per band) and its band layout is ~1/W of the whole index grid."""
    assert _bytes(gf.Params.xsbench(355, 238847, gf.UNIONIZED))[0] == 4
    assert _bytes(gf.Params.xsbench(355, 238847, gf.UNIONIZED, n_bands=2, band=0))[0] == 4
    st, gb8, _ = _bytes(gf.Params.xsbench(355, 238847, gf.UNIONIZED, n_bands=8, band=3))
    assert st == 0
    ig8 = 355 * (355 * 238847 / 8) * 2
    assert ig8 < gb8 < ig8 * 1.1 + 355 * 238847 * (48 + 8 + 8 + 128) + 64e6
    assert _bytes(gf.Params.xsbench(68, 11303, gf.HASH, n_bands=2, band=0))[0] == 1
    assert _bytes(gf.Params.xsbench(68, 11303, gf.UNIONIZED, n_bands=2, band=2))[0] == 1
    assert _bytes(gf.Params.xsbench(68, 11303, gf.UNIONIZED, n_bands=4, band=1))[0] == 0


def test_pagerank_abi_exports_and_checks():
    """include/gf_pr.h (NEXT-4): every declared function is exported; argument checks run before any
    CUDA call."""
    import os as _os
    src = open(_os.path.join(_os.path.dirname(HEADER), "gf_pr.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = sorted(set(re.findall(r"\b(gf_pr_\w+)\s*\(", src)))
    assert len(names) == 6
    out = subprocess.run(["nm", "-D", "--defined-only", gfbuild.LIB], capture_output=True, text=True).stdout
    assert set(names) <= set(re.findall(r"\bT (gf_pr_\w+)", out))
    L = gf.lib()
    gb, sb = C.c_size_t(), C.c_size_t()
    assert L.gf_pr_graph_bytes(1 << 24, 16, C.byref(gb), C.byref(sb)) == 0
    assert gb.value >= (1 << 24) * 31 * 4
    assert L.gf_pr_graph_bytes(0, 16, C.byref(gb), C.byref(sb)) == 1
    assert L.gf_pr_graph_bytes(100, 33, C.byref(gb), C.byref(sb)) == 1
    assert L.gf_pr_propagate(None, None, None, None, None) == 1
    assert L.gf_pr_last_error()


def test_amg_abi_exports_and_checks():
    """include/gf_amg.h (NEXT-4): exports, the closed-form nonzero count, argument checks."""
    import os as _os
    src = open(_os.path.join(_os.path.dirname(HEADER), "gf_amg.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = sorted(set(re.findall(r"\b(gf_amg_\w+)\s*\(", src)))
    assert len(names) == 6
    out = subprocess.run(["nm", "-D", "--defined-only", gfbuild.LIB], capture_output=True, text=True).stdout
    assert set(names) <= set(re.findall(r"\bT (gf_amg_\w+)", out))
    import oracle as O
    L = gf.lib()
    b, nnz = C.c_size_t(), C.c_int64()
    for dims in ((5, 4, 3), (1, 1, 1), (1, 7, 2), (64, 64, 64)):
        assert L.gf_amg_matrix_bytes(*dims, C.byref(b), C.byref(nnz)) == 0
        if dims[0] * dims[1] * dims[2] < 10000:
            assert nnz.value == len(O.amg_matrix(*dims)[1])
    assert nnz.value == 64 ** 3 * 27 - 6 * 64 * 64 * 9 + 12 * 64 * 3 - 8  # inclusion-exclusion, 27-point stencil
    assert L.gf_amg_matrix_bytes(0, 4, 4, C.byref(b), C.byref(nnz)) == 1
    assert L.gf_amg_relax(None, None, None, None, None) == 1
    assert L.gf_amg_last_error()
