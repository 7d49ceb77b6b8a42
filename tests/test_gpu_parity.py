"""GPU parity: the CUDA path (through the C ABI) against the plain CPU oracle, element by element.

XSBench: grid arrays bit-identical; per-lookup macro xs bit-identical (0 ulp; north_star allows
1e-12 relative, R-FP makes it exact); raw hash sums equal.  RSBench: data bit-identical; macro xs
within 1e-10 * S (R-UNIQ, S = the oracle's cancellation scale); raw hash sums equal.
Run on a B200 via gpurun:  python -m pytest tests -m gpu -x -q
"""
import json
import math
import os

import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_HASHES = os.path.join(HERE, "golden", "oracle_hashes.json")


@pytest.fixture(scope="module")
def torch():
    import torch as T
    if not T.cuda.is_available():
        pytest.fail("no CUDA device: the gpu tests must run on a B200 (no CPU fallback exists)")
    return T


@pytest.fixture(scope="module")
def gf(torch):
    import paper_2306_11686_b200 as G
    from paper_2306_11686_b200 import build
    build.build()
    return G


def golden():
    return json.load(open(ORACLE_HASHES))


def tiny_tables(n_iso):
    rows = [[0, 2, 4], [1], [3, 0], [2], [4], [0], [4, 3, 2, 1, 0], [1, 3], [0], [1], [2], [3]]
    nn = np.zeros(12, dtype=np.int32)
    mats = np.zeros((12, 5), dtype=np.int32)
    for m, r in enumerate(rows):
        r = list(dict.fromkeys(x % n_iso for x in r))
        nn[m] = len(r)
        mats[m, :len(r)] = r
    return nn, mats


def make_pair(gf, n_iso, n_gp, grid_type, bins=10000, custom=False, seed=42):
    if custom:
        nn, mats = tiny_tables(n_iso)
        o = O.XSOracle(n_iso, n_gp, grid_type, bins=bins, seed=seed, num_nucs=nn, mats=mats)
        g = gf.Grid(gf.Params.xsbench(n_iso, n_gp, grid_type, bins, seed), num_nucs=nn, mats=mats)
    else:
        o = O.XSOracle(n_iso, n_gp, grid_type, bins=bins, seed=seed)
        g = gf.Grid(gf.Params.xsbench(n_iso, n_gp, grid_type, bins, seed))
    return o, g


def check_arrays(o, g, full_ig=True):
    n_iso, n_gp = o.n_iso, o.n_gp
    G = g.array("nuclide_grid")[0].cpu().numpy().reshape(n_iso, n_gp, 6)
    assert np.array_equal(G, o.nuclide_grid())
    R = g.array("recip_width")[0].cpu().numpy().reshape(n_iso, n_gp)
    w = np.diff(G[:, :, 0], axis=1)
    with np.errstate(divide="ignore"):
        assert np.array_equal(R[:, :-1], 1.0 / w)  # correctly rounded reciprocal widths
    assert g.fastdiv == bool(np.all(w >= 2.0 ** -960))
    Ed = g.array("energy")[0].cpu().numpy().reshape(n_iso, n_gp)
    assert np.array_equal(Ed, o.nuclide_grid()[:, :, 0])
    if o.grid_type != O.NUCLIDE or n_gp < 65536:  # interval records: every stored value is one RN numpy operation
        XR = g.array("intervals")[0].cpu().numpy().reshape(n_iso, n_gp, 16)
        lo, hi = G[:, :-1, :], G[:, 1:, :]
        with np.errstate(divide="ignore"):
            want = np.zeros((n_iso, n_gp, 16))
            want[:, :-1, 0] = hi[..., 0]
            want[:, :-1, 1] = hi[..., 0] - lo[..., 0]
            want[:, :-1, 2:12:2] = hi[..., 1:]
            want[:, :-1, 3:12:2] = hi[..., 1:] - lo[..., 1:]
            want[:, :-1, 12] = 1.0 / (hi[..., 0] - lo[..., 0])
            want[:, :-1, 13] = lo[..., 0]
        assert np.array_equal(XR, want)
    nn, mats, concs = o.tables()
    off = g.array("mat_offsets")[0].cpu().numpy()
    gc = g.array("concs")[0].cpu().numpy()
    gn = g.array("mat_nucs")[0].cpu().numpy()
    for m in range(12):
        assert off[m + 1] - off[m] == nn[m]
        assert np.array_equal(gn[off[m]:off[m + 1]], mats[m, :nn[m]])
        assert np.array_equal(gc[off[m]:off[m + 1]], concs[m, :nn[m]])
    T = g.array("thresholds")[0].cpu().numpy()
    assert np.array_equal(T, O.thresholds())
    if o.grid_type == O.UNIONIZED:
        U = g.array("unionized")[0].cpu().numpy()
        assert np.array_equal(U, o.unionized())
        ub = g.array("union_bins")[0].cpu().numpy().astype(np.int64)
        edges = np.arange(2 ** 20 + 1) / 2.0 ** 20
        want_ub = np.searchsorted(o.unionized(), edges, side="left")
        want_ub[-1] = len(U)
        assert np.array_equal(ub, want_ub)
        IG, pitch = g.array("index_grid")
        IG = IG.view(n_iso, pitch)
        nu = n_iso * n_gp
        if full_ig:
            want = o.ig_rows(0, nu)                          # energy-major [e][i]
            assert np.array_equal(IG[:, :nu].cpu().numpy().T, want)
        else:
            rng = np.random.default_rng(11)
            es = rng.integers(0, nu, 4000)
            ii = rng.integers(0, n_iso, 4000)
            import torch
            got = IG[torch.from_numpy(ii).to(IG.device), torch.from_numpy(es).to(IG.device)].cpu().numpy()
            want = np.array([o.ig_entry(int(e), int(i)) for e, i in zip(es, ii)])
            assert np.array_equal(got, want)
    if o.grid_type == O.HASH:
        HG, pitch = g.array("hash_grid")
        HG = HG.view(n_iso, pitch)[:, :o.bins].cpu().numpy()
        assert np.array_equal(HG.T, o.hash_grid())


def check_lookups(o, g, first, n, sort=True, seed=1070):
    raw_o, m_o = o.lookup_batch(first, n, seed=seed, want_macro=True)
    raw_g, m_g = g.lookup_batch(first, n, seed=seed, sort=sort, want_macro=True)
    m_g = m_g.cpu().numpy()
    bad = np.argwhere(m_g != m_o)
    assert bad.size == 0, f"{len(bad)} mismatching entries, first {bad[:3]}: {m_g[tuple(bad[0])]} vs {m_o[tuple(bad[0])]}"
    assert raw_g == raw_o
    return raw_g


# ------------------------------------------------------------------------------------------ tiny grids
@pytest.mark.parametrize("grid_type", [0, 1, 2])
@pytest.mark.parametrize("n_iso,n_gp,bins", [(5, 40, 16), (3, 2, 1), (1, 7, 3), (4, 1000, 300), (5, 33, 997)])
def test_tiny_grid_arrays_and_lookups(gf, grid_type, n_iso, n_gp, bins):
    o, g = make_pair(gf, n_iso, n_gp, grid_type, bins=bins, custom=True)
    check_arrays(o, g)
    for sort in (True, False):
        check_lookups(o, g, 0, 3001, sort=sort)  # several CTAs and a ragged tail
    check_lookups(o, g, 12345, 517)


def test_n_zero_and_flags(gf, torch):
    o, g = make_pair(gf, 5, 40, 1, custom=True)
    assert g.lookup_batch(0, 0) == 0
    v = torch.zeros(1, dtype=torch.int64, device="cuda")
    with pytest.raises(gf.GFError) as e:
        import ctypes as C
        sc = g._get_scratch(g.scratch_bytes(10, 0))
        gf._check(gf.lib().gf_xs_lookup_batch(g.h, 0, 10, 1070, gf.HISTORY, None, C.c_void_p(v.data_ptr()),
                                              C.c_void_p(sc.data_ptr()), sc.numel(), None))
    assert e.value.status == 4
    with pytest.raises(gf.GFError) as e:
        gf._check(gf.lib().gf_xs_lookup_batch(g.h, 0, 1 << 32, 1070, 0, None, C.c_void_p(v.data_ptr()),
                                              C.c_void_p(sc.data_ptr()), sc.numel(), None))
    assert e.value.status == 1


def test_div_rn_matches_ieee(gf, torch):
    """The lookup kernels' reciprocal division (q0 = a y, two FMA corrections, y = RN(1/b)) equals
    IEEE a / b bit for bit: random operands, binade-edge adversarial operands, and the real (a, b)
    pairs of a large grid's intervals."""
    import ctypes as C
    rng = np.random.default_rng(12)
    n = 2_000_000
    a1 = rng.uniform(-4, 4, n)
    b1 = np.ldexp(1 + rng.random(n), rng.integers(-900, 3, n))
    # b just above a power of two, a/b just below the next one (the worst case of q0 = RN(a y))
    e = rng.integers(-60, 1, n)
    b2 = np.ldexp(1 + rng.random(n) * 2.0 ** -20, e)
    x = np.ldexp(2 - rng.random(n) * 2.0 ** -20, rng.integers(-6, 2, n))
    a2 = np.clip(x * b2, -4, 4)
    o = O.XSOracle(355, 11303, O.NUCLIDE)
    G = o.nuclide_grid()[:, :, 0]
    nuc = rng.integers(0, 355, n)
    k = rng.integers(0, 11302, n)
    lo, hi = G[nuc, k], G[nuc, k + 1]
    E = lo + (hi - lo) * rng.uniform(-0.5, 1.5, n)
    b3 = hi - lo
    a3 = hi - E
    # (a = -0.0 is outside div_rn's domain -- it returns +0.0 -- and never occurs in the lookup, where
    #  a = RN(hi.E - E) and RN(x - x) = +0.0)
    a = np.concatenate([a1, a2, a3, [0.0, 4.0, -4.0, 1e-300]])
    b = np.concatenate([b1, b2, b3, [1.0, 3.0, 2.0 ** -900, 1.0 - 2.0 ** -53]])
    a[a == 0] = 0.0  # +0.0 only
    keep = b >= 2.0 ** -960
    a, b = a[keep], b[keep]
    da, db = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
    out, ref = torch.empty_like(da), torch.empty_like(da)
    gf._check(gf.lib().gf_xs_selftest_div(C.c_void_p(da.data_ptr()), C.c_void_p(db.data_ptr()),
                                          C.c_void_p(out.data_ptr()), C.c_void_p(ref.data_ptr()), len(a), None))
    out, ref = out.cpu().numpy(), ref.cpu().numpy()
    bad = np.flatnonzero(out.view(np.int64) != ref.view(np.int64))
    assert bad.size == 0, [(a[i].hex(), b[i].hex(), out[i], ref[i]) for i in bad[:5]]
    assert np.array_equal(ref, a / b)  # numpy's division is IEEE RN too


# ------------------------------------------------------------------------------------------ paper shapes
def test_C1_small_nuclide_full(gf):
    o, g = make_pair(gf, 68, 11303, O.NUCLIDE)
    check_arrays(o, g)
    raw = check_lookups(o, g, 0, 100_000)
    assert raw == golden()["C1"]["raw"] and gf.verify(raw) == golden()["C1"]["hash"]
    assert check_lookups(o, g, 0, 100_000, sort=False) == raw


def test_C2_small_unionized(gf):
    o, g = make_pair(gf, 68, 11303, O.UNIONIZED)
    check_arrays(o, g, full_ig=True)
    check_lookups(o, g, 0, 1_000_000)
    check_lookups(o, g, 16_000_000, 1_000_000, sort=False)
    raw = g.lookup_batch(0, 17_000_000)
    assert raw == golden()["C2"]["raw"] and gf.verify(raw) == golden()["C2"]["hash"]


@pytest.mark.parametrize("kernel,grid", [("thread", 1), ("group", 1), ("tile", 1), ("tilenb", 1),
                                         ("thread", 0), ("warp", 0), ("tile", 0), ("group", 2), ("tile", 2)])
def test_alternative_sorted_kernels_match(gf, kernel, grid):
    """gf_xs_debug_set_kernel forces one kernel of the sorted path for every batch size (the per-thread kernel, the 4-lookups-per-thread group kernel, the warp-tile
    kernel with index-grid or NB runs, the warp-cooperative nuclide search); each must give the
    oracle's bits.  At 200 k lookups a tile spans many intervals per nuclide, so the tile kernel's
    runs overflow kNbMax and its per-lookup search fallback runs too."""
    o = O.XSOracle(355, 11303, grid)
    g = gf.Grid(gf.Params.xsbench(355, 11303, grid))
    g.set_kernel(kernel)
    if kernel == "tile" and grid == 1:
        g.set_prep_min(1_000_000)  # the 2.125 M batch below takes the per-tile-index variant, 200 k the other
    for first, n in ((3_000_000, 200_000), (0, 2_125_000)):
        r1, m1 = o.lookup_batch(first, n, want_macro=True)
        r2, m2 = g.lookup_batch(first, n, want_macro=True)
        assert r1 == r2 and np.array_equal(m1, m2.cpu().numpy()), (first, n)


def test_small_hash_grid(gf):
    o, g = make_pair(gf, 68, 11303, O.HASH)
    check_arrays(o, g)
    check_lookups(o, g, 0, 300_000)
    check_lookups(o, g, 5_000_000, 100_000, sort=False)


def sampled_indices(n, k, seed):
    rng = np.random.default_rng(seed)
    idx = np.unique(np.concatenate([rng.integers(0, n, k), [0, 1, n - 2, n - 1], np.arange(0, n, n // 997)]))
    return idx


def check_sampled_full_size(gf, torch, o, g, n, seed=7):
    """At full size, in the bench launch configuration (sorted, one batch of n): per-lookup outputs at
    sampled indices equal the oracle's, which computes them one by one."""
    raw_g, m_g = g.lookup_batch(0, n, want_macro=True)
    idx = sampled_indices(n, 3000, seed)
    raw_o, m_o = o.lookup_indices(idx)
    got = m_g[torch.from_numpy(idx).to(m_g.device)].cpu().numpy()
    assert np.array_equal(got, m_o)
    assert raw_g == g.lookup_batch(0, n)  # the output path does not change the hash
    return raw_g


def test_C3_large_unionized_full_size(gf, torch):
    o, g = make_pair(gf, 355, 11303, O.UNIONIZED)
    check_arrays(o, g, full_ig=False)
    raw = check_sampled_full_size(gf, torch, o, g, 17_000_000)
    gold = golden()["C3"]
    assert raw == gold["raw"] and gf.verify(raw) == gold["hash"]
    check_lookups(o, g, 0, 200_000)
    check_lookups(o, g, 9_876_543, 50_000, sort=False)
    # shard additivity: 8 virtual shards (the multi-GPU partition) sum to the full raw
    tot = 0
    for r in range(8):
        lo, cnt = gf.shard_range(17_000_000, r, 8)
        tot += g.lookup_batch(lo, cnt)
    assert tot == raw


def test_C4_large_hash_170M(gf, torch):
    o, g = make_pair(gf, 355, 11303, O.HASH)
    check_arrays(o, g)
    check_lookups(o, g, 0, 100_000)
    raw = 0
    for r in range(8):  # the 8-GPU shards, each one batch (21.25 M)
        lo, cnt = gf.shard_range(170_000_000, r, 8)
        raw += g.lookup_batch(lo, cnt)
    gold = golden()["C4"]
    assert raw == gold["raw"] and gf.verify(raw) == gold["hash"]
    idx = sampled_indices(170_000_000, 2000, 5)
    lo, cnt = gf.shard_range(170_000_000, 7, 8)
    raw7, m7 = g.lookup_batch(lo, cnt, want_macro=True)
    sel = idx[(idx >= lo) & (idx < lo + cnt)]
    _, m_o = o.lookup_indices(sel)
    assert np.array_equal(m7[torch.from_numpy(sel - lo).to(m7.device)].cpu().numpy(), m_o)


# ------------------------------------------------------------------------------------------ energies API
def edge_energies(o, n_rand, seed):
    """Seeded synthetic particle states plus the method's degenerate energies: 0, 1, exact gridpoints
    of several nuclides, their 1-ulp neighbours, the unionized grid ends and hash-bin edges."""
    rng = np.random.default_rng(seed)
    G = o.nuclide_grid()
    Es = [0.0, 1.0, math.nextafter(1.0, 0), 5e-324, 0.5]
    for nuc in (0, 1, o.n_iso - 1):
        for k in (0, 1, o.n_gp // 2, o.n_gp - 2, o.n_gp - 1):
            e = float(G[nuc, k, 0])
            Es += [e, math.nextafter(e, 0), math.nextafter(e, 2)]
    for b in (1, 2, 77, 9999):
        e = b * (1.0 / 10000)
        Es += [e, math.nextafter(e, 0), math.nextafter(e, 2)]
    Es = np.array(Es + list(rng.random(n_rand)))
    mats = np.concatenate([np.arange(len(Es) - n_rand) % 12, rng.integers(0, 12, n_rand)]).astype(np.uint8)
    return Es, mats


@pytest.mark.parametrize("grid_type", [0, 1, 2])
def test_energies_api_device_and_host(gf, torch, grid_type):
    o, g = make_pair(gf, 68, 11303, grid_type)
    E, mats = edge_energies(o, 5000, 3)
    raw_o, m_o = o.lookup_energies(E, mats.astype(np.int32))
    for sort in (True, False):
        raw_g, m_g = g.lookup_energies(torch.from_numpy(E).cuda(), torch.from_numpy(mats).cuda(), sort=sort)
        assert raw_g == raw_o and np.array_equal(m_g.cpu().numpy(), m_o)
    Eh = torch.from_numpy(E).pin_memory()
    mh = torch.from_numpy(mats).pin_memory()
    raw_h, m_h = g.lookup_energies(Eh, mh)
    assert raw_h == raw_o and np.array_equal(m_h.numpy(), m_o)


def test_energies_async_stream(gf, torch):
    """gf_xs_lookup_energies_async: back-to-back batches from pinned host memory on two streams (one scratch
    each) add the oracle's raw sum to the device accumulators; invalid inputs set bit 63; a short scratch
    is refused."""
    o, g = make_pair(gf, 68, 11303, O.UNIONIZED)
    rng = np.random.default_rng(5)
    n = 300_000
    E = rng.random(n)
    mat = rng.integers(0, 12, n).astype(np.uint8)
    raw_o, _ = o.lookup_energies(E, mat.astype(np.int32))
    Eh, mh = torch.from_numpy(E).pin_memory(), torch.from_numpy(mat).pin_memory()
    need = g.scratch_bytes(n, gf.SORT_LOCALITY | gf.HOST_IO, whole=True)
    scr = [torch.empty(need, dtype=torch.uint8, device="cuda") for _ in range(2)]
    sts = [torch.cuda.Stream(), torch.cuda.Stream()]
    dv = torch.zeros(2, dtype=torch.int64, device="cuda")
    for k in range(4):
        with torch.cuda.stream(sts[k % 2]):
            g.lookup_energies_async(Eh, mh, dv[k % 2:k % 2 + 1], scr[k % 2], stream=sts[k % 2])
    torch.cuda.synchronize()
    assert dv.tolist() == [2 * raw_o, 2 * raw_o]
    mh[7] = 12
    d1 = torch.zeros(1, dtype=torch.int64, device="cuda")
    g.lookup_energies_async(Eh, mh, d1, scr[0])
    torch.cuda.synchronize()
    assert int(d1.item()) < 0  # bit 63: the invalid-input flag
    with pytest.raises(gf.GFError):
        g.lookup_energies_async(Eh, mh, d1, scr[0][:1024])


@pytest.mark.parametrize("grid_type", [1, 2])
def test_sorted_groups_at_interval_edges(gf, torch, grid_type):
    """Sorted lookups share record pairs and (hash grid) the interval shortcut R-SHORT, which takes
    lookup 0's interval for a group-mate strictly inside it.  Clusters of one material around exact
    gridpoints, hash-bin edges and repeated energies put ties, 1-ulp neighbours and interval
    crossings inside the same groups of 4; every macro xs must still equal the oracle's bitwise."""
    o, g = make_pair(gf, 68, 11303, grid_type)
    rng = np.random.default_rng(77)
    G = o.nuclide_grid()
    Es = []
    for nuc in (0, 2, 5, 41, 60, 67):
        for k in list(rng.integers(0, o.n_gp - 1, 6)) + [0, o.n_gp - 2, o.n_gp - 1]:
            e = float(G[nuc, k, 0])
            Es += [e, e, math.nextafter(e, 0), math.nextafter(e, 2), e, math.nextafter(e, 2)]
            Es += list(e + (rng.random(10) - 0.5) * 2e-4)
    for b in list(rng.integers(1, 10000, 20)) + [1, 9999]:
        e = b * (1.0 / 10000)
        Es += [e, math.nextafter(e, 0), math.nextafter(e, 2), e, math.nextafter(math.nextafter(e, 0), 0)]
    for b in list(rng.integers(1, 2 ** 17, 30)) + [1, 2 ** 17 - 1]:  # bin-summary bin edges
        e = float(b) * 2.0 ** -17
        Es += [e, math.nextafter(e, 0), math.nextafter(e, 2), e, math.nextafter(math.nextafter(e, 2), 2)]
    for nuc in (3, 33):  # gridpoints and neighbours within 2^-32 of the bin position (ambiguous q)
        for k in rng.integers(0, o.n_gp - 1, 10):
            e = float(G[nuc, k, 0])
            Es += [e + d * 2.0 ** -40 for d in (-3, -1, 0, 1, 3)]
    Es += list(0.3 + rng.random(20000) * 1e-3)  # dense: about 20 lookups per interval per nuclide
    E = np.clip(np.array(Es), 0.0, 1.0)
    for kern, prep in (("auto", 0), ("tile", 0), ("tile", 1 << 23), ("group", 0)):  # R-TILE runs see the clusters
        g.set_kernel(kern)
        if grid_type == 1:
            g.set_prep_min(prep)  # 0: per-tile union indices and the bisection fallback even for this small batch
        for mat in (0, 4, 7):
            mats = np.full(len(E), mat, dtype=np.uint8)
            raw_o, m_o = o.lookup_energies(E, mats.astype(np.int32))
            raw_g, m_g = g.lookup_energies(torch.from_numpy(E).cuda(), torch.from_numpy(mats).cuda(), sort=True)
            assert raw_g == raw_o, (kern, mat)
            assert np.array_equal(m_g.cpu().numpy(), m_o), f"{kern} mat {mat}"


def test_nuclide_warp_search_edges(gf, torch):
    """The nuclide-grid sorted kernels: the warp-cooperative search (once per warp, 32-ary over the
    warp's [Emin, Emax], then a shuffle search per lane) and the NB-bracket kernel (auto).  Exact
    gridpoints and their 1-ulp neighbours inside one warp, dense clusters (narrow warps), a sparse
    spread (wide warps that end in the per-lane fallback), the grid ends, energies outside [0, 1],
    -0.0 and subnormals must all give the oracle's bits."""
    o, g = make_pair(gf, 68, 11303, O.NUCLIDE)
    rng = np.random.default_rng(5)
    G = o.nuclide_grid()
    Es = []
    for nuc in (0, 2, 41, 67):
        for k in list(rng.integers(0, o.n_gp - 1, 8)) + [0, 1, o.n_gp - 2, o.n_gp - 1]:
            e = float(G[nuc, k, 0])
            Es += [e, math.nextafter(e, -1), math.nextafter(e, 2), e] + list(e + (rng.random(12) - 0.5) * 1e-6)
    Es += list(0.25 + rng.random(3000) * 1e-4)            # narrow warps
    Es += list(rng.random(40))                             # wide warps
    Es += [0.0, 1.0, -0.5, 3.0, 1e300, -1e300, 5e-324, -0.0]
    E = np.array(Es)
    for kern, mat in [("warp", 0), ("warp", 4), ("warp", 7), ("auto", 0), ("auto", 7)]:  # auto: NB brackets
        g.set_kernel(kern)
        mats = np.full(len(E), mat, dtype=np.uint8)
        raw_o, m_o = o.lookup_energies(E, mats.astype(np.int32))
        raw_g, m_g = g.lookup_energies(torch.from_numpy(E).cuda(), torch.from_numpy(mats).cuda(), sort=True)
        assert raw_g == raw_o and np.array_equal(m_g.cpu().numpy(), m_o), (kern, mat)


@pytest.mark.parametrize("bench,grid_type", [("xs", 0), ("xs", 1), ("xs", 2), ("rs", None)])
def test_invalid_caller_inputs(gf, torch, bench, grid_type):
    """Caller states outside the input domain (material id > 11, NaN, +-inf) are errors on both sides:
    the oracle rejects the batch, the device path sets the invalid-input bit of the raw sum (the
    binding raises GF_E_INVAL; gf_xs_verify rejects the raw), the host-I/O path returns GF_E_INVAL.
    Valid batches around them are unaffected."""
    g = gf.Grid(gf.Params.xsbench(68, 11303, grid_type) if bench == "xs" else gf.Params.rsbench(68))
    rng = np.random.default_rng(3)
    E = rng.random(5000)
    mats = rng.integers(0, 12, 5000).astype(np.uint8)
    ok = g.lookup_energies(torch.from_numpy(E).cuda(), torch.from_numpy(mats).cuda(), want_macro=False)
    for bad_e, bad_m in ((math.nan, 0), (math.inf, 0), (-math.inf, 3), (0.5, 12), (0.5, 255)):
        E2, m2 = E.copy(), mats.copy()
        E2[1234], m2[1234] = bad_e, bad_m
        if bench == "xs":
            with pytest.raises(ValueError):
                O.XSOracle(68, 11303, grid_type).lookup_energies(E2, m2.astype(np.int32))
        for sort in (True, False):
            with pytest.raises(gf.GFError) as e:
                g.lookup_energies(torch.from_numpy(E2).cuda(), torch.from_numpy(m2).cuda(), sort=sort, want_macro=False)
            assert e.value.status == 1
        with pytest.raises(gf.GFError) as e:
            g.lookup_energies(torch.from_numpy(E2).pin_memory(), torch.from_numpy(m2).pin_memory(), want_macro=False)
        assert e.value.status == 1
    assert g.lookup_energies(torch.from_numpy(E).cuda(), torch.from_numpy(mats).cuda(), want_macro=False) == ok
    with pytest.raises(gf.GFError):
        gf.verify(ok | (1 << 63))


def test_host_io_pipeline_chunks(gf, torch):
    """GF_HOST_IO pipelines chunks of 2^22 lookups over two slots and three streams; with several
    chunks and a ragged last one the outputs equal the device-resident call's, and the oracle's.
    Without per-lookup outputs the call runs the whole-batch mode (chunk copies overlap the sort's
    counting pass; one sort and one lookup pass): its raw sum equals the oracle's over the batch."""
    o, g = make_pair(gf, 68, 11303, O.UNIONIZED)
    rng = np.random.default_rng(21)
    n = 2 * (1 << 22) + 12345
    E = rng.random(n)
    mats = rng.integers(0, 12, n).astype(np.uint8)
    raw_d, m_d = g.lookup_energies(torch.from_numpy(E).cuda(), torch.from_numpy(mats).cuda())
    raw_h, m_h = g.lookup_energies(torch.from_numpy(E).pin_memory(), torch.from_numpy(mats).pin_memory())
    assert raw_h == raw_d
    assert np.array_equal(m_h.numpy(), m_d.cpu().numpy())
    sel = np.unique(np.concatenate([rng.integers(0, n, 3000), [0, (1 << 22) - 1, 1 << 22, n - 1]]))
    _, m_o = o.lookup_energies(E[sel], mats[sel].astype(np.int32))
    assert np.array_equal(m_h.numpy()[sel], m_o)
    raw_w = g.lookup_energies(torch.from_numpy(E).pin_memory(), torch.from_numpy(mats).pin_memory(), want_macro=False)
    raw_o, _ = o.lookup_energies(E, mats.astype(np.int32))
    assert raw_w == raw_d == raw_o


# ------------------------------------------------------------------------------------------ RSBench
def rs_pair(gf, n_nuc=355):
    o = O.RSOracle(n_nuc, 1000, 100, 4)
    g = gf.Grid(gf.Params.rsbench(n_nuc))
    return o, g


def check_rs_data(o, g):
    d = o.data()
    npo, nwi = o.counts()
    poff = g.array("rs_pole_off")[0].cpu().numpy()
    woff = g.array("rs_win_off")[0].cpu().numpy()
    assert np.array_equal(np.diff(poff), npo) and np.array_equal(np.diff(woff), nwi)
    assert np.array_equal(g.array("rs_poles")[0].cpu().numpy().reshape(-1, 8), d["pole"])
    assert np.array_equal(g.array("rs_pole_l")[0].cpu().numpy(), d["pole_l"])
    W = g.array("rs_windows")[0].cpu().numpy().reshape(-1, 4)
    assert np.array_equal(W[:, :3], d["win"])
    se = W[:, 3].copy().view(np.int32).reshape(-1, 2)
    assert np.array_equal(se[:, 0], d["win_start"]) and np.array_equal(se[:, 1], d["win_end"])
    assert np.array_equal(g.array("rs_K0RS")[0].cpu().numpy().reshape(-1, 4), d["K0RS"])
    nn, mats = O.builtin_tables(o.n_nuc)
    gc = g.array("concs")[0].cpu().numpy()
    off = g.array("mat_offsets")[0].cpu().numpy()
    for m in range(12):
        assert np.array_equal(gc[off[m]:off[m + 1]], d["concs"][m, :nn[m]])


def check_rs_lookups(o, g, first, n, sort=True):
    raw_o, m_o, S = o.lookup_batch(first, n, want_macro=True)
    raw_g, m_g = g.lookup_batch(first, n, sort=sort, want_macro=True)
    err = np.abs(m_g.cpu().numpy() - m_o) / S[:, None]
    assert err.max() <= 1e-10, err.max()
    assert raw_g == raw_o
    return err.max()


def test_rs_large_data_and_lookups(gf, torch):
    o, g = rs_pair(gf, 355)
    check_rs_data(o, g)
    check_rs_lookups(o, g, 0, 20_000)
    check_rs_lookups(o, g, 123_457, 5_001, sort=False)
    raw_g, m_g = g.lookup_batch(0, 10_200_000, want_macro=True)
    gold = golden()["C5"]
    assert raw_g == gold["raw"] and gf.verify(raw_g) == gold["hash"]
    idx = sampled_indices(10_200_000, 1500, 9)
    _, m_o, S = o.lookup_indices(idx)
    got = m_g[torch.from_numpy(idx).to(m_g.device)].cpu().numpy()
    assert (np.abs(got - m_o) / S[:, None]).max() <= 1e-10


def test_rs_small(gf):
    o, g = rs_pair(gf, 68)
    check_rs_data(o, g)
    check_rs_lookups(o, g, 0, 50_000)
    assert g.lookup_batch(0, 1_000_000) == golden()["RS_small_1M"]["raw"]


def test_rs_energies_api(gf, torch):
    o, g = rs_pair(gf, 355)
    rng = np.random.default_rng(4)
    E = np.concatenate([[0.0, 1.0, 0.5, 1e-300, math.nextafter(1.0, 0)], rng.random(3000)])
    mats = rng.integers(0, 12, len(E)).astype(np.uint8)
    raw_g, m_g = g.lookup_energies(torch.from_numpy(E).cuda(), torch.from_numpy(mats).cuda())
    m_g = m_g.cpu().numpy()
    raw_o = 0
    for t in range(len(E)):
        m, S = o.macro(float(E[t]), int(mats[t]))
        assert np.all(np.abs(m_g[t] - m) <= 1e-10 * max(S, 1e-300)), t
        raw_o += O.argmax4_plus1(m)
    assert raw_g == raw_o
    # host I/O: the chunked pipeline (with per-lookup outputs) and the whole-batch mode (raw only)
    Eh, mh = torch.from_numpy(E).pin_memory(), torch.from_numpy(mats).pin_memory()
    raw_h, m_h = g.lookup_energies(Eh, mh)
    assert raw_h == raw_o and np.array_equal(m_h.numpy(), m_g)
    assert g.lookup_energies(Eh, mh, want_macro=False) == raw_o


@pytest.mark.parametrize("n_iso", [68, 355])
def test_rs_zero_kelvin(gf, torch, n_iso):
    """NEXT-3: the 0 K pole kernel (doppler = 0, R-RS0): data identical to the Doppler grid's, macro xs
    within 1e-10 S of the oracle (R-UNIQ), raw sums equal, event (sorted / unsorted) and history."""
    o = O.RSOracle(n_iso, doppler=0)
    g = gf.Grid(gf.Params.rsbench(n_iso, doppler=0))
    n = 20_000 if n_iso == 355 else 50_000
    raw_o, m_o, S = o.lookup_batch(3_000_000, n, want_macro=True)
    for sort in (True, False):
        raw_g, m_g = g.lookup_batch(3_000_000, n, sort=sort, want_macro=True)
        assert raw_g == raw_o
        assert (np.abs(m_g.cpu().numpy() - m_o) / S[:, None]).max() <= 1e-10
    raw_h, m_h, S_h = o.history_batch(11, 200, 34, want_macro=True)
    for mode in ("direct", "sorted"):
        r, m = g.history_batch(11, 200, 34, mode=mode, want_macro=True)
        assert r == raw_h
        assert (np.abs(m.cpu().numpy() - m_h) / S_h[..., None]).max() <= 1e-10


@pytest.mark.parametrize("grid_type", [0, 1, 2])
def test_large_custom_tables_need_big_smem(gf, grid_type):
    """3,600 table entries: the SMEM-staged tables exceed the 48 KB default (opt-in path); history too."""
    rng = np.random.default_rng(3)
    n_iso = 355
    nn = np.full(12, 300, dtype=np.int32)
    mats = np.stack([rng.permutation(n_iso)[:300] for _ in range(12)]).astype(np.int32)
    o = O.XSOracle(n_iso, 200, grid_type, bins=97, num_nucs=nn, mats=mats)
    g = gf.Grid(gf.Params.xsbench(n_iso, 200, grid_type, 97), num_nucs=nn, mats=mats)
    for sort in (True, False):
        check_lookups(o, g, 777, 20_000, sort=sort)
    raw_o, m_o = o.history_batch(5, 300, 6, want_macro=True)
    for mode in ("direct", "sorted"):
        raw_g, m_g = g.history_batch(5, 300, 6, mode=mode, want_macro=True)
        assert raw_g == raw_o and np.array_equal(m_g.cpu().numpy(), m_o)


def test_integer_material_thresholds(gf, torch):
    """The samplers decide the material on the integer LCG state: roll = RN(s) 2^-63 < T[m] iff
    s < S[m].  S[m] (stored after T in the thresholds block) must be the least s with
    float(s) 2^-63 >= T[m] (Python's int -> float conversion rounds to nearest)."""
    o, g = make_pair(gf, 68, 40, O.UNIONIZED, custom=True)
    t, _ = g.array("thresholds")
    off = t.data_ptr() - g.buf.data_ptr()
    raw = g.buf[off:off + 24 * 8].cpu().numpy()
    T = raw[:96].view(np.float64)
    S = raw[96:].view(np.uint64)
    assert np.array_equal(T, O.thresholds())
    for m in range(1, 12):
        s = int(S[m])
        assert float(s) * 2.0 ** -63 >= T[m] and float(s - 1) * 2.0 ** -63 < T[m], m


@pytest.mark.parametrize("grid_type,n_iso,n_gp", [(0, 5, 40000), (1, 4, 40000), (2, 5, 40000), (2, 3, 70000),
                                                   (0, 3, 70000)])
def test_large_gridpoint_grids(gf, torch, grid_type, n_iso, n_gp):
    """NEXT-2 point counts: grids above the one-CTA SMEM sort (chunked sort + segment merges) and, above
    65,536 points, u32 hash-grid entries.  Arrays and lookups bit-identical to the oracle."""
    o, g = make_pair(gf, n_iso, n_gp, grid_type, bins=997, custom=True)
    check_arrays(o, g)
    for sort in (True, False):
        check_lookups(o, g, 0, 30_001, sort=sort)


@pytest.mark.parametrize("grid_type", [0, 2])
def test_xl_gridpoints(gf, torch, grid_type):
    """XSBench XL point count (238,847 per nuclide) with the 68-nuclide
    tables: energy column and hash grid identical to the oracle's, 200 k lookups bit-exact."""
    o, g = make_pair(gf, 68, 238847, grid_type)
    Ed = g.array("energy")[0].cpu().numpy().reshape(68, 238847)
    assert np.array_equal(Ed, o.nuclide_grid()[:, :, 0])
    if grid_type == O.HASH:
        HG, pitch = g.array("hash_grid")
        HG = HG.cpu().numpy().reshape(68, pitch)[:, :10000]
        assert np.array_equal(HG.T, o.hash_grid())
    raw = check_lookups(o, g, 5_000_000, 200_000)
    assert check_lookups(o, g, 5_000_000, 200_000, sort=False) == raw


def band_of(E, W):
    r = np.floor(np.asarray(E) * W).astype(np.int64)
    return np.clip(r, 0, W - 1)


def check_bands(gf, torch, o, mk_grid, W, first, n):
    """Run every band replica over the same lookups: each keeps the lookups of its band (rows of the
    others stay NaN), the raw sums add up to the oracle's, every row equals the oracle's bitwise."""
    raw_o, m_o = o.lookup_batch(first, n, want_macro=True)
    E = np.array([O.sample(first + i)[0] for i in range(n)])
    bands = band_of(E, W)
    raw_sum = 0
    for r in range(W):
        g = mk_grid(r)
        vs = torch.zeros(1, dtype=torch.int64, device="cuda")
        m = torch.full((n, 5), float("nan"), dtype=torch.float64, device="cuda")
        g.lookup_batch_async(first, n, vs, macro_out=m)
        raw_sum += int(vs.item())
        m = m.cpu().numpy()
        mine = bands == r
        assert np.array_equal(m[mine], m_o[mine]), r
        assert np.isnan(m[~mine]).all(), r
        with pytest.raises(gf.GFError):  # unsorted / energies / history calls are refused on band grids
            g.lookup_batch(0, 10, sort=False)
        del g
        torch.cuda.empty_cache()
    assert raw_sum == raw_o


@pytest.mark.parametrize("W", [2, 3, 5])
def test_energy_bands_small(gf, torch, W):
    """NEXT-2 energy-band sharding of the unionized grid (tiny custom grid, several bands)."""
    nn, mats = tiny_tables(5)
    o = O.XSOracle(5, 4000, O.UNIONIZED, num_nucs=nn, mats=mats)
    check_bands(gf, torch, o, lambda r: gf.Grid(gf.Params.xsbench(5, 4000, gf.UNIONIZED, n_bands=W, band=r),
                                                 num_nucs=nn, mats=mats), W, 777, 30_001)


def test_energy_bands_unionized_beyond_u16(gf, torch):
    """100,000 points per nuclide: the whole unionized index grid would need u32 intervals; four bands
    of ~25 k points each keep u16 and reproduce the oracle (its nuclide grid: identical results)."""
    o = O.XSOracle(68, 100_000, O.NUCLIDE)
    assert gf.lib  # the whole-grid unionized request is refused:
    with pytest.raises(gf.GFError):
        gf.Grid(gf.Params.xsbench(68, 100_000, gf.UNIONIZED))
    check_bands(gf, torch, o, lambda r: gf.Grid(gf.Params.xsbench(68, 100_000, gf.UNIONIZED, n_bands=4, band=r)),
                4, 1_000_000, 100_000)


def test_full_size_golden_C6_C5D0(gf, torch):
    """Whole-batch raw sums against the oracle's full-size values (tests/golden/make_golden.py --extra):
    C6 XSBench XL hash grid, 17 M lookups (NEXT-2); C5D0 RSBench 0 K, 10.2 M lookups (NEXT-3)."""
    gold = golden()
    g = gf.Grid(gf.Params.xsbench(355, 238847, gf.HASH))
    assert g.lookup_batch(0, 17_000_000) == gold["C6"]["raw"]
    del g
    torch.cuda.empty_cache()
    r = gf.Grid(gf.Params.rsbench(355, doppler=0))
    assert r.lookup_batch(0, 10_200_000) == gold["C5D0"]["raw"]


def test_C7_bands_sum_to_xl(gf, torch):
    """C7: the eight energy-band replicas of the XL unionized grid together reproduce the XL batch's raw
    sum (the oracle's C6 value: the hash and unionized grids give identical intervals), and one band's
    per-lookup outputs equal the oracle's nuclide-grid results bitwise."""
    gold = golden()
    n, W, raw = 17_000_000, 8, 0
    for b in range(W):
        g = gf.Grid(gf.Params.xsbench(355, 238847, gf.UNIONIZED, n_bands=W, band=b))
        raw += g.lookup_batch(0, n)
        if b == 3:
            o = O.XSOracle(355, 238847, O.NUCLIDE)
            check_bands_one(gf, torch, o, g, W, b, 2_000_000, 50_000)
            del o
        del g
        torch.cuda.empty_cache()
    assert raw == gold["C6"]["raw"]


@pytest.mark.parametrize("W,b", [(8, 0), (8, 5), (8, 7), (3, 2)])
def test_band_tile_path_per_lookup(gf, torch, W, b):
    """A C3 band replica through the warp-tile kernel with the per-tile union indices the sort's scatter
    writes (sort-bin edges, TixSpec) and the compacted in-band list of the band sort: every in-band row
    equals the oracle's bitwise (its nuclide grid gives identical intervals), the others stay untouched."""
    o = O.XSOracle(355, 11303, O.NUCLIDE)
    g = gf.Grid(gf.Params.xsbench(355, 11303, gf.UNIONIZED, n_bands=W, band=b))
    g.set_kernel("tile")
    g.set_prep_min(0)
    check_bands_one(gf, torch, o, g, W, b, 5_000_000, 400_000)


def test_C8_xxl_bands_sum(gf, torch):
    """NEXT-2 XXL (R-XXL: 355 x 501,579 gridpoints, 2.1 x XL): the 16 energy-band replicas of the unionized
    grid (16 so that a band's index grid stays below 65,536 points per nuclide) together reproduce the
    oracle's XXL raw sum (tests/golden/make_golden.py --xxl, on its hash grid: identical intervals)."""
    gold = golden()
    n, W, raw = 17_000_000, 16, 0
    for b in range(W):
        g = gf.Grid(gf.Params.xsbench(355, 501579, gf.UNIONIZED, n_bands=W, band=b))
        raw += g.lookup_batch(0, n)
        del g
        torch.cuda.empty_cache()
    assert raw == gold["C8"]["raw"]


def check_bands_one(gf, torch, o, g, W, b, first, n):
    raw_o, m_o = o.lookup_batch(first, n, want_macro=True)
    E = np.array([O.sample(first + i)[0] for i in range(n)])
    mine = band_of(E, W) == b
    vs = torch.zeros(1, dtype=torch.int64, device="cuda")
    m = torch.full((n, 5), float("nan"), dtype=torch.float64, device="cuda")
    g.lookup_batch_async(first, n, vs, macro_out=m)
    m = m.cpu().numpy()
    assert mine.sum() > 0 and np.array_equal(m[mine], m_o[mine]) and np.isnan(m[~mine]).all()


def test_argmax_robustness_report(gf, torch):
    """SURVEY.md 8(c) c.4 'argmax robustness': the smallest top-2 relative gap of the macro xs over the
    first 2 M lookups of C3 (XS, compared bitwise anyway) and over 500 k of C5 (RS, whose macro xs are
    only 1e-10 S-close to the oracle's, so the hash needs the gap above that) -- printed and bounded."""
    g = gf.Grid(gf.Params.xsbench(355, 11303, gf.UNIONIZED))
    _, m = g.lookup_batch(0, 2_000_000, want_macro=True)
    s = torch.sort(m, dim=1).values
    gap_xs = ((s[:, -1] - s[:, -2]) / s[:, -1].abs()).min().item()
    del g, m, s
    torch.cuda.empty_cache()
    r = gf.Grid(gf.Params.rsbench(355))
    _, m = r.lookup_batch(0, 500_000, want_macro=True)
    s = torch.sort(m, dim=1).values
    gap_rs = ((s[:, -1] - s[:, -2]) / s[:, -1].abs()).min().item()
    print(f"min top-2 relative gap: XS C3 2M {gap_xs:.3e}, RS C5 500k {gap_rs:.3e}")
    assert gap_xs > 1e-12 and gap_rs > 1e-8


@pytest.mark.parametrize("n_iso,grid_type", [(68, 1), (355, 1), (355, 0)])
def test_nuclide_bin_search_sparse_batches(gf, torch, n_iso, grid_type):
    """Sparse batches on a unionized grid (below the group kernel's 4 M threshold) search the
    per-nuclide bin tables NB (#{E_nuc <= b 2^-14}) instead of the index grid.  The table is checked
    against a plain count over the device's energy column, and the lookups -- at NB bin edges, their
    ulp neighbours, exact gridpoints and outside [0, 1), where the kernel falls back to the index
    grid -- against the oracle, with the NB search on and off."""
    o, g = make_pair(gf, n_iso, 11303, grid_type)  # (355: the fuel's 321 nuclides take the 3-stage NB ring;
    #                                                   nuclide grids use NB for every sorted batch)
    nbt, pitch = g.array("nuclide_bins")
    nb = nbt.cpu().numpy().astype(np.int64).reshape(n_iso, pitch)
    Ed = g.array("energy")[0].cpu().numpy().reshape(n_iso, 11303)
    edges = np.ldexp(np.arange(2 ** 14 + 1, dtype=np.float64), -14)
    for nuc in (0, 1, 33, n_iso - 1):
        assert np.array_equal(nb[nuc, :2 ** 14 + 1], np.searchsorted(Ed[nuc], edges, side="right"))
    rng = np.random.default_rng(14)
    E, mats = edge_energies(o, 4000, 5)
    extra = [-0.25, -5e-324, 1.0, 1.5, math.nextafter(1.0, 2)]
    for b in list(rng.integers(1, 2 ** 14, 40)) + [1, 2 ** 14 - 1]:
        e = float(b) * 2.0 ** -14
        extra += [e, math.nextafter(e, 0), math.nextafter(e, 2)]
    G = o.nuclide_grid()
    for nuc in (2, 40):
        for k in rng.integers(0, o.n_gp - 1, 20):
            e = float(G[nuc, k, 0])
            extra += [e, math.nextafter(e, 0), math.nextafter(e, 2)]
    E = np.concatenate([E, np.array(extra)])
    mats = np.concatenate([mats, rng.integers(0, 12, len(extra)).astype(np.uint8)])
    raw_o, m_o = o.lookup_energies(E, mats.astype(np.int32))
    for flag in ("1", "0"):
        g.set_kernel("auto", nb=flag == "1")
        raw_g, m_g = g.lookup_energies(torch.from_numpy(E).cuda(), torch.from_numpy(mats).cuda(), sort=True)
        assert raw_g == raw_o and np.array_equal(m_g.cpu().numpy(), m_o), flag


@pytest.mark.parametrize("config,split,hash_", [("C3", "index", 113528), ("C3", "band", 113528),
                                                ("C5", "index", 662460)])
def test_torchrun_two_ranks_strong_split(gf, config, split, hash_):
    """The product's N > 1 path end to end: bench.py under torchrun with 2 ranks (gloo, both on this one
    GPU: GF_DIST_BACKEND), strong split of the config's lookups (index ranges on a
    replicated grid, or energy bands: rank r builds band r of the unionized grid and keeps the batch's
    lookups in it), one int64 all-reduce of the raw sums per step -- the all-reduced hash must be the full
    batch's golden hash (the band run also runs its end-to-end leg)."""
    import subprocess
    import sys
    env = dict(os.environ, GF_DIST_BACKEND="gloo", PYTHONPATH=os.path.dirname(HERE))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29611", os.path.join(os.path.dirname(HERE), "bench.py"),
           "--gpus", "2", "--config", config, "--steps", "3", "--warmup", "3", "--no-cpu-baseline", "--split", split]
    if split == "index":
        cmd.append("--no-e2e")
    res = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=900)
    assert res.returncode == 0, res.stderr[-3000:]
    line = json.loads([ln for ln in res.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["scaling"] == "strong" and line["config"]["lookups_per_rank"] * 2 in (
        line["config"]["n_lookups"], line["config"]["n_lookups"] + 1)
    assert line["hash"] == hash_ and line["config"]["split"] == split
    if split == "band":
        assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["value"] > 0


@pytest.mark.parametrize("grid_type", [0, 1, 2])
def test_ieee_division_path_matches(gf, torch, grid_type):
    """The FAST = false instantiations of every sorted kernel (tile, group, thread, NB, warp search) and of
    the unsorted kernel: forced IEEE __ddiv_rn division (the path a grid with a zero-width interval
    takes; LCG grids never have one) must give the oracle's bits, like the exact reciprocal scheme."""
    o, g = make_pair(gf, 355 if grid_type else 68, 11303, grid_type)
    assert g.fastdiv
    g.set_ieee_division(True)
    kernels = ["auto", "thread", "warp"] if grid_type == 0 else ["tile", "group", "thread"]
    for kern in kernels:
        g.set_kernel(kern)
        check_lookups(o, g, 1_000_000, 150_000)
    check_lookups(o, g, 0, 50_000, sort=False)
    g.set_ieee_division(False)
    g.set_kernel("auto")
