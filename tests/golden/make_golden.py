"""Writes tests/golden/oracle_hashes.json: full-size raw sums computed by oracle/ ONLY.

The GPU parity tests compare the CUDA path against these oracle values (the oracle itself is pinned
to SURVEY.md A.8's independent golden values and to the closed-form / brute-force pins in
tests/test_oracle_*.py).  Nothing here touches the CUDA path.  Run: python tests/golden/make_golden.py
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "oracle_hashes.json")


def chunked(o, n, chunk):
    raw, first = 0, 0
    while first < n:
        k = min(chunk, n - first)
        raw += o.lookup_batch(first, k)
        first += k
    return raw


def extra():
    """Later configs (merged into the existing file): C6 XL hash grid (NEXT-2), C5D0 RS 0 K (NEXT-3),
    H2 / H3 / H5 history mode (NEXT-1) at full size."""
    res = json.load(open(OUT))
    t = time.time()
    o = O.XSOracle(355, 238847, O.HASH, bins=10000)
    raw = chunked(o, 17_000_000, 5_000_000)
    res["C6"] = {"n_iso": 355, "n_gp": 238847, "grid": O.HASH, "n": 17_000_000, "raw": raw, "hash": raw % O.HASH_MOD}
    print("C6", res["C6"], f"{time.time() - t:.1f}s", flush=True)
    del o
    rs0 = O.RSOracle(355, 1000, 100, 4, doppler=0)
    raw = chunked(rs0, 10_200_000, 1_000_000)
    res["C5D0"] = {"n_iso": 355, "doppler": 0, "n": 10_200_000, "raw": raw, "hash": raw % O.HASH_MOD}
    print("C5D0", res["C5D0"], f"{time.time() - t:.1f}s", flush=True)
    del rs0
    for name, n_iso in (("H2", 68), ("H3", 355)):
        o = O.XSOracle(n_iso, 11303, O.UNIONIZED)
        raw = o.history_batch(0, 500_000, 34)
        res[name] = {"n_iso": n_iso, "grid": O.UNIONIZED, "particles": 500_000, "L": 34, "raw": raw,
                     "hash": raw % O.HASH_MOD}
        print(name, res[name], f"{time.time() - t:.1f}s", flush=True)
        del o
    rs = O.RSOracle(355, 1000, 100, 4)
    raw = rs.history_batch(0, 300_000, 34)
    res["H5"] = {"n_iso": 355, "particles": 300_000, "L": 34, "raw": raw, "hash": raw % O.HASH_MOD}
    print("H5", res["H5"], f"{time.time() - t:.1f}s", flush=True)
    json.dump(res, open(OUT, "w"), indent=1)


def main():
    res = {"_source": "oracle/ (plain C, -O2 -ffp-contract=off) via tests/golden/make_golden.py; no CUDA code involved",
           "threads": O.max_threads()}
    t = time.time()
    cfgs = [
        ("C1", dict(n_iso=68, grid=O.NUCLIDE), 100_000),
        ("C2", dict(n_iso=68, grid=O.UNIONIZED), 17_000_000),
        ("C3", dict(n_iso=355, grid=O.UNIONIZED), 17_000_000),
        ("C4", dict(n_iso=355, grid=O.HASH), 170_000_000),
    ]
    for name, c, n in cfgs:
        o = O.XSOracle(c["n_iso"], 11303, c["grid"], bins=10000)
        raw = chunked(o, n, 5_000_000)
        res[name] = {"n_iso": c["n_iso"], "grid": c["grid"], "n": n, "raw": raw, "hash": raw % O.HASH_MOD}
        print(name, res[name], f"{time.time() - t:.1f}s", flush=True)
        del o
    rs = O.RSOracle(355, 1000, 100, 4)
    raw = chunked(rs, 10_200_000, 1_000_000)
    res["C5"] = {"n_iso": 355, "n": 10_200_000, "raw": raw, "hash": raw % O.HASH_MOD}
    print("C5", res["C5"], f"{time.time() - t:.1f}s", flush=True)
    rs68 = O.RSOracle(68, 1000, 100, 4)
    raw = chunked(rs68, 1_000_000, 1_000_000)
    res["RS_small_1M"] = {"n_iso": 68, "n": 1_000_000, "raw": raw, "hash": raw % O.HASH_MOD}
    json.dump(res, open(OUT, "w"), indent=1)
    print("wrote", OUT)


def xxl():
    """C8: XSBench XXL (355 x 501,579 gridpoints: 2.1 x XL, R-XXL in DESIGN.md), 17 M lookups on the hash grid
    (the unionized grid's energy bands give identical intervals; the GPU test sums its 16 bands)."""
    res = json.load(open(OUT))
    t = time.time()
    o = O.XSOracle(355, 501579, O.HASH, bins=10000)
    raw = chunked(o, 17_000_000, 5_000_000)
    res["C8"] = {"n_iso": 355, "n_gp": 501579, "grid": O.HASH, "n": 17_000_000, "raw": raw, "hash": raw % O.HASH_MOD}
    print("C8", res["C8"], f"{time.time() - t:.1f}s", flush=True)
    json.dump(res, open(OUT, "w"), indent=1)


if __name__ == "__main__":
    if "--xxl" in sys.argv:
        xxl()
    elif "--extra" in sys.argv:
        extra()
    else:
        main()
