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


if __name__ == "__main__":
    main()
