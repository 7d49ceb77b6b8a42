"""Mean per-launch duration by kernel from an ncu --metrics gpu__time_duration.sum --csv launch list."""
import csv
import sys
from collections import defaultdict


def table(path):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[start]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    d = defaultdict(list)
    for r in rows[start + 1:]:
        if len(r) > vi:
            d[r[ki][:70]].append(float(r[vi].replace(",", "")))
    return d


if __name__ == "__main__":
    for k, v in table(sys.argv[1]).items():
        print(f"{len(v):4d} {sum(v) / len(v) / 1e3:10.3f} us  {k}")
