"""Top SASS lines of an ncu report by warp-stall samples (needs --import-source / -lineinfo)."""
import csv
import subprocess
import sys


def main(rep, top=30):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h = rows[1]
    ai, si = h.index("Address"), h.index("Source")
    wi, ei = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
    data = []
    for r in rows[2:]:
        try:
            data.append((int(r[wi] or 0), int(r[ei] or 0), r[ai][-5:], r[si]))
        except (ValueError, IndexError):
            pass
    tot = sum(d[0] for d in data) or 1
    print("samples", tot, "instructions", sum(d[1] for d in data))
    for d in sorted(data, reverse=True)[:int(top)]:
        print(f"{d[0]:8d} {100 * d[0] / tot:5.1f}% {d[1]:11d} {d[2]} {d[3][:100]}")


if __name__ == "__main__":
    main(*sys.argv[1:])
