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


def reasons(rep, top=10):
    """Per-instruction stall-reason breakdown of the hottest SASS lines."""
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h = rows[1]
    wi, si, ai = h.index("Warp Stall Sampling (All Samples)"), h.index("Source"), h.index("Address")
    cols = [i for i, x in enumerate(h) if x.startswith("stall_") and "Not Issued" not in x]
    data = []
    for r in rows[2:]:
        try:
            data.append((int(r[wi] or 0), r))
        except (ValueError, IndexError):
            pass
    for w, r in sorted(data, key=lambda x: -x[0])[:int(top)]:
        br = sorted(((int(r[i] or 0), h[i]) for i in cols), reverse=True)[:3]
        print(f"{w:8d} {r[ai][-5:]} {r[si][:60]:60s} " + " ".join(f"{n[6:]}={v}" for v, n in br))
