"""Summarise an ncu report (one kernel) into the numbers DESIGN.md / profiles/ quote."""
import csv
import re
import subprocess
import sys

KEYS = [
    r"^gpu__time_duration\.sum$", r"^dram__bytes_read\.sum$", r"^dram__bytes_write\.sum$",
    r"^dram__throughput\.avg\.pct_of_peak_sustained_elapsed$", r"^lts__t_sector_hit_rate\.pct$",
    r"^lts__throughput\.avg\.pct_of_peak_sustained_elapsed$", r"^lts__t_sectors_srcunit_tex_op_read\.sum$",
    r"^l1tex__t_sector_hit_rate\.pct$", r"^l1tex__t_requests_pipe_lsu_mem_global_op_ld\.sum$",
    r"^l1tex__t_sectors_pipe_lsu_mem_global_op_ld\.sum$", r"^l1tex__throughput\.avg\.pct_of_peak_sustained_active$",
    r"^sm__pipe_fp64_cycles_active\.avg\.pct_of_peak_sustained_active$",
    r"^sm__inst_executed_pipe_fp64\.avg\.pct_of_peak_sustained_active$",
    r"^smsp__inst_executed\.sum$", r"^sm__warps_active\.avg\.pct_of_peak_sustained_active$",
    r"^smsp__issue_active\.avg\.pct_of_peak_sustained_active$",
    r"^launch__registers_per_thread$", r"^launch__grid_size$", r"^launch__block_size$",
    r"^smsp__average_warps_issue_stalled_.*_per_issue_active\.ratio$",
]


def main(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    for row in rows[2:]:
        name = row[hdr.index("Kernel Name")]
        print(f"== {name[:100]}")
        stalls = []
        for k, u, v in zip(hdr, units, row):
            if any(re.search(p, k) for p in KEYS):
                if "stalled" in k:
                    try:
                        stalls.append((float(v), k))
                    except ValueError:
                        pass
                else:
                    print(f"  {k:70s} {v:>18s} {u}")
        for v, k in sorted(stalls, reverse=True)[:8]:
            print(f"  stall {k.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', ''):40s} {v:8.2f}")


if __name__ == "__main__":
    main(sys.argv[1])
