"""Turn ncu captures (gpurun_out/*.ncu-rep) into the committed evidence under profiles/.

    python tools/make_profile_summary.py r01 C3=gpurun_out/prof_lookup.ncu-rep C3_nosort=gpurun_out/prof_C3_direct.ncu-rep ...

Writes profiles/ncu_<round>_<key>.txt (the raw metrics we quote) and merges per-launch DRAM bytes
and durations into profiles/ncu_summary.json (read by bench.py for roofline.traffic).
"""
import csv
import json
import os
import re
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sectors_srcunit_tex_op_read.sum",
    "l1tex__t_sector_hit_rate.pct", "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum",
    "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "l1tex__throughput.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "launch__shared_mem_per_block_dynamic", "sm__inst_executed_pipe_adu.avg.pct_of_peak_sustained_active",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
]
UNIT = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "ms": 1e-3, "us": 1e-6, "ns": 1e-9, "s": 1.0}


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    return rows[0], rows[1], rows[2:]


def main(rnd, *pairs):
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    summ_path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    summ = json.load(open(summ_path)) if os.path.exists(summ_path) else {}
    for pair in pairs:
        key, rep = pair.split("=", 1)
        hdr, units, rows = raw(rep)
        row = rows[0]
        vals = dict(zip(hdr, row))
        unit = dict(zip(hdr, units))
        lines = [f"# ncu --set full capture, round {rnd}, {key}: {vals.get('Kernel Name', '')[:160]}",
                 f"# source: {os.path.basename(rep)} (gpurun_out/, not committed)"]
        stalls = []
        for k in hdr:
            if k in KEYS:
                lines.append(f"{k:70s} {vals[k]:>20s} {unit.get(k, '')}")
            m = re.match(r"smsp__average_warps_issue_stalled_(\w+)_per_issue_active\.ratio$", k)
            if m:
                try:
                    stalls.append((float(vals[k]), m.group(1)))
                except ValueError:
                    pass
        lines.append("# top warp stall reasons (per issue):")
        for v, n in sorted(stalls, reverse=True)[:8]:
            lines.append(f"stall_{n:60s} {v:10.2f}")
        open(os.path.join(ROOT, "profiles", f"ncu_{rnd}_{key}.txt"), "w").write("\n".join(lines) + "\n")

        def num(k):
            try:
                return float(vals[k]) * UNIT.get(unit.get(k, ""), 1.0)
            except (KeyError, ValueError):
                return None
        rd, wr = num("dram__bytes_read.sum"), num("dram__bytes_write.sum")
        summ[key] = {"kernel": vals.get("Kernel Name", "")[:120], "duration_s": num("gpu__time_duration.sum"),
                     "dram_bytes": (rd or 0) + (wr or 0), "dram_read_bytes": rd, "dram_write_bytes": wr,
                     "fp64_pipe_pct": num("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
                     "dram_pct": num("dram__throughput.avg.pct_of_peak_sustained_elapsed"),
                     "lts_pct": num("lts__throughput.avg.pct_of_peak_sustained_elapsed"),
                     "l2_hit_pct": num("lts__t_sector_hit_rate.pct"),
                     "l1_hit_pct": num("l1tex__t_sector_hit_rate.pct"),
                     "src": f"profiles/ncu_{rnd}_{key}.txt"}
        print(key, summ[key])
    json.dump(summ, open(summ_path, "w"), indent=1)


if __name__ == "__main__":
    main(*sys.argv[1:])
