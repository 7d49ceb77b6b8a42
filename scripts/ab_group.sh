#!/bin/bash
# A/B of the group kernel's lookups-per-thread (built on the box with extra nvcc defines).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for cfg in "4 3" "2 4" "2 5" "8 2" "4 2"; do
  set -- $cfg
  rm -f paper_2306_11686_b200/libgfxs.so
  GF_EXTRA_NVCC="-DGF_GROUP_L=$1 -DGF_GROUP_MINB=$2" python -c "from paper_2306_11686_b200 import build; build.build(force=True)" > gpurun_out/build_L$1.log 2>&1
  grep -A3 "xs_lookup_group" paper_2306_11686_b200/ptxas_report.txt | grep -E "registers|spill" >> gpurun_out/build_L$1.log
  timeout 600 python bench.py --config C3 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ab_L$1_B$2.json 2>&1
  echo "L=$1 B=$2 $(python -c "import json; d=json.load(open('gpurun_out/ab_L$1_B$2.json')); print(d['value'], d['stage_ms'])" 2>&1 | tail -1)"
done
