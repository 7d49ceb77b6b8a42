#!/bin/bash
# A/B of compile-time variants: AB_CONFIG=C4 AB_VARIANTS="name1:-DX=1 -DY=2;name2:" bash scripts/ab.sh
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
IFS=';' read -ra VS <<< "$AB_VARIANTS"
for v in "${VS[@]}"; do
  name="${v%%:*}"; defs="${v#*:}"
  rm -f paper_2306_11686_b200/libgfxs.so
  GF_EXTRA_NVCC="$defs" python -c "from paper_2306_11686_b200 import build; build.build(force=True)" > gpurun_out/build_$name.log 2>&1
  grep -A3 "xs_lookup_group" paper_2306_11686_b200/ptxas_report.txt | grep -E "registers|spill" >> gpurun_out/build_$name.log
  for c in ${AB_CONFIG:-C4}; do
    timeout ${AB_BENCH_TIMEOUT:-120} python bench.py --config $c --steps ${AB_STEPS:-5} --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ab_${name}_$c.json 2>gpurun_out/ab_${name}_$c.err
    echo "$name $c $(python -c "import json; d=json.load(open('gpurun_out/ab_${name}_$c.json')); print(d['value'], d['stage_ms'])" 2>&1 | tail -1)"
  done
done
