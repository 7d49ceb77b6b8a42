#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/${OUT:-r02bd}; mkdir -p $O; rm -f $O/*
for v in "-DGF_PDL=0" "" "-DGF_PDL=0" ""; do
  GF_EXTRA_NVCC="$v" python -c "from paper_2306_11686_b200 import build; build.build()" > $O/build.log 2>&1
  for c in H2; do
    timeout 600 python bench.py --config $c --steps 5 --no-e2e --no-cpu-baseline --no-proxy > $O/b.json 2>/dev/null
    python -c "import json; d=json.load(open('$O/b.json')); print('[$v] $c', d['value'], d['ms_per_step'])" >> $O/ab.txt
  done
  timeout 300 python tools/ab_batch_n.py C3 tile 17000000 >> $O/ab.txt 2>&1
  timeout 300 python tools/band_proxy.py 8 >> $O/ab.txt 2>&1
done
python -c "from paper_2306_11686_b200 import build; build.build()" > $O/build.log 2>&1
cat $O/ab.txt
