#!/bin/bash
# RS sorted kernel register-cap / unroll A/B (C5, C5D0)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/${OUT:-r02ar}; mkdir -p $O; rm -f $O/*
for v in "-DGF_RS_MINB=1" "-DGF_RS_MINB=5" "-DGF_RS_MINB=6" "-DGF_RS_MINB=5 -DGF_RS_POLE_UNROLL=1" "-DGF_RS_MINB=4 -DGF_RS_POLE_UNROLL=3"; do
  GF_EXTRA_NVCC="$v" python -c "from paper_2306_11686_b200 import build; build.build()" > $O/build.log 2>&1
  grep -A3 "rs_lookup_sorted" paper_2306_11686_b200/ptxas_report.txt | grep -E "registers|spill" >> $O/ab.txt
  for c in C5 C5D0; do
    echo "== $v $c" >> $O/ab.txt
    timeout 600 python bench.py --config $c --steps 3 --no-e2e --no-cpu-baseline --no-proxy 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['hash'] if 'hash' in d else '')" >> $O/ab.txt 2>&1
  done
done
python -c "from paper_2306_11686_b200 import build; build.build()" > $O/build_default.log 2>&1
cat $O/ab.txt
