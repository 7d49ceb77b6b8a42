#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/${OUT:-r02as}; mkdir -p $O; rm -f $O/*
python -c "from paper_2306_11686_b200 import build; build.build()" > $O/build.log 2>&1
grep -A3 "rs_lookup_sorted" paper_2306_11686_b200/ptxas_report.txt | grep -E "registers|spill" >> $O/ab.txt
for c in C5 C3; do
  timeout 600 python bench.py --config $c --steps 3 --no-e2e --no-cpu-baseline --no-proxy > $O/bench_$c.json 2> $O/bench_$c.err
  python -c "import json; d=json.load(open('$O/bench_$c.json')); print('$c', d['value'], d['ms_per_step'], d['roofline']['frac'], d.get('clocks'), d.get('stage_ms'))" >> $O/ab.txt 2>&1
done
GF_SCATTER_SLICES=1 timeout 600 python bench.py --config C5 --steps 3 --no-e2e --no-cpu-baseline --no-proxy > $O/bench_C5_s1.json 2>&1
python -c "import json; d=json.load(open('$O/bench_C5_s1.json')); print('C5 s1', d['value'], d['ms_per_step'], d.get('stage_ms'))" >> $O/ab.txt 2>&1
cat $O/ab.txt
