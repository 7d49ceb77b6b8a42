#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/${OUT:-r02bi}; mkdir -p $O; rm -f $O/*
python -c "from paper_2306_11686_b200 import build; build.build()" > $O/build.log 2>&1
for a in "" "--no-sort"; do
  for c in C1 C2; do
    timeout 600 python bench.py --config $c --steps 10 --no-e2e --no-cpu-baseline --no-proxy $a > $O/b.json 2>/dev/null
    python -c "import json; d=json.load(open('$O/b.json')); print('$c [$a]', d['value'], d['ms_per_step'], d['hash'], d['roofline']['kernel'])" >> $O/ab.txt 2>&1
  done
done
cat $O/ab.txt
