#!/bin/bash
# XL / XXL band grids: tile vs group kernel
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/${OUT:-r02ax}; mkdir -p $O; rm -f $O/*
python -c "from paper_2306_11686_b200 import build; build.build()" > $O/build.log 2>&1
for c in C7 C8; do
  for k in tile group; do
    GF_XS_KERNEL=$k timeout 900 python bench.py --config $c --steps 3 --no-e2e --no-cpu-baseline > $O/bench_${c}_$k.json 2> $O/bench_${c}_$k.err
    python -c "import json; d=json.load(open('$O/bench_${c}_$k.json')); print('$c $k', d['value'], d['ms_per_step'], d['hash'])" >> $O/ab.txt 2>&1
  done
done
cat $O/ab.txt
