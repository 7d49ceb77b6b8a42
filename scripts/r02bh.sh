#!/bin/bash
# history waves: forced tile / group vs auto (thread)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/${OUT:-r02bh}; mkdir -p $O; rm -f $O/*
python -c "from paper_2306_11686_b200 import build; build.build()" > $O/build.log 2>&1
for c in H2 H3; do
  for k in auto tile group tilenb; do
    if [ $k = auto ]; then unset GF_XS_KERNEL; else export GF_XS_KERNEL=$k; fi
    timeout 600 python bench.py --config $c --steps 3 --no-e2e --no-cpu-baseline --no-proxy > $O/b.json 2>/dev/null
    python -c "import json; d=json.load(open('$O/b.json')); print('$c $k', d['value'], d['ms_per_step'], d['hash'])" >> $O/ab.txt 2>&1
  done
  unset GF_XS_KERNEL
done
cat $O/ab.txt
