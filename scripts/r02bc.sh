#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/${OUT:-r02bc}; mkdir -p $O; rm -f $O/*
python -c "from paper_2306_11686_b200 import build; build.build()" > $O/build.log 2>&1
for c in H2 H3; do
  timeout 600 python bench.py --config $c --steps 5 --no-e2e --no-cpu-baseline --no-proxy > $O/b.json 2>/dev/null
  python -c "import json; d=json.load(open('$O/b.json')); print('$c', d['value'], d['ms_per_step'], d['hash'])" >> $O/ab.txt
done
GF_XS_KERNEL=thread timeout 600 python bench.py --config H2 --steps 5 --no-e2e --no-cpu-baseline --no-proxy > $O/b.json 2>/dev/null
python -c "import json; d=json.load(open('$O/b.json')); print('H2 forced thread', d['value'], d['ms_per_step'])" >> $O/ab.txt
cat $O/ab.txt
