#!/bin/bash
# bisect the H2 regression (3.76 -> 4.32 ms)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=$PWD/gpurun_out/r02bb; mkdir -p $O; rm -f $O/*
for c in 100f27d 2d4b08d 59c92e5; do
  (cd bisect/$c && python -c "from paper_2306_11686_b200 import build; build.build()" > $O/build_$c.log 2>&1 && \
   timeout 600 python bench.py --config H2 --steps 5 --no-e2e --no-cpu-baseline --no-proxy > $O/h2_$c.json 2>/dev/null; \
   python -c "import json; d=json.load(open('$O/h2_$c.json')); print('$c H2', d['value'], d['ms_per_step'], d.get('stage_ms'))" >> $O/ab.txt)
done
cat $O/ab.txt
