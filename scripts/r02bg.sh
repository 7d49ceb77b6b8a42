#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/${OUT:-r02bg}; mkdir -p $O; rm -f $O/*
python -c "from paper_2306_11686_b200 import build; build.build()" > $O/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q -k "rs or RS or C5 or H5 or history" > $O/pytest.log 2>&1; echo "pytest=$? $(tail -1 $O/pytest.log)" >> $O/ab.txt
for c in C5 C5D0; do
  timeout 600 python bench.py --config $c --steps 3 --no-e2e --no-cpu-baseline --no-proxy > $O/b.json 2>/dev/null
  python -c "import json; d=json.load(open('$O/b.json')); print('$c', d['value'], d['ms_per_step'], d['roofline']['frac'], d['hash'])" >> $O/ab.txt
done
cat $O/ab.txt
