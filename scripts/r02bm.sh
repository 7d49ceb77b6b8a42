#!/bin/bash
# last-block scan prefix: tests + launch lists + bench
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/${OUT:-r02bm}; mkdir -p $O; rm -f $O/*
S=$O/status.txt
python -c "from paper_2306_11686_b200 import build; build.build()" > $O/build.log 2>&1
timeout 1700 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo "pytest=$? $(tail -1 $O/pytest.log)" >> $S
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $O/launches_C3.csv python bench.py --config C3 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-proxy > /dev/null 2>&1
python tools/parse_ncu_csv.py $O/launches_C3.csv > $O/launches_C3.txt 2>&1
timeout 600 python tools/band_proxy.py 1,8 > $O/band_proxy.txt 2>&1
timeout 600 python bench.py --config H2 --steps 5 --no-e2e --no-cpu-baseline --no-proxy > $O/h2.json 2>/dev/null
python -c "import json; d=json.load(open('$O/h2.json')); print('H2', d['value'], d['ms_per_step'])" >> $S
cat $S; grep -v "^\[" $O/launches_C3.txt | tail -7; cat $O/band_proxy.txt
