#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/${OUT:-r02bf}; mkdir -p $O; rm -f $O/*
python -c "from paper_2306_11686_b200 import build; build.build()" > $O/build.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:rs_lookup_sorted -s 2 -c 1 -o $O/rs python bench.py --config C5 --steps 1 --warmup 2 --no-cpu-baseline --no-e2e --no-proxy > /dev/null 2>&1; echo "ncu=$?" >> $O/status.txt
ncu -i $O/rs.ncu-rep --page source --csv --print-source sass > $O/rs_sass.csv 2>/dev/null
ncu -i $O/rs.ncu-rep --page source --csv --print-source cuda > $O/rs_cuda.csv 2>/dev/null
cat $O/status.txt
