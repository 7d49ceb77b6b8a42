#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/${OUT:-r02bn}; mkdir -p $O; rm -f $O/*
S=$O/status.txt
python -c "from paper_2306_11686_b200 import build; build.build()" > $O/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "C3_large or alternative_sorted or interval_edges or band or C7 or C2_small" > $O/pytest.log 2>&1; echo "pytest=$? $(tail -1 $O/pytest.log)" >> $S
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $O/launches_C3.csv python bench.py --config C3 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-proxy > /dev/null 2>&1
python tools/parse_ncu_csv.py $O/launches_C3.csv > $O/launches_C3.txt 2>&1
timeout 600 python tools/band_proxy.py 1,8 > $O/band_proxy.txt 2>&1
cat $S; grep -v "^\[" $O/launches_C3.txt | tail -7; cat $O/band_proxy.txt
