#!/bin/bash
# one-pass look-back scan: full GPU suite, band proxy, bench, launch lists
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/${OUT:-r02ao}; mkdir -p $O; rm -f $O/*
S=$O/status.txt
python -c "from paper_2306_11686_b200 import build; build.build()" > $O/build.log 2>&1
timeout 900 python tools/band_proxy.py 1,8 > $O/band_proxy.txt 2>&1; echo "band=$?" >> $S
timeout 600 python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo "bench_default=$?" >> $S
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_C3.csv python bench.py --config C3 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-proxy > /dev/null 2>&1; echo "ncu_launch=$?" >> $S
python tools/parse_ncu_csv.py $O/launches_C3.csv > $O/launches_C3.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_band8.csv python tools/band_proxy.py 8 > /dev/null 2>&1; echo "ncu_launch_band=$?" >> $S
python tools/parse_ncu_csv.py $O/launches_band8.csv > $O/launches_band8.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo "pytest=$? $(tail -1 $O/pytest.log)" >> $S
cat $S
