#!/bin/bash
# per-warp band segments: tests, band proxy, launch list; C6 kernel A/B
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/${OUT:-r02ak}; mkdir -p $O; rm -f $O/*
S=$O/status.txt
python -c "from paper_2306_11686_b200 import build; build.build()" > $O/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "band or C7 or torchrun" > $O/pytest.log 2>&1; echo "pytest=$? $(tail -1 $O/pytest.log)" >> $S
timeout 900 python tools/band_proxy.py 1,8 > $O/band_proxy.txt 2>&1; echo "band=$?" >> $S
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_band8.csv python tools/band_proxy.py 8 > /dev/null 2>&1; echo "ncu_launch_band=$?" >> $S
python tools/parse_ncu_csv.py $O/launches_band8.csv > $O/launches_band8.txt 2>&1
for k in tile group thread; do
  GF_XS_KERNEL=$k timeout 600 python bench.py --config C6 --steps 3 --no-e2e --no-cpu-baseline --no-proxy > $O/bench_C6_$k.json 2> $O/bench_C6_$k.err; echo "C6_$k=$?" >> $S
done
cat $S
