#!/bin/bash
# Re-entry baseline: default bench line, band proxy split, launch list of the W=8 band shard
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/r02z; mkdir -p $O; rm -f $O/*
S=$O/status.txt
python -c "from paper_2306_11686_b200 import build; build.build()" > $O/build.log 2>&1
timeout 600 python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo "bench_default=$?" >> $S
timeout 600 python tools/band_proxy.py 1,8 > $O/band_proxy.txt 2>&1; echo "band=$?" >> $S
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_band8.csv python tools/band_proxy.py 8 > /dev/null 2>&1; echo "ncu_launch=$?" >> $S
python tools/parse_ncu_csv.py $O/launches_band8.csv > $O/launches_band8.txt 2>&1
cat $S
