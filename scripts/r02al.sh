#!/bin/bash
# scatter slices A/B (full C3), launch list with 2 slices, C6 auto kernel
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/${OUT:-r02al}; mkdir -p $O; rm -f $O/*
S=$O/status.txt
python -c "from paper_2306_11686_b200 import build; build.build()" > $O/build.log 2>&1
for k in 1 2 3 4 1 2; do
  echo "== GF_SCATTER_SLICES=$k" >> $O/ab.txt
  GF_SCATTER_SLICES=$k timeout 300 python tools/ab_batch_n.py C3 tile 17000000 >> $O/ab.txt 2>&1
done
echo "ab=$?" >> $S
GF_SCATTER_SLICES=2 timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/launches_C3_s2.csv python bench.py --config C3 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-proxy > /dev/null 2>&1; echo "ncu_launch=$?" >> $S
python tools/parse_ncu_csv.py $O/launches_C3_s2.csv > $O/launches_C3_s2.txt 2>&1
timeout 600 python bench.py --config C6 --steps 3 --no-e2e --no-cpu-baseline --no-proxy > $O/bench_C6.json 2> $O/bench_C6.err; echo "C6=$?" >> $S
cat $S
