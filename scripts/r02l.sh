#!/bin/bash
# Round-2 evidence (late): full GPU tests, smoke, bench lines for every config, launch lists, ncu captures.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/${OUT:-r02l}; mkdir -p $O; rm -f $O/*
S=$O/status.txt
python -c "from paper_2306_11686_b200 import build; build.build()" > $O/build.log 2>&1
timeout 1700 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest=$? $(tail -1 $O/pytest_gpu.log)" >> $S
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke=$?" >> $S
timeout 600 python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo "bench_default=$?" >> $S
for c in ${CONFIGS:-C1 C2 C4 C5 C5D0 C3N C6 C7 C8 H2 H3 P1 A1}; do
  timeout 900 python bench.py --config $c --steps 5 --no-e2e --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err; echo "bench_$c=$?" >> $S
done
timeout 300 python bench.py --impl reference --config C3 --steps 2 --warmup 1 > $O/bench_reference_C3.json 2> $O/bench_reference_C3.err; echo "reference=$?" >> $S
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $O/launches_C3.csv python bench.py --config C3 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-proxy > /dev/null 2>&1; echo "ncu_launch=$?" >> $S
python tools/parse_ncu_csv.py $O/launches_C3.csv > $O/launches_C3.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_band8.csv python tools/band_proxy.py 8 > /dev/null 2>&1; echo "ncu_launch_band=$?" >> $S
python tools/parse_ncu_csv.py $O/launches_band8.csv > $O/launches_band8.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:xs_lookup_tile -s 3 -c 1 -o $O/prof_C3 python bench.py --config C3 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-proxy > /dev/null 2>&1; echo "ncu_C3=$?" >> $S
timeout 600 ncu --set full --clock-control none -k regex:xs_lookup_tile -s 3 -c 1 -o $O/prof_C4 python bench.py --config C4 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-proxy > /dev/null 2>&1; echo "ncu_C4=$?" >> $S
timeout 600 ncu --set full --clock-control none -k regex:xs_lookup_tile -s 2 -c 1 -o $O/prof_band8 python tools/band_proxy.py 8 > /dev/null 2>&1; echo "ncu_band8=$?" >> $S
for k in sort_count sort_scatter; do
  timeout 300 ncu --set full --clock-control none -k regex:"^$k\$" -s 1 -c 1 -o $O/prof_C3_$k python bench.py --config C3 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-proxy > /dev/null 2>&1; echo "ncu_C3_$k=$?" >> $S
done
for k in sort_count_band sort_scatter_band; do
  timeout 300 ncu --set full --clock-control none -k regex:$k -s 2 -c 1 -o $O/prof_band8_$k python tools/band_proxy.py 8 > /dev/null 2>&1; echo "ncu_band8_$k=$?" >> $S
done
timeout 600 ncu --set full --clock-control none -k regex:rs_lookup_sorted -s 3 -c 1 -o $O/prof_C5 python bench.py --config C5 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-proxy > /dev/null 2>&1; echo "ncu_C5=$?" >> $S
for f in $O/prof_*.ncu-rep; do python tools/ncu_summary.py $f > ${f%.ncu-rep}.txt 2>&1; done
cat $S
