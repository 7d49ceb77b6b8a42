#!/bin/bash
# Round-2 evidence on the current code: full GPU tests, smoke, bench lines, launch list, ncu captures.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/r02e; mkdir -p $O; rm -f $O/*
S=$O/status.txt
python -c "from paper_2306_11686_b200 import build; build.build()" > $O/build.log 2>&1
timeout 1700 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest=$? $(tail -1 $O/pytest_gpu.log)" >> $S
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke=$?" >> $S
timeout 600 python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo "bench_default=$?" >> $S
for c in ${CONFIGS:-C1 C2 C4 C5 C3N H3}; do
  timeout 900 python bench.py --config $c --steps 5 --no-e2e --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err; echo "bench_$c=$?" >> $S
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $O/launches_C3.csv python bench.py --config C3 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-proxy > /dev/null 2>&1; echo "ncu_launch=$?" >> $S
timeout 600 ncu --set full --clock-control none --import-source on -k regex:xs_lookup_tile -s 3 -c 1 -o $O/prof_C3 python bench.py --config C3 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-proxy > /dev/null 2>&1; echo "ncu_C3=$?" >> $S
timeout 600 ncu --set full --clock-control none -k regex:xs_lookup_tile -s 3 -c 1 -o $O/prof_C4 python bench.py --config C4 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-proxy > /dev/null 2>&1; echo "ncu_C4=$?" >> $S
cat $S
