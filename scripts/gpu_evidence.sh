#!/bin/bash
# Round evidence: full GPU tests, smoke, every bench line, launch list and ncu captures of the dominant
# kernels.  Outputs under gpurun_out/ev/ (copied to profiles/<round>/ afterwards).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/ev; mkdir -p $O
S=$O/status.txt; : > $S
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest=$? $(tail -1 $O/pytest_gpu.log)" >> $S
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke=$?" >> $S
timeout 600 python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo "bench_default=$?" >> $S
for c in C1 C2 C4 C5 C5D0 C3N C6 C7 H2 H3 H5 P1 A1; do
  timeout 900 python bench.py --config $c --steps 5 --no-e2e --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err; echo "bench_$c=$?" >> $S
done
timeout 300 python bench.py --config C3 --steps 3 --no-sort --no-e2e --no-cpu-baseline > $O/bench_C3_nosort.json 2> $O/bench_C3_nosort.err; echo "bench_C3_nosort=$?" >> $S
timeout 300 python bench.py --impl reference --config C3 --steps 2 --warmup 1 > $O/bench_reference_C3.json 2> $O/bench_reference_C3.err; echo "reference=$?" >> $S
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file $O/launches_C3.csv python bench.py --config C3 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo "ncu_launch=$?" >> $S
timeout 600 ncu --set full --clock-control none --import-source on -k regex:xs_lookup_group -s 3 -c 1 -o $O/prof_C3 python bench.py --config C3 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo "ncu_C3=$?" >> $S
timeout 600 ncu --set full --clock-control none -k regex:xs_lookup_group -s 3 -c 1 -o $O/prof_C4 python bench.py --config C4 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo "ncu_C4=$?" >> $S
timeout 600 ncu --set full --clock-control none -k regex:xs_lookup_direct -s 3 -c 1 -o $O/prof_C3_nosort python bench.py --config C3 --steps 1 --warmup 3 --no-sort --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo "ncu_C3_nosort=$?" >> $S
timeout 600 ncu --set full --clock-control none -k regex:rs_lookup_sorted -s 3 -c 1 -o $O/prof_C5 python bench.py --config C5 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo "ncu_C5=$?" >> $S
timeout 600 ncu --set full --clock-control none -k regex:pr_gather -s 3 -c 1 -o $O/prof_P1 python bench.py --config P1 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo "ncu_P1=$?" >> $S
timeout 600 ncu --set full --clock-control none -k regex:amg_relax -s 3 -c 1 -o $O/prof_A1 python bench.py --config A1 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo "ncu_A1=$?" >> $S
timeout 600 ncu --set full --clock-control none -k regex:xs_lookup_sorted -s 3 -c 1 -o $O/prof_C1 python bench.py --config C1 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo "ncu_C1=$?" >> $S
cat $S
