#!/bin/bash
# Bench lines for every config + ncu captures of each config's dominant kernel.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
S=gpurun_out/status_all.txt; : > $S
for c in C3 C2 C1 C4 C5; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-e2e ${EXTRA:-} > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo bench_$c=$? >> $S
done
timeout 600 python bench.py --config C3 --steps 5 --warmup 3 --no-sort --no-e2e --no-cpu-baseline > gpurun_out/bench_C3_nosort.json 2> gpurun_out/bench_C3_nosort.err; echo bench_C3_nosort=$? >> $S
if [ "${NCU:-1}" = 1 ]; then
  timeout 900 ncu --set full --clock-control none -k regex:xs_lookup_direct -s 3 -c 1 -o gpurun_out/prof_C3_direct python bench.py --config C3 --steps 1 --warmup 3 --no-sort --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo ncu_direct=$? >> $S
  timeout 900 ncu --set full --clock-control none -k regex:xs_lookup_sorted -s 3 -c 1 -o gpurun_out/prof_C4 python bench.py --config C4 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo ncu_C4=$? >> $S
  timeout 900 ncu --set full --clock-control none -k regex:rs_lookup -s 3 -c 1 -o gpurun_out/prof_C5 python bench.py --config C5 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo ncu_C5=$? >> $S
fi
cat $S
