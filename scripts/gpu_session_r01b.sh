cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python tools/roofline_probe.py gpurun_out/roofline_probe.json > gpurun_out/probe.log 2>&1; echo probe=$?
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
for c in C3 C4 C5; do timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo bench_$c=$?; done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:xs_lookup_group -s 3 -c 1 -o gpurun_out/prof_C3 python bench.py --config C3 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo ncu_C3=$?
timeout 900 ncu --set full --clock-control none -k regex:xs_lookup_group -s 3 -c 1 -o gpurun_out/prof_C4 python bench.py --config C4 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo ncu_C4=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:rs_lookup -s 3 -c 1 -o gpurun_out/prof_C5 python bench.py --config C5 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo ncu_C5=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_C3.csv python bench.py --config C3 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo ncu_launch=$?
