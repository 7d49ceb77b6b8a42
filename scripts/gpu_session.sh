#!/bin/bash
# One gpurun session: smoke, roofline probe, GPU tests, bench, ncu launch list + full capture.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
S=gpurun_out/status.txt; : > $S
nvidia-smi > gpurun_out/nvidia-smi.txt 2>&1
nproc >> gpurun_out/nvidia-smi.txt
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$? >> $S
if [ "${SKIP_PROBE:-0}" != 1 ]; then
  timeout 300 python tools/roofline_probe.py gpurun_out/roofline_probe.json > gpurun_out/probe.log 2>&1; echo probe=$? >> $S
fi
if [ "${SKIP_TESTS:-0}" != 1 ]; then
  timeout ${TEST_TIMEOUT:-1500} python -m pytest tests -m gpu -x -q ${PYTEST_ARGS:-} > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$? >> $S
fi
timeout 600 python bench.py --steps 10 --warmup 3 ${BENCH_ARGS:-} > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$? >> $S
if [ "${SKIP_NCU:-0}" != 1 ]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 120 --csv --log-file gpurun_out/launches.csv \
     python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e ${BENCH_ARGS:-} > gpurun_out/ncu_launch.log 2>&1; echo ncu_launch=$? >> $S
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:${NCU_KERNEL:-xs_lookup_sorted} -s 3 -c 1 \
     -o gpurun_out/prof_lookup python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e ${BENCH_ARGS:-} > gpurun_out/ncu_full.log 2>&1; echo ncu_full=$? >> $S
fi
cat $S
