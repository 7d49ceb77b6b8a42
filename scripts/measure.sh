#!/bin/bash
# One measurement session: GPU tests, benches, launch list, one full ncu capture of the C3 lookup kernel.
# MEAS_CONFIGS="C3 C4" MEAS_TESTS=1 MEAS_NCU=1 bash scripts/measure.sh
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
if [ "${MEAS_TESTS:-1}" = 1 ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$? $(tail -1 gpurun_out/pytest_gpu.log)"
fi
for c in ${MEAS_CONFIGS:-C3}; do
  timeout 900 python bench.py --config $c --steps ${MEAS_STEPS:-10} --warmup 3 ${MEAS_BENCH_ARGS:---no-cpu-baseline --no-e2e} > gpurun_out/$c.json 2>gpurun_out/$c.err
  echo "$c $(python -c "import json; d=json.load(open('gpurun_out/$c.json')); print(d['value'], d['stage_ms'], d['roofline']['frac'])" 2>&1 | tail -1)"
done
if [ "${MEAS_NCU:-0}" = 1 ]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches_${MEAS_NCU_CFG:-C3}.csv \
     python bench.py --config ${MEAS_NCU_CFG:-C3} --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch.log 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:${MEAS_NCU_KERNEL:-xs_lookup_group} -s 3 -c 1 \
     -o gpurun_out/prof_${MEAS_NCU_CFG:-C3} python bench.py --config ${MEAS_NCU_CFG:-C3} --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full.log 2>&1
  echo "ncu rc=$?"
fi
