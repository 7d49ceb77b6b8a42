# QB_CONFIGS="C3 H2 H3" QB_K="test name expression" bash scripts/quick_bench.sh
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
if [ -n "${QB_K:-}" ]; then
  timeout 600 python -m pytest tests -m gpu -x -q -k "$QB_K" > gpurun_out/pytest_qb.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_qb.log
fi
for c in ${QB_CONFIGS:-C3}; do
  timeout 300 python bench.py --config $c --steps ${QB_STEPS:-10} --no-cpu-baseline --no-e2e > gpurun_out/qb_$c.json 2>gpurun_out/qb_$c.err
  python -c "import json; d=json.load(open('gpurun_out/qb_$c.json')); print('$c', '%.4e'%d['value'], d['stage_ms'], d['hash'])" 2>&1 | tail -1
done
