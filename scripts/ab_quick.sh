# usage: AB_VARIANTS="a:;b:-DX=1" AB_CONFIG="C3" AB_TESTS=1 bash scripts/ab_quick.sh
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
if [ "${AB_TESTS:-1}" = 1 ]; then
  timeout ${AB_TEST_TIMEOUT:-300} python -m pytest tests/test_gpu_parity.py -x -q -k "${AB_K:-C3 or C2 or C4 or groups or energies or tiny or large_custom or host_io or alternative}" > gpurun_out/pytest_ab.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_ab.log
fi
bash scripts/ab.sh
for f in gpurun_out/ab_*_C*.json; do python -c "import json,sys; d=json.load(open('$f')); print('$f', d['hash'])"; done
