#!/bin/bash
# GPU tests (full suite) + default bench line
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/r02t; mkdir -p $O
timeout 1700 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo "pytest=$? $(tail -1 $O/pytest_gpu.log)" > $O/status.txt
timeout 300 python bench.py --steps 10 --no-cpu-baseline > $O/bench_C3.json 2> $O/bench_C3.err
timeout 600 python bench.py --config C4 --steps 5 --no-cpu-baseline --no-e2e > $O/bench_C4.json 2> $O/bench_C4.err
cat $O/status.txt; tail -3 $O/pytest_gpu.log; head -c 300 $O/bench_C3.json; echo; head -c 300 $O/bench_C4.json
