#!/bin/bash
# Round 2: full GPU tests, default bench line (strong proxies), K6 probe, compute-sanitizer.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/r02s; mkdir -p $O
python -c "from paper_2306_11686_b200 import build; build.build()" > $O/build.log 2>&1
timeout 1700 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo "pytest=$? $(tail -1 $O/pytest_gpu.log)" > $O/status.txt
timeout 400 python bench.py --steps 10 > $O/bench_C3.json 2> $O/bench_C3.err; echo "bench=$?" >> $O/status.txt
timeout 300 python tools/roofline_probe.py > $O/probe.log 2>&1; echo "probe=$?" >> $O/status.txt
cp profiles/roofline_probe.json $O/ 2>/dev/null
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_small.py > $O/san_$tool.log 2>&1; echo "san_$tool=$?" >> $O/status.txt
done
cat $O/status.txt; tail -2 $O/san_*.log
