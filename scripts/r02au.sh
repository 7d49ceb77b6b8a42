#!/bin/bash
# XXL (C8) test + bench; compute-sanitizer on the small workload (new sort kernels, PDL)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/${OUT:-r02au}; mkdir -p $O; rm -f $O/*
S=$O/status.txt
python -c "from paper_2306_11686_b200 import build; build.build()" > $O/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "C8 or C7" > $O/pytest_c8.log 2>&1; echo "pytest_c8=$? $(tail -1 $O/pytest_c8.log)" >> $S
timeout 900 python bench.py --config C8 --steps 3 --no-e2e --no-cpu-baseline > $O/bench_C8.json 2> $O/bench_C8.err; echo "bench_C8=$?" >> $S
for t in memcheck racecheck synccheck; do
  GF_SAN_N=40000 timeout 1500 compute-sanitizer --tool $t --print-limit 20 python tools/sanitize_small.py > $O/sanitizer_$t.txt 2>&1; echo "san_$t=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' $O/sanitizer_$t.txt | tail -1)" >> $S
done
cat $S
