#!/bin/bash
# quick iteration: parity subset, C3 / C4 batch-size A/B (raw sums must agree across kernels), ncu of the tile kernel
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/r02q; mkdir -p $O; rm -f $O/*
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "alternative or interval_edges or C3_large or C4_large or ieee" > $O/pytest.log 2>&1; echo "pytest=$? $(tail -1 $O/pytest.log)"
timeout 300 python tools/ab_batch_n.py C3 tile,group ${AB_N:-2125000,4250000,8500000,17000000} > $O/ab_C3.txt 2>&1
timeout 300 python tools/ab_batch_n.py C4 tile,group 2125000,21250000 > $O/ab_C4.txt 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:xs_lookup_tile -s ${NCU_S:-3} -c 1 -o $O/prof_C3 python bench.py --config C3 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-proxy > $O/ncu.log 2>&1
cat $O/ab_C3.txt $O/ab_C4.txt
