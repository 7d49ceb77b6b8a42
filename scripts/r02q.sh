#!/bin/bash
# quick perf iteration: C3 / C4 batch-size A/B (raw sums must agree across kernels) + ncu of the tile kernel
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/r02q; mkdir -p $O
timeout 300 python tools/ab_batch_n.py C3 tile,group 2125000,8500000,17000000 > $O/ab_C3.txt 2>&1
timeout 300 python tools/ab_batch_n.py C4 tile,group 21250000 > $O/ab_C4.txt 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:xs_lookup_tile -s 3 -c 1 -o $O/prof_C3 python bench.py --config C3 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu.log 2>&1
cat $O/ab_C3.txt $O/ab_C4.txt
