#!/bin/bash
# Round-2 first call: the round-1 code on this round's box (default bench line + batch-size sweep).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/r02a; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt 2>&1
timeout 300 python bench.py --steps 10 --no-cpu-baseline > $O/bench_default.json 2> $O/bench_default.err
timeout 300 python tools/ab_batch_n.py C3 > $O/ab_batch_n_C3.txt 2>&1
timeout 300 python bench.py --config C4 --steps 5 --no-e2e --no-cpu-baseline > $O/bench_C4.json 2> $O/bench_C4.err
tail -3 $O/*.json $O/ab_batch_n_C3.txt
