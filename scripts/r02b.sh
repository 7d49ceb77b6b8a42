#!/bin/bash
# Round 2: warp-tile kernel -- parity of the forced kernels, batch-size A/B, C3 / C4 bench lines.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/r02b; mkdir -p $O
python -c "from paper_2306_11686_b200 import build; build.build()" > $O/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "alternative or interval_edges or C3_large or nuclide_bin or warp_search" > $O/pytest.log 2>&1; echo "pytest=$?" >> $O/status.txt
timeout 300 python tools/ab_batch_n.py C3 tile,tilenb,group,thread > $O/ab_C3.txt 2>&1
timeout 300 python tools/ab_batch_n.py C4 tile,group,thread 2125000,21250000 > $O/ab_C4.txt 2>&1
timeout 300 python bench.py --steps 10 --no-cpu-baseline --no-e2e > $O/bench_C3.json 2> $O/bench_C3.err
timeout 300 ncu --set full --clock-control none --import-source on -k regex:xs_lookup_tile -s 3 -c 1 -o $O/prof_C3 python bench.py --config C3 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu.log 2>&1
tail -2 $O/pytest.log; cat $O/ab_C3.txt $O/ab_C4.txt; head -c 400 $O/bench_C3.json
