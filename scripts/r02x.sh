#!/bin/bash
# quick: parity subset + per-shard timings of the 8-way C3 split + C4 + C3 17M
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/r02x; mkdir -p $O; rm -f $O/*
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "alternative or interval_edges or C3_large or C4_large or ieee or energies or host_io or invalid" > $O/pytest.log 2>&1; echo "pytest=$? $(tail -1 $O/pytest.log)"
timeout 300 python tools/shard_times.py C3 8 > $O/shards_C3.txt 2>&1
timeout 300 python tools/ab_batch_n.py C3 tile 2125000,17000000 > $O/ab_C3.txt 2>&1
timeout 300 python tools/ab_batch_n.py C4 tile 2125000,21250000 > $O/ab_C4.txt 2>&1
cat $O/shards_C3.txt $O/ab_C3.txt $O/ab_C4.txt
