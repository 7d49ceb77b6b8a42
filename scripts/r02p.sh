#!/bin/bash
# ncu of the tile kernel at a small batch (the strong-split per-rank size)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/r02p; mkdir -p $O; rm -f $O/*
timeout 600 ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-xs_lookup_tile} -s 2 -c 1 -o $O/prof_small python tools/ab_batch_n.py C3 ${KERN:-tile} ${N:-2125000} > $O/ncu.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv python tools/ab_batch_n.py C3 ${KERN:-tile} ${N:-2125000} > /dev/null 2>&1
tail -3 $O/ncu.log
