#!/bin/bash
# batch-size sweep of the sorted kernels (thresholds of the auto choice)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/r02w; mkdir -p $O; rm -f $O/*
timeout 600 python tools/ab_batch_n.py C3 tile,group,thread 250000,500000,1000000,1500000,2125000,4250000 > $O/ab_C3.txt 2>&1
timeout 600 python tools/ab_batch_n.py C4 tile,group,thread 250000,500000,1000000,2125000,4250000,21250000 > $O/ab_C4.txt 2>&1
timeout 600 python tools/ab_batch_n.py C2 tile,group,thread 500000,2125000,17000000 > $O/ab_C2.txt 2>&1
cat $O/ab_*.txt
