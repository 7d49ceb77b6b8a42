#!/bin/bash
# ncu launch list of one C3 17M batch (cold, serialised)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/r02l; mkdir -p $O; rm -f $O/*
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv python tools/ab_batch_n.py C3 tile ${N:-17000000} > /dev/null 2>&1
python tools/launch_table.py $O/launches.csv | tail -12
