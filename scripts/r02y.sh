#!/bin/bash
# sort-bin resolution A/B on the 8-way C3 shard and the full batch
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/r02y; mkdir -p $O; rm -f $O/*
for b in 13 14 15 16 17; do
  echo "== GF_SORT_BITS=$b" >> $O/ab.txt
  GF_SORT_BITS=$b timeout 300 python tools/ab_batch_n.py C3 tile 2125000,17000000 >> $O/ab.txt 2>&1
done
cat $O/ab.txt
