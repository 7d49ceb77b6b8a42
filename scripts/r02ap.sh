#!/bin/bash
# ncu with source: band count / scatter / tile kernels (W=8 band 0)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/${OUT:-r02ap}; mkdir -p $O; rm -f $O/*
S=$O/status.txt
python -c "from paper_2306_11686_b200 import build; build.build()" > $O/build.log 2>&1
for k in sort_count_band sort_scatter_band xs_lookup_tile; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 -o $O/b_$k python tools/band_proxy.py 8 > /dev/null 2>&1; echo "ncu_$k=$?" >> $S
  ncu -i $O/b_$k.ncu-rep --page source --csv --print-source sass > $O/b_${k}_sass.csv 2>/dev/null
  python tools/ncu_summary.py $O/b_$k.ncu-rep > $O/b_$k.txt 2>&1
done
cat $S
