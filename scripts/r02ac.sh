#!/bin/bash
# ncu captures: band sort kernels (W=8), full-batch sort kernels and the tile kernel (C3) with source counters
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/${OUT:-r02ac}; mkdir -p $O; rm -f $O/*
S=$O/status.txt
python -c "from paper_2306_11686_b200 import build; build.build()" > $O/build.log 2>&1
for k in sort_count_band sort_scatter_band scan_add; do
  timeout 300 ncu --set full --clock-control none -k regex:$k -s 2 -c 1 -o $O/band_$k python tools/band_proxy.py 8 > /dev/null 2>&1; echo "ncu_band_$k=$?" >> $S
  ncu -i $O/band_$k.ncu-rep --page raw --csv > $O/band_$k.csv 2>/dev/null
done
for k in sort_count sort_scatter; do
  timeout 300 ncu --set full --clock-control none -k regex:"^gf::$k\$|$k\(" -s 2 -c 1 -o $O/full_$k python bench.py --config C3 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-proxy > /dev/null 2>&1; echo "ncu_full_$k=$?" >> $S
  ncu -i $O/full_$k.ncu-rep --page raw --csv > $O/full_$k.csv 2>/dev/null
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:xs_lookup_tile -s 3 -c 1 -o $O/tile_C3 python bench.py --config C3 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-proxy > /dev/null 2>&1; echo "ncu_tile=$?" >> $S
ncu -i $O/tile_C3.ncu-rep --page raw --csv > $O/tile_C3_raw.csv 2>/dev/null
ncu -i $O/tile_C3.ncu-rep --page source --csv --print-source sass > $O/tile_C3_sass.csv 2>/dev/null
ls -la $O >> $S
cat $S
