#!/bin/bash
# ncu: band W=8 tile kernel (tail / SM balance) and the full C3 tile kernel after the header fast paths
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/${OUT:-r02ag}; mkdir -p $O; rm -f $O/*
S=$O/status.txt
python -c "from paper_2306_11686_b200 import build; build.build()" > $O/build.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:xs_lookup_tile -s 2 -c 1 -o $O/tile_band8 python tools/band_proxy.py 8 > /dev/null 2>&1; echo "ncu_band=$?" >> $S
ncu -i $O/tile_band8.ncu-rep --page raw --csv > $O/tile_band8_raw.csv 2>/dev/null
timeout 600 ncu --set full --clock-control none --import-source on -k regex:xs_lookup_tile -s 3 -c 1 -o $O/tile_C3 python bench.py --config C3 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-proxy > /dev/null 2>&1; echo "ncu_tile=$?" >> $S
ncu -i $O/tile_C3.ncu-rep --page raw --csv > $O/tile_C3_raw.csv 2>/dev/null
ncu -i $O/tile_C3.ncu-rep --page source --csv --print-source sass > $O/tile_C3_sass.csv 2>/dev/null
timeout 300 ncu --set full --clock-control none -k regex:sort_scatter_band -s 2 -c 1 -o $O/scatter_band python tools/band_proxy.py 8 > /dev/null 2>&1; echo "ncu_scat=$?" >> $S
cat $S
