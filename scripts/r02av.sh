#!/bin/bash
# tile prefetch A/B: C3 step and band W=8 with GF_TILE_PF=0 / 1
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/${OUT:-r02av}; mkdir -p $O; rm -f $O/*
for v in "-DGF_TILE_PF=0" "" "-DGF_TILE_PF=0" ""; do
  GF_EXTRA_NVCC="$v" python -c "from paper_2306_11686_b200 import build; build.build()" > $O/build.log 2>&1
  echo "== [$v]" >> $O/ab.txt
  timeout 300 python tools/ab_batch_n.py C3 tile 17000000 >> $O/ab.txt 2>&1
  timeout 300 python tools/band_proxy.py 8 >> $O/ab.txt 2>&1
  timeout 300 python tools/ab_batch_n.py C4 tile 170000000 >> $O/ab.txt 2>&1
done
cat $O/ab.txt
