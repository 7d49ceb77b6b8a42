#!/bin/bash
# tile occupancy / buffer A/B
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/${OUT:-r02bj}; mkdir -p $O; rm -f $O/*
for v in "" "-DGF_TILE_MINB=5 -DGF_TILE_CAP=28" "-DGF_TILE_CAP=32" ""; do
  GF_EXTRA_NVCC="$v" python -c "from paper_2306_11686_b200 import build; build.build()" > $O/build.log 2>&1
  echo "== [$v]" >> $O/ab.txt
  timeout 300 python tools/ab_batch_n.py C3 tile 17000000 >> $O/ab.txt 2>&1
  timeout 300 python tools/ab_batch_n.py C2 tile 17000000 >> $O/ab.txt 2>&1
done
python -c "from paper_2306_11686_b200 import build; build.build()" > $O/build.log 2>&1
cat $O/ab.txt
