#!/bin/bash
# tile reserve-next + L1 prefetch A/B
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/${OUT:-r02bl}; mkdir -p $O; rm -f $O/*
python -c "from paper_2306_11686_b200 import build; build.build()" > $O/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "C3_large or alternative_sorted or interval_edges or C4 or C2_small or band" > $O/pytest.log 2>&1; echo "pytest=$? $(tail -1 $O/pytest.log)" >> $O/ab.txt
for v in "-DGF_TILE_RESERVE=0" "" "-DGF_TILE_RESERVE=0" ""; do
  GF_EXTRA_NVCC="$v" python -c "from paper_2306_11686_b200 import build; build.build()" > $O/build.log 2>&1
  echo "== [$v]" >> $O/ab.txt
  timeout 300 python tools/ab_batch_n.py C3 tile 17000000 >> $O/ab.txt 2>&1
  timeout 300 python tools/ab_batch_n.py C2 tile 17000000 >> $O/ab.txt 2>&1
  timeout 300 python tools/ab_batch_n.py C4 tile 170000000 >> $O/ab.txt 2>&1
done
python -c "from paper_2306_11686_b200 import build; build.build()" > $O/build.log 2>&1
cat $O/ab.txt
