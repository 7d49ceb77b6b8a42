#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/${OUT:-r02bp}; mkdir -p $O; rm -f $O/*
python -c "from paper_2306_11686_b200 import build; build.build()" > $O/build.log 2>&1
for b in 17 18 17 18; do
  echo "== GF_SORT_BITS=$b" >> $O/ab.txt
  GF_SORT_BITS=$b timeout 300 python tools/ab_batch_n.py C2 tile 17000000 >> $O/ab.txt 2>&1
  GF_SORT_BITS=$b timeout 300 python tools/ab_batch_n.py C3 tile 17000000 >> $O/ab.txt 2>&1
  GF_SORT_BITS=$b timeout 300 python tools/ab_batch_n.py C4 tile 170000000 >> $O/ab.txt 2>&1
  GF_SORT_BITS=$b timeout 300 python tools/band_proxy.py 8 >> $O/ab.txt 2>&1
done
cat $O/ab.txt
