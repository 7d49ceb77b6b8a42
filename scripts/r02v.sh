#!/bin/bash
# A/B of compile-time variants of the tile kernel (VARIANTS="name:defs;name:defs"), C3 / C4 batch sizes
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/r02v; mkdir -p $O; rm -f $O/*
IFS=';' read -ra VS <<< "$VARIANTS"
for v in "${VS[@]}"; do
  name="${v%%:*}"; defs="${v#*:}"
  GF_EXTRA_NVCC="$defs" python -c "from paper_2306_11686_b200 import build; build.build()" > $O/build_$name.log 2>&1
  echo "== $name ($defs)" >> $O/ab.txt
  GF_EXTRA_NVCC="$defs" timeout 300 python tools/ab_batch_n.py C3 tile ${AB_N:-2125000,17000000} >> $O/ab.txt 2>&1
  GF_EXTRA_NVCC="$defs" timeout 300 python tools/ab_batch_n.py C4 tile 2125000,21250000 >> $O/ab.txt 2>&1
done
python -c "from paper_2306_11686_b200 import build; build.build()" > /dev/null 2>&1
cat $O/ab.txt
