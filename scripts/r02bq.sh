#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/${OUT:-r02bq}; mkdir -p $O; rm -f $O/*
S=$O/status.txt
python -c "from paper_2306_11686_b200 import build; build.build()" > $O/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "band or C7 or C8 or torchrun" > $O/pytest.log 2>&1; echo "pytest=$? $(tail -1 $O/pytest.log)" >> $S
for r in 1 2; do timeout 600 python tools/band_proxy.py 1,8 >> $O/band_proxy.txt 2>&1; done
timeout 600 python bench.py --config C7 --steps 3 --no-e2e --no-cpu-baseline > $O/c7.json 2>/dev/null
python -c "import json; d=json.load(open('$O/c7.json')); print('C7', d['value'], d['ms_per_step'], d['hash'])" >> $S
cat $S; cat $O/band_proxy.txt
