#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/${OUT:-r02ay}; mkdir -p $O; rm -f $O/*
python -c "from paper_2306_11686_b200 import build; build.build()" > $O/build.log 2>&1
timeout 600 python tools/e2e_modes.py > $O/e2e_modes.txt 2>&1
timeout 600 python tools/e2e_probe.py > $O/e2e_probe.txt 2>&1
cat $O/e2e_modes.txt $O/e2e_probe.txt
