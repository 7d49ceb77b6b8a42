#!/bin/bash
# nuclide grid on the tile kernel: parity + C3N / C1 lines
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/r02n; mkdir -p $O; rm -f $O/*
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "alternative or nuclide or C1 or tiny or energies" > $O/pytest.log 2>&1; echo "pytest=$? $(tail -1 $O/pytest.log)"
timeout 600 python bench.py --config C3N --steps 5 --no-e2e --no-cpu-baseline > $O/bench_C3N.json 2> $O/bench_C3N.err
timeout 600 python bench.py --config C1 --steps 5 --no-e2e --no-cpu-baseline > $O/bench_C1.json 2> $O/bench_C1.err
python -c "
import json
for c in ('C3N','C1'):
    d=json.load(open('$O/bench_'+c+'.json')); print(c, '%.3e'%d['value'], d['ms_per_step'], d['hash'], d['roofline']['kernel'][:50], {k:(round(v['max_shard_ms'],3),round(v['speedup'],2)) for k,v in (d.get('strong_proxy') or {}).items() if isinstance(v,dict)})
"
