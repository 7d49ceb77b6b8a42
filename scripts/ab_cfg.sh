# AB_VARIANTS="base:;m6:-DGF_SORTED_MINB=6" AB_CONFIGS="H2 H3" AB_K="nuclide_bin" bash scripts/ab_cfg.sh
# Rebuilds per variant, runs the GPU tests selected by AB_K, then each config's bench line (ms, hash).
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
IFS=';' read -ra VS <<< "$AB_VARIANTS"
for v in "${VS[@]}"; do
  name="${v%%:*}"; defs="${v#*:}"
  rm -f paper_2306_11686_b200/libgfxs.so
  GF_EXTRA_NVCC="$defs" python -c "from paper_2306_11686_b200 import build; build.build(force=True)" > /dev/null 2>&1
  t=skip
  if [ -n "${AB_K:-}" ]; then timeout 600 python -m pytest tests -m gpu -x -q -k "$AB_K" > gpurun_out/pt_$name.log 2>&1; t=$?; fi
  for c in ${AB_CONFIGS:-C3}; do
    timeout 300 python bench.py --config $c --steps ${AB_STEPS:-5} --no-cpu-baseline --no-e2e > gpurun_out/abc_${name}_$c.json 2>&1
    echo "$name tests=$t $c $(python -c "import json; d=json.loads(open('gpurun_out/abc_${name}_$c.json').read().strip().splitlines()[-1]); print('%.4e'%d['value'], '%.3f'%d['ms_per_step'], d.get('hash'))" 2>&1 | tail -1)"
  done
done
