# AB_VARIANTS="c21:-DGF_IO_CHUNK_LOG2=21;c22:-DGF_IO_CHUNK_LOG2=22" bash scripts/ab_e2e.sh  (host-IO e2e leg of C3)
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
IFS=';' read -ra VS <<< "$AB_VARIANTS"
for v in "${VS[@]}"; do
  name="${v%%:*}"; defs="${v#*:}"
  rm -f paper_2306_11686_b200/libgfxs.so
  GF_EXTRA_NVCC="$defs" python -c "from paper_2306_11686_b200 import build; build.build(force=True)" > /dev/null 2>&1
  timeout 300 python -m pytest tests -m gpu -x -q -k "host" > gpurun_out/pt_$name.log 2>&1; t=$?
  timeout 300 python bench.py --config ${AB_CONFIG:-C3} --steps 3 --no-cpu-baseline > gpurun_out/abe_$name.json 2>&1
  echo "$name tests=$t $(tail -1 gpurun_out/pt_$name.log) $(python -c "import json; d=json.loads(open('gpurun_out/abe_$name.json').read().strip().splitlines()[-1]); print('%.3e'%d['value'], '%.3e'%d['e2e']['value'], '%.3e'%d['e2e']['with_macro']['value'])" 2>&1 | tail -1)"
done
