# AB_VARIANTS="g4:;g8:-DGF_PR_G=8" bash scripts/ab_pr.sh  (kernel variants of a NEXT-4 bench; tests each)
# AB_TEST (default tests/test_gpu_pagerank.py) and AB_CONFIG (default P1) pick the test file and bench config.
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
IFS=';' read -ra VS <<< "$AB_VARIANTS"
for v in "${VS[@]}"; do
  name="${v%%:*}"; defs="${v#*:}"
  rm -f paper_2306_11686_b200/libgfxs.so
  GF_EXTRA_NVCC="$defs" python -c "from paper_2306_11686_b200 import build; build.build(force=True)" > /dev/null 2>&1
  timeout 300 python -m pytest "${AB_TEST:-tests/test_gpu_pagerank.py}" -x -q -k "bit_exact" > gpurun_out/pt_$name.log 2>&1; t=$?
  timeout 120 python bench.py --config "${AB_CONFIG:-P1}" --steps 5 --no-cpu-baseline --no-e2e > gpurun_out/abp_$name.json 2>&1
  echo "$name tests=$t $(python -c "import json; d=json.load(open('gpurun_out/abp_$name.json')); print(d['value'], d['ms_per_step'], d['roofline']['frac'])" 2>&1 | tail -1)"
done
