# A/B of kernel variants (build/variants/libbdm_<v>.so, built here with tools/build_variant.sh):
# parity + half-shell tests with the in-tree build, then cfg3 benches alternating the variants.
# VARIANTS="a b" REPS=2 TESTS="tests/test_gpu_parity.py ..." bash tools/gpu/r2_abv.sh
mkdir -p gpurun_out
make -s all 2>&1 | tail -2
BDM_LIBRARY=${TESTLIB:-} timeout 900 python -m pytest ${TESTS:-tests/test_gpu_parity.py tests/test_gpu_half.py} -x -q > gpurun_out/pytest_ab.log 2>&1; echo pytest rc=$?
tail -2 gpurun_out/pytest_ab.log
for rep in $(seq ${REPS:-2}); do
for v in ${VARIANTS}; do
  BDM_LIBRARY=build/variants/libbdm_$v.so timeout 300 python bench.py --no-cpu-baseline --steps 20 ${BENCH_ARGS} > gpurun_out/ab_$v.log 2>&1
  rc=$?; python -c "import json;d=json.loads(open('gpurun_out/ab_$v.log').read().strip().splitlines()[-1]);print('$v', $rc, d['ms_per_step'],d['roofline']['passes_ms'],d['roofline_rebuild']['ms_per_step'])" 2>&1 | tail -1
done; done
