set -x
mkdir -p gpurun_out
make -s all 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pytest_parity.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_parity.log
for v in ${VARIANTS:-nostage stage}; do
  BDM_LIBRARY=build/variants/libbdm_$v.so timeout 300 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/ab_$v.log 2>&1
  echo $v; python -c "import json;d=json.loads(open('gpurun_out/ab_$v.log').read().strip().splitlines()[-1]);print(d['ms_per_step'],d['roofline']['ms_per_launch'],d['roofline_rebuild']['ms_per_step'])"
done
