# A/B of programmatic dependent launch (BDM_PDL): full pytest -m gpu, then cfg3 and cfg2 benches
mkdir -p gpurun_out
make -s all 2>&1 | tail -2
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_gpu.log
show() { python -c "import json;d=json.loads(open('$1').read().strip().splitlines()[-1]);print(d['ms_per_step'],d['roofline']['ms_per_launch'],d['roofline_rebuild']['ms_per_step'],d['value'])" 2>&1 | tail -1; }
for cfg in 3 2; do
for rep in 1 2; do
for p in 1 0; do
  BDM_PDL=$p timeout 300 python bench.py --no-cpu-baseline --steps 20 --config $cfg > gpurun_out/pdl_${cfg}_$p.log 2>&1
  echo "cfg$cfg pdl=$p rc=$?"; show gpurun_out/pdl_${cfg}_$p.log
done; done; done
