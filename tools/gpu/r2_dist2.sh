make -s all 2>&1 | tail -3
timeout 900 python -m pytest tests/test_gpu_dist.py -q > gpurun_out/r2_dist2.log 2>&1; echo dist rc=$?
tail -3 gpurun_out/r2_dist2.log
ab() { echo "$1"; python -c "import json;d=json.loads(open('$2').read().strip().splitlines()[-1]);print(d['ms_per_step'],d['roofline']['passes_ms'],d.get('dist',{}).get('host_syncs'))"; }
for rep in 1 2; do
timeout 300 python bench.py --no-cpu-baseline --steps 20 --warmup 5 --e2e-steps 1 > gpurun_out/r2_d_a.log 2>&1; ab single gpurun_out/r2_d_a.log
timeout 300 python bench.py --slabs --no-cpu-baseline --steps 20 --warmup 5 --e2e-steps 1 > gpurun_out/r2_d_b.log 2>&1; ab dist1 gpurun_out/r2_d_b.log
done
