make -s all 2>&1 | tail -3
timeout 600 python -m pytest tests/test_gpu_half.py tests/test_gpu_parity.py tests/test_gpu_dist.py tests/test_gpu_neurite.py -x -q > gpurun_out/r2_slow_pytest.log 2>&1; echo pytest rc=$?; tail -1 gpurun_out/r2_slow_pytest.log
ab() { echo "$1"; python -c "import json;d=json.loads(open('$2').read().strip().splitlines()[-1]);print(d['ms_per_step'],d['roofline']['passes_ms'],d['roofline_rebuild']['ms_per_step'])"; }
for rep in 1 2; do
timeout 300 python bench.py --no-cpu-baseline --steps 20 --warmup 5 --e2e-steps 1 > gpurun_out/r2_v0.log 2>&1; ab warp_slow gpurun_out/r2_v0.log
done
