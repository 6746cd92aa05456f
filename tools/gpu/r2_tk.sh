make -s all 2>&1 | tail -3
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_half.py tests/test_gpu_dist.py tests/test_gpu_single_path.py tests/test_gpu_skip.py -x -q > gpurun_out/r2_tk_pytest.log 2>&1; echo pytest rc=$?
tail -2 gpurun_out/r2_tk_pytest.log
ab() { echo "$1"; python -c "import json;d=json.loads(open('$2').read().strip().splitlines()[-1]);print(d['ms_per_step'],d['roofline']['passes_ms'],d['roofline_rebuild']['ms_per_step'])"; }
for rep in 1 2; do
timeout 300 python bench.py --no-cpu-baseline --steps 20 --warmup 5 --e2e-steps 1 > gpurun_out/r2_tk.log 2>&1; ab striped gpurun_out/r2_tk.log
done
timeout 900 python tools/dist_virtual_bench.py > gpurun_out/r02_dist_virtual.json 2> gpurun_out/r02_dist_virtual.err; cat gpurun_out/r02_dist_virtual.json
