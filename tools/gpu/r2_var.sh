make -s all 2>&1 | tail -3
ab() { echo "$1"; python -c "import json;d=json.loads(open('$2').read().strip().splitlines()[-1]);print(d['ms_per_step'],d['roofline']['passes_ms'],d['roofline_rebuild']['ms_per_step'])"; }
for rep in 1 2; do
timeout 300 python bench.py --no-cpu-baseline --steps 20 --warmup 5 --e2e-steps 1 > gpurun_out/r2_v0.log 2>&1; ab base gpurun_out/r2_v0.log
for v in pl128 pl512 sc8 sc32; do
BDM_LIBRARY=build/variants/libbdm_$v.so timeout 300 python bench.py --no-cpu-baseline --steps 20 --warmup 5 --e2e-steps 1 > gpurun_out/r2_v_$v.log 2>&1; ab $v gpurun_out/r2_v_$v.log
done
done
