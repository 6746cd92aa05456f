make -s all 2>&1 | tail -3
ab() { echo "$1"; python -c "import json;d=json.loads(open('$2').read().strip().splitlines()[-1]);print(d['ms_per_step'],d['roofline']['passes_ms'],d['roofline_rebuild']['ms_per_step'])"; }
for rep in 1 2; do
BDM_BANDS=1 timeout 300 python bench.py --no-cpu-baseline --steps 20 --warmup 5 --e2e-steps 1 > gpurun_out/r2_bands_1.log 2>&1; ab new gpurun_out/r2_bands_1.log
BDM_LIBRARY=build/variants/libbdm_head.so timeout 300 python bench.py --no-cpu-baseline --steps 20 --warmup 5 --e2e-steps 1 > gpurun_out/r2_bands_h.log 2>&1; ab head gpurun_out/r2_bands_h.log
done
