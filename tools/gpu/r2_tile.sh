make -s all 2>&1 | tail -3
ab() { echo "$1"; python -c "import json;d=json.loads(open('$2').read().strip().splitlines()[-1]);print(d['ms_per_step'],d['roofline']['passes_ms'],d['roofline_rebuild']['ms_per_step'])"; }
BDM_LIBRARY=build/variants/libbdm_nostage.so BDM_HTILE=1 timeout 300 python bench.py --no-cpu-baseline --steps 20 --warmup 5 --e2e-steps 1 > gpurun_out/r2_tile_c.log 2>&1; ab tile_nostage gpurun_out/r2_tile_c.log
