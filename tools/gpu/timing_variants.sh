# bench.py (no CPU baseline, no parity) per kernel variant; prints step / force / pass times
for v in "$@"; do
  BDM_LIBRARY=build/variants/libbdm_$v.so timeout 300 python bench.py --no-cpu-baseline --steps 10 ${BENCH_ARGS} > gpurun_out/tv_$v.log 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/tv_$v.log').read().strip().splitlines()[-1]);print('$v',round(d['ms_per_step'],4),round(d['roofline']['ms_per_launch'],4),{k:round(x,4) for k,x in d['roofline']['passes_ms'].items()},round(d['roofline_rebuild']['ms_per_step'],4))" 2>&1 | tail -1
done
