# A/B of run-time switches: pytest -m gpu, then bench.py (no CPU baseline) per "NAME=ENV" argument
mkdir -p gpurun_out
make -s all 2>&1 | tail -2
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_gpu.log
for v in "$@"; do
  name=${v%%=*}; envs=${v#*=}
  env $envs timeout 300 python bench.py --no-cpu-baseline --steps 10 ${BENCH_ARGS} > gpurun_out/ab_$name.log 2>&1
  echo "$name rc=$?"; python -c "import json;d=json.loads(open('gpurun_out/ab_$name.log').read().strip().splitlines()[-1]);print(d['ms_per_step'],d['roofline']['ms_per_launch'],d['roofline_rebuild']['ms_per_step'])" 2>&1 | tail -1
done
