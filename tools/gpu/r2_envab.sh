# A/B of run-time environment switches on one library: ENVS="NAME=VAR=val,... NAME2=..." LIB=path REPS=n
mkdir -p gpurun_out
make -s all 2>&1 | tail -2
for rep in $(seq ${REPS:-2}); do
for v in ${ENVS}; do
  name=${v%%=*}; envs=${v#*=}; envs=${envs//,/ }
  env $envs BDM_LIBRARY=${LIB:-} timeout 300 python bench.py --no-cpu-baseline --steps 20 ${BENCH_ARGS} > gpurun_out/envab_$name.log 2>&1
  echo "$name rc=$?"; python -c "import json;d=json.loads(open('gpurun_out/envab_$name.log').read().strip().splitlines()[-1]);print(d['ms_per_step'],d['roofline']['passes_ms'],d['roofline_rebuild']['ms_per_step'])" 2>&1 | tail -1
done; done
