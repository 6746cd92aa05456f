# profiles/ evidence of round 2 (cfg3): fp64 pipe microbenchmark, bench launch list of the timed steps, full
# captures of the force-phase and rebuild kernels, launch list of the distributed runtime (--slabs, 1 rank)
mkdir -p gpurun_out
make -s all 2>&1 | tail -2
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp64_microbench tools/fp64_microbench.cu && ./tools/fp64_microbench > gpurun_out/r02_fp64_microbench.txt 2>&1; echo fp64 rc=$?
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/r02_bench_plain.log 2>&1 && \
BDM_PROFILE_TIMED=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
  --log-file gpurun_out/r02_bench_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/r02_bench_ncu.log 2>&1
echo launches rc=$?
python tools/profile_step.py --steps 2 > gpurun_out/r02_ps.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:k_half -c 2 \
  -o gpurun_out/r02_half -f python tools/profile_step.py --steps 2 > gpurun_out/r02_ncu_half.log 2>&1; echo half rc=$?
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off \
  -k "regex:k_key_hist|k_scatter|k_place|k_scan|k_table_zero" -c 6 \
  -o gpurun_out/r02_rebuild -f python tools/profile_step.py --steps 2 > gpurun_out/r02_ncu_rebuild.log 2>&1; echo rebuild rc=$?
python bench.py --slabs --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/r02_slabs_plain.log 2>&1 && \
BDM_PROFILE_TIMED=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
  --log-file gpurun_out/r02_dist_launches.csv python bench.py --slabs --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/r02_dist_ncu.log 2>&1
echo dist launches rc=$?
