# profiles/ evidence of the current kernels (cfg3): bench launch list of the timed steps, full captures
# of the force-phase and rebuild kernels (steady-state step without the dp write, as the bench times)
mkdir -p gpurun_out
make -s all 2>&1 | tail -2
BDM_PROFILE_TIMED=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
  --log-file gpurun_out/bench_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_ncu.log 2>&1
echo launches rc=$?
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:k_half -c 2 \
  -o gpurun_out/half -f python tools/profile_step.py --steps 2 > gpurun_out/ncu_half.log 2>&1; echo half rc=$?
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off \
  -k "regex:k_key_hist|k_scatter|k_place|k_scan|k_table_zero" -c 6 \
  -o gpurun_out/rebuild -f python tools/profile_step.py --steps 2 > gpurun_out/ncu_rebuild.log 2>&1; echo rebuild rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/nb_launches.csv \
  python tools/neurite_bench.py --steps 2 --warmup 1 > gpurun_out/ncu_nb.log 2>&1; echo neurite launches rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:k_el_update|k_sc_rows" -s 2 -c 2 \
  -o gpurun_out/elu -f python tools/neurite_bench.py --steps 2 --warmup 1 > gpurun_out/ncu_elu.log 2>&1; echo neurite kernels rc=$?
