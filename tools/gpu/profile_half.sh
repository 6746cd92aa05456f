# launch list of steady-state cfg3 steps + full captures of the half-shell kernels
mkdir -p gpurun_out
make -s all 2>&1 | tail -2
timeout 300 python tools/profile_step.py --steps 2 > gpurun_out/prof_plain.log 2>&1; echo plain rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
  --log-file gpurun_out/launches.csv python tools/profile_step.py --steps 2 > gpurun_out/ncu_launch.log 2>&1; echo launch rc=$?
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:k_half -c 2 \
  -o gpurun_out/half -f python tools/profile_step.py --steps 2 > gpurun_out/ncu_half.log 2>&1; echo half rc=$?
