# launch list of steady-state cfg3 steps + one full capture of the force kernel (tools/profile_step.py)
set -x
mkdir -p gpurun_out
make -s all 2>&1 | tail -2
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
tail -2 gpurun_out/smoke.log
timeout 300 python tools/profile_step.py --steps 2 > gpurun_out/prof_plain.log 2>&1; echo plain rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
  --log-file gpurun_out/launches.csv python tools/profile_step.py --steps 2 > gpurun_out/ncu_launch.log 2>&1; echo launch rc=$?
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:k_force -c 1 \
  -o gpurun_out/force -f python tools/profile_step.py --steps 1 > gpurun_out/ncu_force.log 2>&1; echo force rc=$?
