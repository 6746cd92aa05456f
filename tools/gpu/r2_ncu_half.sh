make -s all 2>&1 | tail -2
python tools/profile_step.py --steps 2 > gpurun_out/r02_ps.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:k_half -c 2 \
  -o gpurun_out/${OUT:-r02_half} -f python tools/profile_step.py --steps 2 > gpurun_out/r02_ncu_half.log 2>&1; echo half rc=$?
