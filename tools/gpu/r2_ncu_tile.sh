make -s all 2>&1 | tail -3
python tools/profile_step.py --steps 1 > gpurun_out/ps_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:k_half_search -c 1 \
  -o gpurun_out/r2_tile -f python tools/profile_step.py --steps 1 > gpurun_out/ncu_tile.log 2>&1; echo tile rc=$?
BDM_HTILE=0 python tools/profile_step.py --steps 1 > gpurun_out/ps_plain0.log 2>&1 && \
BDM_HTILE=0 timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:k_half_search -c 1 \
  -o gpurun_out/r2_notile -f python tools/profile_step.py --steps 1 > gpurun_out/ncu_notile.log 2>&1; echo notile rc=$?
