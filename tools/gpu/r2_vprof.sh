make -s all 2>&1 | tail -3
BDM_DIST_NOGRAPH=1 python tools/dist_virtual_profile.py --ranks 8 > gpurun_out/vp_plain.log 2>&1 && \
BDM_DIST_NOGRAPH=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
  --log-file gpurun_out/r02_dist_virtual8_launches.csv python tools/dist_virtual_profile.py --ranks 8 > gpurun_out/vp_ncu.log 2>&1; echo rc=$?
