mkdir -p gpurun_out
make -s all >/dev/null 2>&1
timeout 900 ncu --set full --clock-control none --profile-from-start off -k "regex:k_key_hist|k_scatter|k_place|k_scan|k_table_zero" -c 6 \
  -o gpurun_out/rebuild -f python tools/profile_step.py --steps 1 > gpurun_out/ncu_rebuild.log 2>&1; echo rebuild rc=$?
