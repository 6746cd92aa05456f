make -s all 2>&1 | tail -3
for v in 0 1 2 3; do
BDM_DIST_SYNC=$v timeout 600 python -m pytest tests/test_gpu_dist.py -q > gpurun_out/r2_dbg_sync$v.log 2>&1; echo sync=$v rc=$?
grep -E "BdmError:|passed|failed" gpurun_out/r2_dbg_sync$v.log | head -5
done
