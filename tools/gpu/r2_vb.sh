make -s all 2>&1 | tail -3
timeout 900 python -m pytest tests/test_gpu_dist.py -q > gpurun_out/r2_dist3.log 2>&1; echo dist rc=$?
tail -3 gpurun_out/r2_dist3.log
timeout 900 python tools/dist_virtual_bench.py > gpurun_out/r02_dist_virtual.json 2> gpurun_out/r02_dist_virtual.err; echo rc=$?
cat gpurun_out/r02_dist_virtual.json; tail -3 gpurun_out/r02_dist_virtual.err
BDM_DIST_NOGRAPH=1 timeout 900 python tools/dist_virtual_bench.py > gpurun_out/r02_dist_virtual_nograph.json 2>/dev/null; cat gpurun_out/r02_dist_virtual_nograph.json
