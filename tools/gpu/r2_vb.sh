make -s all 2>&1 | tail -3
timeout 900 python tools/dist_virtual_bench.py --ranks 2 8 > gpurun_out/r02_dist_virtual.json 2> gpurun_out/r02_dist_virtual.err; echo rc=$?
cat gpurun_out/r02_dist_virtual.json; tail -3 gpurun_out/r02_dist_virtual.err
