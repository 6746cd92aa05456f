make -s all 2>&1 | tail -3
timeout 600 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_dist.py -q -x -k "overflow" > gpurun_out/r2_memcheck_dist.log 2>&1; echo rc=$?
head -80 gpurun_out/r2_memcheck_dist.log
