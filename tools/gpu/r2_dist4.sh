make -s all 2>&1 | tail -3
timeout 900 python -m pytest tests/test_gpu_dist.py -q > gpurun_out/r2_dist4.log 2>&1; echo dist rc=$?
tail -15 gpurun_out/r2_dist4.log
