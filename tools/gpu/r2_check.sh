set -x
make -s all 2>&1 | tail -3
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/r2_pytest1.log 2>&1; echo pytest rc=$?
tail -5 gpurun_out/r2_pytest1.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke1.log 2>&1; echo smoke rc=$?
tail -3 gpurun_out/r2_smoke1.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r2_bench1.log 2>&1; echo bench rc=$?
tail -2 gpurun_out/r2_bench1.log | cut -c1-3000
