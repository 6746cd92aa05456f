set -x
make -s all 2>&1 | tail -3
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r2_pytest_final.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/r2_pytest_final.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke_final.log 2>&1; echo smoke rc=$?
tail -1 gpurun_out/r2_smoke_final.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r2_bench_final.log 2>&1; echo bench rc=$?
tail -1 gpurun_out/r2_bench_final.log | cut -c1-4000
