set -x
make -s all 2>&1 | tail -3
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/r2_pytest3.log 2>&1; echo pytest rc=$?
tail -15 gpurun_out/r2_pytest3.log
timeout 900 python bench.py --slabs --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2_bench_slabs.log 2>&1; echo slabs rc=$?
grep -v NCCL gpurun_out/r2_bench_slabs.log | tail -3 | cut -c1-2500
