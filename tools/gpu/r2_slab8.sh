make -s all 2>&1 | tail -2
timeout 1500 python bench.py --slabs --config 5 --slab-of 8 --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/r02_cfg5_slab8.log 2>&1; echo rc=$?
grep -v "NCCL INFO" gpurun_out/r02_cfg5_slab8.log | tail -2 | cut -c1-4000
