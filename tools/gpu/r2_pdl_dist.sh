# distributed runtime with PDL: dist + slab tests, then the virtual-rank fixed cost with BDM_PDL=0 / 1
mkdir -p gpurun_out
make -s all 2>&1 | tail -3
timeout 900 python -m pytest tests/test_gpu_dist.py tests/test_gpu_slabs.py -x -q > gpurun_out/pytest_dist.log 2>&1; echo pytest rc=$?
tail -2 gpurun_out/pytest_dist.log
for p in 1 0 1; do
  BDM_PDL=$p timeout 600 python tools/dist_virtual_bench.py --ranks 8 > gpurun_out/vb_pdl$p.json 2> gpurun_out/vb_pdl$p.err; echo "pdl=$p rc=$?"
  cat gpurun_out/vb_pdl$p.json | python -c "import json,sys; d=json.load(sys.stdin); print({k: d[k] for k in d if k!='runs'} if isinstance(d, dict) else d)" 2>&1 | tail -3
done
