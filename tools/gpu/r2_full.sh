make -s all 2>&1 | tail -3
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r2_full_pytest.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/r2_full_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke.log 2>&1; echo smoke rc=$?; tail -1 gpurun_out/r2_smoke.log
