# the GPU test suite against the bounds-checked build (device asserts; compute-sanitizer is closed here)
make -s all 2>&1 | tail -2
./tools/build_variant.sh checked -DBDM_CHECK=1 > /dev/null 2>&1
BDM_LIBRARY=build/variants/libbdm_checked.so timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r02_checked_pytest.log 2>&1; echo checked rc=$?
tail -5 gpurun_out/r02_checked_pytest.log
BDM_LIBRARY=build/variants/libbdm_checked.so BDM_HTILE=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_half.py tests/test_gpu_dist.py -q > gpurun_out/r02_checked_tile_pytest.log 2>&1; echo checked_tile rc=$?
tail -3 gpurun_out/r02_checked_tile_pytest.log
