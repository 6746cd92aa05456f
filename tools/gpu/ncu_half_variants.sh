# full ncu capture of the half-shell kernels for each variant (build/variants/libbdm_<v>.so)
mkdir -p gpurun_out
for v in "$@"; do
  BDM_LIBRARY=build/variants/libbdm_$v.so timeout 600 ncu --set full --clock-control none --import-source on \
    --profile-from-start off -k regex:k_half -c 2 -o gpurun_out/half_$v -f python tools/profile_step.py --steps 1 \
    > gpurun_out/ncu_$v.log 2>&1; echo $v rc=$?
done
