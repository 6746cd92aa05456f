# full ncu capture of k_force for each kernel variant given as arguments (build/variants/libbdm_<v>.so)
mkdir -p gpurun_out
for v in "$@"; do
  BDM_LIBRARY=build/variants/libbdm_$v.so timeout 600 ncu --set full --clock-control none --import-source on \
    --profile-from-start off -k regex:k_force -c 1 -o gpurun_out/force_$v -f python tools/profile_step.py --steps 1 \
    > gpurun_out/ncu_$v.log 2>&1; echo $v rc=$?
done
