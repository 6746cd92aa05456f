#!/bin/bash
# build a kernel variant of libbdm.so: tools/build_variant.sh <name> <extra nvcc flags...>
# -> build/variants/libbdm_<name>.so (select it at run time with BDM_LIBRARY=...)
set -e
cd "$(dirname "$0")/.."
name=$1; shift
mkdir -p build/variants
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -fmad=false -Xcompiler -fPIC -Xptxas -v \
  "$@" -shared -o build/variants/libbdm_$name.so paper_2006_06775_b200/csrc/bdm_capi.cu 2> build/variants/ptxas_$name.log
grep -A2 "k_forceILb0" build/variants/ptxas_$name.log | grep -E "spill|Used" | sed "s/^/$name: /"
