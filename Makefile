# libbdm.so: the C-ABI library (sm_100a).  -fmad=false keeps every fp64 +,-,* separately rounded
# (bit-identical per-pair arithmetic with the oracle reading).
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -fmad=false -Xcompiler -fPIC -Xptxas -v
PKG := paper_2006_06775_b200
SRC := $(PKG)/csrc/bdm_capi.cu
HDR := $(PKG)/csrc/bdm_kernels.cuh $(PKG)/csrc/bdm_dist.cuh include/bdm.h

all: $(PKG)/libbdm.so oracle/liboracle.so

$(PKG)/libbdm.so: $(SRC) $(HDR)
	$(NVCC) $(NVFLAGS) -shared -o $@ $(SRC) -ldl 2> $(PKG)/csrc/ptxas.log || (cat $(PKG)/csrc/ptxas.log; false)

oracle/liboracle.so: oracle/bdm_oracle.c
	gcc -O2 -ffp-contract=off -fno-fast-math -fopenmp -fPIC -shared -o $@ $< -lm

sass: $(PKG)/libbdm.so
	cuobjdump -sass $< > $(PKG)/csrc/libbdm.sass

clean:
	rm -f $(PKG)/libbdm.so oracle/liboracle.so

.PHONY: all clean sass
