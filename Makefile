# libkm (the product, sm_100a) and liboracle (test infrastructure, plain C).
NVCC    ?= /usr/local/cuda/bin/nvcc
ARCH    := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := -O3 -lineinfo -std=c++17 $(ARCH) -Xcompiler -fPIC,-O2 -Xptxas -v
PKG     := paper_2412_02244_b200
SRC     := $(PKG)/csrc/km_api.cu
DEPS    := $(wildcard $(PKG)/csrc/*.cu $(PKG)/csrc/*.cuh) include/km.h

all: $(PKG)/libkm.so oracle/liboracle.so

$(PKG)/libkm.so: $(DEPS)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -shared -o $@ $(SRC) 2> build/ptxas.log || (cat build/ptxas.log; exit 1)
	@grep -E "registers|spill" build/ptxas.log | sed 's/^ptxas info    : //' > build/ptxas_summary.txt || true

oracle/liboracle.so: oracle/lloyd_oracle.c
	gcc -O2 -fPIC -shared -fopenmp -ffp-contract=off -fno-fast-math -std=c11 $< -o $@ -lm

# tuning / profiling variants: make var VAR=prof DEFS=-DKM_PROF -> build/var/libkm_prof.so
var: $(DEPS)
	@mkdir -p build/var
	$(NVCC) $(NVFLAGS) $(DEFS) -shared -o build/var/libkm_$(VAR).so $(SRC) 2> build/var/ptxas_$(VAR).log || (cat build/var/ptxas_$(VAR).log; exit 1)

sass: $(PKG)/libkm.so
	/usr/local/cuda/bin/cuobjdump -sass $< > build/libkm.sass

clean:
	rm -f $(PKG)/libkm.so oracle/liboracle.so build/*

.PHONY: all clean sass var
