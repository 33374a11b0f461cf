# Build the product library (libcil.so, CUDA sm_100a) and the test oracle (liboracle.so).
# The two share no sources, headers or flags files.
NVCC   ?= /usr/local/cuda/bin/nvcc
CUDA   ?= /usr/local/cuda
ARCH   := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -fvisibility=hidden \
           -Iinclude --expt-relaxed-constexpr -Xptxas -v

PKG    := paper_1807_00399_b200
CSRC   := $(wildcard $(PKG)/csrc/*.cu)
CHDR   := $(wildcard $(PKG)/csrc/*.cuh) include/cil.h

all: cil oracle

cil: $(PKG)/libcil.so
oracle: oracle/liboracle.so

$(PKG)/libcil.so: $(CSRC) $(CHDR)
	$(NVCC) $(NVFLAGS) -shared -o $@ $(CSRC) -lcudart 2> $(PKG)/ptxas.log || (cat $(PKG)/ptxas.log; exit 1)

oracle/liboracle.so: oracle/oracle.c
	gcc -O2 -ffp-contract=off -fno-fast-math -fopenmp -shared -fPIC -o $@ $< -lm

clean:
	rm -f $(PKG)/libcil.so oracle/liboracle.so $(PKG)/ptxas.log

.PHONY: all cil oracle clean
