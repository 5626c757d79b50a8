# Builds the B200 product library (sm_100a) and the parity checker.
NVCC ?= /usr/local/cuda/bin/nvcc
PKG := paper_2410_12614_b200
LIB := $(PKG)/lib/libmpfem_b200.so
SRCS := $(PKG)/csrc/capi.cu $(PKG)/csrc/assembly_capi.cu $(PKG)/csrc/host_setup.cpp $(PKG)/csrc/host_mesh.cpp
HDRS := $(wildcard $(PKG)/csrc/*.cuh) $(wildcard $(PKG)/csrc/*.hpp) include/mpfem_b200.h
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-ffp-contract=off -shared \
           --expt-relaxed-constexpr -Xptxas -v

all: $(LIB) oracle

$(LIB): $(SRCS) $(HDRS)
	mkdir -p $(PKG)/lib
	$(NVCC) $(NVFLAGS) -o $@ $(SRCS) 2> $(PKG)/lib/ptxas.log || (cat $(PKG)/lib/ptxas.log; exit 1)

oracle:
	$(MAKE) -s -C oracle all

clean:
	rm -f $(LIB)

.PHONY: all oracle clean
