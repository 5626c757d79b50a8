# Builds the B200 product library (sm_100a) and the parity checker.
NVCC ?= /usr/local/cuda/bin/nvcc
PKG := paper_2410_12614_b200
LIB := $(PKG)/lib/libmpfem_b200.so
OBJDIR := $(PKG)/lib/obj
CU_SRCS := capi assembly_capi launch_geom launch_geom_box launch_fused launch_action launch_bounds geom_tensor assembly_host
CPP_SRCS := host_setup host_mesh
OBJS := $(addprefix $(OBJDIR)/,$(addsuffix .o,$(CU_SRCS) $(CPP_SRCS)))
HDRS := $(wildcard $(PKG)/csrc/*.cuh) $(wildcard $(PKG)/csrc/*.hpp) include/mpfem_b200.h
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-ffp-contract=off \
           --expt-relaxed-constexpr -Xptxas -v

all: $(LIB) oracle

# kernel_bounds on the GPU: binary64 without FMA contraction (the reference's roundings)
$(OBJDIR)/launch_bounds.o: $(PKG)/csrc/launch_bounds.cu $(HDRS)
	@mkdir -p $(OBJDIR)
	$(NVCC) $(NVFLAGS) --fmad=false -c -o $@ $< 2> $@.ptxas.log || (cat $@.ptxas.log; exit 1)

$(OBJDIR)/%.o: $(PKG)/csrc/%.cu $(HDRS)
	@mkdir -p $(OBJDIR)
	$(NVCC) $(NVFLAGS) -c -o $@ $< 2> $@.ptxas.log || (cat $@.ptxas.log; exit 1)

$(OBJDIR)/%.o: $(PKG)/csrc/%.cpp $(HDRS)
	@mkdir -p $(OBJDIR)
	$(NVCC) $(NVFLAGS) -c -o $@ $< 2> $@.ptxas.log || (cat $@.ptxas.log; exit 1)

$(LIB): $(OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS)
	cat $(OBJDIR)/*.ptxas.log > $(PKG)/lib/ptxas.log

oracle:
	$(MAKE) -s -C oracle all

# Diagnostic variant (not shipped): K2 epilogue without global stores, to separate the
# operand feed from the output write path. Load with MPFEM_B200_LIB=<path>.
DIAG_LIB := $(PKG)/lib/diag/libmpfem_b200_nostore.so
diag: $(OBJS)
	@mkdir -p $(PKG)/lib/diag
	$(NVCC) $(NVFLAGS) -DMPFEM_TC2_NOSTORE -c -o $(PKG)/lib/diag/capi.o $(PKG)/csrc/capi.cu 2> /dev/null
	$(NVCC) $(ARCH) -shared -o $(DIAG_LIB) $(PKG)/lib/diag/capi.o $(filter-out $(OBJDIR)/capi.o,$(OBJS))

clean:
	rm -rf $(LIB) $(OBJDIR)

.PHONY: all oracle clean diag
