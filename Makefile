# Builds the B200 product library (sm_100a only) and the CPU oracle.
#   make            -> paper_2212_14318_b200/libqtensor_b200.so + oracle/liboracle.so
#   make ref        -> oracle/_ref/* (needs /root/reference; test infrastructure only)
NVCC      ?= nvcc
ARCH      := -gencode arch=compute_100a,code=sm_100a
NVFLAGS   := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -Wall --expt-relaxed-constexpr
PKG       := paper_2212_14318_b200
CSRC      := $(PKG)/csrc
LIB       := $(PKG)/libqtensor_b200.so
OBJDIR    := build/obj
SRCS_CU   := $(CSRC)/qt_fft.cu $(CSRC)/qt_gemm.cu $(CSRC)/qt_ozaki.cu $(CSRC)/qt_naive.cu $(CSRC)/qt_io.cu $(CSRC)/qt_api.cu $(CSRC)/qt_multi.cu $(CSRC)/qt_nccl.cu $(CSRC)/qt_rank.cu $(CSRC)/qt_small.cu
SRCS_CPP  := $(CSRC)/qt_rng.cpp
OBJS      := $(patsubst $(CSRC)/%.cu,$(OBJDIR)/%.o,$(SRCS_CU)) $(patsubst $(CSRC)/%.cpp,$(OBJDIR)/%.o,$(SRCS_CPP))

all: $(LIB) oracle

$(OBJDIR)/%.o: $(CSRC)/%.cu $(CSRC)/qt_internal.cuh $(CSRC)/qt_dmma_tile.cuh $(CSRC)/qt_fft_reg.cuh $(CSRC)/qt_nccl.h include/qtensor_b200.h
	@mkdir -p $(OBJDIR)
	$(NVCC) $(NVFLAGS) -Xptxas -v -c $< -o $@ 2> $(OBJDIR)/$*.ptxas.txt || (cat $(OBJDIR)/$*.ptxas.txt; false)

$(OBJDIR)/%.o: $(CSRC)/%.cpp include/qtensor_b200.h
	@mkdir -p $(OBJDIR)
	g++ -O3 -std=c++17 -fPIC -Wall -c $< -o $@

$(LIB): $(OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS) -ldl -lpthread

oracle:
	$(MAKE) -C oracle

ref:
	$(MAKE) -C oracle ref

clean:
	rm -rf build $(LIB)
	$(MAKE) -C oracle clean

.PHONY: all oracle ref clean
