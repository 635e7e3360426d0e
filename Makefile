# Builds the sm_100a C-ABI library in-tree (paper_2212_13459_b200/libspst.so).
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
CSRC := paper_2212_13459_b200/csrc
SRCS := $(CSRC)/conv_tc.cu $(CSRC)/gram_tc.cu $(CSRC)/simt.cu $(CSRC)/metrics.cu $(CSRC)/first_bwd_tc.cu $(CSRC)/runtime.cu
FLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Iinclude --expt-relaxed-constexpr
LIB := paper_2212_13459_b200/libspst.so

all: $(LIB)

$(LIB): $(SRCS) $(CSRC)/common.cuh $(CSRC)/sm100.cuh include/spst.h
	$(NVCC) $(FLAGS) -shared $(SRCS) -o $@

ptxas: $(SRCS)
	$(NVCC) $(FLAGS) -Xptxas -v -c $(CSRC)/conv_tc.cu -o /tmp/conv_tc.o 2>&1 | grep -E "registers|spill|smem" | head -20

clean:
	rm -f $(LIB)

.PHONY: all clean ptxas
