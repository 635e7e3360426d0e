# Builds the sm_100a C-ABI library in-tree (paper_2212_13459_b200/libspst.so).
# Each translation unit compiles separately (make -j), then one link.
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
CSRC := paper_2212_13459_b200/csrc
UNITS := conv_tc gram_tc simt metrics first_bwd_tc api runtime
SRCS := $(addprefix $(CSRC)/,$(addsuffix .cu,$(UNITS)))
HDRS := $(CSRC)/common.cuh $(CSRC)/sm100.cuh include/spst.h
FLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Iinclude --expt-relaxed-constexpr
LIB := paper_2212_13459_b200/libspst.so
OBJDIR := build/obj$(if $(NAME),_$(NAME),)
OBJS := $(addprefix $(OBJDIR)/,$(addsuffix .o,$(UNITS)))

all: $(LIB)

$(OBJDIR)/%.o: $(CSRC)/%.cu $(HDRS)
	@mkdir -p $(OBJDIR)
	$(NVCC) $(FLAGS) $(XFLAGS) -c $< -o $@

$(LIB): $(OBJS)
	$(NVCC) $(ARCH) -shared $(OBJS) -o $@

# numerics variants for tools/error_budget.py:
#   make variant NAME=drain1 XFLAGS="-DSPST_CONV_DRAIN=1 -DSPST_CONV_DRAIN64=1"
variant: build/libspst_$(NAME).so
build/libspst_$(NAME).so: $(OBJS)
	$(NVCC) $(ARCH) -shared $(OBJS) -o $@

ptxas: $(SRCS)
	$(NVCC) $(FLAGS) -Xptxas -v -c $(CSRC)/conv_tc.cu -o /tmp/conv_tc.o 2>&1 | grep -E "registers|spill|smem" | head -20

clean:
	rm -rf $(LIB) build/obj*

.PHONY: all clean ptxas variant
