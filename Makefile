# Builds the sm_100a C-ABI library in-tree: paper_2211_15841_b200/libmoe.so
NVCC    ?= /usr/local/cuda/bin/nvcc
ARCH    := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := -O3 -std=c++17 -lineinfo $(ARCH) -Xcompiler -fPIC,-O3,-Wall -Xptxas -v --expt-relaxed-constexpr $(EXTRA)
SRCDIR  := paper_2211_15841_b200/csrc
SRCS    := $(wildcard $(SRCDIR)/*.cu)
OBJS    := $(patsubst $(SRCDIR)/%.cu,build/%.o,$(SRCS))
HDRS    := $(wildcard $(SRCDIR)/*.cuh) include/moe.h
LIB     := paper_2211_15841_b200/libmoe.so

all: $(LIB)

build/%.o: $(SRCDIR)/%.cu $(HDRS)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> build/$*.ptxas.log || (cat build/$*.ptxas.log; exit 1)

$(LIB): $(OBJS)
	$(NVCC) $(ARCH) -shared -cudart static -o $@ $(OBJS)

clean:
	rm -rf build $(LIB)

.PHONY: all clean
