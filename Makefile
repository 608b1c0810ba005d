# Builds the sm_100a C-ABI library (in-tree so it travels with gpurun) and the
# oracle helpers.  `python -c "import __graft_entry__ as g; g.build()"` runs it.
NVCC ?= /usr/local/cuda/bin/nvcc
CSRC := paper_2510_02080_b200/csrc
LIB := paper_2510_02080_b200/libec3r_b200.so
SRCS := $(wildcard $(CSRC)/*.cu)
OBJS := $(patsubst $(CSRC)/%.cu,build/%.o,$(SRCS))
HDRS := $(wildcard $(CSRC)/*.cuh) include/ec3r_b200.h
NVFLAGS := -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
           -Xcompiler -fPIC -Xcompiler -fvisibility=hidden --expt-relaxed-constexpr \
           -Iinclude -Xptxas -warn-spills

all: $(LIB)

build/%.o: $(CSRC)/%.cu $(HDRS)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -dc -c $< -o $@

$(LIB): $(OBJS)
	$(NVCC) -gencode arch=compute_100a,code=sm_100a -shared -o $@ $(OBJS) -lcudart_static -lrt -ldl -lpthread

clean:
	rm -rf build $(LIB)

.PHONY: all clean
