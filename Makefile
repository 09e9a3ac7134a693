# Builds libdpipe.so (sm_100a kernels + C ABI) in-tree so it travels with gpurun snapshots.
NVCC ?= /usr/local/cuda/bin/nvcc
PKG := paper_2405_01248_b200
SRC := $(wildcard $(PKG)/csrc/*.cu)
OBJ := $(patsubst $(PKG)/csrc/%.cu,build/%.o,$(SRC))
HDR := $(wildcard $(PKG)/csrc/*.cuh) include/dpipe.h
LIB := $(PKG)/libdpipe.so

NVFLAGS := -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
           -Xcompiler -fPIC -Iinclude -I$(PKG)/csrc --expt-relaxed-constexpr -Xptxas -v

all: $(LIB)

build/%.o: $(PKG)/csrc/%.cu $(HDR)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> build/$*.ptxas.log || (cat build/$*.ptxas.log; false)

$(LIB): $(OBJ)
	$(NVCC) -shared -gencode arch=compute_100a,code=sm_100a -o $@ $(OBJ)

clean:
	rm -rf build $(LIB)

.PHONY: all clean
