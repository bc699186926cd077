# Builds the sm_100a native library in-tree (travels to the GPU box with the snapshot).
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -Wall --expt-relaxed-constexpr
SRC := $(wildcard paper_1810_06860_b200/csrc/*.cu)
OBJ := $(patsubst paper_1810_06860_b200/csrc/%.cu,build/%.o,$(SRC))
LIB := paper_1810_06860_b200/_native/liblowrank_b200.so

all: $(LIB)

build/%.o: paper_1810_06860_b200/csrc/%.cu paper_1810_06860_b200/csrc/lr_common.cuh include/lowrank_b200.h
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(LIB): $(OBJ)
	@mkdir -p $(dir $(LIB))
	$(NVCC) $(ARCH) -shared -o $@ $(OBJ)

clean:
	rm -rf build $(LIB)

.PHONY: all clean
