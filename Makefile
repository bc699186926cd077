# Builds the sm_100a native library in-tree (travels to the GPU box with the snapshot).
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -Wall --expt-relaxed-constexpr
SRC := $(wildcard paper_1810_06860_b200/csrc/*.cu)
CSRC := $(wildcard paper_1810_06860_b200/csrc/*.c)
OBJ := $(patsubst paper_1810_06860_b200/csrc/%.cu,build/%.o,$(SRC)) $(patsubst paper_1810_06860_b200/csrc/%.c,build/%.c.o,$(CSRC))
# host C (the parity Omega's uniforms / Box-Muller): strict IEEE, numpy's operation order
CFLAGS_HOST := -O2 -fPIC -fno-fast-math -ffp-contract=off -Wall
LIB := paper_1810_06860_b200/_native/liblowrank_b200.so

all: $(LIB)

build/%.o: paper_1810_06860_b200/csrc/%.cu paper_1810_06860_b200/csrc/lr_common.cuh include/lowrank_b200.h
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c $< -o $@

build/%.c.o: paper_1810_06860_b200/csrc/%.c
	@mkdir -p build
	$(CC) $(CFLAGS_HOST) -c $< -o $@

$(LIB): $(OBJ)
	@mkdir -p $(dir $(LIB))
	$(NVCC) $(ARCH) -shared -o $@ $(OBJ) -lm

clean:
	rm -rf build $(LIB)

.PHONY: all clean
