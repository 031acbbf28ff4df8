# Builds the in-tree C-ABI library paper_1703_01175_b200/libh2b.so for sm_100a (B200).
# One object per CUDA source (compiled in parallel with -j), linked into one shared library.
NVCC ?= /usr/local/cuda/bin/nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := -O3 -std=c++17 -lineinfo --extended-lambda $(ARCH) -Xcompiler -fPIC,-O3,-Wall -Xptxas -v
SRC := $(wildcard paper_1703_01175_b200/csrc/*.cu)
HDR := $(wildcard paper_1703_01175_b200/csrc/*.cuh) $(wildcard paper_1703_01175_b200/csrc/*.inc) include/h2b.h
OBJ := $(patsubst paper_1703_01175_b200/csrc/%.cu,build/%.o,$(SRC))
LIB := paper_1703_01175_b200/libh2b.so

all: $(LIB)

build/%.o: paper_1703_01175_b200/csrc/%.cu $(HDR) | build
	$(NVCC) $(NVFLAGS) -c -o $@ $< 2> build/$*.ptxas.log || (cat build/$*.ptxas.log; false)

$(LIB): $(OBJ)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJ)
	cat build/*.ptxas.log > build/ptxas.log

build:
	mkdir -p build

clean:
	rm -f $(LIB) build/*.o
.PHONY: all clean
