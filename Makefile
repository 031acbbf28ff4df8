# Builds the in-tree C-ABI library paper_1703_01175_b200/libh2b.so for sm_100a (B200).
NVCC ?= /usr/local/cuda/bin/nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := -O3 -std=c++17 -lineinfo --extended-lambda $(ARCH) -Xcompiler -fPIC,-O3,-Wall -Xptxas -v
SRC := $(wildcard paper_1703_01175_b200/csrc/*.cu)
HDR := $(wildcard paper_1703_01175_b200/csrc/*.cuh) include/h2b.h
LIB := paper_1703_01175_b200/libh2b.so

all: $(LIB)

$(LIB): $(SRC) $(HDR)
	$(NVCC) $(NVFLAGS) -shared -o $@ $(SRC) 2> build/ptxas.log || (cat build/ptxas.log; false)

$(SRC): | build
build:
	mkdir -p build

clean:
	rm -f $(LIB)
.PHONY: all clean
