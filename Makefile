# Native build of the sidecar data plane (sm_100a only).
#   make            libfsx.so (+ SASS/resource report in build/)
#   make oracle     checker libraries (oracle/Makefile)
NVCC ?= /usr/local/cuda/bin/nvcc
CXX ?= g++
ARCH := -gencode arch=compute_100a,code=sm_100a
PKG := paper_2603_12118_b200
CSRC := $(PKG)/csrc
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-Wall -Iinclude -I$(CSRC) \
           -Xptxas -v -cudart static
LIB := $(PKG)/libfsx.so
OBJS := build/fsx_kernels.o build/fsx_runtime.o

all: $(LIB)

build:
	mkdir -p build

build/fsx_kernels.o: $(CSRC)/fsx_kernels.cu $(CSRC)/fsx_kernels.cuh include/fsx.h | build
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> build/fsx_kernels.ptxas.txt || { cat build/fsx_kernels.ptxas.txt; exit 1; }

build/fsx_runtime.o: $(CSRC)/fsx_runtime.cu $(CSRC)/fsx_kernels.cuh include/fsx.h | build
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> build/fsx_runtime.ptxas.txt || { cat build/fsx_runtime.ptxas.txt; exit 1; }

$(LIB): $(OBJS)
	$(NVCC) $(ARCH) -shared -cudart static -o $@ $(OBJS)

oracle:
	$(MAKE) -C oracle all

sass: $(LIB)
	/usr/local/cuda/bin/cuobjdump -sass $(LIB) > build/libfsx.sass.txt

clean:
	rm -rf build $(LIB)

.PHONY: all oracle sass clean
