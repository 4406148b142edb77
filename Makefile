# Builds the device library, the host C++ library and the test oracle.
#   make            -> paper_2507_14051_b200/lib/librhp_cuda.so, librhpdhg.so, oracle/liboracle.so
#   make ref        -> oracle/_ref/librhpdhg_ref.so (needs /root/reference; test infrastructure)
NVCC     ?= /usr/local/cuda/bin/nvcc
CXX      := /usr/bin/g++  # the system toolchain nvcc also uses (one libstdc++ per process)
PKG      := paper_2507_14051_b200
LIB      := $(PKG)/lib
ARCH     := -gencode arch=compute_100a,code=sm_100a
NVFLAGS  := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Iinclude -Xptxas -v \
            --expt-relaxed-constexpr -DRHP_WITH_NCCL
CXXFLAGS := -std=c++20 -O2 -fPIC -Wall -Wextra -Iinclude -I$(PKG)/host -isystem /usr/local/cuda/include

CU_SRCS  := $(PKG)/csrc/rhp_cuda.cu $(PKG)/csrc/layout.cu $(PKG)/csrc/ingest.cu $(PKG)/csrc/segments.cu $(PKG)/csrc/ops.cu
CU_HDRS  := $(wildcard $(PKG)/csrc/*.cuh) include/rhpdhg_cuda.h include/rhpdhg_c.h
HOST_SRCS:= $(wildcard $(PKG)/host/*.cpp)
HOST_HDRS:= $(wildcard $(PKG)/host/*.hpp) $(wildcard include/rhpdhg/*.hpp) include/rhpdhg_c.h include/rhpdhg_cuda.h

.PHONY: all oracle ref clean
all: $(LIB)/librhp_cuda.so $(LIB)/librhpdhg.so oracle

$(LIB)/librhp_cuda.so: $(CU_SRCS) $(CU_HDRS)
	@mkdir -p $(LIB)
	$(NVCC) $(NVFLAGS) -shared -o $@ $(CU_SRCS) -ldl 2> $(LIB)/ptxas.log || (cat $(LIB)/ptxas.log; exit 1)

$(LIB)/librhpdhg.so: $(HOST_SRCS) $(HOST_HDRS) $(LIB)/librhp_cuda.so
	$(CXX) $(CXXFLAGS) -shared -o $@ $(HOST_SRCS) -L$(LIB) -lrhp_cuda -lz -ldl -pthread -Wl,-rpath,'$$ORIGIN'

oracle:
	$(MAKE) -C oracle oracle

ref:
	$(MAKE) -C oracle ref

clean:
	rm -f $(LIB)/*.so $(LIB)/ptxas.log
	$(MAKE) -C oracle clean
