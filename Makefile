# Build of the in-tree native libraries (run by __graft_entry__.build()).
#   libpmg_cuda.so : the sm_100a solve path behind include/pmg_cuda.h
#   libiga_host.so : host discretization (input generation, include/iga_host.h)
#   libiga_pmg.so  : the C++ API (include/iga/pmg.hpp) over the C ABI
#   oracle         : CPU oracle (test infrastructure, oracle/_build)
# -fmad=false / -ffp-contract=off: no multiply-add contraction anywhere, so the kernels
# round exactly like the oracle.
NVCC     ?= /usr/local/cuda/bin/nvcc
CXX      ?= g++
PKG      := paper_1901_01685_b200
LIBDIR   := $(PKG)/lib
CU_SRC   := $(wildcard $(PKG)/csrc/cuda/*.cu)
CU_CPP   := $(wildcard $(PKG)/csrc/cuda/*.cpp)
CU_HDR   := $(wildcard $(PKG)/csrc/cuda/*.cuh) $(wildcard $(PKG)/csrc/cuda/*.hpp) include/pmg_cuda.h
HOST_SRC := $(wildcard $(PKG)/csrc/host/*.cpp)
API_SRC  := $(wildcard $(PKG)/csrc/api/*.cpp)
ARCH     := -gencode arch=compute_100a,code=sm_100a
NVFLAGS  := -std=c++17 -O3 -lineinfo $(ARCH) -fmad=false -Xcompiler -fPIC -Xcompiler -ffp-contract=off -Xptxas -v
CXXFLAGS := -std=c++20 -O2 -fPIC -ffp-contract=off -Wall -Wextra -Wno-unused-parameter

all: $(LIBDIR)/libpmg_cuda.so $(LIBDIR)/libiga_host.so $(LIBDIR)/libiga_pmg.so oracle

$(LIBDIR)/libpmg_cuda.so: $(CU_SRC) $(CU_CPP) $(CU_HDR)
	@mkdir -p $(LIBDIR) build/cuda
	$(NVCC) $(NVFLAGS) -shared -o $@ $(CU_SRC) $(CU_CPP) 2> build/cuda/ptxas.log || (cat build/cuda/ptxas.log; exit 1)

$(LIBDIR)/libiga_host.so: $(HOST_SRC) $(wildcard $(PKG)/csrc/host/*.hpp) include/iga_host.h
	@mkdir -p $(LIBDIR)
	$(CXX) $(CXXFLAGS) -shared -o $@ $(HOST_SRC) -lpthread

$(LIBDIR)/libiga_pmg.so: $(API_SRC) include/iga/pmg.hpp include/pmg_cuda.h include/iga_host.h $(LIBDIR)/libpmg_cuda.so $(LIBDIR)/libiga_host.so
	@mkdir -p $(LIBDIR)
	$(CXX) $(CXXFLAGS) -Iinclude -shared -o $@ $(API_SRC) -L$(LIBDIR) -lpmg_cuda -liga_host -Wl,-rpath,'$$ORIGIN'

oracle:
	$(MAKE) -C oracle

clean:
	rm -rf $(LIBDIR)/*.so build oracle/_build

.PHONY: all oracle clean
