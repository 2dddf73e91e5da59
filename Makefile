# graphvx-b200 build: sm_100a device runtime + C++ graph API + C facade.
# Everything builds in-tree (the .so files travel with the repo snapshot).

CUDA_HOME ?= /usr/local/cuda
NVCC      ?= $(CUDA_HOME)/bin/nvcc
CXX       ?= g++
PKG       := paper_2008_11476_b200
LIB       := $(PKG)/lib
ARCH      := -gencode arch=compute_100a,code=sm_100a

NVCCFLAGS := $(ARCH) -lineinfo -O3 -std=c++17 -Xcompiler -fPIC -Iinclude -I$(PKG)/csrc/cuda \
             -Xptxas -v --resource-usage
CXXFLAGS  := -std=c++20 -O2 -fPIC -ffp-contract=off -Wall -Wextra -Wno-unused-parameter -Iinclude \
             -I$(CUDA_HOME)/include

CUDA_SRC  := $(wildcard $(PKG)/csrc/cuda/*.cu)
CUDA_OBJ  := $(patsubst $(PKG)/csrc/cuda/%.cu,build/cuda/%.o,$(CUDA_SRC))
HOST_SRC  := $(wildcard $(PKG)/csrc/host/*.cpp)
HOST_OBJ  := $(patsubst $(PKG)/csrc/host/%.cpp,build/host/%.o,$(HOST_SRC))
CAPI_SRC  := $(wildcard $(PKG)/csrc/capi/*.cpp)
CAPI_OBJ  := $(patsubst $(PKG)/csrc/capi/%.cpp,build/capi/%.o,$(CAPI_SRC))

all: $(LIB)/libgvx_cuda.so $(LIB)/libgraphvx.so tests/cpp/bin/test_graphvx

build/cuda/%.o: $(PKG)/csrc/cuda/%.cu $(wildcard $(PKG)/csrc/cuda/*.cuh) include/gvxb.h
	@mkdir -p build/cuda
	$(NVCC) $(NVCCFLAGS) -c $< -o $@ 2> build/cuda/$*.ptxas.log || (cat build/cuda/$*.ptxas.log; false)

$(LIB)/libgvx_cuda.so: $(CUDA_OBJ)
	@mkdir -p $(LIB)
	$(NVCC) $(ARCH) -shared -Xcompiler -fPIC $^ -o $@ -L$(CUDA_HOME)/lib64 -lnvrtc -ldl \
	    -Xlinker -rpath,$(CUDA_HOME)/lib64

build/host/%.o: $(PKG)/csrc/host/%.cpp $(wildcard include/graphvx/*.hpp) $(wildcard $(PKG)/csrc/host/*.hpp) include/gvxb.h
	@mkdir -p build/host
	$(CXX) $(CXXFLAGS) -c $< -o $@

build/capi/%.o: $(PKG)/csrc/capi/%.cpp $(wildcard include/graphvx/*.hpp) $(wildcard include/*.h)
	@mkdir -p build/capi
	$(CXX) $(CXXFLAGS) -I$(PKG)/csrc/host -c $< -o $@

$(LIB)/libgraphvx.so: $(HOST_OBJ) $(CAPI_OBJ) $(LIB)/libgvx_cuda.so
	$(CXX) -shared $(HOST_OBJ) $(CAPI_OBJ) -o $@ -L$(LIB) -lgvx_cuda -Wl,-rpath,'$$ORIGIN' -lpthread

clean:
	rm -rf build $(LIB)/*.so

.PHONY: all clean

# C++ API / fusion tests (doctest stand-in); pytest runs them
tests/cpp/bin/test_graphvx: tests/cpp/test_graphvx.cpp tests/cpp/doctest.h $(LIB)/libgraphvx.so $(PKG)/csrc/configs/config_graphs.hpp
	@mkdir -p tests/cpp/bin
	$(CXX) -std=c++20 -O1 -Iinclude -Itests/cpp $< -o $@ -L$(LIB) -lgraphvx -Wl,-rpath,'$$ORIGIN/../../../$(LIB)'

tests: tests/cpp/bin/test_graphvx
.PHONY: tests
