# gdi-b200 build: sm_100a kernels + C ABI (libgdi.so), the C++ solver API
# (libising.so) and the pyising binding, all in-tree so the .so files travel
# with the gpurun snapshot. `make oracle` builds the test-only checkers.

PKG      := paper_1908_00210_b200
CSRC     := $(PKG)/csrc
LIBDIR   := $(PKG)/lib
BUILD    := build
NVCC     ?= nvcc
CXX      ?= g++
ARCH     := -gencode arch=compute_100a,code=sm_100a
NVFLAGS  := -std=c++17 $(ARCH) -lineinfo -O3 -Xcompiler -fPIC -Xcompiler -Wall -Iinclude -I$(CSRC)
CXXFLAGS := -std=c++20 -O3 -fPIC -Wall -Wextra -Iinclude -I$(CSRC)
PYINC    := $(shell python3 -m pybind11 --includes)
PYEXT    := $(shell python3-config --extension-suffix)

CU_SRC   := $(wildcard $(CSRC)/*.cu)
CU_OBJ   := $(patsubst $(CSRC)/%.cu,$(BUILD)/%.o,$(CU_SRC))
HOST_SRC := $(wildcard $(CSRC)/host/*.cpp)
HOST_OBJ := $(patsubst $(CSRC)/host/%.cpp,$(BUILD)/host/%.o,$(HOST_SRC))
CU_HDR   := $(wildcard $(CSRC)/*.cuh) $(wildcard $(CSRC)/*.hpp) include/gdi.h
HOST_HDR := $(wildcard include/ising/*.hpp) $(wildcard $(CSRC)/host/*.hpp) include/gdi.h

LIBGDI   := $(LIBDIR)/libgdi.so
LIBISING := $(LIBDIR)/libising.so
PYMOD    := $(PKG)/pyising$(PYEXT)

.PHONY: all oracle clean sass

all: $(LIBGDI) $(LIBISING) $(PYMOD)

$(BUILD)/%.o: $(CSRC)/%.cu $(CU_HDR)
	@mkdir -p $(dir $@)
	$(NVCC) $(NVFLAGS) -Xptxas -v -c $< -o $@ 2> $(BUILD)/$*.ptxas.txt || (cat $(BUILD)/$*.ptxas.txt; exit 1)

$(LIBGDI): $(CU_OBJ)
	@mkdir -p $(LIBDIR)
	$(NVCC) $(ARCH) -shared -cudart static -o $@ $^

$(BUILD)/host/%.o: $(CSRC)/host/%.cpp $(HOST_HDR)
	@mkdir -p $(dir $@)
	$(CXX) $(CXXFLAGS) -c $< -o $@

$(LIBISING): $(HOST_OBJ) $(LIBGDI)
	$(CXX) -shared -o $@ $(HOST_OBJ) -L$(LIBDIR) -lgdi -Wl,-rpath,'$$ORIGIN'

$(PYMOD): $(CSRC)/python/pyising.cpp $(HOST_HDR) $(LIBISING)
	$(CXX) $(CXXFLAGS) $(PYINC) -shared $< -o $@ -L$(LIBDIR) -lising -lgdi -Wl,-rpath,'$$ORIGIN/lib'

oracle:
	$(MAKE) -C oracle all

sass: $(LIBGDI)
	cuobjdump -sass $(LIBGDI) > $(BUILD)/libgdi.sass

clean:
	rm -rf $(BUILD) $(LIBDIR) $(PKG)/pyising*.so
