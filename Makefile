# prism-b200 build: one shared library with the host C++ runtime, the C-ABI
# and the sm_100a kernels. No GPU is needed to build (nvcc cross-compiles).
#
#   make            -> paper_2505_04021_b200/libprism_b200.so
#   make oracle     -> oracle/_ref/* (reference + restatement; see oracle/Makefile)
#   make clean

CUDA      ?= /usr/local/cuda
NVCC      ?= $(CUDA)/bin/nvcc
CXX       ?= g++
PKG       := paper_2505_04021_b200
SRC       := $(PKG)/csrc
BUILD     := build
LIB       := $(PKG)/libprism_b200.so

ARCH      := -gencode arch=compute_100a,code=sm_100a
CXXFLAGS  := -std=c++20 -O2 -g -fPIC -Wall -Wextra -Wno-unused-parameter -DPRISM_PRODUCT \
             -Iinclude -I$(SRC) -I$(CUDA)/include -fvisibility=default
NVFLAGS   := -std=c++20 -O3 $(ARCH) -lineinfo -Xcompiler -fPIC -DPRISM_PRODUCT -Iinclude -I$(SRC) \
             --expt-relaxed-constexpr -Xptxas -v
LDFLAGS   := -shared -Xlinker -Bsymbolic-functions -Xlinker --no-undefined -lcudart_static -lrt -ldl -lpthread

HOST_SRCS := $(wildcard $(SRC)/host/*.cpp) $(SRC)/capi_host.cpp $(SRC)/capi_device.cpp $(SRC)/simcore.cpp
CU_SRCS   := $(wildcard $(SRC)/cuda/*.cu)
HOST_OBJS := $(patsubst $(SRC)/%.cpp,$(BUILD)/%.o,$(HOST_SRCS))
CU_OBJS   := $(patsubst $(SRC)/%.cu,$(BUILD)/%.o,$(CU_SRCS))
HEADERS   := $(wildcard include/*.h include/msim/*.hpp $(SRC)/*.hpp $(SRC)/host/*.hpp $(SRC)/cuda/*.cuh)

.PHONY: all oracle clean
all: $(LIB)
	$(MAKE) -C oracle

$(BUILD)/%.o: $(SRC)/%.cpp $(HEADERS)
	@mkdir -p $(dir $@)
	$(CXX) $(CXXFLAGS) -c $< -o $@

$(BUILD)/%.o: $(SRC)/%.cu $(HEADERS)
	@mkdir -p $(dir $@)
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> $@.ptxas.txt || (cat $@.ptxas.txt; false)

$(LIB): $(HOST_OBJS) $(CU_OBJS)
	$(NVCC) $(ARCH) -o $@ $^ $(LDFLAGS)

oracle: $(LIB)
	$(MAKE) -C oracle

clean:
	rm -rf $(BUILD) $(LIB)
	$(MAKE) -C oracle clean
