# Builds the B200-native hot-path library in-tree (the .so travels to the GPU
# box with the repo snapshot) and the oracle libraries under oracle/.
CUDA     ?= /usr/local/cuda
NVCC     ?= $(CUDA)/bin/nvcc
CXX      ?= g++
ARCH     := -gencode arch=compute_100a,code=sm_100a
PKG      := paper_1805_10167_b200
CSRC     := $(PKG)/csrc
BUILD    := build/obj
LIB      := $(PKG)/libhyteg_b200.so

# -fmad=false / -ffp-contract=off: every product and sum rounds separately, as
# in the reference's baseline x86-64 build (bitwise parity).
NVFLAGS  := $(ARCH) -O3 -lineinfo -fmad=false -std=c++17 -Xcompiler -fPIC -Xptxas -v
CXXFLAGS := -O2 -std=c++20 -fPIC -ffp-contract=off -Wall -Wextra -I$(CUDA)/include
LDFLAGS  := -shared -Wl,--no-undefined -static-libstdc++ -static-libgcc -Wl,--exclude-libs,ALL -L$(CUDA)/lib64 -lcudart_static -ldl -lpthread -lrt

HDRS := $(wildcard $(CSRC)/*.hpp) $(wildcard $(CSRC)/*.cuh) include/hyteg_b200.h
OBJS := $(BUILD)/kernels.o $(BUILD)/setup.o $(BUILD)/domain.o $(BUILD)/exchange.o $(BUILD)/plan.o $(BUILD)/coarse.o $(BUILD)/ops.o $(BUILD)/serialize.o $(BUILD)/stokes.o $(BUILD)/p2.o $(BUILD)/controller.o $(BUILD)/capi.o

.PHONY: all lib oracle clean
all: lib oracle

lib: $(LIB)

$(BUILD):
	mkdir -p $(BUILD)

$(BUILD)/kernels.o: $(CSRC)/kernels.cu $(HDRS) | $(BUILD)
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> $(BUILD)/ptxas.log || (cat $(BUILD)/ptxas.log; exit 1)

$(BUILD)/%.o: $(CSRC)/%.cpp $(HDRS) | $(BUILD)
	$(CXX) $(CXXFLAGS) -c $< -o $@

$(LIB): $(OBJS)
	$(CXX) -o $@ $(OBJS) $(LDFLAGS)

oracle:
	$(MAKE) -C oracle

clean:
	rm -rf build $(LIB)
	$(MAKE) -C oracle clean
