# Builds the in-tree C-ABI library paper_2605_11517_b200/libgrinder_b200.so
# (sm_100a kernels + host preprocessing) and the oracle's C helpers.
NVCC ?= /usr/local/cuda/bin/nvcc
CXX ?= g++
PKG := paper_2605_11517_b200
SRC := $(PKG)/csrc
OUT := $(PKG)/libgrinder_b200.so
BUILD := build
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-fopenmp -Xptxas -v
CXXFLAGS := -O3 -std=c++17 -fPIC -fopenmp -ffp-contract=off -Wall -Wno-unused-function

CU_SRCS := $(wildcard $(SRC)/*.cu)
CPP_SRCS := $(wildcard $(SRC)/*.cpp)
OBJS := $(patsubst $(SRC)/%.cu,$(BUILD)/%.cu.o,$(CU_SRCS)) $(patsubst $(SRC)/%.cpp,$(BUILD)/%.cpp.o,$(CPP_SRCS))

all: $(OUT)

$(BUILD)/%.cu.o: $(SRC)/%.cu $(SRC)/*.h include/grinder_b200.h | $(BUILD)
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> $(BUILD)/$*.ptxas.txt || (cat $(BUILD)/$*.ptxas.txt; false)

$(BUILD)/%.cpp.o: $(SRC)/%.cpp $(SRC)/*.h include/grinder_b200.h | $(BUILD)
	$(CXX) $(CXXFLAGS) -I/usr/local/cuda/include -c $< -o $@

$(OUT): $(OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS) -Xcompiler -fopenmp -lgomp

$(BUILD):
	mkdir -p $(BUILD)

clean:
	rm -rf $(BUILD) $(OUT)

.PHONY: all clean
