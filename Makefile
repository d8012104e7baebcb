# librlb.so: the B200 (sm_100a) rollout data path behind include/rlb.h.
NVCC ?= /usr/local/cuda/bin/nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-Wall -Iinclude --expt-relaxed-constexpr
SRC_DIR := paper_2510_19225_b200/csrc
SRCS := $(wildcard $(SRC_DIR)/*.cu)
OBJS := $(patsubst $(SRC_DIR)/%.cu,build/%.o,$(SRCS))
LIB := paper_2510_19225_b200/librlb.so

all: $(LIB)

build/%.o: $(SRC_DIR)/%.cu $(SRC_DIR)/*.cuh $(SRC_DIR)/*.h include/rlb.h
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(LIB): $(OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS) -lcudart -ldl

clean:
	rm -rf build $(LIB)

.PHONY: all clean
