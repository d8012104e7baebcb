# librlb.so: the B200 (sm_100a) rollout data path behind include/rlb.h.
# `make checked`: librlb_checked.so with device-side bounds checks (RLB_CHECKED)
NVCC ?= /usr/local/cuda/bin/nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-Wall -Iinclude --expt-relaxed-constexpr
SRC_DIR := paper_2510_19225_b200/csrc
SRCS := $(wildcard $(SRC_DIR)/*.cu)
OBJS := $(patsubst $(SRC_DIR)/%.cu,build/%.o,$(SRCS))
COBJS := $(patsubst $(SRC_DIR)/%.cu,build/checked/%.o,$(SRCS))
LIB := paper_2510_19225_b200/librlb.so
CLIB := paper_2510_19225_b200/librlb_checked.so

all: $(LIB)

checked: $(CLIB)

build/%.o: $(SRC_DIR)/%.cu $(SRC_DIR)/*.cuh $(SRC_DIR)/*.h include/rlb.h
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c $< -o $@

build/checked/%.o: $(SRC_DIR)/%.cu $(SRC_DIR)/*.cuh $(SRC_DIR)/*.h include/rlb.h
	@mkdir -p build/checked
	$(NVCC) $(NVFLAGS) -DRLB_CHECKED -c $< -o $@

$(LIB): $(OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS) -lcudart -ldl

$(CLIB): $(COBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(COBJS) -lcudart -ldl

clean:
	rm -rf build $(LIB) $(CLIB)

.PHONY: all checked clean
