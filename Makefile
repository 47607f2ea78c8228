# Builds the product library (sm_100a) and the CPU oracle (test infrastructure).
#   make            -> paper_1701_06600_b200/libcprand_b200.so + oracle/build/liborc.so
#   make lib        -> product only
NVCC     ?= /usr/local/cuda/bin/nvcc
ARCH     ?= -gencode arch=compute_100a,code=sm_100a
NVFLAGS  ?= -O3 -lineinfo -std=c++20 $(ARCH) -Xcompiler -fPIC,-O3 -Xptxas -v --expt-relaxed-constexpr
SRC_DIR  := paper_1701_06600_b200/csrc
OBJ_DIR  := build/obj
LIB      := paper_1701_06600_b200/libcprand_b200.so
SRCS     := $(wildcard $(SRC_DIR)/*.cu)
OBJS     := $(patsubst $(SRC_DIR)/%.cu,$(OBJ_DIR)/%.o,$(SRCS))
HDRS     := $(wildcard $(SRC_DIR)/*.cuh) $(wildcard $(SRC_DIR)/*.hpp) include/cprand_b200.h

all: lib oracle

lib: $(LIB)

$(OBJ_DIR)/%.o: $(SRC_DIR)/%.cu $(HDRS)
	@mkdir -p $(OBJ_DIR)
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> $@.log || (cat $@.log; exit 1)

$(LIB): $(OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS) -lnccl -lcudart

# device-check build (bounds asserts, flag-wait time-outs; tests/test_gpu_checked.py)
CHK_DIR  := build/objc
CHK_OBJS := $(patsubst $(SRC_DIR)/%.cu,$(CHK_DIR)/%.o,$(SRCS))
CHK_LIB  := paper_1701_06600_b200/libcprand_b200_check.so
checklib: $(CHK_LIB)
$(CHK_DIR)/%.o: $(SRC_DIR)/%.cu $(HDRS)
	@mkdir -p $(CHK_DIR)
	$(NVCC) $(NVFLAGS) -DCPB_DEVICE_CHECKS -c $< -o $@ 2> $@.log || (cat $@.log; exit 1)
$(CHK_LIB): $(CHK_OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(CHK_OBJS) -lnccl -lcudart
.PHONY: checklib

oracle:
	$(MAKE) -s -C oracle

clean:
	rm -rf build $(LIB)

.PHONY: all lib oracle clean

DROPIN := build/dropin_smoke
dropin: $(DROPIN)
$(DROPIN): tests/cpp/dropin_smoke.cpp include/cprand_b200/cprand.hpp $(LIB)
	@mkdir -p build
	g++ -std=c++20 -O2 -Iinclude -o $@ $< -Lpaper_1701_06600_b200 -lcprand_b200 -Wl,-rpath,'$$ORIGIN/../paper_1701_06600_b200'
.PHONY: dropin

CLI := build/cprand_b200
cli: $(CLI)
$(CLI): tools/cprand_b200_cli.cpp include/cprand_b200/cprand.hpp include/cprand_b200/io.hpp $(LIB)
	@mkdir -p build
	g++ -std=c++20 -O2 -Iinclude -o $@ $< -Lpaper_1701_06600_b200 -lcprand_b200 -Wl,-rpath,'$$ORIGIN/../paper_1701_06600_b200'
.PHONY: cli
