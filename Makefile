# Builds the product libraries in-tree (they travel to the GPU box with the
# gpurun snapshot; *.so is git-ignored):
#
#   paper_1508_05488_b200/libchgpu.so     C ABI (include/chgpu.h): sm_100a kernels
#                                          + host finisher + generator
#   paper_1508_05488_b200/libchainhull.so  the reference's C++ API
#                                          (include/chainhull/*.hpp) over libchgpu
#   build/chainhull                        the reference CLI (hull/gen/verify/bench)
#                                          over libchainhull
#   build/acceptance_b200                  the reference acceptance gate relinked
#                                          against libchainhull (only when
#                                          /root/reference is present)
#
# Device code: -fmad=false keeps cross() free of FMA contraction (the
# predicate also spells out __dmul_rn/__dsub_rn); host finisher code:
# -ffp-contract=off for the same reason.

NVCC     ?= /usr/local/cuda/bin/nvcc
CXX      ?= g++
ARCH     := -gencode arch=compute_100a,code=sm_100a
PKG      := paper_1508_05488_b200
CSRC     := $(PKG)/csrc
BUILD    := build
NVFLAGS  := $(ARCH) -O3 -lineinfo -fmad=false -std=c++17 -Xcompiler -fPIC -Iinclude -I$(CSRC) \
            -Xptxas -warn-spills
CXXFLAGS := -O3 -std=gnu++20 -fPIC -ffp-contract=off -Wall -Wextra -Iinclude -I$(CSRC) \
            -I/usr/local/cuda/include
REF      ?= /root/reference/proj

CU_SRCS  := $(CSRC)/k_discard.cu $(CSRC)/k_sort.cu $(CSRC)/k_spa.cu \
            $(CSRC)/k_filter.cu $(CSRC)/k_convex.cu \
            $(CSRC)/pipeline.cu
CXX_SRCS := $(CSRC)/finisher.cpp $(CSRC)/datasets.cpp
CU_OBJS  := $(patsubst $(CSRC)/%.cu,$(BUILD)/%.o,$(CU_SRCS))
CXX_OBJS := $(patsubst $(CSRC)/%.cpp,$(BUILD)/%.o,$(CXX_SRCS))
HDRS     := $(wildcard $(CSRC)/*.h $(CSRC)/*.cuh include/*.h)

API_SRCS := $(wildcard $(PKG)/cpp/*.cpp)
API_OBJS := $(patsubst $(PKG)/cpp/%.cpp,$(BUILD)/api_%.o,$(API_SRCS))
API_HDRS := $(wildcard include/chainhull/*.hpp)

all: $(PKG)/libchgpu.so $(PKG)/libchainhull.so acceptance $(BUILD)/io_probe_b200 $(BUILD)/chainhull

$(BUILD)/%.o: $(CSRC)/%.cu $(HDRS)
	@mkdir -p $(BUILD)
	$(NVCC) $(NVFLAGS) -c -o $@ $<

$(BUILD)/%.o: $(CSRC)/%.cpp $(HDRS)
	@mkdir -p $(BUILD)
	$(CXX) $(CXXFLAGS) -c -o $@ $<

$(PKG)/libchgpu.so: $(CU_OBJS) $(CXX_OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $^ -Xlinker -soname=libchgpu.so

$(BUILD)/api_%.o: $(PKG)/cpp/%.cpp $(API_HDRS) include/chgpu.h
	@mkdir -p $(BUILD)
	$(CXX) $(CXXFLAGS) -c -o $@ $<

$(PKG)/libchainhull.so: $(API_OBJS) $(PKG)/libchgpu.so
	$(CXX) -shared -o $@ $(API_OBJS) -L$(PKG) -lchgpu -Wl,-rpath,'$$ORIGIN' -lpthread

ifneq ($(wildcard $(REF)/tests/acceptance.cpp),)
acceptance: $(BUILD)/acceptance_b200
$(BUILD)/acceptance_b200: $(REF)/tests/acceptance.cpp $(PKG)/libchainhull.so $(API_HDRS)
	$(CXX) -O3 -std=gnu++20 -ffp-contract=off -Iinclude -I$(REF)/tests -o $@ $< \
	  -L$(PKG) -lchainhull -lchgpu -Wl,-rpath,'$$ORIGIN/../$(PKG)' -lpthread
else
acceptance:
	@echo "acceptance: /root/reference absent; using prebuilt build/acceptance_b200 if any"
endif

# I/O parity probe against the drop-in (tests/test_io_parity.py).
$(BUILD)/io_probe_b200: tests/io_probe.cpp $(PKG)/libchainhull.so $(API_HDRS)
	$(CXX) -O2 -std=gnu++20 -ffp-contract=off -Iinclude -o $@ $< \
	  -L$(PKG) -lchainhull -lchgpu -Wl,-rpath,'$$ORIGIN/../$(PKG)' -lpthread

# The reference command line (tools/src/main.cpp) over the drop-in.
$(BUILD)/chainhull: $(PKG)/tools/chainhull_cli.cpp $(PKG)/libchainhull.so $(API_HDRS)
	$(CXX) -O2 -std=gnu++20 -Wall -Wextra -Iinclude -o $@ $< \
	  -L$(PKG) -lchainhull -lchgpu -Wl,-rpath,'$$ORIGIN/../$(PKG)' -lpthread

sass: $(PKG)/libchgpu.so
	/usr/local/cuda/bin/cuobjdump -sass $< > $(BUILD)/libchgpu.sass

clean:
	rm -rf $(BUILD) $(PKG)/libchgpu.so $(PKG)/libchainhull.so

.PHONY: all acceptance sass clean
