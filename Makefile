# Builds the product (libcarve_cuda.so, sm_100a only), the drop-in C++ tools,
# and the CPU checkers under oracle/ (test infrastructure).
NVCC ?= nvcc
CXX ?= g++
ARCH := -gencode arch=compute_100a,code=sm_100a
# -fmad=false: no FMA contraction anywhere (FP64 bit-exactness)
NVFLAGS := -O3 -std=c++17 $(ARCH) -lineinfo -fmad=false -Xcompiler -fPIC -Xptxas -v -Iinclude
PKG := paper_2410_21207_b200
LIB := $(PKG)/libcarve_cuda.so
# the DP variant instances compile in their own translation units (in parallel: make -j)
SRCS := $(PKG)/csrc/carve_cuda.cu $(PKG)/csrc/dp_variants_a.cu $(PKG)/csrc/dp_variants_b.cu $(PKG)/csrc/dp_variants_c.cu \
        $(PKG)/csrc/dp_variants_d.cu
OBJS := $(patsubst $(PKG)/csrc/%.cu,build/%.o,$(SRCS))
HDR := $(wildcard $(PKG)/csrc/*.cuh) $(wildcard $(PKG)/csrc/*.h) include/carve_cuda.h

all: $(LIB) oracle tools

build/%.o: $(PKG)/csrc/%.cu $(HDR) | build
	$(NVCC) $(NVFLAGS) -c -o $@ $< 2> build/$*.ptxas.log || (cat build/$*.ptxas.log; false)

$(LIB): $(OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS)
	cat build/*.ptxas.log > build/ptxas.log

build:
	@mkdir -p build

$(LIB): | build

tools: build/carve build/carve_parity

build/carve: tools/carve_main.cpp $(wildcard include/carve/*.hpp) $(LIB) | build
	$(CXX) -std=c++20 -O2 -Iinclude -o $@ tools/carve_main.cpp -L$(PKG) -lcarve_cuda -lz -Wl,-rpath,'$$ORIGIN/../$(PKG)'

build/carve_parity: tools/carve_parity.cpp $(wildcard include/carve/*.hpp) $(LIB) | build
	$(CXX) -std=c++20 -O2 -Iinclude -o $@ tools/carve_parity.cpp -L$(PKG) -lcarve_cuda -lz -Wl,-rpath,'$$ORIGIN/../$(PKG)'

oracle:
	$(MAKE) -s -C oracle

clean:
	rm -rf build $(LIB)
	$(MAKE) -s -C oracle clean

.PHONY: all oracle tools clean
