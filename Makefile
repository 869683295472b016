# Build of the B200-native anti-lopsided NNLS hot path.
#   make            -> paper_1502_01645_b200/lib/libalnnls.so (sm_100a kernels + C ABI)
#                      paper_1502_01645_b200/lib/libalnnls_gen.so (seeded input generator)
#                      oracle/ (test-only parity checkers, see oracle/Makefile)
#                      build/tests/facade_tests (C++ facade tests)
NVCC ?= /usr/local/cuda/bin/nvcc
CXX ?= g++
CC ?= gcc

PKG := paper_1502_01645_b200
LIB := $(PKG)/lib
ARCH := -gencode arch=compute_100a,code=sm_100a
# --fmad=false: no FMA contraction anywhere in the exact path
NVFLAGS := $(ARCH) -O3 -lineinfo --fmad=false -std=c++17 -Xcompiler -fPIC -Xptxas -v \
           -Xcompiler -Wall $(EXTRA)
CU_SRCS := $(PKG)/csrc/nqp.cu $(PKG)/csrc/setup.cu $(PKG)/csrc/capi.cu $(PKG)/csrc/batched.cu \
           $(PKG)/csrc/dmma.cu $(PKG)/csrc/fastloop.cu $(PKG)/csrc/small.cu
CU_HDRS := $(wildcard $(PKG)/csrc/*.cuh) include/alnnls.h
CU_OBJS := $(patsubst $(PKG)/csrc/%.cu,build/obj/%.o,$(CU_SRCS))

.PHONY: all lib gen oracle facade clean
all: lib gen oracle facade

lib: $(LIB)/libalnnls.so
gen: $(LIB)/libalnnls_gen.so

build/obj/%.o: $(PKG)/csrc/%.cu $(CU_HDRS)
	@mkdir -p build/obj
	$(NVCC) $(NVFLAGS) -c -o $@ $< 2> build/obj/$*.ptxas.log || (cat build/obj/$*.ptxas.log; false)

$(LIB)/libalnnls.so: $(CU_OBJS)
	@mkdir -p $(LIB)
	$(NVCC) $(ARCH) -shared -o $@ $(CU_OBJS) -lcudart_static -lrt -ldl -lpthread

$(LIB)/libalnnls_gen.so: $(PKG)/csrc/instgen.c
	@mkdir -p $(LIB)
	$(CC) -O2 -std=c11 -fPIC -shared -ffp-contract=off -o $@ $< -lm -pthread

oracle: lib gen
	$(MAKE) -C oracle

facade: build/tests/facade_tests

build/tests/facade_tests: tests/cpp/facade_tests.cpp $(wildcard include/antilop/*.hpp) include/alnnls.h $(LIB)/libalnnls.so
	@mkdir -p build/tests
	$(CXX) -O2 -std=c++20 -Iinclude -o $@ tests/cpp/facade_tests.cpp -L$(LIB) -lalnnls \
	  -Wl,-rpath,'$$ORIGIN/../../$(LIB)'

clean:
	rm -rf build $(LIB)
	$(MAKE) -C oracle clean
