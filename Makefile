# Build of the product library (sm_100a) and the test-only CPU checkers.
#
#   make            -> paper_2602_20826_b200/_lib/libdagsched_b200.so   (product)
#                      oracle/_build/libdagsched_oracle.so               (checker)
#                      oracle/_ref/libdagsched_ref.so  (only if /root/reference exists)
# nvcc cross-compiles for sm_100a here; no GPU is needed to build.

NVCC    ?= /usr/local/cuda/bin/nvcc
CXX     ?= g++
ARCH    := -gencode arch=compute_100a,code=sm_100a
PKG     := paper_2602_20826_b200
LIBDIR  := $(PKG)/_lib
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-fvisibility=hidden -Xptxas -v --expt-relaxed-constexpr
CXXFLAGS:= -std=c++17 -O3 -fPIC -fopenmp -fvisibility=hidden -I/usr/local/cuda/include -Wall -Wno-comment
LDOMP   := -L/usr/lib/gcc/x86_64-linux-gnu/13 -lgomp -lpthread

CU_OBJS := $(LIBDIR)/capi.o $(LIBDIR)/k1_main.o $(LIBDIR)/k1_detail.o $(LIBDIR)/k3_executor.o
CU_DEPS := $(wildcard $(PKG)/csrc/*.cuh) $(wildcard $(PKG)/csrc/*.h) include/dagsched_b200.h

.PHONY: all product oracle ref clean
all: product oracle ref

product: $(LIBDIR)/libdagsched_b200.so

$(LIBDIR)/%.o: $(PKG)/csrc/%.cu $(CU_DEPS) $(PKG)/csrc/k1_main.cu
	@mkdir -p $(LIBDIR)
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> $(LIBDIR)/ptxas_$*.txt || (cat $(LIBDIR)/ptxas_$*.txt; false)

$(LIBDIR)/host_gen.o: $(PKG)/csrc/host_gen.cpp include/dagsched_b200.h
	@mkdir -p $(LIBDIR)
	$(CXX) $(CXXFLAGS) -c $< -o $@

$(LIBDIR)/libdagsched_b200.so: $(CU_OBJS) $(LIBDIR)/host_gen.o
	$(NVCC) $(ARCH) -shared -o $@ $^ -Xlinker --exclude-libs,ALL $(LDOMP)

oracle:
	$(MAKE) -C oracle oracle

ref:
	@if [ -d /root/reference/proj ]; then $(MAKE) -C oracle ref; else echo "no /root/reference: using prebuilt oracle/_ref if present"; fi

clean:
	rm -rf $(LIBDIR)
	$(MAKE) -C oracle clean
