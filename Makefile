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

CU_OBJS := $(LIBDIR)/capi.o $(LIBDIR)/k1_main.o $(LIBDIR)/k1_detail.o $(LIBDIR)/k1_small.o $(LIBDIR)/k3_executor.o $(LIBDIR)/k4_validate.o $(LIBDIR)/k5_generate.o $(LIBDIR)/k6_greedy.o $(LIBDIR)/k1_big8.o $(LIBDIR)/k1_big16_u32.o $(LIBDIR)/k1_big16_u64.o $(LIBDIR)/k1_big16_u128.o
CU_DEPS := $(wildcard $(PKG)/csrc/*.cuh) $(wildcard $(PKG)/csrc/*.h) include/dagsched_b200.h

.PHONY: all product oracle ref clean
all: product cppapi oracle ref

product: $(LIBDIR)/libdagsched_b200.so

$(LIBDIR)/%.o: $(PKG)/csrc/%.cu $(CU_DEPS) $(PKG)/csrc/k1_main.cu
	@mkdir -p $(LIBDIR)
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> $(LIBDIR)/ptxas_$*.txt || (cat $(LIBDIR)/ptxas_$*.txt; false)

$(LIBDIR)/host_gen.o: $(PKG)/csrc/host_gen.cpp $(PKG)/csrc/k5_generate_host.h include/dagsched_b200.h
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

# ---------------------------------------------------------------- C++ API
CPP_SRCS := $(wildcard $(PKG)/cpp/*.cpp)
CPP_OBJS := $(patsubst $(PKG)/cpp/%.cpp,$(LIBDIR)/cpp_%.o,$(CPP_SRCS))
API_INC  := -Iinclude -I$(PKG)/cpp
REFPROJ  ?= /root/reference/proj

cppapi: $(LIBDIR)/libdagsched_cpp.so $(LIBDIR)/api_parity $(LIBDIR)/api_division_dump $(LIBDIR)/api_bench $(LIBDIR)/api_rational_check $(LIBDIR)/api_drivers_dump $(if $(wildcard $(REFPROJ)/tests),$(LIBDIR)/api_test_dag_model $(LIBDIR)/api_test_exec_model)

$(LIBDIR)/cpp_%.o: $(PKG)/cpp/%.cpp $(wildcard include/dagsched/*.hpp) $(PKG)/cpp/device.hpp include/dagsched_b200.h
	@mkdir -p $(LIBDIR)
	$(CXX) -std=c++20 -O2 -fPIC -Wall -Wno-comment $(API_INC) -c $< -o $@

$(LIBDIR)/libdagsched_cpp.so: $(CPP_OBJS) $(LIBDIR)/libdagsched_b200.so
	$(CXX) -shared -o $@ $(CPP_OBJS) -L$(LIBDIR) -ldagsched_b200 -Wl,-rpath,'$$ORIGIN'

$(LIBDIR)/api_parity: tests/cpp/api_parity.cpp $(LIBDIR)/libdagsched_cpp.so
	$(CXX) -std=c++20 -O2 $(API_INC) $< -o $@ -L$(LIBDIR) -ldagsched_cpp -ldagsched_b200 -Wl,-rpath,'$$ORIGIN'

$(LIBDIR)/api_rational_check: tests/cpp/rational_check.cpp $(LIBDIR)/libdagsched_cpp.so
	$(CXX) -std=c++20 -O2 $(API_INC) $< -o $@ -L$(LIBDIR) -ldagsched_cpp -ldagsched_b200 -Wl,-rpath,'$$ORIGIN'

$(LIBDIR)/api_drivers_dump: tests/cpp/drivers_dump.cpp $(LIBDIR)/libdagsched_cpp.so
	$(CXX) -std=c++20 -O2 $(API_INC) $< -o $@ -L$(LIBDIR) -ldagsched_cpp -ldagsched_b200 -Wl,-rpath,'$$ORIGIN'

$(LIBDIR)/api_bench: tests/cpp/api_bench.cpp $(LIBDIR)/libdagsched_cpp.so
	$(CXX) -std=c++20 -O2 -DDS_API_BENCH_RAW $(API_INC) $< -o $@ -L$(LIBDIR) -ldagsched_cpp -ldagsched_b200 -Wl,-rpath,'$$ORIGIN'

$(LIBDIR)/api_division_dump: tests/cpp/division_dump.cpp $(LIBDIR)/libdagsched_cpp.so
	$(CXX) -std=c++20 -O2 $(API_INC) $< -o $@ -L$(LIBDIR) -ldagsched_cpp -ldagsched_b200 -Wl,-rpath,'$$ORIGIN'

# the reference's own unit tests (proj/tests, read in place) against this API
$(LIBDIR)/api_test_%: $(REFPROJ)/tests/test_%.cpp $(LIBDIR)/libdagsched_cpp.so
	$(CXX) -std=c++20 -O2 $(API_INC) -Ioracle/shim -I$(REFPROJ)/tests -DDOCTEST_CONFIG_IMPLEMENT_WITH_MAIN \
	    -include oracle/shim/doctest.h $< -o $@ -L$(LIBDIR) -ldagsched_cpp -ldagsched_b200 -Wl,-rpath,'$$ORIGIN'
