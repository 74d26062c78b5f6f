# vgpu-b200 build. `make` builds the product (.so + tools), the C++ unit
# tests and the C oracle; `make ref` additionally compiles the reference
# oracle into oracle/_ref when /root/reference is present (never shipped).
#
#   paper_1511_07658_b200/lib/libvgpu_cuda.so   device backend (nvcc, sm_100a, static cudart)
#   paper_1511_07658_b200/lib/libvgpu.so        C++ host stack + C-ABI (links the backend)
#   paper_1511_07658_b200/bin/{vgpud,vgpu-spmd,payload-bench,vgpu-launch}
#   tests/_bin/vgpu-tests                       C++ unit / parity tests
#   oracle/_build/libvgpu_oracle.so             CPU oracle (test infrastructure)

PKG      := paper_1511_07658_b200
CSRC     := $(PKG)/csrc
LIBDIR   := $(PKG)/lib
BINDIR   := $(PKG)/bin
OBJDIR   := build/obj
TESTBIN  := tests/_bin

NVCC     ?= nvcc
CXX      ?= g++
CC       ?= gcc
ARCH     := -gencode arch=compute_100a,code=sm_100a
NVFLAGS  := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Iinclude -Xptxas -v
CUDA_HOME ?= /usr/local/cuda
CXXFLAGS := -O2 -g -std=c++20 -fPIC -Wall -Wextra -pthread -Iinclude -I$(CUDA_HOME)/include
CFLAGS   := -O2 -g -fPIC -ffp-contract=off -std=c11 -Wall -Wextra -Wno-unknown-pragmas
# the oracle's batch loops are OpenMP-parallel when the system gcc has libgomp
# (the image's CC wrapper does not); results do not depend on the thread count
OCC      := $(shell test -x /usr/bin/gcc && echo /usr/bin/gcc || echo $(CC))
OMP      := $(shell echo 'int main(void){return 0;}' | $(OCC) -fopenmp -x c - -o /dev/null 2>/dev/null && echo -fopenmp)

HOST_SRC := $(wildcard $(CSRC)/host/*.cpp)
HOST_OBJ := $(patsubst $(CSRC)/host/%.cpp,$(OBJDIR)/host/%.o,$(HOST_SRC))
CUDA_HDR := $(wildcard $(CSRC)/cuda/*.cuh) $(wildcard $(CSRC)/common/*.h) include/vgpu_cuda.h
HDRS     := $(wildcard include/vgpu/*.hpp) include/vgpu_cuda.h include/vgpu_c.h
TEST_SRC := $(wildcard tests/cpp/*.cpp)

RPATH_LIB := -Wl,-rpath,'$$ORIGIN'
RPATH_BIN := -Wl,-rpath,'$$ORIGIN/../lib'
RPATH_TST := -Wl,-rpath,'$$ORIGIN/../../$(LIBDIR)'

.PHONY: all product tests oracle ref clean tsan
all: product tests oracle

product: $(LIBDIR)/libvgpu_cuda.so $(LIBDIR)/libvgpu.so \
         $(BINDIR)/vgpud $(BINDIR)/vgpu-spmd $(BINDIR)/payload-bench $(BINDIR)/vgpu-launch

$(OBJDIR)/cuda/backend.o: $(CSRC)/cuda/backend.cu $(CUDA_HDR)
	@mkdir -p $(dir $@)
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> $(OBJDIR)/cuda/ptxas.log || (cat $(OBJDIR)/cuda/ptxas.log; false)

$(LIBDIR)/libvgpu_cuda.so: $(OBJDIR)/cuda/backend.o
	@mkdir -p $(LIBDIR)
	$(NVCC) $(ARCH) -shared -cudart static -o $@ $< -ldl -lrt -lpthread

$(OBJDIR)/host/%.o: $(CSRC)/host/%.cpp $(HDRS)
	@mkdir -p $(dir $@)
	$(CXX) $(CXXFLAGS) -c $< -o $@

$(LIBDIR)/libvgpu.so: $(HOST_OBJ) $(LIBDIR)/libvgpu_cuda.so
	$(CXX) -shared -o $@ $(HOST_OBJ) -L$(LIBDIR) -lvgpu_cuda $(RPATH_LIB) -pthread -lrt

$(BINDIR)/%: $(CSRC)/tools/%.cpp $(CSRC)/tools/workloads.hpp $(LIBDIR)/libvgpu.so $(HDRS)
	@mkdir -p $(BINDIR)
	$(CXX) $(CXXFLAGS) -o $@ $< -L$(LIBDIR) -lvgpu -lvgpu_cuda $(RPATH_BIN) -lrt

tests: $(TESTBIN)/vgpu-tests

$(TESTBIN)/vgpu-tests: $(TEST_SRC) tests/cpp/minitest.hpp $(LIBDIR)/libvgpu.so oracle/_build/libvgpu_oracle.so
	@mkdir -p $(TESTBIN)
	$(CXX) $(CXXFLAGS) -Itests/cpp -Ioracle -o $@ $(TEST_SRC) \
	    -L$(LIBDIR) -lvgpu -lvgpu_cuda -Loracle/_build -lvgpu_oracle \
	    $(RPATH_TST) -Wl,-rpath,'$$ORIGIN/../../oracle/_build' -lrt

oracle: oracle/_build/libvgpu_oracle.so

oracle/_build/libvgpu_oracle.so: oracle/vgpu_oracle.c oracle/vgpu_oracle.h $(wildcard $(CSRC)/common/*.h)
	@mkdir -p oracle/_build
	$(OCC) $(CFLAGS) $(OMP) -shared -o $@ oracle/vgpu_oracle.c -lm

# ThreadSanitizer build of the host layer (GVM, transports, client SDK,
# model) and its C++ tests; the CUDA backend stays uninstrumented. Run the
# CPU cases: `make tsan && TSAN_OPTIONS=halt_on_error=1 tests/_bin/vgpu-tests-tsan --exclude-gpu`
TSAN_FLAGS := -O1 -g -std=c++20 -fPIC -pthread -fsanitize=thread -Iinclude -I$(CUDA_HOME)/include
TSAN_CXX := $(shell test -x /usr/bin/g++ && echo /usr/bin/g++ || echo $(CXX))
tsan: $(TESTBIN)/vgpu-tests-tsan

$(TESTBIN)/vgpu-tests-tsan: $(HOST_SRC) $(TEST_SRC) tests/cpp/minitest.hpp $(LIBDIR)/libvgpu_cuda.so oracle/_build/libvgpu_oracle.so $(HDRS)
	@mkdir -p $(TESTBIN)
	$(TSAN_CXX) $(TSAN_FLAGS) -Itests/cpp -Ioracle -o $@ $(HOST_SRC) $(TEST_SRC) \
	    -L$(LIBDIR) -lvgpu_cuda -Loracle/_build -lvgpu_oracle \
	    $(RPATH_TST) -Wl,-rpath,'$$ORIGIN/../../oracle/_build' -lrt

ref:
	$(MAKE) -f oracle/Makefile.ref

clean:
	rm -rf build $(LIBDIR) $(BINDIR) $(TESTBIN) oracle/_build
