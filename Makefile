# Build of the B200 SRM library (sm_100a only) and the CPU checker (oracle/).
#   make            -> paper_2605_18254_b200/libsrm_b200.so + oracle libraries
#   make lib        -> the product library only
#   make shimtest   -> tests/cpp/shim_test (C++ drop-in shim over the C ABI)
NVCC ?= /usr/local/cuda/bin/nvcc
PKG := paper_2605_18254_b200
CSRC := $(PKG)/csrc
LIB := $(PKG)/libsrm_b200.so
REF ?= /root/reference/proj

ARCH := -gencode arch=compute_100a,code=sm_100a
# --fmad=false: no FMA contraction, so every double operation rounds like the
# reference's plain x86-64 build (bit-exact keys, decisions and positions)
NVFLAGS := $(ARCH) -O3 -lineinfo --fmad=false -std=c++17 -Xcompiler -fPIC,-ffp-contract=off \
           --expt-relaxed-constexpr -Xptxas -v
CXXFLAGS := -O2 -std=c++17 -fPIC -ffp-contract=off
# nlohmann::json 3.11.3 (header only; the reference's JSON library and version) for the
# snapshot header -- the copy vendored in the image's cudnn_frontend package
JSON_INC ?= $(firstword $(wildcard /opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty))

all: lib oracle microbench
	@if [ -d "$(REF)/core/include" ]; then $(MAKE) shimtest; else echo "shimtest: $(REF) absent, keeping prebuilt binary (if any)"; fi

lib: $(LIB)

$(CSRC)/srm_capi.o: $(CSRC)/srm_capi.cu $(wildcard $(CSRC)/*.cuh) include/srm_b200.h
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> $(CSRC)/ptxas.log || (cat $(CSRC)/ptxas.log; exit 1)

$(CSRC)/srm_selftest.o: $(CSRC)/srm_selftest.cu $(CSRC)/srm_device.cuh include/srm_b200.h
	$(NVCC) $(ARCH) -O3 -lineinfo --fmad=false -std=c++17 -Xcompiler -fPIC -c $< -o $@

$(CSRC)/srm_rsa.o: $(CSRC)/srm_rsa.cpp include/srm_b200.h
	g++ $(CXXFLAGS) -c $< -o $@

$(CSRC)/srm_snapshot.o: $(CSRC)/srm_snapshot.cpp include/srm_b200.h
	g++ $(CXXFLAGS) -I$(JSON_INC) -c $< -o $@

$(LIB): $(CSRC)/srm_capi.o $(CSRC)/srm_selftest.o $(CSRC)/srm_rsa.o $(CSRC)/srm_snapshot.o
	$(NVCC) $(ARCH) -shared -o $@ $^ -lcudart

oracle:
	$(MAKE) -f oracle/Makefile REF=$(REF) JSON_INC=$(JSON_INC)

shimtest: tests/cpp/shim_test

# (the reference side of the comparisons -- spherodisk.cpp, recipes.cpp -- from the
#  checker library oracle/_ref/libsrm_ref.so, built from the reference's own sources)
tests/cpp/shim_test: tests/cpp/shim_test.cpp include/srm/b200/engine.hpp include/srm_b200.h $(LIB) oracle
	g++ -std=gnu++20 -O2 -I$(REF)/core/include -Iinclude -o $@ tests/cpp/shim_test.cpp \
	    -L$(PKG) -lsrm_b200 -Loracle/_ref -lsrm_ref \
	    -Wl,-rpath,'$$ORIGIN/../../$(PKG)' -Wl,-rpath,'$$ORIGIN/../../oracle/_ref'

# memory-system ceiling of the migrate step's access patterns
microbench: tools/random_access_bench

tools/random_access_bench: tools/random_access_bench.cu
	$(NVCC) $(ARCH) -O3 -lineinfo -std=c++17 -o $@ $<

clean:
	rm -f $(CSRC)/*.o $(LIB) $(CSRC)/ptxas.log tests/cpp/shim_test
	$(MAKE) -f oracle/Makefile clean

.PHONY: all lib oracle shimtest microbench clean

