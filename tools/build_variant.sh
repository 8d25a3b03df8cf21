#!/bin/bash
# Build a tuning variant of libsrm_b200.so: tools/build_variant.sh NAME -DSRM_...=V ...
# -> exp/libsrm_b200_NAME.so (select it with SRM_B200_LIB=...; tools/ experiments only).
set -e
cd "$(dirname "$0")/.."
make -s lib >/dev/null
name=$1; shift
mkdir -p exp
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo --fmad=false -std=c++17 \
  -Xcompiler -fPIC,-ffp-contract=off --expt-relaxed-constexpr -Xptxas -v "$@" \
  -c paper_2605_18254_b200/csrc/srm_capi.cu -o exp/capi_$name.o 2> exp/ptxas_$name.log
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o exp/libsrm_b200_$name.so exp/capi_$name.o \
  paper_2605_18254_b200/csrc/srm_selftest.o paper_2605_18254_b200/csrc/srm_rsa.o paper_2605_18254_b200/csrc/srm_snapshot.o -lcudart
grep -A2 k_near_tiles exp/ptxas_$name.log | grep -E "Used|spill" | head -2 | sed "s/^/$name: /"
