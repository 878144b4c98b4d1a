#!/bin/bash
# Builds an experimental variant of the engine library: tools/build_variant.sh NAME "-DFLAG=V ..."
# -> paper_2510_20499_b200/variants/libbp_NAME.so (select with BP_LIB=...).
set -e
NAME=$1; shift
D=paper_2510_20499_b200/csrc
mkdir -p paper_2510_20499_b200/variants
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo --fmad=false -std=c++17 -Xcompiler -fPIC \
  $@ -shared -o paper_2510_20499_b200/variants/libbp_$NAME.so \
  $D/bp_propagate.cu $D/bp_probe.cu $D/bp_cache.cu $D/bp_round.cu $D/bp_capi.cu $D/bp_build.cu $D/bp_lp.cu
