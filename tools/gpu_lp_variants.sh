#!/bin/bash
# PDHG iteration A/B on the C2 matrix: default build vs library variants.
TAG=${1:-lpv}
O=gpurun_out/$TAG
mkdir -p $O
timeout 300 python tools/ncu_lp_target.py time > $O/default.log 2>&1
for v in $(ls paper_2510_20499_b200/variants/ 2>/dev/null | sed 's/libbp_//; s/\.so//'); do
  BP_LIB=paper_2510_20499_b200/variants/libbp_$v.so timeout 300 python tools/ncu_lp_target.py time > $O/$v.log 2>&1
done
