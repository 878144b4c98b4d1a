#!/bin/bash
# Probe-kernel A/B on C3 (all 200k binaries): default build vs library variants.
TAG=${1:-pv}
O=gpurun_out/$TAG
mkdir -p $O
timeout 300 python tools/ncu_probe_target.py > $O/default.log 2>&1
for v in $(ls paper_2510_20499_b200/variants/ 2>/dev/null | sed 's/libbp_//; s/\.so//'); do
  BP_LIB=paper_2510_20499_b200/variants/libbp_$v.so timeout 300 python tools/ncu_probe_target.py > $O/$v.log 2>&1
done
echo done > $O/DONE
