#!/bin/bash
# A/B on C2: default build (split SELL off/on), stream-hint variants, L2 persistence knob.
TAG=${1:-ab}
O=gpurun_out/$TAG
mkdir -p $O
run() {  # name
  timeout 300 python tools/phase_profile.py --workload C2 > $O/phase_$1.log 2>&1
}
BP_SPLIT_SELL=0 run nosplit
BP_SPLIT_SELL=0 BP_L2_PERSIST=16 run persist16
BP_SPLIT_SELL=0 BP_L2_PERSIST=64 run persist64
for v in $(ls paper_2510_20499_b200/variants/ 2>/dev/null | sed 's/libbp_//; s/\.so//'); do
  BP_SPLIT_SELL=0 BP_LIB=paper_2510_20499_b200/variants/libbp_$v.so run $v
done
echo done > $O/DONE
