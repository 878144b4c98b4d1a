#!/bin/bash
# A/B on C2: default build vs library variants (phase profile + task counters).
TAG=${1:-ab}
O=gpurun_out/$TAG
mkdir -p $O
run() {  # name
  timeout 300 python tools/phase_profile.py --workload C2 > $O/phase_$1.log 2>&1
  BP_DEBUG=1 timeout 300 python tools/ncu_target.py --workload C2 --reps 1 > $O/dbg_$1.log 2>&1
}
run default
for v in $(ls paper_2510_20499_b200/variants/ 2>/dev/null | sed 's/libbp_//; s/\.so//'); do
  BP_LIB=paper_2510_20499_b200/variants/libbp_$v.so run $v
done
echo done > $O/DONE
