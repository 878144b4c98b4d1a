#!/bin/bash
# A/B on C2: variants + the full-round threshold knob (BP_FULL_PCT).
TAG=${1:-ab}
O=gpurun_out/$TAG
mkdir -p $O
run() { timeout 300 python tools/phase_profile.py --workload C2 > $O/phase_$1.log 2>&1; }
run default
BP_FULL_PCT=20 run pct20
BP_FULL_PCT=60 run pct60
for v in $(ls paper_2510_20499_b200/variants/ 2>/dev/null | sed 's/libbp_//; s/\.so//'); do
  BP_LIB=paper_2510_20499_b200/variants/libbp_$v.so run $v
done
echo done > $O/DONE
