#!/bin/bash
O=gpurun_out/${1:-pct}; mkdir -p $O
for p in 20 35 50; do for W in C2 C1; do
  BP_FULL_PCT=$p timeout 300 python tools/phase_profile.py --workload $W > $O/phase_${W}_$p.log 2>&1
done; done
echo done > $O/DONE
