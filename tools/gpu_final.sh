#!/bin/bash
# Round evidence: session (tests, smoke, bench, ncu launch list, k_rows_full full capture),
# DRAM traffic per launch, C2 phase profile, k_probe full capture.
TAG=${1:-final}
bash tools/gpu_session.sh $TAG
bash tools/gpu_traffic.sh $TAG
O=gpurun_out/$TAG
timeout 300 python tools/phase_profile.py --workload C2 > $O/phase_C2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_probe -c 1 -o $O/k_probe_C3 \
   python tools/ncu_probe_target.py > $O/ncu_probe.log 2>&1
echo done > $O/DONE2
