#!/bin/bash
# A/B of engine build variants on C2 (phase profile + task counters), plus the default build with
# BP_SPLIT_SELL=0, after the propagation parity tests on the default build.
TAG=${1:-ab}
O=gpurun_out/$TAG
mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_propagation.py tests/test_gpu_probing.py -x -q > $O/pytest.log 2>&1; echo "pytest exit $?" >> $O/pytest.log
run() {  # name
  timeout 300 python tools/phase_profile.py --workload C2 > $O/phase_$1.log 2>&1
  BP_DEBUG=1 timeout 300 python tools/ncu_target.py --workload C2 --reps 1 > $O/dbg_$1.log 2>&1
}
run default
BP_SPLIT_SELL=0 run nosplit
for v in $(ls paper_2510_20499_b200/variants/ 2>/dev/null | sed 's/libbp_//; s/\.so//'); do
  BP_LIB=paper_2510_20499_b200/variants/libbp_$v.so run $v
done
echo done > $O/DONE
