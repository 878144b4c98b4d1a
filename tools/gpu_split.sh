#!/bin/bash
O=gpurun_out/${1:-split}; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_propagation.py tests/test_gpu_probing.py tests/test_gpu_rounding.py -x -q > $O/pytest.log 2>&1; echo "pytest exit $?" >> $O/pytest.log
timeout 300 python tools/phase_profile.py --workload C2 > $O/phase_split.log 2>&1
BP_NO_SPLIT_ROWS=1 timeout 300 python tools/phase_profile.py --workload C2 > $O/phase_nosplit.log 2>&1
BP_DEBUG=1 timeout 300 python tools/ncu_target.py --workload C2 --reps 1 > $O/dbg_split.log 2>&1
echo done > $O/DONE
