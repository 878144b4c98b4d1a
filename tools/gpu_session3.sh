#!/bin/bash
# Parity + default bench (all sections) + C2 phase profile.
TAG=${1:-r01d}
O=gpurun_out/$TAG
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
timeout 300 python tools/phase_profile.py --workload C2 > $O/phase_C2.log 2>&1
BP_DEBUG=1 timeout 300 python tools/ncu_target.py --workload C2 --reps 1 > $O/dbg_C2.log 2>&1
time timeout 900 python bench.py > $O/bench.log 2> $O/bench.err; echo "exit $?" >> $O/bench.err
echo done > $O/DONE
