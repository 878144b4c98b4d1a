#!/bin/bash
# Quick engine iteration: parity (propagation + probing + rounding), C2 phases, BP bench line.
TAG=${1:-q}
O=gpurun_out/$TAG
mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_propagation.py tests/test_gpu_probing.py tests/test_gpu_rounding.py -x -q > $O/pytest.log 2>&1; echo "pytest exit $?" >> $O/pytest.log
timeout 300 python tools/phase_profile.py --workload C2 > $O/phase_C2.log 2>&1
BP_DEBUG=1 timeout 300 python tools/ncu_target.py --workload C2 --reps 1 > $O/dbg_C2.log 2>&1
timeout 300 python bench.py --steps 10 --warmup 3 --no-probing --no-rounding --no-batch --no-cpu-baseline > $O/bench_bp.log 2> $O/bench_bp.err
echo done > $O/DONE
