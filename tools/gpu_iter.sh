#!/bin/bash
# Engine iteration on the GPU box: parity (selected test files), C2 phase profile, BP bench line.
#   tools/gpu_iter.sh TAG "tests/test_gpu_propagation.py ..." [extra bench args]
TAG=${1:-iter}
TESTS=${2:-tests/test_gpu_propagation.py}
O=gpurun_out/$TAG
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/gpu.txt 2>&1
[ "$TESTS" != "none" ] && { timeout 900 python -m pytest $TESTS -x -q > $O/pytest.log 2>&1; echo "pytest exit $?" >> $O/pytest.log; }
timeout 300 python tools/phase_profile.py --workload C2 > $O/phase_C2.log 2>&1
timeout 400 python bench.py --steps 20 --warmup 3 --no-probing --no-rounding --no-batch --no-lp --no-build --no-cpu-baseline $3 > $O/bench_bp.log 2> $O/bench_bp.err
echo done > $O/DONE
