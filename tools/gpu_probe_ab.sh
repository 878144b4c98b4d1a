#!/bin/bash
# Probing parity tests + the bench's probing section (C3) with the host step profile.
TAG=${1:-pr}
O=gpurun_out/$TAG
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_probing.py tests/test_gpu_rounding.py tests/test_gpu_dropin.py -x -q > $O/pytest.log 2>&1; echo "exit $?" >> $O/pytest.log
BP_PROBE_PROFILE=1 timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-rounding --no-batch --e2e-steps 1 > $O/bench.log 2> $O/bench.err
echo done > $O/DONE
