#!/bin/bash
# End-of-round style check: GPU tests, smoke, drop-in criteria, the driver's default bench command.
TAG=${1:-check}
O=gpurun_out/$TAG
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q --durations=15 > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?" >> $O/smoke.log
timeout 1500 python bench.py > $O/bench.log 2> $O/bench.err; echo "bench exit $?" >> $O/bench.err
echo done > $O/DONE
