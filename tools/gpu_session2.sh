#!/bin/bash
# Diagnostic session: new tests, drop-in binary, bench sections one at a time (timed), C2 phases.
TAG=${1:-r01b}
O=gpurun_out/$TAG
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
timeout 600 python tools/phase_profile.py --workload C2 > $O/phase_C2.log 2>&1
/usr/bin/time -v timeout 600 python bench.py --steps 10 --warmup 3 --no-probing --no-rounding > $O/bench_bp.log 2> $O/bench_bp.err; echo "exit $?" >> $O/bench_bp.err
/usr/bin/time -v timeout 900 python bench.py --steps 3 --warmup 3 --no-rounding --no-cpu-baseline --e2e-steps 1 > $O/bench_probe.log 2> $O/bench_probe.err; echo "exit $?" >> $O/bench_probe.err
/usr/bin/time -v timeout 1200 python bench.py --steps 3 --warmup 3 --no-probing --no-cpu-baseline --e2e-steps 1 > $O/bench_round.log 2> $O/bench_round.err; echo "exit $?" >> $O/bench_round.err
echo done > $O/DONE
