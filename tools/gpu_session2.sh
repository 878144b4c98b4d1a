#!/bin/bash
# Diagnostic session: new tests, drop-in binary, bench sections one at a time (timed), C2 phases.
TAG=${1:-r01b}
O=gpurun_out/$TAG
mkdir -p $O
BP_DEBUG=1 timeout 300 python tools/ncu_target.py --workload C2 --reps 2 > $O/dbg_C2.log 2>&1

time timeout 600 python bench.py --steps 10 --warmup 3 --no-probing --no-rounding > $O/bench_bp.log 2> $O/bench_bp.err; echo "exit $?" >> $O/bench_bp.err
time timeout 900 python bench.py --steps 3 --warmup 3 --no-rounding --no-cpu-baseline --e2e-steps 1 > $O/bench_probe.log 2> $O/bench_probe.err; echo "exit $?" >> $O/bench_probe.err
time timeout 1200 python bench.py --steps 3 --warmup 3 --no-probing --no-cpu-baseline --e2e-steps 1 > $O/bench_round.log 2> $O/bench_round.err; echo "exit $?" >> $O/bench_round.err
echo done > $O/DONE
