#!/bin/bash
# bench sections other than BP: probing (C3), rounding (C4), batch (C5); no CPU baselines.
O=gpurun_out/${1:-sec}; mkdir -p $O
timeout 1200 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 --no-rounding > $O/bench.log 2> $O/bench.err; echo "exit $?" >> $O/bench.err
echo done > $O/DONE
