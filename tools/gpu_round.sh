#!/bin/bash
O=gpurun_out/${1:-rnd}; mkdir -p $O
BP_ROUND_PROFILE=1 timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 --no-probing --no-batch > $O/bench.log 2> $O/bench.err; echo "exit $?" >> $O/bench.err
echo done > $O/DONE
