#!/bin/bash
# A/B of two engine builds on the same box: BP-only bench lines, alternating (BP_LIB selects the .so).
# usage: tools/gpu_ab.sh TAG path/to/variant.so
O=gpurun_out/${1:-ab}; V=$2; mkdir -p $O
for i in 1 2 3; do
  timeout 300 python bench.py --steps 20 --warmup 3 --no-probing --no-rounding --no-batch --no-lp --no-build --no-cpu-baseline > $O/base_$i.log 2>/dev/null
  BP_LIB=$V timeout 300 python bench.py --steps 20 --warmup 3 --no-probing --no-rounding --no-batch --no-lp --no-build --no-cpu-baseline > $O/var_$i.log 2>/dev/null
done
for f in $O/base_*.log $O/var_*.log; do python -c "import json,sys; d=json.loads(open('$f').read()); print('$f', round(d['ms_per_step'],3))"; done > $O/summary.txt
