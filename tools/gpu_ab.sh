#!/bin/bash
# A/B of engine builds / settings on the same box: BP-only bench lines, interleaved.
# usage: tools/gpu_ab.sh TAG "ENV=.. BP_LIB=a.so" "ENV=.. BP_LIB=b.so" [...]   (3 runs each)
O=gpurun_out/${1:-ab}; shift; mkdir -p $O
for i in 1 2 3; do
  j=0
  for cfg in "$@"; do
    j=$((j+1))
    env $cfg timeout 300 python bench.py --steps 20 --warmup 3 --no-probing --no-rounding --no-batch --no-lp --no-build --no-cpu-baseline > $O/v${j}_$i.log 2>/dev/null
  done
done
j=0
for cfg in "$@"; do
  j=$((j+1))
  echo "$cfg: $(for f in $O/v${j}_*.log; do python -c "import json; print(round(json.loads(open('$f').read())['ms_per_step'],3), end=' ')"; done)" >> $O/summary.txt
done
