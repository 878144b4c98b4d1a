#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over tools/sanitize_target.py (profiles/r02/).
O=gpurun_out/sanitize; mkdir -p $O
for tool in memcheck racecheck synccheck; do
  for t in prop probe round; do
    timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_target.py $t > $O/${tool}_$t.log 2>&1
    echo "exit $?" >> $O/${tool}_$t.log
  done
done
echo done > $O/DONE
