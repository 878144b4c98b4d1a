#!/bin/bash
O=gpurun_out/${1:-trf}; mkdir -p $O
for W in C2 C1; do
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file $O/traffic_$W.csv python tools/ncu_target.py --workload $W --reps 1 > $O/traffic_$W.log 2>&1
done
echo done > $O/DONE
