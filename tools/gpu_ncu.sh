#!/bin/bash
# ncu: launch list of a C2 propagate + one --set full capture of the given kernel (regex).
TAG=${1:-ncu}; K=${2:-k_rows_full}; W=${3:-C2}
O=gpurun_out/$TAG
mkdir -p $O
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_$W.csv \
   python tools/ncu_target.py --workload $W --reps 1 > $O/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s 3 -c 1 -o $O/${K}_$W \
   python tools/ncu_target.py --workload $W --reps 1 > $O/ncu_full.log 2>&1
echo done > $O/DONE
