#!/bin/bash
# --set full captures (with source) of an early and a late k_rows_full launch of C2 + a launch list.
#   tools/gpu_ncu_rows.sh TAG
O=gpurun_out/${1:-ncu_rows}; mkdir -p $O
ncu --set full --clock-control none --import-source on -k regex:k_rows_full -s 1 -c 1 -o $O/rows_r2 python tools/ncu_target.py --workload C2 --reps 1 > $O/ncu_r2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_rows_full -s ${LATE:-20} -c 1 -o $O/rows_late python tools/ncu_target.py --workload C2 --reps 1 > $O/ncu_late.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv python tools/ncu_target.py --workload C2 --reps 1 > /dev/null 2>&1
echo done > $O/DONE
