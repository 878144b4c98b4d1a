ncu --set full --clock-control none --import-source on -k regex:k_rows_full -s 21 -c 1 -o gpurun_out/rows_late python tools/ncu_target.py --workload C2 --reps 1 > gpurun_out/ncu_late.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_rows_full -s 5 -c 1 -o gpurun_out/rows_r6 python tools/ncu_target.py --workload C2 --reps 1 > gpurun_out/ncu_r6.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_df.csv python tools/ncu_target.py --workload C2 --reps 1 > /dev/null 2>&1
