#!/bin/bash
# Round-2 evidence: launch lists + `ncu --set full` captures of every hot kernel (profiles/r02/).
O=gpurun_out/prof; mkdir -p $O
N="ncu --clock-control none"
# C2 propagate: per-launch time + DRAM bytes
timeout 900 $N --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv --log-file $O/launches_C2.csv python tools/ncu_target.py --workload C2 --reps 1 > /dev/null 2>&1
# k_rows_full and k_rows_sell: an early (round 2, all rows) and a late (round 20, dirty-filtered)
# launch; k_engine in a dirty-filtered round (12: finalize over the touched vars + marks)
timeout 900 $N --set full --import-source on -k regex:k_rows_full -s 1 -c 1 -o $O/k_rows_full_C2_r2 python tools/ncu_target.py --workload C2 --reps 1 > $O/n1.log 2>&1
timeout 900 $N --set full --import-source on -k regex:k_rows_full -s 19 -c 1 -o $O/k_rows_full_C2_r20 python tools/ncu_target.py --workload C2 --reps 1 > $O/n2.log 2>&1
timeout 900 $N --set full --import-source on -k regex:k_rows_sell -s 1 -c 1 -o $O/k_rows_sell_C2_r2 python tools/ncu_target.py --workload C2 --reps 1 > $O/n3.log 2>&1
timeout 900 $N --set full --import-source on -k regex:k_rows_sell -s 19 -c 1 -o $O/k_rows_sell_C2_r20 python tools/ncu_target.py --workload C2 --reps 1 > $O/n4.log 2>&1
timeout 900 $N --set full --import-source on -k regex:k_engine -s 11 -c 1 -o $O/k_engine_C2_r12 python tools/ncu_target.py --workload C2 --reps 1 > $O/n8.log 2>&1
# probing: the warp kernel on C3, the block kernel on a scaled C4
timeout 900 $N --set full --import-source on -k regex:k_probe -c 1 -o $O/k_probe_C3 python tools/ncu_probe_target.py > $O/n5.log 2>&1
timeout 1200 $N --set full --import-source on -k regex:k_probe_block -c 1 -o $O/k_probe_block_C4s python tools/ncu_c4probe_target.py > $O/n6.log 2>&1
# PDHG products
timeout 900 $N --set full --import-source on -k regex:spmv -c 2 -o $O/lp_spmv_C2 python tools/ncu_lp_target.py > $O/n7.log 2>&1
# summaries on the box (the reports together exceed gpurun's 64 MiB copy-back): ncu_summary.py text
# + the per-source-line stall table of each capture; the reports themselves are removed
for r in $O/*.ncu-rep; do
  b=$(basename $r .ncu-rep)
  python tools/ncu_summary.py $r $O/ncu_$b > /dev/null 2>&1
  ncu -i $r --page source --print-source cuda,sass --csv > $O/src.csv 2>/dev/null && python tools/ncu_lines.py $O/src.csv 40 > $O/lines_$b.txt 2>&1
  rm -f $O/src.csv
done
python tools/ncu_traffic.py $O/launches_C2.csv --workload C2 > $O/traffic_C2.txt 2>&1
rm -f $O/*.ncu-rep
echo done > $O/DONE
