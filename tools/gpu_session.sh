#!/bin/bash
# One gpurun session: host info, GPU tests, smoke, bench, ncu launch list + full capture of the engine.
# Usage (from the repo root on the box): bash tools/gpu_session.sh [tag]
TAG=${1:-r01}
O=gpurun_out/$TAG
mkdir -p $O
(uname -m; nproc; lscpu | grep "Model name"; nvidia-smi -L) > $O/host.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?" >> $O/smoke.log
timeout 1200 python bench.py --steps 20 --warmup 3 > $O/bench.log 2>&1; echo "bench exit $?" >> $O/bench.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv \
   python bench.py --steps 2 --warmup 3 --no-probing --no-rounding --no-cpu-baseline --e2e-steps 1 > $O/ncu_launch_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_rows_full -s 3 -c 1 -o $O/k_rows_full_C2 \
   python tools/ncu_target.py --workload C2 --reps 3 > $O/ncu_full.log 2>&1
echo done > $O/DONE
