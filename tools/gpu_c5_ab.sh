mkdir -p gpurun_out/c5a
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/c5a/pytest.log 2>&1; echo "exit $?" >> gpurun_out/c5a/pytest.log
for cfg in "8 8192" "1 8192" "8 0" "1 0"; do
  set -- $cfg
  BP_GRID_NNZ=$2 timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-probing --no-rounding --no-lp --no-build --e2e-steps 1 --c5-streams $1 > gpurun_out/c5a/bench_$1_$2.log 2> gpurun_out/c5a/bench_$1_$2.err
done
