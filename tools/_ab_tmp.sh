O=gpurun_out/pshard; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_multi.py tests/test_gpu_probing.py -x -q > $O/pytest.log 2>&1; echo "pytest exit $?" >> $O/pytest.log
for i in 1 2; do timeout 900 python bench.py --steps 3 --warmup 3 --no-rounding --no-batch --no-lp --no-build --no-cpu-baseline > $O/b$i.log 2> $O/b$i.err; done
