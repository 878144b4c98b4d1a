O=gpurun_out/bld; mkdir -p $O
timeout 600 python bench.py --steps 3 --warmup 3 --no-probing --no-rounding --no-batch --no-lp --no-cpu-baseline > $O/b1.log 2> $O/b1.err
timeout 900 python bench.py --steps 3 --warmup 3 --no-probing --no-rounding --no-lp --no-cpu-baseline > $O/b2.log 2> $O/b2.err
