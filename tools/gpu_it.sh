O=gpurun_out/it8; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_probing.py tests/test_gpu_rounding.py -x -q --durations=8 > $O/pytest.log 2>&1; echo "pytest exit $?" >> $O/pytest.log
timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python tools/sanitize_target.py probe > $O/racecheck_probe.log 2>&1
BP_PROBE_PROFILE=1 timeout 900 python tools/round_profile.py --deadline 30 > $O/round.log 2>&1; echo "round exit $?" >> $O/round.log
