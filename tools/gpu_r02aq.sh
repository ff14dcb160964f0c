mkdir -p gpurun_out/r02aq
timeout 900 python -m pytest tests/test_gpu_policy.py tests/test_gpu_a2c.py -x -q -k "tag or multi" > gpurun_out/r02aq/pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/r02aq/pytest.log
timeout 300 python bench.py --workload C4T --no-cpu-baseline --sustain-s 0.3 > gpurun_out/r02aq/bench_C4T.log 2>&1
