mkdir -p gpurun_out/r02am
timeout 900 python -m pytest tests/test_gpu_user_env.py -x -q > gpurun_out/r02am/pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/r02am/pytest.log
timeout 300 python bench.py --workload C2U --no-cpu-baseline --sustain-s 0.3 > gpurun_out/r02am/bench_C2U.log 2>&1
