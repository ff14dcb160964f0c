mkdir -p gpurun_out/r02ab
timeout 900 python -m pytest tests/test_gpu_user_env.py tests/test_gpu_policy.py -x -q > gpurun_out/r02ab/pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/r02ab/pytest.log
timeout 300 python bench.py --workload C2U --no-cpu-baseline --sustain-s 0.3 > gpurun_out/r02ab/bench_C2U.log 2>&1
