mkdir -p gpurun_out/r02bc
timeout 900 python -m pytest tests/test_gpu_user_env.py tests/test_gpu_kernels.py tests/test_gpu_parity.py tests/test_gpu_policy.py -x -q > gpurun_out/r02bc/pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/r02bc/pytest.log
timeout 300 python bench.py --workload C2U --no-cpu-baseline --sustain-s 0.3 > gpurun_out/r02bc/bench_C2U.log 2>&1
python tools/time_rollout.py cartpole 10000 1000 100 > gpurun_out/r02bc/time_C2.log 2>&1
