mkdir -p gpurun_out/r02ai
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py tests/test_gpu_policy.py tests/test_gpu_user_env.py -x -q > gpurun_out/r02ai/pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/r02ai/pytest.log
python bench.py --no-cpu-baseline > gpurun_out/r02ai/bench_C2.log 2>&1
python tools/time_rollout.py cartpole 10000 1000 50 > gpurun_out/r02ai/time_C2.log 2>&1
timeout 300 python bench.py --workload C2P --no-cpu-baseline --sustain-s 0.3 > gpurun_out/r02ai/bench_C2P.log 2>&1
