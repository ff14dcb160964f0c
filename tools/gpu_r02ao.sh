mkdir -p gpurun_out/r02ao
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py tests/test_gpu_policy.py tests/test_gpu_staged.py -x -q -k "pendulum or angle or gauss or C3b or continuous or env_parity or Gaussian or gaussian" > gpurun_out/r02ao/pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/r02ao/pytest.log
timeout 300 python bench.py --workload C3b --no-cpu-baseline --sustain-s 0.3 > gpurun_out/r02ao/bench_C3b.log 2>&1
