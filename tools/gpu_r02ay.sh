mkdir -p gpurun_out/r02ay
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kernels.py tests/test_gpu_staged.py tests/test_gpu_policy.py -x -q -k "pendulum or gaussian or C3b or env_parity or single_step or staged" > gpurun_out/r02ay/pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/r02ay/pytest.log
timeout 300 python bench.py --workload C3b --no-cpu-baseline --sustain-s 0.3 > gpurun_out/r02ay/bench_C3b.log 2>&1
