mkdir -p gpurun_out/r02y
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kernels.py tests/test_gpu_staged.py tests/test_gpu_policy.py -x -q -k "surface or C5 or gaussian or pendulum or gauss" > gpurun_out/r02y/pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/r02y/pytest.log
timeout 300 python bench.py --workload C5 --no-cpu-baseline --sustain-s 0.3 > gpurun_out/r02y/bench_C5.log 2>&1
bash tools/prof_one.sh C5 k_plan_gauss r02y_C5plan
