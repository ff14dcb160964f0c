mkdir -p gpurun_out/r02ax
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kernels.py tests/test_gpu_staged.py -x -q -k "surface or C5 or gaussian" > gpurun_out/r02ax/pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/r02ax/pytest.log
timeout 300 python bench.py --workload C5 --no-cpu-baseline --sustain-s 0.3 > gpurun_out/r02ax/bench_C5.log 2>&1
