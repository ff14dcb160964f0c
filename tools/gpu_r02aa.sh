mkdir -p gpurun_out/r02aa
timeout 600 python -m pytest tests/test_gpu_multirank.py tests/test_gpu_kernels.py -x -q > gpurun_out/r02aa/pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/r02aa/pytest.log
python bench.py > gpurun_out/r02aa/bench_default.log 2>&1
timeout 300 python bench.py --workload C5 --no-cpu-baseline --sustain-s 0.3 > gpurun_out/r02aa/bench_C5.log 2>&1
