mkdir -p gpurun_out/r02ap
timeout 900 python -m pytest tests/test_gpu_a2c.py tests/test_gpu_a2c_dp.py -x -q > gpurun_out/r02ap/pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/r02ap/pytest.log
timeout 300 python bench.py --workload C2T --no-cpu-baseline --sustain-s 0.3 > gpurun_out/r02ap/bench_C2T.log 2>&1
timeout 300 python bench.py --workload C2O --no-cpu-baseline --sustain-s 0.3 > gpurun_out/r02ap/bench_C2O.log 2>&1
