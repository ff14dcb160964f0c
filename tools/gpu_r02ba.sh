mkdir -p gpurun_out/r02ba
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "host" > gpurun_out/r02ba/pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/r02ba/pytest.log
python bench.py --no-cpu-baseline > gpurun_out/r02ba/bench_C2.log 2>&1
