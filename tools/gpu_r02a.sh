set -x
python bench.py > gpurun_out/r02a_bench_C2.log 2>&1; tail -1 gpurun_out/r02a_bench_C2.log
python bench.py --workload C5 --no-cpu-baseline > gpurun_out/r02a_bench_C5.log 2>&1; tail -1 gpurun_out/r02a_bench_C5.log | cut -c1-600
python -m pytest tests/test_gpu_multirank.py tests/test_gpu_a2c_dp.py -x -q > gpurun_out/r02a_pytest.log 2>&1; tail -3 gpurun_out/r02a_pytest.log
tools/ncu_table.sh r02a C2 C3a C3b C4 C5 D0 C2S C3S
