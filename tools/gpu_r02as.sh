mkdir -p gpurun_out/r02as
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multirank.py tests/test_gpu_checkpoint.py -x -q > gpurun_out/r02as/pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/r02as/pytest.log
python bench.py --no-cpu-baseline > gpurun_out/r02as/bench_C2.log 2>&1
python tools/time_rollout.py acrobot 12500 500 20 > gpurun_out/r02as/time_C3a_shard.log 2>&1
python tools/time_rollout.py cartpole 10000 1000 100 > gpurun_out/r02as/time_C2.log 2>&1
