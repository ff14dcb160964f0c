mkdir -p gpurun_out/r02at
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/r02at/pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/r02at/pytest.log
python tools/time_rollout.py acrobot 12500 500 20 > gpurun_out/r02at/time_C3a_shard.log 2>&1
python tools/time_rollout.py cartpole 10000 1000 100 > gpurun_out/r02at/time_C2.log 2>&1
python tools/time_rollout.py dummy 10000 1000 100 > gpurun_out/r02at/time_dummy.log 2>&1
