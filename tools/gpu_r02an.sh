mkdir -p gpurun_out/r02an
timeout 900 python -m pytest tests/test_gpu_a2c.py -x -q -k "ppo" > gpurun_out/r02an/pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/r02an/pytest.log
