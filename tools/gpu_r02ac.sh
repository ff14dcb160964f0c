mkdir -p gpurun_out/r02ac
timeout 900 python -m pytest tests/test_gpu_policy.py tests/test_gpu_parity.py tests/test_gpu_checkpoint.py -x -q > gpurun_out/r02ac/pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/r02ac/pytest.log
timeout 300 python tools/time_policy_graph.py 10000 1000 5 > gpurun_out/r02ac/policy_graph.log 2>&1
