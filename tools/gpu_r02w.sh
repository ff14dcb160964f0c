mkdir -p gpurun_out/r02w
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kernels.py tests/test_gpu_staged.py -x -q -k "surface or C5 or gaussian" > gpurun_out/r02w/pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/r02w/pytest.log
timeout 300 python tools/time_rollout.py surface 2000 200 50 > gpurun_out/r02w/time_C5.log 2>&1
bash tools/prof_one.sh C5 k_rollout_surface r02w_C5
