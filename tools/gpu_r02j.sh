timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/r02j_parity.log 2>&1; tail -2 gpurun_out/r02j_parity.log
for E in 12500 100000 400000; do python tools/time_rollout.py acrobot $E 500 5; done
python tools/time_rollout.py cartpole 10000 1000 20
