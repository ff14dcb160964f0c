# round-2 re-entry check: full GPU suite + default bench line on the restored tree
mkdir -p gpurun_out/r02t
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02t/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/r02t/pytest_gpu.log
python bench.py --no-cpu-baseline > gpurun_out/r02t/bench_default.log 2>&1
python tools/time_rollout.py cartpole 10000 1000 50 > gpurun_out/r02t/time_rollout.log 2>&1
