mkdir -p gpurun_out/r02ag
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multirank.py tests/test_gpu_checkpoint.py -x -q > gpurun_out/r02ag/pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/r02ag/pytest.log
python bench.py --no-cpu-baseline > gpurun_out/r02ag/bench_C2.log 2>&1
for w in C2S C3a; do
  timeout 300 python bench.py --workload $w --no-cpu-baseline --sustain-s 0.3 > gpurun_out/r02ag/bench_$w.log 2>&1
done
python tools/time_rollout.py cartpole 10000 1000 50 > gpurun_out/r02ag/time_C2.log 2>&1
