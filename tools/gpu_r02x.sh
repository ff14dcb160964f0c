mkdir -p gpurun_out/r02x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02x/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/r02x/pytest_gpu.log
for w in C5 C2P C2T; do
  timeout 300 python bench.py --workload $w --no-cpu-baseline --sustain-s 0.3 > gpurun_out/r02x/bench_$w.log 2>&1
done
