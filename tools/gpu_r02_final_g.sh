# round-2 final evidence, part G: the training / GAE workload lines after the GAE and packed-pair gradient changes
mkdir -p gpurun_out/r02_final
for w in C2G C4G C2T C2O C3T C4T; do
  timeout 600 python bench.py --workload $w --no-cpu-baseline --sustain-s 0.5 > gpurun_out/r02_final/bench_g_$w.log 2>&1
done
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/r02_final/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/r02_final/pytest_gpu.log
