mkdir -p gpurun_out/r02aw
timeout 900 python -m pytest tests/test_gpu_gae.py tests/test_gpu_a2c.py -x -q > gpurun_out/r02aw/pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/r02aw/pytest.log
for w in C2G C4G C2T; do timeout 300 python bench.py --workload $w --no-cpu-baseline --sustain-s 0.3 > gpurun_out/r02aw/bench_$w.log 2>&1; done
