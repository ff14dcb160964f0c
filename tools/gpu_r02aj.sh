mkdir -p gpurun_out/r02aj
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "surface or C5 or gaussian" > gpurun_out/r02aj/pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/r02aj/pytest.log
timeout 300 python bench.py --workload C5 --no-cpu-baseline --sustain-s 0.3 > gpurun_out/r02aj/bench_C5.log 2>&1
python tools/time_rollout.py surface 2000 200 50 > gpurun_out/r02aj/time_C5.log 2>&1
