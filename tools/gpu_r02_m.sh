# sincos_c assembled in fp32 (quadrant swap / sign after the rounding): GPU suite on the new
# library, A/B against the previous one (lib/old) on the sincos-heavy workloads
mkdir -p gpurun_out/r02_m
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r02_m/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/r02_m/pytest_gpu.log
for rep in 1 2; do
for w in C3a C3S C3b C3T C5; do
  timeout 600 python bench.py --workload $w --no-cpu-baseline --sustain-s 0.5 2>/dev/null | tail -1 >> gpurun_out/r02_m/new.jsonl
  WS_LIBWS=$PWD/paper_2408_00930_b200/lib/old/libws.so timeout 600 python bench.py --workload $w --no-cpu-baseline --sustain-s 0.5 2>/dev/null | tail -1 >> gpurun_out/r02_m/old.jsonl
done
done
timeout 300 python tools/time_rollout.py acrobot 12500 500 100 > gpurun_out/r02_m/time_C3a_shard.log 2>&1
