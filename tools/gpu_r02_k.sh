# composer: out-of-line wide-angle sincos -- A/B of C2U against the library before (lib/old);
# the reduction worst-case test and the composer tests on the new library
mkdir -p gpurun_out/r02_k
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_user_env.py -m gpu -q > gpurun_out/r02_k/pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/r02_k/pytest.log
for rep in 1 2 3; do
  timeout 600 python bench.py --workload C2U --no-cpu-baseline --sustain-s 0.5 2>/dev/null | tail -1 >> gpurun_out/r02_k/new.jsonl
  WS_LIBWS=$PWD/paper_2408_00930_b200/lib/old/libws.so timeout 600 python bench.py --workload C2U --no-cpu-baseline --sustain-s 0.5 2>/dev/null | tail -1 >> gpurun_out/r02_k/old.jsonl
done
