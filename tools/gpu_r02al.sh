mkdir -p gpurun_out/r02al
python tools/time_rollout.py surface 2000 200 50 > gpurun_out/r02al/time_C5_k8.log 2>&1
WS_LIBWS=$PWD/paper_2408_00930_b200/lib/exp16/libws.so python tools/time_rollout.py surface 2000 200 50 > gpurun_out/r02al/time_C5_k16.log 2>&1
WS_LIBWS=$PWD/paper_2408_00930_b200/lib/exp16/libws.so timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "surface or C5 or gaussian" > gpurun_out/r02al/pytest_k16.log 2>&1; echo "pytest exit $?" >> gpurun_out/r02al/pytest_k16.log
WS_LIBWS=$PWD/paper_2408_00930_b200/lib/exp16/libws.so timeout 300 python bench.py --workload C5 --no-cpu-baseline --sustain-s 0.3 > gpurun_out/r02al/bench_C5_k16.log 2>&1
