mkdir -p gpurun_out/r02ar
for i in 1 2; do
python tools/time_rollout.py cartpole 10000 1000 100 > gpurun_out/r02ar/base_$i.log 2>&1
WS_LIBWS=$PWD/paper_2408_00930_b200/lib/exp64/libws.so python tools/time_rollout.py cartpole 10000 1000 100 > gpurun_out/r02ar/exp64_$i.log 2>&1
done
WS_LIBWS=$PWD/paper_2408_00930_b200/lib/exp64/libws.so timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "c2 or C2 or tiny or truncation" > gpurun_out/r02ar/pytest_exp64.log 2>&1; echo "exit $?" >> gpurun_out/r02ar/pytest_exp64.log
