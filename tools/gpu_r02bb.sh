mkdir -p gpurun_out/r02bb
for i in 1 2; do
python tools/time_rollout.py cartpole 10000 1000 100 > gpurun_out/r02bb/base_$i.log 2>&1
WS_LIBWS=$PWD/paper_2408_00930_b200/lib/pc64/libws.so python tools/time_rollout.py cartpole 10000 1000 100 > gpurun_out/r02bb/pc64_$i.log 2>&1
WS_LIBWS=$PWD/paper_2408_00930_b200/lib/pc32/libws.so python tools/time_rollout.py cartpole 10000 1000 100 > gpurun_out/r02bb/pc32_$i.log 2>&1
done
