mkdir -p gpurun_out/r02bd
for i in 1 2 3; do
python tools/time_rollout.py cartpole 10000 1000 100 > gpurun_out/r02bd/new_$i.log 2>&1
WS_LIBWS=$PWD/paper_2408_00930_b200/lib/old/libws.so python tools/time_rollout.py cartpole 10000 1000 100 > gpurun_out/r02bd/old_$i.log 2>&1
done
