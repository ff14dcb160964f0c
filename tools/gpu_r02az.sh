mkdir -p gpurun_out/r02az
for b in 128 64 32 256 128; do python tools/time_rollout.py surface 2000 200 100 $b; done > gpurun_out/r02az/blocks.log 2>&1
for b in 128 64 32 128; do python tools/time_rollout.py acrobot 12500 500 20 $b; done >> gpurun_out/r02az/blocks.log 2>&1
