mkdir -p gpurun_out/r02av
for b in 128 64 32 128; do python tools/time_rollout.py cartpole 10000 1000 100 $b; done > gpurun_out/r02av/blocks.log 2>&1
