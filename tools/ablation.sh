#!/bin/bash
# C2 ablation: build the WS_EXP variants here (CPU), then run this on the GPU.
#   for x in 2 4 8 16 30; do python paper_2408_00930_b200/build.py -DWS_EXP=$x \
#       --out=paper_2408_00930_b200/lib/exp/libws_$x.so; done
# WS_EXP bits: 1 fast CartPole dynamics everywhere, 2 no statistics, 4 no stores, 8 no reset
# refill, 16 fp32 hardware sin (breaks parity: timing only).
echo "base"; python tools/sweep.py cartpole 10000,160000 128 1000
for x in 16 2 4 8 30; do
  echo "WS_EXP=$x"; WS_LIBWS=$PWD/paper_2408_00930_b200/lib/exp/libws_$x.so python tools/sweep.py cartpole 10000,160000 128 1000
done
