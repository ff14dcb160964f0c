#!/bin/bash
echo "EXP base"; python tools/sweep.py cartpole 10000,160000 128 1000
for x in 16 2 4 8 30; do
  echo "EXP $x"; WS_LIBWS=$PWD/paper_2408_00930_b200/lib/exp/libws_$x.so python tools/sweep.py cartpole 10000,160000 128 1000
done
