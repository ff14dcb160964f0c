#!/bin/bash
echo "EXP base"; python tools/sweep.py cartpole 10000,160000 128 1000
echo "EXP 32"; WS_LIBWS=$PWD/paper_2408_00930_b200/lib/exp/libws_32.so python tools/sweep.py cartpole 10000,160000 128 1000
