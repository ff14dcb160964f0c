#!/bin/bash
# plan chunk (pc64/pc32) and roll-out min-blocks (mb5/mb6) experiments
L=$PWD/paper_2408_00930_b200/lib/exp
echo "== default"; timeout 300 python tools/sweep.py cartpole 10000,640000 128 1000; timeout 300 python tools/sweep.py acrobot 12500,100000 128 500
for x in pc64 pc32; do echo "== $x"; WS_LIBWS=$L/libws_$x.so timeout 300 python tools/sweep.py cartpole 10000,640000 128 1000; done
for x in mb5 mb6; do echo "== $x"; WS_LIBWS=$L/libws_$x.so timeout 300 python tools/sweep.py acrobot 12500,100000 128 500; WS_LIBWS=$L/libws_$x.so timeout 300 python tools/sweep.py cartpole 10000,640000 128 1000; done
