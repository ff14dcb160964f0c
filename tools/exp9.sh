#!/bin/bash
L=$PWD/paper_2408_00930_b200/lib/exp
for x in "" a16_5 a8_6 a32_1; do
  if [ -n "$x" ]; then export WS_LIBWS=$L/libws_$x.so; fi
  echo "== ${x:-default}"; timeout 300 python tools/sweep.py acrobot 12500,100000 128 500
done
unset WS_LIBWS
timeout 300 python tools/sweep.py cartpole 10000,640000 128 1000
timeout 300 python tools/sweep.py pendulum 100000 128 200
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
