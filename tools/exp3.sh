#!/bin/bash
# A/B: warp-specialised group kernel (default) vs plan + single-warp roll-out (WS_EXP=64)
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
echo "== group"; timeout 300 python tools/sweep.py cartpole 10000,40000,640000 96,192 1000
timeout 300 python tools/sweep.py acrobot 12500,100000 96,192 500
timeout 300 python tools/sweep.py dummy 1000000 96,192 100
echo "== old"; WS_LIBWS=$PWD/paper_2408_00930_b200/lib/exp/libws_64.so timeout 300 python tools/sweep.py cartpole 10000,640000 128 1000
timeout 900 python -m pytest tests -m gpu -x -q ${PYARGS} 2>&1 | tail -15
