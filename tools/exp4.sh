#!/bin/bash
# group kernel R=1 (exp 128) and R=2 (exp 256) vs the default (plan + single-warp roll-out)
L=$PWD/paper_2408_00930_b200/lib/exp
echo "== default"; timeout 300 python tools/sweep.py cartpole 10000,40000,640000 128 1000
for x in 128 256; do
  echo "== exp $x"; WS_LIBWS=$L/libws_$x.so timeout 300 python tools/sweep.py cartpole 10000,20000,40000,640000 96,192 1000
done
for x in 256 128; do
  echo "== parity exp $x"; WS_LIBWS=$L/libws_$x.so timeout 900 python -m pytest tests -m gpu -x -q --deselect tests/test_gpu_multirank.py::test_two_rank_bench_matches_oracle 2>&1 | tail -4
done
