#!/bin/bash
L=$PWD/paper_2408_00930_b200/lib/exp
for x in "" w16 w32; do
  if [ -n "$x" ]; then export WS_LIBWS=$L/libws_$x.so; fi
  echo "== ${x:-default}"; timeout 300 python bench.py --workload C3b --steps 10 --warmup 3 --no-cpu-baseline | python -c "import json,sys; d=json.load(sys.stdin); r=d['roofline']; print(d['ms_per_step'], r['kernel_ms'], r['frac'])"
  timeout 300 python tools/sweep.py pendulum 100000,400000 128,256 200
done
unset WS_LIBWS
timeout 600 python -m pytest tests -m gpu -x -q -k "pendulum or C3b or statistics or single_step" 2>&1 | tail -2
