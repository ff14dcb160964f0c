#!/bin/bash
L=$PWD/paper_2408_00930_b200/lib/exp
for x in ""; do
  if [ -n "$x" ]; then export WS_LIBWS=$L/libws_$x.so; fi
  echo "== ${x:-default}"; timeout 300 python bench.py --workload C5 --steps 10 --warmup 3 --no-cpu-baseline | python -c "import json,sys; d=json.load(sys.stdin); r=d['roofline']; print(d['ms_per_step'], r['kernel_ms'], r['other_kernels'])"
done
timeout 600 python -m pytest tests -m gpu -x -q -k "surface or C5" 2>&1 | tail -2
