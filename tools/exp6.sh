#!/bin/bash
L=$PWD/paper_2408_00930_b200/lib/exp
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for x in "" tag5 tag4; do
  if [ -n "$x" ]; then export WS_LIBWS=$L/libws_$x.so; fi
  echo "== ${x:-default}"; timeout 300 python bench.py --workload C4 --steps 10 --warmup 3 --no-cpu-baseline | python -c "import json,sys; d=json.load(sys.stdin); print(d['ms_per_step'], d['roofline']['kernel_ms'], d['roofline']['frac'])"
done
