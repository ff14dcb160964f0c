#!/bin/bash
for w in ${WORKLOADS:-C1 C2 C3a C3b C4 C5 D0 C2P C2G C4G C2T C2X}; do
  timeout 600 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err
  echo "$w rc=$?"; python -c "
import json,sys
d=json.load(open('gpurun_out/bench_$w.json')); r=d['roofline']
print('$w', round(d['value']/1e9,3), 'Gsteps/s', 'ms', round(d['ms_per_step'],3), 'kernel', r['kernel'], round(r['kernel_ms'],3), 'ms', r['achieved'], 'GB/s', r['frac'])
" 2>&1 | tail -1
done
