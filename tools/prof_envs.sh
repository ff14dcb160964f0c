#!/bin/bash
mkdir -p gpurun_out
for w in C3a C4 C5; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_rollout|k_tag" -s 1 -c 1 \
      -o gpurun_out/prof_env_$w -f python bench.py --workload $w --steps 1 --warmup 1 --ncu > gpurun_out/ncu_env_$w.log 2>&1
  echo "$w rc=$?"
done
