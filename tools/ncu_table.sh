#!/bin/bash
# ncu_table.sh <tag> [workloads...]: one `ncu --set full` capture of the dominant roll-out kernel of
# each workload (second launch: after one warm-up roll-out), exported to csv pages on the box
# (raw metrics + source page), for tools/ncu_table.py -> profiles/ncu_inst.json
tag=$1; shift
mkdir -p gpurun_out/ncu_$tag
for w in "${@:-C2 C3a C3b C4 C5 D0 C2S C3S}"; do
  k="k_rollout|k_tag|k_user_rollout"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$k" -s 1 -c 1 \
      -o gpurun_out/ncu_$tag/$w -f python bench.py --workload $w --steps 1 --warmup 1 --ncu \
      > gpurun_out/ncu_$tag/$w.log 2>&1
  echo "$w rc=$?"
  ncu -i gpurun_out/ncu_$tag/$w.ncu-rep --page raw --csv > gpurun_out/ncu_$tag/$w.raw.csv 2>/dev/null
  ncu -i gpurun_out/ncu_$tag/$w.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu_$tag/$w.src.csv 2>/dev/null
  ncu -i gpurun_out/ncu_$tag/$w.ncu-rep --page details --csv > gpurun_out/ncu_$tag/$w.details.csv 2>/dev/null
  rm -f gpurun_out/ncu_$tag/$w.ncu-rep
done
