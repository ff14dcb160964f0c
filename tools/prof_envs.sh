#!/bin/bash
# full ncu captures of the roll-out kernel of several workloads (+ the Gaussian plan of C3b)
mkdir -p gpurun_out
for w in ${WL:-C3a C3b C4 C5}; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_rollout|k_tag" -s 1 -c 1 \
      -o gpurun_out/prof_env_$w -f python bench.py --workload $w --steps 1 --warmup 1 --ncu > gpurun_out/ncu_env_$w.log 2>&1
  echo "$w rc=$?"
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_plan" -s 1 -c 1 \
    -o gpurun_out/prof_plan_C3b -f python bench.py --workload C3b --steps 1 --warmup 1 --ncu > gpurun_out/ncu_plan_C3b.log 2>&1
echo "plan C3b rc=$?"
# export the pages here (the reports themselves are too large to bring back together)
for f in gpurun_out/prof_env_*.ncu-rep gpurun_out/prof_plan_*.ncu-rep; do
  b=${f%.ncu-rep}
  ncu -i $f --page raw --csv > $b.raw.csv 2>/dev/null
  ncu -i $f --page source --csv --print-source sass > $b.src.csv 2>/dev/null
  ncu -i $f --page details --csv > $b.details.csv 2>/dev/null
  rm -f $f
done
ls -la gpurun_out
