#!/bin/bash
# prof_one.sh <workload> <kernel regex> <tag>: one full ncu capture, exported to csv pages on the box
mkdir -p gpurun_out
w=$1; k=$2; tag=$3
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"$k" -s 1 -c 1 \
    -o gpurun_out/prof_$tag -f python bench.py --workload $w --steps 1 --warmup 1 --ncu > gpurun_out/ncu_$tag.log 2>&1
echo "$tag rc=$?"
ncu -i gpurun_out/prof_$tag.ncu-rep --page raw --csv > gpurun_out/prof_$tag.raw.csv 2>/dev/null
ncu -i gpurun_out/prof_$tag.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_$tag.src.csv 2>/dev/null
ncu -i gpurun_out/prof_$tag.ncu-rep --page details --csv > gpurun_out/prof_$tag.details.csv 2>/dev/null
rm -f gpurun_out/prof_$tag.ncu-rep
