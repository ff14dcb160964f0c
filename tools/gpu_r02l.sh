mkdir -p gpurun_out/ncu_r02l
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_rollout_policy" -s 1 -c 1 -o gpurun_out/ncu_r02l/C2P -f python bench.py --workload C2P --steps 1 --warmup 1 --ncu > gpurun_out/ncu_r02l/C2P.log 2>&1
ncu -i gpurun_out/ncu_r02l/C2P.ncu-rep --page raw --csv > gpurun_out/ncu_r02l/C2P.raw.csv 2>/dev/null
ncu -i gpurun_out/ncu_r02l/C2P.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu_r02l/C2P.src.csv 2>/dev/null
rm -f gpurun_out/ncu_r02l/C2P.ncu-rep
