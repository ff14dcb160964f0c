# round-2 end measurements: default bench line, every workload, launch list, ncu tables
mkdir -p gpurun_out/r02_end
python bench.py > gpurun_out/r02_end/bench_default.log 2>&1; tail -1 gpurun_out/r02_end/bench_default.log > gpurun_out/r02_end/bench_default.jsonl
python bench.py --impl reference > gpurun_out/r02_end/bench_reference.log 2>&1; tail -1 gpurun_out/r02_end/bench_reference.log > gpurun_out/r02_end/bench_reference.jsonl
for w in C1 C2S C3a C3S C3b C4 C5 D0 C2P C2G C4G C2T C2O C3T C4T C2X C2U; do
  timeout 600 python bench.py --workload $w --no-cpu-baseline --sustain-s 0.5 > gpurun_out/r02_end/bench_$w.log 2>&1
  tail -1 gpurun_out/r02_end/bench_$w.log >> gpurun_out/r02_end/workloads.jsonl
done
ncu --metrics gpu__time_duration.sum --clock-control none -s 15 -c 12 --csv --log-file gpurun_out/r02_end/launches_C2.csv python bench.py --steps 5 --warmup 3 --ncu > /dev/null 2>&1
mkdir -p gpurun_out/ncu_r02_end
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_plan" -s 1 -c 1 -o gpurun_out/ncu_r02_end/plan_C2 -f python bench.py --workload C2 --steps 1 --warmup 1 --ncu > gpurun_out/ncu_r02_end/plan_C2.log 2>&1
ncu -i gpurun_out/ncu_r02_end/plan_C2.ncu-rep --page raw --csv > gpurun_out/ncu_r02_end/plan_C2.raw.csv 2>/dev/null
ncu -i gpurun_out/ncu_r02_end/plan_C2.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu_r02_end/plan_C2.src.csv 2>/dev/null
rm -f gpurun_out/ncu_r02_end/plan_C2.ncu-rep
bash tools/ncu_table.sh r02_end C2 C2S C3a C3S C3b C4 C5 D0 C2U
