# round-2 final evidence, part E (after the per-warp statistics flushes): ncu of the changed roll-out kernels, C2 launch list
mkdir -p gpurun_out/r02_final
bash tools/ncu_table.sh r02_final C2 C5 C1 > gpurun_out/r02_final/ncu_table_e.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -s 15 -c 12 --csv --log-file gpurun_out/r02_final/launches_C2.csv python bench.py --steps 5 --warmup 3 --ncu > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -s 15 -c 12 --csv --log-file gpurun_out/r02_final/launches_C5.csv python bench.py --workload C5 --steps 5 --warmup 3 --ncu > /dev/null 2>&1
