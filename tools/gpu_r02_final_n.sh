# round-2 final evidence, part N: after the fp32 sincos assembly -- ncu tables of the changed
# roll-out kernels, issue-view counts refreshed on the box, then their workload lines
mkdir -p gpurun_out/r02_final_n
bash tools/ncu_table.sh r02_final C3a C3S C3b C5 > gpurun_out/r02_final_n/ncu_table.log 2>&1
python tools/ncu_table.py r02_final > gpurun_out/r02_final_n/ncu_table_py.log 2>&1
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r02_final_n/smoke.log 2>&1
for w in C3a C3S C3b C3T C5; do
  timeout 600 python bench.py --workload $w --no-cpu-baseline --sustain-s 0.5 > gpurun_out/r02_final_n/bench_$w.log 2>&1
  tail -1 gpurun_out/r02_final_n/bench_$w.log >> gpurun_out/r02_final_n/workloads.jsonl
done
ncu --metrics gpu__time_duration.sum --clock-control none -s 15 -c 12 --csv --log-file gpurun_out/r02_final_n/launches_C5.csv python bench.py --workload C5 --steps 5 --warmup 3 --ncu > /dev/null 2>&1
