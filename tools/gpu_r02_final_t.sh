# round-2 final evidence, part T: the workload lines that use Box-Muller draws, after its change
mkdir -p gpurun_out/r02_final_t
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r02_final_t/smoke.log 2>&1
for w in C3b C3T C5; do
  timeout 600 python bench.py --workload $w --no-cpu-baseline --sustain-s 0.5 > gpurun_out/r02_final_t/bench_$w.log 2>&1
  tail -1 gpurun_out/r02_final_t/bench_$w.log >> gpurun_out/r02_final_t/workloads.jsonl
done
python bench.py > gpurun_out/r02_final_t/bench_default.log 2>&1; tail -1 gpurun_out/r02_final_t/bench_default.log > gpurun_out/r02_final_t/bench_default.jsonl
