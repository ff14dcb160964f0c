# round-2 final evidence, part F: bench lines of the workloads the per-warp flushes changed, the default line
mkdir -p gpurun_out/r02_final
python bench.py > gpurun_out/r02_final/bench_default.log 2>&1; tail -1 gpurun_out/r02_final/bench_default.log > gpurun_out/r02_final/bench_default.jsonl
for w in C1 C5 C2G C2S D0; do
  timeout 600 python bench.py --workload $w --no-cpu-baseline --sustain-s 0.5 > gpurun_out/r02_final/bench_f_$w.log 2>&1
done
