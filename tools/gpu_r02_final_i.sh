# round-2 final evidence, part I: the full set on the final code -- GPU suite, smoke, default line
# (with the CPU baseline), the reference arm, every workload line
mkdir -p gpurun_out/r02_final
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r02_final/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/r02_final/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r02_final/smoke.log 2>&1
python bench.py > gpurun_out/r02_final/bench_default.log 2>&1; tail -1 gpurun_out/r02_final/bench_default.log > gpurun_out/r02_final/bench_default.jsonl
python bench.py --impl reference > gpurun_out/r02_final/bench_reference.log 2>&1; tail -1 gpurun_out/r02_final/bench_reference.log > gpurun_out/r02_final/bench_reference.jsonl
rm -f gpurun_out/r02_final/workloads.jsonl
for w in C1 C2S C3a C3S C3b C4 C5 D0 C2P C2G C4G C2T C2O C3T C4T C2X C2U; do
  timeout 600 python bench.py --workload $w --no-cpu-baseline --sustain-s 0.5 > gpurun_out/r02_final/bench_$w.log 2>&1
  tail -1 gpurun_out/r02_final/bench_$w.log >> gpurun_out/r02_final/workloads.jsonl
done
