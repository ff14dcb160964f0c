# round-2 final evidence, part H: lines changed by the last plan-kernel edits; the GPU suite
mkdir -p gpurun_out/r02_final
for w in C3b C5 C3T; do
  timeout 600 python bench.py --workload $w --no-cpu-baseline --sustain-s 0.5 > gpurun_out/r02_final/bench_h_$w.log 2>&1
done
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/r02_final/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/r02_final/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r02_final/smoke.log 2>&1
