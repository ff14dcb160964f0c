# Box-Muller fp32-side signs, gauss_z's swap condition fixed: GPU suite, A/B against lib/old
mkdir -p gpurun_out/r02_s
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r02_s/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/r02_s/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r02_s/smoke.log 2>&1
for rep in 1 2; do
for w in C3b C5 C3T; do
  timeout 600 python bench.py --workload $w --no-cpu-baseline --sustain-s 0.5 2>/dev/null | tail -1 >> gpurun_out/r02_s/new.jsonl
  WS_LIBWS=$PWD/paper_2408_00930_b200/lib/old/libws.so timeout 600 python bench.py --workload $w --no-cpu-baseline --sustain-s 0.5 2>/dev/null | tail -1 >> gpurun_out/r02_s/old.jsonl
done
done
