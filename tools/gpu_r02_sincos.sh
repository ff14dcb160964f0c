# minimax sincos64: GPU suite on the new library, then A/B of the fp64-trig workloads against the
# previous library (lib/old) on the same box, alternating
mkdir -p gpurun_out/r02_sincos
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r02_sincos/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/r02_sincos/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r02_sincos/smoke.log 2>&1
for rep in 1 2; do
for w in C3a C3S C3T C4 C4T C5 C2U; do
  timeout 600 python bench.py --workload $w --no-cpu-baseline --sustain-s 0.5 2>/dev/null | tail -1 >> gpurun_out/r02_sincos/new.jsonl
  WS_LIBWS=$PWD/paper_2408_00930_b200/lib/old/libws.so timeout 600 python bench.py --workload $w --no-cpu-baseline --sustain-s 0.5 2>/dev/null | tail -1 >> gpurun_out/r02_sincos/old.jsonl
done
done
