# minimax small-angle sincos (CartPole, composer): GPU suite on the new library, then A/B of the
# CartPole workloads against the library with only the sincos64 change (lib/s64), alternating
mkdir -p gpurun_out/r02_sincos_b
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r02_sincos_b/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/r02_sincos_b/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r02_sincos_b/smoke.log 2>&1
for rep in 1 2 3; do
for w in C2 C2P C2G C2O C2T C2U; do
  timeout 600 python bench.py --workload $w --no-cpu-baseline --sustain-s 0.5 2>/dev/null | tail -1 >> gpurun_out/r02_sincos_b/new.jsonl
  WS_LIBWS=$PWD/paper_2408_00930_b200/lib/s64/libws.so timeout 600 python bench.py --workload $w --no-cpu-baseline --sustain-s 0.5 2>/dev/null | tail -1 >> gpurun_out/r02_sincos_b/s64.jsonl
done
done
