# Box-Muller with the quadrant swap before the products and the signs on the rounded fp32 bits
# (no wide-argument check): GPU suite on the new library, A/B against the previous one (lib/old)
mkdir -p gpurun_out/r02_r
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r02_r/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/r02_r/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r02_r/smoke.log 2>&1
for rep in 1 2; do
for w in C3b C5 C3T C2U; do
  timeout 600 python bench.py --workload $w --no-cpu-baseline --sustain-s 0.5 2>/dev/null | tail -1 >> gpurun_out/r02_r/new.jsonl
  WS_LIBWS=$PWD/paper_2408_00930_b200/lib/old/libws.so timeout 600 python bench.py --workload $w --no-cpu-baseline --sustain-s 0.5 2>/dev/null | tail -1 >> gpurun_out/r02_r/old.jsonl
done
done
