# round-2 final evidence, part J (after the near-minimax sincos polynomials and the three-FMA
# reduction): GPU suite, A/B of the reduction against the previous library (lib/old), smoke, the
# default line (with the CPU baseline), the reference arm, every workload line, ncu tables of the
# kernels whose code changed, the C2 / C5 launch lists
mkdir -p gpurun_out/r02_final gpurun_out/r02_reduc
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r02_final/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/r02_final/pytest_gpu.log
for rep in 1 2; do
for w in C3a C3S C3T C5; do
  timeout 600 python bench.py --workload $w --no-cpu-baseline --sustain-s 0.5 2>/dev/null | tail -1 >> gpurun_out/r02_reduc/new.jsonl
  WS_LIBWS=$PWD/paper_2408_00930_b200/lib/old/libws.so timeout 600 python bench.py --workload $w --no-cpu-baseline --sustain-s 0.5 2>/dev/null | tail -1 >> gpurun_out/r02_reduc/old.jsonl
done
done
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r02_final/smoke.log 2>&1
python bench.py > gpurun_out/r02_final/bench_default.log 2>&1; tail -1 gpurun_out/r02_final/bench_default.log > gpurun_out/r02_final/bench_default.jsonl
python bench.py --impl reference > gpurun_out/r02_final/bench_reference.log 2>&1; tail -1 gpurun_out/r02_final/bench_reference.log > gpurun_out/r02_final/bench_reference.jsonl
rm -f gpurun_out/r02_final/workloads.jsonl
for w in C1 C2S C3a C3S C3b C4 C5 D0 C2P C2G C4G C2T C2O C3T C4T C2X C2U; do
  timeout 600 python bench.py --workload $w --no-cpu-baseline --sustain-s 0.5 > gpurun_out/r02_final/bench_$w.log 2>&1
  tail -1 gpurun_out/r02_final/bench_$w.log >> gpurun_out/r02_final/workloads.jsonl
done
bash tools/ncu_table.sh r02_final C2 C3a C3S C2P C3b C5 > gpurun_out/r02_final/ncu_table_j.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -s 15 -c 12 --csv --log-file gpurun_out/r02_final/launches_C2.csv python bench.py --steps 5 --warmup 3 --ncu > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -s 15 -c 12 --csv --log-file gpurun_out/r02_final/launches_C5.csv python bench.py --workload C5 --steps 5 --warmup 3 --ncu > /dev/null 2>&1
