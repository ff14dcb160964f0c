# round-2 final evidence, part P (after the kTrig padding): ncu tables of the kernels whose code moved (C5, C2U),
# the issue-view counts refreshed on the box before any bench line, then the GPU suite, smoke, the
# default line (with the CPU baseline), the reference arm, every workload line, the launch lists
mkdir -p gpurun_out/r02_final
bash tools/ncu_table.sh r02_final C5 C2U > gpurun_out/r02_final/ncu_table_p.log 2>&1
python tools/ncu_table.py r02_final > gpurun_out/r02_final/ncu_table_p_py.log 2>&1
cp profiles/ncu_inst.json gpurun_out/r02_final/ncu_inst_box.json
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r02_final/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/r02_final/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r02_final/smoke.log 2>&1
python bench.py > gpurun_out/r02_final/bench_default.log 2>&1; tail -1 gpurun_out/r02_final/bench_default.log > gpurun_out/r02_final/bench_default.jsonl
python bench.py --impl reference > gpurun_out/r02_final/bench_reference.log 2>&1; tail -1 gpurun_out/r02_final/bench_reference.log > gpurun_out/r02_final/bench_reference.jsonl
rm -f gpurun_out/r02_final/workloads.jsonl
for w in C1 C2S C3a C3S C3b C4 C5 D0 C2P C2G C4G C2T C2O C3T C4T C2X C2U; do
  timeout 600 python bench.py --workload $w --no-cpu-baseline --sustain-s 0.5 > gpurun_out/r02_final/bench_$w.log 2>&1
  tail -1 gpurun_out/r02_final/bench_$w.log >> gpurun_out/r02_final/workloads.jsonl
done
ncu --metrics gpu__time_duration.sum --clock-control none -s 15 -c 12 --csv --log-file gpurun_out/r02_final/launches_C2.csv python bench.py --steps 5 --warmup 3 --ncu > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -s 15 -c 12 --csv --log-file gpurun_out/r02_final/launches_C5.csv python bench.py --workload C5 --steps 5 --warmup 3 --ncu > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_a2c.py -q -k "solved or learns" -s > gpurun_out/r02_final/learning.log 2>&1
