set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/r02b_parity.log 2>&1; tail -3 gpurun_out/r02b_parity.log
for b in 0 64 32; do python bench.py --block $b --no-cpu-baseline --sustain-s 0.5 > gpurun_out/r02b_bench_b$b.log 2>&1; tail -1 gpurun_out/r02b_bench_b$b.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('block', $b, d['ms_per_step'], d['sustained']['ms_per_step'], d['roofline']['kernel_ms'])"; done
WS_FUSED_PLAN_CTAS=0 python bench.py --no-cpu-baseline --sustain-s 0.5 > gpurun_out/r02b_bench_p0.log 2>&1; tail -1 gpurun_out/r02b_bench_p0.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('planctas0', d['ms_per_step'], d['sustained']['ms_per_step'])"
python bench.py --workload C1 --no-cpu-baseline --sustain-s 0.5 > gpurun_out/r02b_bench_C1.log 2>&1; tail -1 gpurun_out/r02b_bench_C1.log | cut -c1-300
ncu --metrics gpu__time_duration.sum --clock-control none -s 10 -c 10 --csv --log-file gpurun_out/r02b_launches.csv python bench.py --steps 5 --warmup 3 --ncu > /dev/null 2>&1
