timeout 900 python -m pytest tests/test_gpu_policy.py -x -q > gpurun_out/r02n_pytest.log 2>&1; tail -2 gpurun_out/r02n_pytest.log
show() { tail -1 $1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$2', round(d['ms_per_step'],4), round(d['sustained']['ms_per_step'],4), r['kernel_ms'], r.get('frac'), r.get('bound'))"; }
timeout 300 python bench.py --workload C2P --no-cpu-baseline --sustain-s 0.3 > gpurun_out/r02n_C2P.log 2>&1; show gpurun_out/r02n_C2P.log C2P
mkdir -p gpurun_out/ncu_r02n
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_rollout_policy" -s 1 -c 1 -o gpurun_out/ncu_r02n/C2P -f python bench.py --workload C2P --steps 1 --warmup 1 --ncu > gpurun_out/ncu_r02n/C2P.log 2>&1
ncu -i gpurun_out/ncu_r02n/C2P.ncu-rep --page raw --csv > gpurun_out/ncu_r02n/C2P.raw.csv 2>/dev/null
ncu -i gpurun_out/ncu_r02n/C2P.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu_r02n/C2P.src.csv 2>/dev/null
rm -f gpurun_out/ncu_r02n/C2P.ncu-rep
