timeout 1500 python -m pytest tests/test_gpu_policy.py tests/test_gpu_a2c.py tests/test_gpu_user_env.py tests/test_gpu_a2c_dp.py -x -q > gpurun_out/r02k_pytest.log 2>&1; tail -3 gpurun_out/r02k_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
show() { tail -1 $1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$2', round(d['ms_per_step'],4), round(d['sustained']['ms_per_step'],4), r['kernel_ms'], r.get('frac'), r.get('bound'))"; }
for w in C2P C2T C3T C4T C2U; do python bench.py --workload $w --no-cpu-baseline --sustain-s 0.3 > gpurun_out/r02k_$w.log 2>&1; show gpurun_out/r02k_$w.log $w; done
