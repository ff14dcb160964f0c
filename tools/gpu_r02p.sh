timeout 900 python -m pytest tests/test_gpu_user_env.py -x -q > gpurun_out/r02p_pytest.log 2>&1; tail -3 gpurun_out/r02p_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
show() { tail -1 $1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$2', round(d['ms_per_step'],4), round(d['sustained']['ms_per_step'],4), r['kernel_ms'], r.get('frac'), r.get('bound'))"; }
timeout 300 python bench.py --workload C2U --no-cpu-baseline --sustain-s 0.3 > gpurun_out/r02p_C2U.log 2>&1; show gpurun_out/r02p_C2U.log C2U
