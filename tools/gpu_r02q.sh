timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r02q_pytest.log 2>&1; tail -2 gpurun_out/r02q_pytest.log
show() { tail -1 $1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$2', round(d['ms_per_step'],4), round(d['sustained']['ms_per_step'],4), r['kernel_ms'], r.get('frac'), r.get('bound'))"; }
for w in C5 C2; do timeout 300 python bench.py --workload $w --no-cpu-baseline --sustain-s 0.3 > gpurun_out/r02q_$w.log 2>&1; show gpurun_out/r02q_$w.log $w; done
