timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/r02i_parity.log 2>&1; tail -2 gpurun_out/r02i_parity.log
show() { tail -1 $1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$2', round(d['ms_per_step'],4), round(d['sustained']['ms_per_step'],4), r['kernel_ms'], r['other_kernels'].get('plan',{}).get('ms'))"; }
for w in C2 C2S C3a C1; do python bench.py --workload $w --no-cpu-baseline --sustain-s 0.3 > gpurun_out/r02i_$w.log 2>&1; show gpurun_out/r02i_$w.log $w; done
