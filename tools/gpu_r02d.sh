timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/r02d_parity.log 2>&1; tail -2 gpurun_out/r02d_parity.log
show() { tail -1 $1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$2', round(d['ms_per_step'],4), round(d['sustained']['ms_per_step'],4), d['roofline']['kernel_ms'], d['roofline'].get('frac'), d['roofline'].get('bound'))"; }
python bench.py --no-cpu-baseline --sustain-s 0.5 > gpurun_out/r02d_f.log 2>&1; show gpurun_out/r02d_f.log fused_geo
WS_LIBWS=paper_2408_00930_b200/lib/exp64/libws.so python bench.py --no-cpu-baseline --sustain-s 0.5 > gpurun_out/r02d_fldg.log 2>&1; show gpurun_out/r02d_fldg.log fused_ldg
WS_FUSED_NOWAIT=1 WS_LIBWS=paper_2408_00930_b200/lib/exp64/libws.so python bench.py --no-cpu-baseline --sustain-s 0.5 > gpurun_out/r02d_fldgnw.log 2>&1; show gpurun_out/r02d_fldgnw.log fused_ldg_nowait
python bench.py --workload C5 --no-cpu-baseline --sustain-s 0.5 > gpurun_out/r02d_C5.log 2>&1; show gpurun_out/r02d_C5.log C5
timeout 900 python -m pytest tests/ -x -q -m gpu -k "surface or C5 or full_size" > gpurun_out/r02d_surf.log 2>&1; tail -2 gpurun_out/r02d_surf.log
