# fused plan+rollout variants (timing only for the NOWAIT ones)
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "fused or c2_cartpole or c1" > gpurun_out/r02c_parity.log 2>&1; tail -2 gpurun_out/r02c_parity.log
show() { tail -1 $1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$2', round(d['ms_per_step'],4), round(d['sustained']['ms_per_step'],4), d['roofline']['kernel_ms'])"; }
python bench.py --no-cpu-baseline --sustain-s 0.5 > gpurun_out/r02c_f.log 2>&1; show gpurun_out/r02c_f.log fused
WS_FUSED_NOWAIT=1 python bench.py --no-cpu-baseline --sustain-s 0.5 > gpurun_out/r02c_fnw.log 2>&1; show gpurun_out/r02c_fnw.log fused_nowait
WS_FUSED_NOWAIT=1 WS_FUSED_PLAN_CTAS=0 python bench.py --no-cpu-baseline --sustain-s 0.5 > gpurun_out/r02c_fnw0.log 2>&1; show gpurun_out/r02c_fnw0.log fused_nowait_noplan
python bench.py --block 64 --no-cpu-baseline --sustain-s 0.5 > gpurun_out/r02c_split64.log 2>&1; show gpurun_out/r02c_split64.log split64
