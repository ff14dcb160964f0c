show() { tail -1 $1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$2', round(d['ms_per_step'],4), round(d['sustained']['ms_per_step'],4), d['roofline']['kernel_ms'])"; }
export WS_LIBWS=paper_2408_00930_b200/lib/exp256/libws.so
for sm in 0 80000 119808; do
WS_FUSED_OFF=1 WS_SPLIT_SMEM=$sm python bench.py --no-cpu-baseline --sustain-s 0.3 > gpurun_out/r02f_$sm.log 2>&1; show gpurun_out/r02f_$sm.log split128_smem$sm
done
WS_FUSED_PLAN_CTAS=0 WS_FUSED_NOWAIT=1 python bench.py --no-cpu-baseline --sustain-s 0.3 > gpurun_out/r02f_fnw.log 2>&1; show gpurun_out/r02f_fnw.log fused_nowait_noplan
