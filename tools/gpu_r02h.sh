timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "grid or c2_cartpole or c1 or per_step or invalid or tiny" > gpurun_out/r02h_parity.log 2>&1; tail -2 gpurun_out/r02h_parity.log
WS_LIBWS=paper_2408_00930_b200/lib/pc32/libws.so timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "grid or c2_cartpole or c1 or per_step or invalid or tiny or launch_shape" > gpurun_out/r02h_parity32.log 2>&1; tail -2 gpurun_out/r02h_parity32.log
show() { tail -1 $1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$2', round(d['ms_per_step'],4), round(d['sustained']['ms_per_step'],4), r['kernel_ms'], r['other_kernels'].get('plan',{}).get('ms'))"; }
for lib in lib pc32 pc64; do
  L=paper_2408_00930_b200/lib/libws.so; [ $lib != lib ] && L=paper_2408_00930_b200/lib/$lib/libws.so
  for w in C2 C2S C3a; do WS_LIBWS=$L python bench.py --workload $w --no-cpu-baseline --sustain-s 0.3 > gpurun_out/r02h_${lib}_$w.log 2>&1; show gpurun_out/r02h_${lib}_$w.log ${lib}_$w; done
done
