# Acrobot throughput build at 6 CTAs/SM (80 registers, no spills since the sincos changes):
# A/B of the WS_ACRO_MINB=6 library (lib/minb6) against the product library (5 CTAs/SM)
mkdir -p gpurun_out/r02_q
for rep in 1 2; do
for w in C3a C3S; do
  WS_LIBWS=$PWD/paper_2408_00930_b200/lib/minb6/libws.so timeout 600 python bench.py --workload $w --no-cpu-baseline --sustain-s 0.5 2>/dev/null | tail -1 >> gpurun_out/r02_q/new.jsonl
  timeout 600 python bench.py --workload $w --no-cpu-baseline --sustain-s 0.5 2>/dev/null | tail -1 >> gpurun_out/r02_q/old.jsonl
done
WS_LIBWS=$PWD/paper_2408_00930_b200/lib/minb6/libws.so timeout 300 python tools/time_rollout.py acrobot 12500 500 100 >> gpurun_out/r02_q/shard_new.log 2>&1
timeout 300 python tools/time_rollout.py acrobot 12500 500 100 >> gpurun_out/r02_q/shard_old.log 2>&1
done
