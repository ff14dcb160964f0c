#!/bin/bash
# NEXT-N2 measurement session: C2T bench line, its launch list, one full ncu capture of the
# A2C gradient kernel and of the critic kernel.
set -x
mkdir -p gpurun_out
timeout 600 python bench.py --workload C2T --steps 10 --warmup 3 > gpurun_out/bench_c2t.json 2> gpurun_out/bench_c2t.err; echo "bench rc=$?"
cat gpurun_out/bench_c2t.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2t.csv \
    python bench.py --workload C2T --steps 3 --warmup 1 --ncu > gpurun_out/ncu_launch_c2t.log 2>&1; echo "ncu list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_a2c_grad -s 1 -c 1 \
    -o gpurun_out/prof_a2c_grad -f python bench.py --workload C2T --steps 2 --warmup 1 --ncu > gpurun_out/ncu_a2c.log 2>&1; echo "ncu grad rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_ac_values -s 2 -c 1 \
    -o gpurun_out/prof_ac_values -f python bench.py --workload C2T --steps 2 --warmup 1 --ncu > gpurun_out/ncu_values.log 2>&1; echo "ncu values rc=$?"
