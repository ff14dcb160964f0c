#!/bin/bash
# NEXT-N1..N3 evidence: full GPU test suite, every workload's bench line, the C2T launch
# list, and full ncu captures of the GAE, critic, gradient and Adam kernels.
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu.log
bash tools/all_workloads.sh
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2t.csv \
    python bench.py --workload C2T --steps 3 --warmup 1 --ncu > gpurun_out/ncu_launch_c2t.log 2>&1; echo "ncu list rc=$?"
for k in k_a2c_grad k_ac_values k_adam k_moments; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 \
      -o gpurun_out/prof_$k -f python bench.py --workload C2T --steps 2 --warmup 1 --ncu > gpurun_out/ncu_$k.log 2>&1; echo "ncu $k rc=$?"
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gae -s 1 -c 1 \
    -o gpurun_out/prof_k_gae -f python bench.py --workload C2G --steps 2 --warmup 1 --ncu > gpurun_out/ncu_gae.log 2>&1; echo "ncu gae rc=$?"
