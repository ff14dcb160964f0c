#!/bin/bash
# End-of-round evidence: smoke, full GPU suite, every workload line, the default bench line,
# learning curves, launch lists of C2 and C2T, ncu captures of the policy / composer kernels.
set -x
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvidia_smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 1500 python -m pytest tests -m gpu -x -q -s > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu.log
WORKLOADS="C1 C2 C3a C3b C4 C5 D0 C2P C2G C4G C2T C2O C3T C4T C2X C2U" bash tools/all_workloads.sh
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
timeout 300 python -m paper_2408_00930_b200.train --envs 10000 --T 32 --iters 3000 --log-every 50 --csv gpurun_out/curve_cartpole.csv
timeout 300 python -m paper_2408_00930_b200.train --env acrobot --envs 10000 --T 128 --iters 1500 --lr 1e-3 --log-every 50 --csv gpurun_out/curve_acrobot.csv
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 3 --warmup 1 --ncu > gpurun_out/ncu_launch_c2.log 2>&1; echo "ncu list c2 rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2t.csv \
    python bench.py --workload C2T --steps 3 --warmup 1 --ncu > gpurun_out/ncu_launch_c2t.log 2>&1; echo "ncu list c2t rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_rollout_policy -s 1 -c 1 \
    -o gpurun_out/prof_k_rollout_policy -f python bench.py --workload C2T --steps 2 --warmup 1 --ncu > gpurun_out/ncu_pol.log 2>&1; echo "ncu pol rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_user_rollout -s 1 -c 1 \
    -o gpurun_out/prof_k_user_rollout -f python bench.py --workload C2U --steps 2 --warmup 1 --ncu > gpurun_out/ncu_user.log 2>&1; echo "ncu user rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_a2c_grad -s 1 -c 1 \
    -o gpurun_out/prof_k_a2c_grad -f python bench.py --workload C2T --steps 2 --warmup 1 --ncu > gpurun_out/ncu_grad.log 2>&1; echo "ncu grad rc=$?"
