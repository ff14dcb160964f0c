#!/bin/bash
# One GPU session: parity tests, bench, launch list, one full ncu capture of the roll-out kernel.
set -x
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvidia_smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 1200 python -m pytest tests -m gpu -x -q ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
cat gpurun_out/bench.json
if [ -n "${NCU}" ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
      python bench.py --steps 3 --warmup 1 --ncu > gpurun_out/ncu_launch_bench.log 2>&1; echo "ncu list rc=$?"
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_rollout -s 1 -c 1 \
      -o gpurun_out/prof_rollout -f python bench.py --steps 2 --warmup 1 --ncu > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_plan -s 1 -c 1 \
      -o gpurun_out/prof_plan -f python bench.py --steps 2 --warmup 1 --ncu > gpurun_out/ncu_plan.log 2>&1; echo "ncu plan rc=$?"
fi
