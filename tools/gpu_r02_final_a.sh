# round-2 final evidence, part A: GPU suite, smoke, ncu tables of the changed kernels, launch list
mkdir -p gpurun_out/r02_final
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r02_final/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/r02_final/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r02_final/smoke.log 2>&1
bash tools/ncu_table.sh r02_final C2 C5 C2P C2S C3a C3b C4 D0 C3S C2U > gpurun_out/r02_final/ncu_table.log 2>&1
bash tools/prof_one.sh C5 k_plan_gauss r02_final_C5plan > /dev/null 2>&1
bash tools/prof_one.sh C2 k_plan_discrete r02_final_C2plan > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -s 15 -c 12 --csv --log-file gpurun_out/r02_final/launches_C2.csv python bench.py --steps 5 --warmup 3 --ncu > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -s 15 -c 12 --csv --log-file gpurun_out/r02_final/launches_C5.csv python bench.py --workload C5 --steps 5 --warmup 3 --ncu > /dev/null 2>&1
