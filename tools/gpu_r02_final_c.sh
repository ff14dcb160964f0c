# round-2 final evidence, part C (after the C5 8-step trips, the composer clean groups, the PPO edge test)
mkdir -p gpurun_out/r02_final
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r02_final/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/r02_final/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r02_final/smoke.log 2>&1
bash tools/ncu_table.sh r02_final C5 C2U > gpurun_out/r02_final/ncu_table_c.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -s 15 -c 12 --csv --log-file gpurun_out/r02_final/launches_C5.csv python bench.py --workload C5 --steps 5 --warmup 3 --ncu > /dev/null 2>&1
python tools/racecheck_r02.py > gpurun_out/r02_final/racecheck_script_plain.log 2>&1; echo "racecheck script exit $?" >> gpurun_out/r02_final/racecheck_script_plain.log
