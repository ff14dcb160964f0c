mkdir -p gpurun_out/sanitizer_r02f
for tool in racecheck synccheck memcheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/racecheck_r02.py > gpurun_out/sanitizer_r02f/$tool.log 2>&1
  echo "$tool rc=$?"; tail -2 gpurun_out/sanitizer_r02f/$tool.log
done
timeout 1500 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_policy.py tests/test_gpu_parity.py -q -x -k "policy or graph or surface or gaussian" > gpurun_out/sanitizer_r02f/memcheck_pytest.log 2>&1
echo "memcheck pytest rc=$?"; tail -3 gpurun_out/sanitizer_r02f/memcheck_pytest.log
