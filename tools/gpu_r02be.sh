mkdir -p gpurun_out/r02be
timeout 900 python -m pytest tests/test_gpu_overlap.py tests/test_gpu_parity.py -x -q > gpurun_out/r02be/pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/r02be/pytest.log
cat > /tmp/ab.py <<'PY'
import sys, os
sys.path.insert(0, os.getcwd())
import torch, wsinputs as W
from paper_2408_00930_b200 import Env
E, T, reps = 10000, 1000, 100
pt = torch.from_numpy(W.uniform_probs(E, 1, 2)).cuda()
for ov in (False, True, False, True):
    g = Env(E, 1, "cartpole", W.SEED, t_capacity=T); g.set_plan_overlap(ov)
    for _ in range(5): g.rollout(T, pt)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    torch.cuda.synchronize(); ev[0].record()
    for _ in range(reps): g.rollout(T, pt)
    ev[1].record(); torch.cuda.synchronize()
    print("overlap", ov, round(ev[0].elapsed_time(ev[1]) / reps, 4), "ms", g.status(), flush=True)
    g.close()
PY
python /tmp/ab.py > gpurun_out/r02be/ab.log 2>&1
python bench.py --no-cpu-baseline > gpurun_out/r02be/bench_C2.log 2>&1
