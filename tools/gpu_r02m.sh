timeout 120 python -c "
import sys,os; sys.path.insert(0,os.getcwd())
import torch, wsinputs as W
from paper_2408_00930_b200 import Env
g=Env(1000,1,'cartpole',1,t_capacity=50); w=torch.from_numpy(W.policy_weights(4,64,2,seed=1,scale=2.0)).cuda()
g.rollout_policy(50,w,64); torch.cuda.synchronize(); print('policy ok', g.status())
" 2>&1 | tail -2; echo "policy rc=$?"
timeout 900 python -m pytest tests/test_gpu_policy.py tests/test_gpu_a2c.py tests/test_gpu_a2c_dp.py -x -q > gpurun_out/r02m_pytest.log 2>&1; tail -3 gpurun_out/r02m_pytest.log
show() { tail -1 $1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$2', round(d['ms_per_step'],4), round(d['sustained']['ms_per_step'],4), r['kernel_ms'], r.get('frac'), r.get('bound'))"; }
for w in C2P C2T; do timeout 300 python bench.py --workload $w --no-cpu-baseline --sustain-s 0.3 > gpurun_out/r02m_$w.log 2>&1; show gpurun_out/r02m_$w.log $w; done
