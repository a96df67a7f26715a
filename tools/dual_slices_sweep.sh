# Tucker-4 MLP block (cfg4 layout, dual gate/up kernel) at M = 8192 vs TNL_DUAL_SLICES
for sl in 0 1 2 3 4 6 8; do
  if [ $sl = 0 ]; then unset TNL_DUAL_SLICES; else export TNL_DUAL_SLICES=$sl; fi
  python -c "
import json, os, sys, torch
sys.path.insert(0, '.')
from paper_2602_01613_b200 import qwen_stack as Q
from paper_2602_01613_b200.mlp import TNMLP
M = 8192
layers = [Q._tn('tucker4', Q.FFN, Q.HIDDEN, seed=1), Q._tn('tucker4', Q.FFN, Q.HIDDEN, seed=2), Q._tn('tucker4', Q.HIDDEN, Q.FFN, seed=3)]
xs = [torch.randn(M, 5120, device='cuda').to(torch.bfloat16) for _ in range(4)]
mlp = TNMLP(*layers)
y = torch.empty(M, 5120, device='cuda', dtype=torch.bfloat16)
for i in range(3): mlp.forward(xs[i % 4], out=y)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for i in range(20): mlp.forward(xs[i % 4], out=y)
e1.record(); torch.cuda.synchronize()
print(json.dumps({'dual_slices': os.environ.get('TNL_DUAL_SLICES', 'auto'), 'ms': e0.elapsed_time(e1) / 20}))
"
done
