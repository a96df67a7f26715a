for sl in 0 1 2 3 4 5 6 8 10; do
  if [ $sl = 0 ]; then unset TNL_MLP_SLICES; else export TNL_MLP_SLICES=$sl; fi
  python -c "
import json, os, sys, torch
sys.path.insert(0, '.')
from paper_2602_01613_b200 import synthetic as S
from paper_2602_01613_b200.mlp import TNMLP
M = 8192
layers = [S.make_layer(*S.CFG3_GATE, seed=30_100), S.make_layer(*S.CFG3_GATE, seed=30_200), S.make_layer(*S.CFG3_DOWN, seed=30_300)]
xs = [torch.randn(M, 5120, device='cuda').to(torch.bfloat16) for _ in range(4)]
mlp = TNMLP(*layers)
y = torch.empty(M, 5120, device='cuda', dtype=torch.bfloat16)
for i in range(3): mlp.forward(xs[i % 4], out=y)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for i in range(30): mlp.forward(xs[i % 4], out=y)
e1.record(); torch.cuda.synchronize()
print(json.dumps({'slices': os.environ.get('TNL_MLP_SLICES', 'auto'), 'ms': e0.elapsed_time(e1) / 30}))
"
done
