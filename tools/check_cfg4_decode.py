"""Debug: every cfg4 projection kind, decode path (M=64) vs prefill path (M=300, first 64 rows)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2602_01613_b200.qwen_stack import QwenTNStack, SHAPES, _tn
from paper_2602_01613_b200.mlp import TNMLP

kinds = {"q": ["tucker2-256"], "k": ["tucker2-128"], "o": ["tucker2-256"],
         "gate": ["tucker2-256", "tt64", "tr4", "tucker4"], "down": ["tucker2-256", "tt64", "tr4", "tucker4"]}
torch.manual_seed(0)
for name, ks in kinds.items():
    rows, cols = SHAPES[name]
    for kd in ks:
        lay = _tn(kd, rows, cols, seed=7)
        p = lay.plan(torch.bfloat16)
        x = torch.randn(300, cols, device="cuda").to(torch.bfloat16)
        ws = torch.zeros(p.workspace_bytes(300), dtype=torch.uint8, device="cuda")
        y300 = p.forward(x, ws=ws)
        ws64 = torch.zeros(p.workspace_bytes(64), dtype=torch.uint8, device="cuda")
        y64 = p.forward(x[:64].contiguous(), ws=ws64)
        y64b = p.forward(x[:64].contiguous(), ws=ws64)  # second call: accumulator back at rest?
        torch.cuda.synchronize()
        ref = y300[:64].float()
        err = lambda y: float((y.float() - ref).norm() / ref.norm())  # noqa: E731
        print(f"{name:5s} {kd:12s} plan={p.info.get('plan_small_name', '?')} fin={bool(torch.isfinite(y64).all())} "
              f"rel64={err(y64):.3e} rel64_again={err(y64b):.3e}", flush=True)
# MLP blocks at decode size
for kd in ["tucker2-256", "tt64", "tr4", "tucker4"]:
    g, u, d = (_tn(kd, *SHAPES[n], seed=11 + i) for i, n in enumerate(("gate", "up", "down")))
    mlp = TNMLP(g, u, d)
    x = torch.randn(300, 5120, device="cuda").to(torch.bfloat16)
    y300 = mlp(x)
    y64 = mlp(x[:64].contiguous())
    torch.cuda.synchronize()
    ref = y300[:64].float()
    print(f"mlp {kd:12s} fused={mlp.fused} fin={bool(torch.isfinite(y64).all())} rel={float((y64.float()-ref).norm()/ref.norm()):.3e}")
