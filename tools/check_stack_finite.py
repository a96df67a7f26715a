"""Debug: per-layer finiteness / magnitude of the cfg4 residual stream, eager, M=64 vs M=300."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2602_01613_b200.qwen_stack import QwenTNStack, HIDDEN

st = QwenTNStack(8)
for m in (64, 300):
    torch.manual_seed(1)
    x = torch.randn(m, HIDDEN, device="cuda").to(torch.bfloat16)
    ws = st.workspace(m)
    b = st._buffers(m)
    for li, blk in enumerate(st.layers):
        st.add_rmsnorm(x, b["d"] if li else None, b["h"])
        stats = {}
        for nm in ("q", "k", "v"):
            blk[nm][2].forward(b["h"], out=b[nm], ws=ws)
        blk["o"][2].forward(b["q"], out=b["o"], ws=ws)
        st.add_rmsnorm(x, b["o"], b["h"])
        blk["mlp"].forward(b["h"], out=b["d"], ws=ws)
        torch.cuda.synchronize()
        f = lambda t: f"{float(t.float().abs().max()):.3g}{'' if bool(torch.isfinite(t).all()) else '!NaN'}"  # noqa: E731
        print(m, li, blk["gate"][0], "h", f(b["h"]), "q", f(b["q"]), "o", f(b["o"]), "d", f(b["d"]), "x", f(x), flush=True)
