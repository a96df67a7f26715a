"""cfg4 prefill (M=8192) per-op breakdown of one decoder layer of each MLP kind."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2602_01613_b200.qwen_stack import QwenTNStack, HIDDEN, QDIM, KVDIM

st = QwenTNStack(4, mlp_kinds=["tt64", "tr4", "tucker4", "tucker2-256"])  # one decoder layer per MLP kind
M = 8192
ws = st.workspace(M)
b = st._buffers(M)
x = torch.randn(M, HIDDEN, device="cuda").to(torch.bfloat16)


def t(fn, it=10):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(it):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / it * 1e3  # us


rms = lambda: b["h"].copy_(torch.nn.functional.rms_norm(x, (HIDDEN,), eps=1e-6))  # noqa: E731
out = {"rms_norm_copy": t(rms), "residual_add": t(lambda: x.add_(b["o"]))}
for l in range(4):
    blk = st.layers[l]
    for name, dst in (("q", "q"), ("k", "k"), ("v", "v")):
        out[f"L{l}_{name}"] = t(lambda: blk[name][2].forward(b["h"], out=b[dst], ws=ws))
    out[f"L{l}_o"] = t(lambda: blk["o"][2].forward(b["q"], out=b["o"], ws=ws))
    out[f"L{l}_mlp_{blk['gate'][0]}_fused{int(blk['mlp'].fused)}"] = t(lambda: blk["mlp"].forward(b["h"], out=b["d"], ws=ws))
print(json.dumps({k: round(v, 1) for k, v in out.items()}))
