"""Launch list of one cfg4 prefill pass (M = 8192) over 3 decoder layers (TT r64 / TR4 / Tucker-4
MLPs): the target of `ncu --nvtx --nvtx-include "pass/"` to attribute the stack time per kernel."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2602_01613_b200.qwen_stack import HIDDEN, QwenTNStack  # noqa: E402

st = QwenTNStack(3, mlp_kinds=["tt64", "tr4", "tucker4"])
M = int(os.environ.get("M", "8192"))
x = torch.randn(M, HIDDEN, device="cuda").to(torch.bfloat16)
b = st._buffers(M)
for _ in range(2):
    st.forward(x.clone(), b)
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("pass")
st.forward(x, b)
torch.cuda.nvtx.range_pop()
torch.cuda.synchronize()
print("ok")
