import sys, json, torch
sys.path.insert(0, ".")
from paper_2602_01613_b200 import qwen_stack as Q
st = Q.QwenTNStack(16)
orig = Q.QwenTNStack.add_rmsnorm
out = {}
for skip in (False, True, False, True):
    Q.QwenTNStack.add_rmsnorm = staticmethod((lambda x, o, h, eps=1e-6: None) if skip else orig)
    for m in (1, 64):
        g = st.capture(m, microbatches=2)
        st.x.normal_()
        for _ in range(3): g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20): g.replay()
        e1.record(); torch.cuda.synchronize()
        out.setdefault(f"skip={skip} m={m}", []).append(round(e0.elapsed_time(e1) / 20, 4))
        del g
print(json.dumps(out))
