import sys; sys.path.insert(0, "/root/repo")
import numpy as np, torch
import paper_2602_01613_b200 as tnl
from oracle import tn_oracle as O
def rel(a,b): a=np.asarray(a,np.float64); b=np.asarray(b,np.float64); return float(np.linalg.norm(a-b)/np.linalg.norm(a))
for spec in [("tt",(12,8,7,12,6),3,(8,6,1,4)), ("tt",(12,8,7,12,6),3,(8,6,2,4)), ("tt",(12,8,8,12,6),3,(8,6,1,4)), ("tt",(16,8,8,12,6),3,(8,6,1,4))]:
    fam, ms, rm, ranks = spec
    L = O.synthetic_layer(fam, ms, rm, ranks, seed=91_000 + 37 * 18)
    kw = dict(family=L.family, mode_shape=L.mode_shape, row_mode_count=L.row_mode_count, cores=[O.round_bf16(c) for c in L.cores])
    lay = tnl.CompressedLayer(**kw); ref = O.OracleLayer(**kw)
    rows, cols = ref.matrix_shape
    for flags, nm in ((tnl.PLAN_AUTO,"auto"), (tnl.PLAN_NO_DECODE,"nodec"), (tnl.PLAN_GEMV,"gemv")):
        p = lay.plan(torch.bfloat16, flags=flags)
        res = []
        for m in (1, 2, 8, 19, 64, 65, 150):
            x = O.round_bf16(O.synthetic_x(m, cols, seed=92_000 + m + 18))
            y = p.forward(torch.tensor(x, dtype=torch.bfloat16, device="cuda")); torch.cuda.synchronize()
            res.append(round(rel(O.forward_torch_orient(ref, x), y.double().cpu().numpy()), 4))
        print(spec, nm, p.info["plan_small_name"], p.info["plan_large_name"], p.info.get("decode_max_m"), res, flush=True)
