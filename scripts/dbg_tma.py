import os, sys, torch, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2504_16922_b200 as gna
from gna_inputs import make_qkv
sp, w, s = (40, 36), (9, 12), (3, 4)
for D in (64, 128):
  for disc in (False, True):
    q, k, v = (t.cuda() for t in make_qkv(2, sp, 2, D, discriminating=disc))
    res = {}
    for ts in ("0", "1"):
        os.environ["GNA_TMA_STORE"] = ts
        res[ts] = gna.forward(q, k, v, w, s)
    torch.cuda.synchronize()
    o0, o1 = res["0"][0].float(), res["1"][0].float()
    d = (o0 - o1).abs()
    print(D, disc, "max diff", d.max().item(), "plan", gna.plan_info(2, 2, D, spatial=sp, window=w, stride=s)["box"])
    if d.max() > 0:
        idx = torch.nonzero(d.amax(-1) > 0)
        print("  differing (b, x, y, h) rows:", idx.shape[0], idx[:8].tolist(), "nan in tma:", torch.isnan(o1).any().item())
