"""Debug: the dilation+causal D=64 ABI case vs the oracle, error location by work item."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle as O
import paper_2504_16922_b200 as gna
from gna_inputs import make_qkv, as_f32_numpy

cases = [((12, 20, 18), (5, 8, 6), (2, 3, 6), (1, 2, 1), (1, 0, 0), 64, 2, 3),
         ((12, 20, 18), (5, 8, 6), (2, 3, 6), (1, 2, 1), (1, 0, 0), 128, 2, 3),
         ((12, 20, 18), (5, 8, 6), (2, 3, 6), (1, 1, 1), (0, 0, 0), 64, 2, 3)]
for sp, w, s, d, c, D, B, H in cases:
    q, k, v = make_qkv(B, sp, H, D, discriminating=True)
    out, lse = gna.forward(q.cuda(), k.cuda(), v.cuda(), w, s, d, c)
    torch.cuda.synchronize()
    ro, rl = O.forward(as_f32_numpy(q), as_f32_numpy(k), as_f32_numpy(v), O.Params(sp, w, s, d, tuple(bool(x) for x in c)))
    o = out.float().cpu().numpy(); l = lse.cpu().numpy()
    e = np.abs(o - ro).max(-1)
    le = np.abs(l - rl)
    bad = np.argwhere(e > 2e-2)
    print(sp, w, s, d, c, D, f"O max {e.max():.3e} LSE max {le.max():.3e} bad rows {len(bad)}", flush=True)
    if len(bad):
        print("  bad (b,h) counts:", {k: int(v) for k, v in zip(*np.unique(bad[:, 0] * 10 + bad[:, -1], return_counts=True))})
        print("  first bad:", bad[:8].tolist())
