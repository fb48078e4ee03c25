"""Quick GPU sanity run: tiny GNA configs vs the oracle, printing error stats."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle as O
import paper_2504_16922_b200 as gna
from gna_inputs import make_qkv, as_f32_numpy

cases = [
    ((128,), (128,), (1,), 1, 1, 128),     # dense 1 tile
    ((256,), (256,), (1,), 1, 1, 128),     # dense 2 tiles
    ((256,), (32,), (8,), 1, 1, 32),
    ((40, 36), (9, 12), (3, 4), 2, 2, 128),
    ((64, 64), (32, 32), (16, 16), 1, 4, 128),
    ((12, 20, 18), (5, 8, 6), (2, 3, 6), 2, 2, 64),
]
bad = 0
for spatial, window, stride, B, H, D in cases:
    q, k, v = make_qkv(B, spatial, H, D, discriminating=True)
    t0 = time.time()
    out, lse = gna.forward(q.cuda(), k.cuda(), v.cuda(), window, stride, flags=1)
    torch.cuda.synchronize()
    dt = time.time() - t0
    ro, rl = O.forward(as_f32_numpy(q), as_f32_numpy(k), as_f32_numpy(v), O.Params(spatial, window, stride))
    o = out.float().cpu().numpy(); l = lse.cpu().numpy()
    e = np.abs(o - ro)
    print(spatial, window, stride, D, f"O max {np.nanmax(e):.3e} mean {np.nanmean(e):.3e} nan {np.isnan(o).sum()} "
          f"LSE max {np.nanmax(np.abs(l-rl)):.3e}  t={dt:.2f}s", flush=True)
    bad += int(not (np.nanmax(e) <= 2e-2 and np.nanmax(np.abs(l - rl)) <= 1e-3 and not np.isnan(o).any()))
sys.exit(1 if bad else 0)
