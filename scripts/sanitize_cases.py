"""Small GNA forwards for compute-sanitizer (memcheck / racecheck / synccheck / initcheck):
C1 (1-D tiny, D=32, permuted route), tiny 2-D / 3-D configs with dilation and causal axes
on the permute-free route, the permuted route with the standalone inverse permute, extra KV
tokens, fp16 and E4M3.  Each result is checked against the fp64 oracle (a run under a
sanitizer is slow, so the shapes are small).

usage: compute-sanitizer --tool memcheck python scripts/sanitize_cases.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import oracle as O
import paper_2504_16922_b200 as gna
from gna_inputs import WORKLOADS, as_f32_numpy, make_qkv, quantize_e4m3
from paper_2504_16922_b200.gna import GNA_FLAG_PERMUTED, GNA_FLAG_UNFUSED_EPILOGUE

CASES = [
    ("c1_tiny1d", dict(spatial=(256,), window=(32,), stride=(8,)), 32, 0),
    ("2d_dil_causal", dict(spatial=(37, 29), window=(8, 7), stride=(8, 7), dilation=(2, 2), causal=(False, True)), 128, 0),
    ("3d_dil_causal", dict(spatial=(12, 20, 18), window=(5, 8, 6), stride=(2, 3, 6), dilation=(1, 2, 1),
                           causal=(True, False, False)), 64, 0),
    ("2d_permuted_unfused", dict(spatial=(40, 36), window=(9, 12), stride=(3, 4)), 128, GNA_FLAG_UNFUSED_EPILOGUE),
    ("3d_permuted_fused", dict(spatial=(12, 20, 18), window=(5, 8, 6), stride=(2, 3, 6), dilation=(1, 2, 1),
                               causal=(True, False, False)), 128, GNA_FLAG_PERMUTED),
    # blocked (every item dense) with more work items (256) than SMs: the persistent multi-item path
    ("3d_blocked_dense_persistent", dict(spatial=(16, 32, 32), window=(8, 16, 16), stride=(8, 16, 16)), 128, 0),
]


def check(name, o, ro, l, rl, omax=2e-2):
    e = np.abs(o.float().cpu().numpy() - ro).max()
    le = np.abs(l.cpu().numpy() - rl).max()
    ok = e <= omax and le <= 1e-3
    print(f"{name}: O max-abs {e:.2e}  LSE {le:.2e}  {'ok' if ok else 'FAIL'}", flush=True)
    return ok


def main():
    torch.cuda.init()
    ok = True
    for name, cfg, D, flags in CASES:
        B, H = 2, 2
        q, k, v = make_qkv(B, cfg["spatial"], H, D, discriminating=True)
        o, l = gna.forward(q.cuda(), k.cuda(), v.cuda(), cfg["window"], cfg["stride"], cfg.get("dilation"),
                           cfg.get("causal"), flags=flags)
        torch.cuda.synchronize()
        p = O.Params(cfg["spatial"], cfg["window"], cfg["stride"], cfg.get("dilation"), cfg.get("causal"))
        ro, rl = O.forward(as_f32_numpy(q), as_f32_numpy(k), as_f32_numpy(v), p)
        ok &= check(name, o, ro, l, rl)
    # extra KV tokens (NEXT-1), fp16
    cfg = CASES[2][1]
    p = O.Params(cfg["spatial"], cfg["window"], cfg["stride"], cfg.get("dilation"), cfg.get("causal"))
    for dt in (torch.bfloat16, torch.float16):
        q, k, v = make_qkv(2, cfg["spatial"], 2, 128, discriminating=True, dtype=dt)
        g = torch.Generator("cpu").manual_seed(3)
        ek = torch.randn((2, 77, 2, 128), generator=g).to(dt)
        ev = torch.randn((2, 77, 2, 128), generator=g).to(dt)
        o, l = gna.forward(q.cuda(), k.cuda(), v.cuda(), cfg["window"], cfg["stride"], cfg["dilation"],
                           cfg["causal"], extra_k=ek.cuda(), extra_v=ev.cuda())
        torch.cuda.synchronize()
        ro, rl = O.forward(as_f32_numpy(q), as_f32_numpy(k), as_f32_numpy(v), p, extra_k=as_f32_numpy(ek),
                           extra_v=as_f32_numpy(ev))
        ok &= check(f"extra_kv_{dt}", o, ro, l, rl)
    # E4M3
    cfg = dict(spatial=(40, 36), window=(9, 12), stride=(3, 4))
    qf, kf, vf = make_qkv(2, cfg["spatial"], 2, 128, discriminating=True, dtype=torch.float32)
    (q8, qs, qd), (k8, ks, kd), (v8, vs, vd) = (quantize_e4m3(t) for t in (qf, kf, vf))
    o, l = gna.forward(q8.cuda(), k8.cuda(), v8.cuda(), cfg["window"], cfg["stride"], scales=(qs, ks, vs))
    torch.cuda.synchronize()
    ro, rl = O.forward(qd.numpy(), kd.numpy(), vd.numpy(), O.Params(cfg["spatial"], cfg["window"], cfg["stride"]))
    ok &= check("e4m3", o, ro, l, rl, omax=0.1)
    print("ALL OK" if ok else "SOME FAILED")
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
