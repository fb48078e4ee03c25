"""GNA forward with E4M3 Q/K/V (GNA_DTYPE_FP8_E4M3)
against the fp64 oracle run on the dequantised inputs.

Tolerance (reading R17), per output element and scaled to the row's own data:
the kernel's only rounding beyond the bf16 path is P -> E4M3 before PV (RNE, 3 mantissa
bits): |dP| <= 2^-4 P for P >= 2^-6 (E4M3 normal range) and <= 2^-10 below.  Hence
    |dO_d| <= 2^-4 * sum_k p_k |v_kd|  +  (subnormal P terms)  +  bf16 output rounding,
with p_k = P_k / l the softmax weights.  A_d = sum_k p_k |v_kd| is exactly the oracle's
forward on |v|, so the bound is computed per element:
    max:  |O - O_ref| <= 2^-4 A + 2^-8 |O_ref| + 4e-3
    mean: mean|O - O_ref| <= 2^-6 mean(A) + 1e-3
(the 4e-3 / 1e-3 absolute terms cover the unbiased subnormal-P rounding, whose sum over
a window grows like sqrt(#keys) x 2^-10).  On the discriminating inputs (|O| ~ 0.1-0.5)
a PV-side error (wrong V box, P->V column mapping, scale) breaks the bound by >10x.
LSE uses only fp32 row sums: 1e-3 as for bf16."""
import numpy as np
import pytest
import torch

import oracle as O
from gna_inputs import make_qkv, quantize_e4m3

@pytest.fixture(scope="module")
def gna():
    import paper_2504_16922_b200 as pkg
    from paper_2504_16922_b200 import build

    build.build()
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    pkg.load()
    return pkg


CFGS = [
    dict(spatial=(256,), window=(32,), stride=(8,)),
    dict(spatial=(40, 36), window=(9, 12), stride=(3, 4)),
    dict(spatial=(37, 29), window=(8, 7), stride=(8, 7), dilation=(2, 2), causal=(False, True)),
    dict(spatial=(12, 20, 18), window=(5, 8, 6), stride=(2, 3, 6), dilation=(1, 2, 1), causal=(True, False, False)),
    dict(spatial=(64, 64), window=(32, 32), stride=(16, 16)),
]


def _ids(c):
    return "x".join(map(str, c["spatial"])) + "_w" + "x".join(map(str, c["window"]))


def _check_fp8(o, ro, ra, l, rl):
    """o: kernel O, ro: oracle O on the dequantised inputs, ra: oracle forward on |v|."""
    err = np.abs(o - ro)
    bound = 2.0 ** -4 * ra + 2.0 ** -8 * np.abs(ro) + 4e-3
    assert np.isfinite(o).all()
    worst = float((err / bound).max())
    assert worst <= 1.0, f"O error exceeds the per-element bound by {worst:.2f}x (max-abs {err.max():.3e})"
    assert err.mean() <= 2.0 ** -6 * ra.mean() + 1e-3, f"O mean-abs {err.mean():.3e} vs mean A {ra.mean():.3e}"
    assert np.abs(l - rl).max() <= 1e-3
    return worst


@pytest.mark.gpu
@pytest.mark.parametrize("disc", [False, True], ids=["normal", "discriminating"])
@pytest.mark.parametrize("cfg", CFGS, ids=_ids)
def test_fp8_forward_vs_oracle(gna, cfg, disc):
    B, H, D = 2, 2, 128
    q, k, v = make_qkv(B, cfg["spatial"], H, D, discriminating=disc, dtype=torch.float32)
    (q8, qs, qd), (k8, ks, kd), (v8, vs, vd) = (quantize_e4m3(t) for t in (q, k, v))
    out, lse = gna.forward(q8.cuda(), k8.cuda(), v8.cuda(), cfg["window"], cfg["stride"], cfg.get("dilation"),
                           cfg.get("causal"), scales=(qs, ks, vs))
    torch.cuda.synchronize()
    assert out.dtype == torch.bfloat16
    params = O.Params(cfg["spatial"], cfg["window"], cfg["stride"], cfg.get("dilation"), cfg.get("causal"))
    ro, rl = O.forward(qd.numpy(), kd.numpy(), vd.numpy(), params)
    ra, _ = O.forward(qd.numpy(), kd.numpy(), np.abs(vd.numpy()), params)
    _check_fp8(out.float().cpu().numpy(), ro, ra, lse.cpu().numpy(), rl)


@pytest.mark.gpu
def test_fp8_rejects_unsupported(gna):
    q, k, v = make_qkv(1, (64,), 1, 64, dtype=torch.float32)
    t8 = [quantize_e4m3(t)[0].cuda() for t in (q, k, v)]
    with pytest.raises(gna.GnaError):
        gna.forward(*t8, (16,), (4,))  # head_dim 64


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["c2b_flux64_s16", "c4a_hunyuan_blocked", "c3_cosmos"])
def test_fp8_full_size_sampled(gna, name):
    """E4M3 forward at BASELINE.json's full sizes (the launch bench.py --dtype fp8 times), on the
    discriminating inputs, sampled rows incl. grid corners vs the oracle on the dequantised
    inputs; same per-element tolerance as above."""
    from gna_inputs import WORKLOADS, sample_rows
    w = WORKLOADS[name]
    f = w.full()
    q, k, v = make_qkv(w.batch, w.spatial, w.heads, w.head_dim, discriminating=True, dtype=torch.float32)
    (q8, qs, qd), (k8, ks, kd), (v8, vs, vd) = (quantize_e4m3(t) for t in (q, k, v))
    out, lse = gna.forward(q8.cuda(), k8.cuda(), v8.cuda(), f["window"], f["stride"], f["dilation"], f["causal"],
                           scales=(qs, ks, vs))
    torch.cuda.synchronize()
    L = list(w.spatial) + [1] * (3 - len(w.spatial))
    corners = [0, L[1] * L[2] - 1, w.n_tokens - 1, (L[0] // 2) * L[1] * L[2] + (L[1] // 2) * L[2] + L[2] // 2]
    rows = sample_rows(w.batch, w.spatial, w.heads, 64, extra_tokens=corners)
    ro, rl, _ = O.forward_rows(qd.numpy(), kd.numpy(), vd.numpy(), O.Params(**f), rows)
    ra, _, _ = O.forward_rows(qd.numpy(), kd.numpy(), np.abs(vd.numpy()), O.Params(**f), rows)
    oo = out.float().cpu().reshape(w.batch, -1, w.heads, w.head_dim)[rows[:, 0], rows[:, 1], rows[:, 2]].numpy()
    ll = lse.cpu().reshape(w.batch, -1, w.heads)[rows[:, 0], rows[:, 1], rows[:, 2]].numpy()
    _check_fp8(oo, ro, ra, ll, rl)


@pytest.mark.gpu
@pytest.mark.parametrize("T", [77, 200])
def test_fp8_extra_kv(gna, T):
    """E4M3 with extra (text) KV tokens (NEXT-1 x NEXT-3): the extra K/V are E4M3 with the same
    per-tensor scales as K/V (amax over the GNA and extra tokens together)."""
    cfg = CFGS[3]
    B, H, D = 2, 2, 128
    q, k, v = make_qkv(B, cfg["spatial"], H, D, discriminating=True, dtype=torch.float32)
    g = torch.Generator("cpu").manual_seed(91)
    ek = torch.randn((B, T, H, D), generator=g)
    ev = torch.rand((B, T, H, D), generator=g) * 2 - 1

    def quant_pair(a, b):
        scale = float(max(a.abs().max(), b.abs().max())) / 448.0
        qa, qb = (a / scale).to(torch.float8_e4m3fn), (b / scale).to(torch.float8_e4m3fn)
        return qa, qb, scale, qa.float() * scale, qb.float() * scale

    q8, qs, qd = quantize_e4m3(q)
    k8, ek8, ks, kd, ekd = quant_pair(k, ek)
    v8, ev8, vs, vd, evd = quant_pair(v, ev)
    out, lse = gna.forward(q8.cuda(), k8.cuda(), v8.cuda(), cfg["window"], cfg["stride"], cfg.get("dilation"),
                           cfg.get("causal"), scales=(qs, ks, vs), extra_k=ek8.cuda(), extra_v=ev8.cuda())
    torch.cuda.synchronize()
    params = O.Params(cfg["spatial"], cfg["window"], cfg["stride"], cfg.get("dilation"), cfg.get("causal"))
    ro, rl = O.forward(qd.numpy(), kd.numpy(), vd.numpy(), params, extra_k=ekd.numpy(), extra_v=evd.numpy())
    ra, _ = O.forward(qd.numpy(), kd.numpy(), np.abs(vd.numpy()), params, extra_k=ekd.numpy(),
                      extra_v=np.abs(evd.numpy()))
    _check_fp8(out.float().cpu().numpy(), ro, ra, lse.cpu().numpy(), rl)
