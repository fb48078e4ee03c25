"""fp16 inputs and output (GNA_DTYPE_FP16) against the fp64 oracle -- the precision of
every throughput the paper quotes and one of the two input types
BASELINE.json's tolerance clause names ("bf16/fp16 inputs").  Same bars as bf16:
O max-abs 2e-2 and mean-abs 2e-3, LSE 1e-3.  Inputs: the seeded recipe cast to fp16
(rounded once; the oracle consumes exactly those values promoted to fp64)."""
import numpy as np
import pytest
import torch

import oracle as O
from gna_inputs import WORKLOADS, as_f32_numpy, make_qkv, sample_rows

pytestmark = pytest.mark.gpu

O_MAX, O_MEAN, LSE_TOL = 2e-2, 2e-3, 1e-3


@pytest.fixture(scope="module")
def gna():
    import paper_2504_16922_b200 as pkg
    from paper_2504_16922_b200 import build

    build.build()
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    pkg.load()
    return pkg


def _close(o, ro, l, rl):
    err = np.abs(o - ro)
    assert np.isfinite(o).all() and np.isfinite(l).all()
    assert err.max() <= O_MAX, f"O max-abs {err.max()}"
    assert err.mean() <= O_MEAN, f"O mean-abs {err.mean()}"
    assert np.abs(l - rl).max() <= LSE_TOL, f"LSE max-abs {np.abs(l - rl).max()}"


CFGS = [
    dict(spatial=(256,), window=(32,), stride=(8,)),
    dict(spatial=(200,), window=(17,), stride=(5,), dilation=(3,), causal=(True,)),
    dict(spatial=(40, 36), window=(9, 12), stride=(3, 4)),
    dict(spatial=(37, 29), window=(8, 7), stride=(8, 7), dilation=(2, 2), causal=(False, True)),
    dict(spatial=(12, 20, 18), window=(5, 8, 6), stride=(2, 3, 6), dilation=(1, 2, 1), causal=(True, False, False)),
    dict(spatial=(16, 16, 16), window=(16, 16, 16), stride=(1, 1, 1)),
]


def _ids(c):
    return "x".join(map(str, c["spatial"])) + "_w" + "x".join(map(str, c["window"])) + \
        "_d" + "x".join(map(str, c.get("dilation", (1,))))


@pytest.mark.parametrize("disc", [False, True], ids=["normal", "discriminating"])
@pytest.mark.parametrize("cfg", CFGS, ids=_ids)
@pytest.mark.parametrize("D", [128, 64, 32])
def test_fp16_forward_small(gna, cfg, disc, D):
    B, H = 2, 2
    q, k, v = make_qkv(B, cfg["spatial"], H, D, discriminating=disc, dtype=torch.float16)
    out, lse = gna.forward(q.cuda(), k.cuda(), v.cuda(), cfg["window"], cfg["stride"], cfg.get("dilation"),
                           cfg.get("causal"))
    torch.cuda.synchronize()
    assert out.dtype == torch.float16
    p = O.Params(cfg["spatial"], cfg["window"], cfg["stride"], cfg.get("dilation"), cfg.get("causal"))
    ro, rl = O.forward(as_f32_numpy(q), as_f32_numpy(k), as_f32_numpy(v), p)
    _close(out.float().cpu().numpy(), ro, lse.cpu().numpy(), rl)


@pytest.mark.parametrize("cfg", CFGS[2:5], ids=_ids)
def test_fp16_routes_bitwise(gna, cfg):
    """Permute-free, permuted + fused epilogue, permuted + unpermute kernel, and the stage
    API all give identical fp16 bytes."""
    from paper_2504_16922_b200.gna import GNA_FLAG_PERMUTED, GNA_FLAG_UNFUSED_EPILOGUE

    args = (cfg["window"], cfg["stride"], cfg.get("dilation"), cfg.get("causal"))
    q, k, v = (t.cuda() for t in make_qkv(2, cfg["spatial"], 3, 128, discriminating=True, dtype=torch.float16))
    res = [gna.forward(q, k, v, *args, flags=f) for f in (0, GNA_FLAG_PERMUTED, GNA_FLAG_UNFUSED_EPILOGUE)]
    o2 = torch.empty_like(q)
    l2 = torch.empty_like(res[0][1])
    gna.permute(q, k, v, o2, *args)
    gna.attention_permuted(q, k, v, o2, *args)
    gna.unpermute(q, k, v, o2, l2, *args)
    torch.cuda.synchronize()
    res.append((o2, l2))
    for o, l in res[1:]:
        assert torch.equal(res[0][0], o) and torch.equal(res[0][1], l)


@pytest.mark.parametrize("T", [77, 300])
def test_fp16_extra_kv(gna, T):
    cfg = CFGS[4]
    B, H, D = 2, 2, 128
    q, k, v = make_qkv(B, cfg["spatial"], H, D, discriminating=True, dtype=torch.float16)
    g = torch.Generator("cpu").manual_seed(78)
    ek = torch.randn((B, T, H, D), generator=g).to(torch.float16)
    ev = (torch.rand((B, T, H, D), generator=g) * 2 - 1).to(torch.float16)
    out, lse = gna.forward(q.cuda(), k.cuda(), v.cuda(), cfg["window"], cfg["stride"], cfg.get("dilation"),
                           cfg.get("causal"), extra_k=ek.cuda(), extra_v=ev.cuda())
    torch.cuda.synchronize()
    p = O.Params(cfg["spatial"], cfg["window"], cfg["stride"], cfg.get("dilation"), cfg.get("causal"))
    ro, rl = O.forward(as_f32_numpy(q), as_f32_numpy(k), as_f32_numpy(v), p, extra_k=as_f32_numpy(ek),
                       extra_v=as_f32_numpy(ev))
    _close(out.float().cpu().numpy(), ro, lse.cpu().numpy(), rl)


@pytest.mark.parametrize("name", ["c4a_hunyuan_blocked", "c2b_flux64_s16"])
def test_fp16_full_size_sampled(gna, name):
    """The fp16 launch bench.py --dtype fp16 times, at full size, discriminating inputs."""
    w = WORKLOADS[name]
    f = w.full()
    q, k, v = make_qkv(w.batch, w.spatial, w.heads, w.head_dim, discriminating=True, dtype=torch.float16)
    out, lse = gna.forward(q.cuda(), k.cuda(), v.cuda(), f["window"], f["stride"], f["dilation"], f["causal"])
    torch.cuda.synchronize()
    L = list(w.spatial) + [1] * (3 - len(w.spatial))
    corners = [0, L[1] * L[2] - 1, w.n_tokens - 1, (L[0] // 2) * L[1] * L[2] + (L[1] // 2) * L[2] + L[2] // 2]
    rows = sample_rows(w.batch, w.spatial, w.heads, 96, extra_tokens=corners)
    ro, rl, _ = O.forward_rows(as_f32_numpy(q), as_f32_numpy(k), as_f32_numpy(v), O.Params(**f), rows)
    o = out.float().cpu().reshape(w.batch, -1, w.heads, w.head_dim)[rows[:, 0], rows[:, 1], rows[:, 2]].numpy()
    l = lse.cpu().reshape(w.batch, -1, w.heads)[rows[:, 0], rows[:, 1], rows[:, 2]].numpy()
    _close(o, ro, l, rl)


def test_fp16_rejects_mixed_dtypes(gna):
    q = torch.zeros(1, 16, 16, 2, 64, dtype=torch.float16, device="cuda")
    kb = torch.zeros(1, 16, 16, 2, 64, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(gna.GnaError):
        gna.forward(q, kb, q, (4, 4))
    with pytest.raises(gna.GnaError):
        gna.forward(q, q, q, (4, 4), out=kb)
