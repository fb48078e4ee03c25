"""GPU parity: the CUDA path (through the C ABI) against the fp64 oracle.

Bars (BASELINE.json north_star): windows and tile visits bit-exact; O within
max-abs 2e-2 and mean-abs 2e-3; LSE within 1e-3 (abs)."""
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
    assert pkg.device_supported(), "device is not sm_100"
    return pkg


def _cfg(spatial, window, stride=None, dilation=None, causal=None):
    n = len(spatial)
    return dict(spatial=tuple(spatial), window=tuple(window), stride=tuple(stride or (1,) * n),
                dilation=tuple(dilation or (1,) * n), causal=tuple(causal or (False,) * n))


SMALL = [
    _cfg((256,), (32,), (8,)),                                    # C1 geometry
    _cfg((200,), (17,), (5,), (3,), (True,)),                     # 1-D ragged, dilation, causal
    _cfg((40, 36), (9, 12), (3, 4)),                              # 2-D ragged
    _cfg((37, 29), (8, 7), (8, 7), (2, 2), (False, True)),        # blocked + dilation + causal
    _cfg((12, 20, 18), (5, 8, 6), (2, 3, 6), (1, 2, 1), (True, False, False)),
    _cfg((16, 16, 16), (16, 16, 16), (1, 1, 1)),                  # dense (window = extent)
    _cfg((64, 64), (32, 32), (16, 16)),                           # C2b geometry
    _cfg((64, 64), (32, 32), (8, 8)),                             # C2a geometry
]


def _ids(c):
    return "x".join(map(str, c["spatial"])) + "_w" + "x".join(map(str, c["window"])) + \
        "_s" + "x".join(map(str, c["stride"])) + "_d" + "x".join(map(str, c["dilation"])) + \
        "_c" + "".join(str(int(x)) for x in c["causal"])


@pytest.mark.parametrize("cfg", SMALL, ids=_ids)
def test_windows_bit_exact(gna, cfg):
    got = gna.debug_windows(**cfg)
    ref = O.windows(O.Params(**cfg))
    np.testing.assert_array_equal(got, ref)


@pytest.mark.parametrize("cfg", SMALL + [_cfg((30, 48, 80), (18, 24, 24), (16, 8, 8)),
                                         _cfg((30, 48, 80), (18, 24, 24), (1, 1, 1))], ids=_ids)
def test_visits_bit_exact(gna, cfg):
    """Per Q sub-tile: the analytic per-axis box ranges reproduce the oracle's
    brute-force visited set exactly, and the uniform full-tile predicate counts
    exactly the brute-force fully attended boxes."""
    p = O.Params(**cfg)
    info = gna.plan_info(1, 1, 128, **cfg)
    recs = gna.debug_visits(**cfg)
    tq, tk = info["q_sub"], info["box"]
    n_cls = info["n_classes"]
    for cls in range(n_cls):
        Lc = O.class_extents(p, cls)
        nq = [-(-Lc[a] // tq[a]) for a in range(3)]
        nk = [-(-Lc[a] // tk[a]) for a in range(3)]
        vis = O.visits_bruteforce(p, tq, tk, cls)
        full = O.full_bruteforce(p, tq, tk, vis, cls) if p.n_tokens <= 20000 else None
        rc = recs[recs[:, 0] == cls]
        # the GPU sub-tile grid is padded to the class-0 extent: map coordinates
        for rec in rc:
            sc = _sub_coords(rec[1], info, p)
            inside = all(sc[a] < nq[a] for a in range(3))
            if not inside:
                assert rec[9] == 0
                continue
            assert rec[9] == 1
            qt = (sc[0] * nq[1] + sc[1]) * nq[2] + sc[2]
            row = vis[qt].reshape(nk)
            lo, hi = rec[2:8:2], rec[3:8:2]
            box = np.zeros(nk, dtype=np.uint8)
            box[lo[0]:hi[0], lo[1]:hi[1], lo[2]:hi[2]] = 1
            np.testing.assert_array_equal(row, box)
            if full is not None:
                assert rec[8] == int(full[qt].sum())


def _sub_coords(sub, info, p):
    # sub-tile grid of the GPU plan: ceil(ceil(L/d) / q_sub) per axis
    nq = [-(-(-(-p.spatial[a] // p.dilation[a])) // info["q_sub"][a]) for a in range(3)]
    return [sub // (nq[1] * nq[2]), (sub // nq[2]) % nq[1], sub % nq[2]]


def _run(gna, cfg, B, H, D, disc, box=None):
    q, k, v = make_qkv(B, cfg["spatial"], H, D, discriminating=disc)
    out, lse = gna.forward(q.cuda(), k.cuda(), v.cuda(), cfg["window"], cfg["stride"], cfg["dilation"],
                           cfg["causal"], box=box)
    torch.cuda.synchronize()
    return (q, k, v), out.float().cpu().numpy(), lse.cpu().numpy()


def _assert_close(o, ro, l, rl):
    err = np.abs(o - ro)
    lerr = np.abs(l - rl)
    assert np.isfinite(o).all() and np.isfinite(l).all()
    assert err.max() <= O_MAX, f"O max-abs {err.max()}"
    assert err.mean() <= O_MEAN, f"O mean-abs {err.mean()}"
    assert lerr.max() <= LSE_TOL, f"LSE max-abs {lerr.max()}"


@pytest.mark.parametrize("disc", [False, True], ids=["normal", "discriminating"])
@pytest.mark.parametrize("cfg", SMALL[:6], ids=_ids)
@pytest.mark.parametrize("D", [128, 64, 32])
def test_forward_small_full(gna, cfg, disc, D):
    B, H = 2, 2
    (q, k, v), o, l = _run(gna, cfg, B, H, D, disc)
    ro, rl = O.forward(as_f32_numpy(q), as_f32_numpy(k), as_f32_numpy(v), O.Params(**cfg))
    _assert_close(o, ro, l, rl)


def test_c1_tiny_full(gna):
    """configs[0]: 1-D tiny, D=32, fp32 inputs rounded once to bf16, full output."""
    w = WORKLOADS["c1_tiny1d"]
    for disc in (False, True):
        (q, k, v), o, l = _run(gna, w.full(), w.batch, w.heads, w.head_dim, disc)
        ro, rl = O.forward(as_f32_numpy(q), as_f32_numpy(k), as_f32_numpy(v), O.Params(**w.full()))
        _assert_close(o, ro, l, rl)


@pytest.mark.parametrize("box", [None, (8, 8, 1), (8, 16, 1), (16, 8, 1)])
def test_c2_flux_sampled(gna, box):
    """configs[1] at full size, both strides, sampled rows (incl. borders)."""
    for name in ("c2a_flux64_s8", "c2b_flux64_s16"):
        w = WORKLOADS[name]
        f = w.full()
        (q, k, v), o, l = _run(gna, f, w.batch, w.heads, w.head_dim, True, box=box)
        border = [0, 63, 64 * 63, 4095, 64 * 31 + 32, 100, 2000]
        rows = sample_rows(w.batch, w.spatial, w.heads, 300, extra_tokens=border)
        ro, rl, _ = O.forward_rows(as_f32_numpy(q), as_f32_numpy(k), as_f32_numpy(v), O.Params(**f), rows)
        oo = o.reshape(w.batch, -1, w.heads, w.head_dim)[rows[:, 0], rows[:, 1], rows[:, 2]]
        ll = l.reshape(w.batch, -1, w.heads)[rows[:, 0], rows[:, 1], rows[:, 2]]
        _assert_close(oo, ro, ll, rl)


@pytest.mark.parametrize("name", ["c3_cosmos", "c4a_hunyuan_blocked", "c4b_hunyuan_na", "x1_hunyuan_s16"])
def test_video_configs_sampled(gna, name):
    """configs[2], configs[3] and the paper's headline shape at full size."""
    w = WORKLOADS[name]
    f = w.full()
    (q, k, v), o, l = _run(gna, f, w.batch, w.heads, w.head_dim, False)
    L = w.spatial
    corners = [0, L[1] * L[2] - 1, w.n_tokens - 1, (L[0] // 2) * L[1] * L[2] + (L[1] // 2) * L[2] + L[2] // 2]
    rows = sample_rows(w.batch, w.spatial, w.heads, 64, extra_tokens=corners)
    ro, rl, _ = O.forward_rows(as_f32_numpy(q), as_f32_numpy(k), as_f32_numpy(v), O.Params(**f), rows)
    oo = o.reshape(w.batch, -1, w.heads, w.head_dim)[rows[:, 0], rows[:, 1], rows[:, 2]]
    ll = l.reshape(w.batch, -1, w.heads)[rows[:, 0], rows[:, 1], rows[:, 2]]
    _assert_close(oo, ro, ll, rl)


def test_stages_equal_forward(gna):
    cfg = SMALL[4]
    B, H, D = 2, 3, 128
    q, k, v = (t.cuda() for t in make_qkv(B, cfg["spatial"], H, D))
    out, lse = gna.forward(q, k, v, cfg["window"], cfg["stride"], cfg["dilation"], cfg["causal"])
    o2 = torch.empty_like(q)
    l2 = torch.empty_like(lse)
    gna.permute(q, k, v, o2, cfg["window"], cfg["stride"], cfg["dilation"], cfg["causal"])
    gna.attention_permuted(q, k, v, o2, cfg["window"], cfg["stride"], cfg["dilation"], cfg["causal"])
    gna.unpermute(q, k, v, o2, l2, cfg["window"], cfg["stride"], cfg["dilation"], cfg["causal"])
    torch.cuda.synchronize()
    assert torch.equal(out, o2) and torch.equal(lse, l2)


@pytest.mark.parametrize("cfg", SMALL, ids=_ids)
def test_direct_fused_permuted_paths_bitwise(gna, cfg):
    """Three routes to the same result, bit for bit: the default permute-free path
    (5-D TMA gathers + epilogue scatter), permute -> attention with the fused
    epilogue (GNA_FLAG_PERMUTED), and permute -> attention -> unpermute kernel
    (GNA_FLAG_UNFUSED_EPILOGUE).  Masked and padded keys get P = 0 exactly (ex2 of
    -inf on the MUFU and, since round 2, on the FMA-pipe polynomial too) and padded V rows
    are zero on both routes (TMA zero fill / permuted zero rows), so they add exact zeros
    and the two sources of padding are indistinguishable."""
    from paper_2504_16922_b200.gna import GNA_FLAG_PERMUTED, GNA_FLAG_UNFUSED_EPILOGUE

    for D in (128, 64, 32):
        q, k, v = (t.cuda() for t in make_qkv(2, cfg["spatial"], 3, D, discriminating=True))
        res = []
        for flags in (0, GNA_FLAG_PERMUTED, GNA_FLAG_UNFUSED_EPILOGUE):
            o, l = gna.forward(q, k, v, cfg["window"], cfg["stride"], cfg["dilation"], cfg["causal"], flags=flags)
            res.append((o, l))
        torch.cuda.synchronize()
        for o, l in res[1:]:
            assert torch.equal(res[0][0], o) and torch.equal(res[0][1], l)


def test_work_range_split_is_bitwise(gna):
    """Q-tile splitting (multi-GPU sharding) over [begin, end) ranges of the work
    list reproduces the single launch bit for bit."""
    cfg = SMALL[2]
    B, H, D = 2, 2, 64
    q, k, v = (t.cuda() for t in make_qkv(B, cfg["spatial"], H, D))
    out, lse = gna.forward(q, k, v, cfg["window"], cfg["stride"])
    info = gna.plan_info(B, H, D, **cfg)
    total = info["n_work"]
    mid = total // 3
    # run both halves through the stage API on one workspace, then unpermute
    import paper_2504_16922_b200.gna as G
    import ctypes
    o2 = torch.empty_like(q)
    l2 = torch.empty_like(lse)
    gna.permute(q, k, v, o2, cfg["window"], cfg["stride"])
    for rng in ((0, mid), (mid, total)):
        a = G._tensor_args(q, k, v, o2, l2, cfg["window"], cfg["stride"], None, None, None, None, rng, None, 0)
        G._check(G.load().gna_attention_permuted(ctypes.byref(a)))
    gna.unpermute(q, k, v, o2, l2, cfg["window"], cfg["stride"])
    torch.cuda.synchronize()
    assert torch.equal(out, o2) and torch.equal(lse, l2)


def test_dense_matches_torch_sdpa(gna):
    """window = extent: the same kernel is dense attention; compare with torch's SDPA
    (fp32 math on the bf16 inputs) as an independent library reference."""
    spatial, H, D = (32, 32), 4, 128
    q, k, v = (t.cuda() for t in make_qkv(1, spatial, H, D))
    out, lse = gna.forward(q, k, v, spatial)
    qf, kf, vf = (t.float().reshape(1, -1, H, D).transpose(1, 2) for t in (q, k, v))
    ref = torch.nn.functional.scaled_dot_product_attention(qf, kf, vf).transpose(1, 2).reshape(out.shape)
    err = (out.float() - ref).abs()
    assert err.max().item() <= O_MAX and err.mean().item() <= O_MEAN


def test_invalid_args_launch_nothing(gna):
    from paper_2504_16922_b200.gna import GnaError

    q = torch.zeros(1, 16, 1, 64, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(GnaError, match="holes"):
        gna.forward(q, q, q, (4,), (5,))


def _extra(B, T, H, D, seed=77):
    g = torch.Generator("cpu").manual_seed(seed)
    ek = torch.randn((B, T, H, D), generator=g).to(torch.bfloat16)
    ev = (torch.rand((B, T, H, D), generator=g) * 2 - 1).to(torch.bfloat16)
    return ek, ev


@pytest.mark.parametrize("T", [1, 77, 128, 300])
@pytest.mark.parametrize("cfg", [SMALL[2], SMALL[4], SMALL[6]], ids=_ids)
def test_extra_kv_tokens(gna, cfg, T):
    """NEXT-1: extra text tokens attended by every query, fused into the same
    kernel as dense stages; both the permute-free and the permuted path vs the oracle."""
    from paper_2504_16922_b200.gna import GNA_FLAG_PERMUTED

    B, H = 2, 2
    for D in (128, 64):
        q, k, v = make_qkv(B, cfg["spatial"], H, D, discriminating=True)
        ek, ev = _extra(B, T, H, D)
        ro, rl = O.forward(as_f32_numpy(q), as_f32_numpy(k), as_f32_numpy(v), O.Params(**cfg),
                           extra_k=as_f32_numpy(ek), extra_v=as_f32_numpy(ev))
        outs = []
        for flags in (0, GNA_FLAG_PERMUTED):
            o, l = gna.forward(q.cuda(), k.cuda(), v.cuda(), cfg["window"], cfg["stride"], cfg["dilation"],
                               cfg["causal"], flags=flags, extra_k=ek.cuda(), extra_v=ev.cuda())
            torch.cuda.synchronize()
            outs.append((o, l))
            _assert_close(o.float().cpu().numpy(), ro, l.cpu().numpy(), rl)
        assert torch.equal(outs[0][0], outs[1][0]) and torch.equal(outs[0][1], outs[1][1])


@pytest.mark.parametrize("name", ["s1_sweep1d", "s2_sweep2d", "s2c_sweep2d_causal", "s3_sweep3d"])
def test_sweep_configs_sampled(gna, name):
    """configs[4]: the batch-8 sweep rows with dilation 2 and per-axis causal masks, at full
    size through the default launch path, on sampled rows (every batch, class corners)."""
    w = WORKLOADS[name]
    f = w.full()
    (q, k, v), o, l = _run(gna, f, w.batch, w.heads, w.head_dim, True)
    L = list(w.spatial) + [1] * (3 - len(w.spatial))
    corners = [0, 1, w.n_tokens - 1, w.n_tokens - 2, (L[0] // 2) * L[1] * L[2] + 1]
    rows = sample_rows(w.batch, w.spatial, w.heads, 48, extra_tokens=corners)
    ro, rl, _ = O.forward_rows(as_f32_numpy(q), as_f32_numpy(k), as_f32_numpy(v), O.Params(**f), rows)
    oo = o.reshape(w.batch, -1, w.heads, w.head_dim)[rows[:, 0], rows[:, 1], rows[:, 2]]
    ll = l.reshape(w.batch, -1, w.heads)[rows[:, 0], rows[:, 1], rows[:, 2]]
    _assert_close(oo, ro, ll, rl)


@pytest.mark.parametrize("cfg", [
    _cfg((1,), (1,), (1,)),                       # a single token: attends itself only
    _cfg((3, 1, 2), (1, 1, 1), (1, 1, 1)),        # window 1: O = V, LSE = logit
    _cfg((5,), (5,), (5,), causal=(True,)),       # one causal block smaller than any box
    _cfg((2, 3, 130), (2, 3, 7), (1, 3, 7)),      # 3-D with a long last axis (boxes beyond 128)
    _cfg((129,), (129,), (1,)),                   # dense, one key past a 128 box
], ids=_ids)
def test_degenerate_shapes(gna, cfg):
    B, H, D = 3, 2, 64
    (q, k, v), o, l = _run(gna, cfg, B, H, D, True)
    ro, rl = O.forward(as_f32_numpy(q), as_f32_numpy(k), as_f32_numpy(v), O.Params(**cfg))
    _assert_close(o, ro, l, rl)


@pytest.mark.gpu
@pytest.mark.parametrize("cfg", [SMALL[2], SMALL[5], SMALL[6], SMALL[3]], ids=_ids)
def test_tma_store_epilogue_bitwise(gna, cfg, monkeypatch):
    """The epilogue's smem + TMA-store route writes exactly what the per-thread stores write
    (same values, no spill into the neighbouring sample or padding rows), on the direct and the
    permuted stage path; GNA_TMA_STORE=0 selects the per-thread stores."""
    B, H, D = 2, 2, 128
    q, k, v = (t.cuda() for t in make_qkv(B, cfg["spatial"], H, D, discriminating=True))
    res = {}
    for ts in ("0", "1"):
        monkeypatch.setenv("GNA_TMA_STORE", ts)
        o, l = gna.forward(q, k, v, cfg["window"], cfg["stride"], cfg.get("dilation"), cfg.get("causal"))
        o2 = torch.empty_like(q)
        l2 = torch.empty_like(l)
        gna.permute(q, k, v, o2, cfg["window"], cfg["stride"], cfg.get("dilation"), cfg.get("causal"))
        gna.attention_permuted(q, k, v, o2, cfg["window"], cfg["stride"], cfg.get("dilation"), cfg.get("causal"))
        gna.unpermute(q, k, v, o2, l2, cfg["window"], cfg["stride"], cfg.get("dilation"), cfg.get("causal"))
        torch.cuda.synchronize()
        res[ts] = (o, l, o2, l2)
    for a, b in zip(res["0"], res["1"]):
        assert torch.equal(a, b)
