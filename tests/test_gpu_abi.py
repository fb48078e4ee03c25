"""GPU tests of the C ABI itself (through ctypes, no binding helpers where it matters):
the north-star 14-argument gna_forward, the unfused inverse-permute route against the
oracle, masking robustness (a masked key's V never reaches O), explicit work ranges,
and the stream / CUDA-graph contract of include/gna.h."""
import ctypes

import numpy as np
import pytest
import torch

import oracle as O
from gna_inputs import as_f32_numpy, make_qkv

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


I3 = ctypes.c_int * 3


@pytest.mark.parametrize("spatial,window,stride,dil,causal,D", [
    ((40, 36, 1), (9, 12, 1), (3, 4, 1), (1, 1, 1), (0, 0, 0), 128),     # permute-free route
    ((12, 20, 18), (5, 8, 6), (2, 3, 6), (1, 2, 1), (1, 0, 0), 64),       # dilation + causal
    ((200, 1, 1), (17, 1, 1), (5, 1, 1), (3, 1, 1), (1, 0, 0), 32),       # head_dim 32: permuted route
])
def test_north_star_gna_forward_14_args(gna, spatial, window, stride, dil, causal, D):
    """gna_forward(q, k, v, out, lse, batch, heads, head_dim, spatial[3], window[3],
    stride[3], dilation[3], causal[3], scale) on the legacy default stream, scale <= 0
    -> 1/sqrt(D), vs the fp64 oracle."""
    lib = gna.load()
    lib.gna_forward.restype = ctypes.c_int
    lib.gna_forward.argtypes = [ctypes.c_void_p] * 4 + [ctypes.c_void_p] + [ctypes.c_int] * 3 + \
        [ctypes.POINTER(ctypes.c_int)] * 5 + [ctypes.c_float]
    B, H = 2, 3
    sp = tuple(x for x in spatial if x > 1) or (1,)
    n = len(sp)
    q, k, v = make_qkv(B, sp, H, D, discriminating=True)
    qd, kd, vd = q.cuda(), k.cuda(), v.cuda()
    out = torch.full_like(qd, float("nan"))
    lse = torch.full(qd.shape[:-1], float("nan"), dtype=torch.float32, device="cuda")
    torch.cuda.synchronize()
    rc = lib.gna_forward(qd.data_ptr(), kd.data_ptr(), vd.data_ptr(), out.data_ptr(), lse.data_ptr(), B, H, D,
                         I3(*spatial), I3(*window), I3(*stride), I3(*dil), I3(*causal), ctypes.c_float(0.0))
    assert rc == 0, lib.gna_last_error()
    torch.cuda.synchronize()
    p = O.Params(sp, window[:n], stride[:n], dil[:n], tuple(bool(c) for c in causal[:n]))
    ro, rl = O.forward(as_f32_numpy(q), as_f32_numpy(k), as_f32_numpy(v), p)
    _close(out.float().cpu().numpy(), ro, lse.cpu().numpy(), rl)
    # invalid arguments: an error code, nothing written
    out.fill_(0)
    rc = lib.gna_forward(qd.data_ptr(), kd.data_ptr(), vd.data_ptr(), out.data_ptr(), lse.data_ptr(), B, H, D,
                         I3(*spatial), I3(*[w + 1000 for w in window]), I3(*stride), I3(*dil), I3(*causal),
                         ctypes.c_float(0.0))
    assert rc == 1 and b"exceeds" in lib.gna_last_error()
    torch.cuda.synchronize()
    assert int(out.abs().sum().item()) == 0


@pytest.mark.parametrize("cfg", [
    dict(spatial=(40, 36), window=(9, 12), stride=(3, 4)),
    dict(spatial=(37, 29), window=(8, 7), stride=(8, 7), dilation=(2, 2), causal=(False, True)),
    dict(spatial=(12, 20, 18), window=(5, 8, 6), stride=(2, 3, 6), dilation=(1, 2, 1), causal=(True, False, False)),
])
@pytest.mark.parametrize("D", [128, 32])
def test_unfused_unpermute_route_vs_oracle(gna, cfg, D):
    """permute -> attention (permuted O, LSE) -> standalone inverse-permute kernel
    (GNA_FLAG_UNFUSED_EPILOGUE), compared with the oracle directly."""
    from paper_2504_16922_b200.gna import GNA_FLAG_UNFUSED_EPILOGUE

    B, H = 2, 2
    q, k, v = make_qkv(B, cfg["spatial"], H, D, discriminating=True)
    o, l = gna.forward(q.cuda(), k.cuda(), v.cuda(), cfg["window"], cfg["stride"], cfg.get("dilation"),
                       cfg.get("causal"), flags=GNA_FLAG_UNFUSED_EPILOGUE)
    torch.cuda.synchronize()
    p = O.Params(cfg["spatial"], cfg["window"], cfg["stride"], cfg.get("dilation"), cfg.get("causal"))
    ro, rl = O.forward(as_f32_numpy(q), as_f32_numpy(k), as_f32_numpy(v), p)
    _close(o.float().cpu().numpy(), ro, l.cpu().numpy(), rl)


@pytest.mark.parametrize("route", ["direct", "permuted"])
def test_masked_keys_never_reach_o(gna, route):
    """Keys with x0 >= 33 of a 64x64 grid hold V = 1e38 (finite, near the bf16 maximum).
    Queries with x0 <= 28 never attend them (window 9: keys up to x0 + 4), but the KV boxes
    of the Q tiles next to the boundary contain them as MASKED keys of partial tiles.  Those
    rows must equal the oracle (computed with the planted values zeroed): a masked key must
    get P = 0 exactly on every exp path (MUFU and the FMA-pipe polynomial), not 2^-126."""
    from paper_2504_16922_b200.gna import GNA_FLAG_PERMUTED

    spatial, window, stride = (64, 64), (9, 9), (1, 1)
    B, H, D = 1, 2, 128
    q, k, v = make_qkv(B, spatial, H, D, discriminating=True)
    v_planted = v.clone()
    v_planted[:, 33:] = 1e38
    o, l = gna.forward(q.cuda(), k.cuda(), v_planted.cuda(), window, stride,
                       flags=GNA_FLAG_PERMUTED if route == "permuted" else 0)
    torch.cuda.synchronize()
    v_zero = v.clone()
    v_zero[:, 33:] = 0
    ro, rl = O.forward(as_f32_numpy(q), as_f32_numpy(k), as_f32_numpy(v_zero), O.Params(spatial, window, stride))
    keep = slice(0, 29)
    oo = o.float().cpu().numpy()[:, keep]
    assert np.isfinite(oo).all()
    _close(oo, ro[:, keep], l.cpu().numpy()[:, keep], rl[:, keep])
    # rows next to the boundary are where the masked keys sit in partial tiles
    err_edge = np.abs(oo[:, 21:29] - ro[:, 21:29]).max()
    assert err_edge <= O_MAX, err_edge


def test_explicit_work_ranges(gna):
    """GNA_FLAG_WORK_RANGE: an empty range launches nothing; disjoint ranges covering
    [0, n_work) reproduce the single launch bit for bit on the default (permute-free) route;
    out-of-range requests are rejected."""
    spatial, window, stride = (40, 36), (9, 12), (3, 4)
    B, H, D = 2, 3, 128
    q, k, v = (t.cuda() for t in make_qkv(B, spatial, H, D, discriminating=True))
    ref_o, ref_l = gna.forward(q, k, v, window, stride)
    n = gna.plan_info(B, H, D, spatial, window, stride)["n_work"]
    o = torch.zeros_like(q)
    l = torch.zeros(q.shape[:-1], dtype=torch.float32, device="cuda")
    gna.forward(q, k, v, window, stride, out=o, lse=l, work_range=(5, 5))
    torch.cuda.synchronize()
    assert int(o.abs().sum().item()) == 0 and int(l.abs().sum().item()) == 0
    gna.forward(q, k, v, window, stride, out=o, lse=l, work_range=(0, 0))
    torch.cuda.synchronize()
    assert int(o.abs().sum().item()) == 0
    cuts = [0, n // 5, n // 2, n - 1, n]
    for a, b in zip(cuts[:-1], cuts[1:]):
        gna.forward(q, k, v, window, stride, out=o, lse=l, work_range=(a, b))
    torch.cuda.synchronize()
    assert torch.equal(o, ref_o) and torch.equal(l, ref_l)
    with pytest.raises(gna.GnaError):
        gna.forward(q, k, v, window, stride, out=o, lse=l, work_range=(0, n + 1))
    with pytest.raises(gna.GnaError):
        gna.forward(q, k, v, window, stride, out=o, lse=l, work_range=(3, 2))


def test_side_stream_and_cuda_graph(gna):
    """Stream-ordered and capture-safe: a call on a side stream, then the same call
    captured in a CUDA graph and replayed, give the default-stream result bit for bit,
    on the permute-free route and on the permuted route with a caller workspace."""
    from paper_2504_16922_b200.gna import GNA_FLAG_PERMUTED

    spatial, window, stride, dil = (24, 20, 12), (7, 6, 5), (3, 2, 5), (1, 1, 2)
    B, H, D = 2, 2, 128
    q, k, v = (t.cuda() for t in make_qkv(B, spatial, H, D, discriminating=True))
    for flags in (0, GNA_FLAG_PERMUTED):
        ref_o, ref_l = gna.forward(q, k, v, window, stride, dil, flags=flags)
        torch.cuda.synchronize()
        ws = torch.empty(gna.workspace_size(B, H, D, spatial, window, stride, dil), dtype=torch.uint8,
                         device="cuda")
        side = torch.cuda.Stream()
        o = torch.empty_like(q)
        l = torch.empty(q.shape[:-1], dtype=torch.float32, device="cuda")
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            gna.forward(q, k, v, window, stride, dil, out=o, lse=l, flags=flags, workspace=ws)
        side.synchronize()
        assert torch.equal(o, ref_o) and torch.equal(l, ref_l)
        o.zero_()
        l.zero_()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(side):
            with torch.cuda.graph(g, stream=side):
                gna.forward(q, k, v, window, stride, dil, out=o, lse=l, flags=flags, workspace=ws)
        torch.cuda.synchronize()
        for _ in range(3):
            g.replay()
        torch.cuda.synchronize()
        assert torch.equal(o, ref_o) and torch.equal(l, ref_l)


def test_first_call_inside_capture_is_refused(gna):
    """A problem never seen on this device cannot be planned inside a capture (the work
    list upload allocates): a clear error, no crash, and the capture stays usable."""
    spatial, window, stride = (26, 22), (5, 7), (1, 7)  # not used by any other test
    q, k, v = (t.cuda() for t in make_qkv(1, spatial, 1, 64))
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    with pytest.raises(gna.GnaError, match="capture"):
        with torch.cuda.stream(s):
            with torch.cuda.graph(g, stream=s):
                gna.forward(q, k, v, window, stride)
    torch.cuda.synchronize()
    o, l = gna.forward(q, k, v, window, stride)
    torch.cuda.synchronize()
    ro, rl = O.forward(as_f32_numpy(q.cpu()), as_f32_numpy(k.cpu()), as_f32_numpy(v.cpu()),
                       O.Params(spatial, window, stride))
    _close(o.float().cpu().numpy(), ro, l.cpu().numpy(), rl)


def test_binding_rejects_mismatched_shapes(gna):
    q = torch.zeros(1, 16, 16, 2, 64, dtype=torch.bfloat16, device="cuda")
    k_small = torch.zeros(1, 16, 8, 2, 64, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(gna.GnaError, match="shape"):
        gna.forward(q, k_small, q, (4, 4))
    with pytest.raises(gna.GnaError, match="lse"):
        gna.forward(q, q, q, (4, 4), lse=torch.zeros(1, 16, 16, dtype=torch.float32, device="cuda"))


def test_release_workspace_then_reuse(gna):
    """gna_release_workspace frees the caches and device work lists; the next call rebuilds."""
    from paper_2504_16922_b200.gna import GNA_FLAG_PERMUTED

    spatial, window, stride = (40, 36), (9, 12), (3, 4)
    q, k, v = (t.cuda() for t in make_qkv(1, spatial, 2, 64, discriminating=True))
    o1, l1 = gna.forward(q, k, v, window, stride, flags=GNA_FLAG_PERMUTED)
    gna.release_workspace()
    o2, l2 = gna.forward(q, k, v, window, stride, flags=GNA_FLAG_PERMUTED)
    torch.cuda.synchronize()
    assert torch.equal(o1, o2) and torch.equal(l1, l2)
