"""GPU parity at BASELINE.json's full sizes with the DISCRIMINATING input set (q x3 so
the softmax is peaky, v ~ U(-1, 1)): SURVEY §8(c) warns that with N(0,1) inputs and
~10^4-key windows |O| ~ 0.01 sits under the 2e-2 O bar, so only LSE would guard the
V side.  Here |O| ~ 0.1-0.5 and a wrong V box or P->V mapping moves O by O(0.1).

Every video config of the bench (C3, C4a, C4b, X1) plus the paper's FLUX-4K shape X2
(Fig.5) runs through the default launch (the one bench.py times);
the rows compared with the fp64 oracle are a uniform sample plus every head of tokens at
grid corners, borders and stride-group boundaries on every axis."""
import itertools

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


def boundary_tokens(w, per_axis=4, seed=5):
    """Tokens whose coordinates sit on borders and stride-group edges of every axis."""
    L = list(w.spatial)
    f = w.full()
    cand = []
    for a, La in enumerate(L):
        s, win = f["stride"][a], f["window"][a]
        xs = {0, La - 1, min(La - 1, s - 1), min(La - 1, s), min(La - 1, win // 2), max(0, La - 1 - win // 2),
              (La // 2 // s) * s, max(0, (La // 2 // s) * s - 1)}
        cand.append(sorted(xs))
    rng = np.random.default_rng(seed)
    combos = list(itertools.product(*cand))
    pick = rng.choice(len(combos), size=min(len(combos), 24), replace=False)
    toks = []
    for i in pick:
        c = combos[i]
        t = 0
        for a in range(len(L)):
            t = t * L[a] + c[a]
        toks.append(int(t))
    return toks


def _check_rows(w, f, q, k, v, out, lse, rows, dtype_out=None):
    ro, rl, _ = O.forward_rows(as_f32_numpy(q), as_f32_numpy(k), as_f32_numpy(v), O.Params(**f), rows)
    o = out.float().cpu().reshape(w.batch, -1, w.heads, w.head_dim)[rows[:, 0], rows[:, 1], rows[:, 2]].numpy()
    l = lse.cpu().reshape(w.batch, -1, w.heads)[rows[:, 0], rows[:, 1], rows[:, 2]].numpy()
    err = np.abs(o - ro)
    lerr = np.abs(l - rl)
    assert np.isfinite(o).all() and np.isfinite(l).all()
    # the discriminating set makes O large enough to be checked at all
    assert np.abs(ro).mean() > 0.05, f"|O| mean {np.abs(ro).mean()}: inputs not discriminating"
    assert err.max() <= O_MAX, f"O max-abs {err.max()}"
    assert err.mean() <= O_MEAN, f"O mean-abs {err.mean()}"
    assert lerr.max() <= LSE_TOL, f"LSE max-abs {lerr.max()}"
    return err.max(), err.mean(), lerr.max()


@pytest.mark.parametrize("name", ["c3_cosmos", "c4a_hunyuan_blocked", "c4b_hunyuan_na", "x1_hunyuan_s16",
                                  "x2_flux4k"])
def test_fullsize_discriminating(gna, name):
    w = WORKLOADS[name]
    f = w.full()
    q, k, v = make_qkv(w.batch, w.spatial, w.heads, w.head_dim, discriminating=True)
    out, lse = gna.forward(q.cuda(), k.cuda(), v.cuda(), f["window"], f["stride"], f["dilation"], f["causal"])
    torch.cuda.synchronize()
    rows = sample_rows(w.batch, w.spatial, w.heads, 96, extra_tokens=boundary_tokens(w))
    mx, mean, lmx = _check_rows(w, f, q, k, v, out, lse, rows)
    print(f"{name}: {len(rows)} rows  O max {mx:.2e} mean {mean:.2e}  LSE {lmx:.2e}")


@pytest.mark.parametrize("name", ["x2_flux4k", "c2b_flux64_s16"])
def test_fullsize_normal_inputs(gna, name):
    """X2 and C2b with the plain N(0,1) recipe too (the bench inputs)."""
    w = WORKLOADS[name]
    f = w.full()
    q, k, v = make_qkv(w.batch, w.spatial, w.heads, w.head_dim)
    out, lse = gna.forward(q.cuda(), k.cuda(), v.cuda(), f["window"], f["stride"], f["dilation"], f["causal"])
    torch.cuda.synchronize()
    rows = sample_rows(w.batch, w.spatial, w.heads, 64, extra_tokens=boundary_tokens(w)[:8])
    ro, rl, _ = O.forward_rows(as_f32_numpy(q), as_f32_numpy(k), as_f32_numpy(v), O.Params(**f), rows)
    o = out.float().cpu().reshape(w.batch, -1, w.heads, w.head_dim)[rows[:, 0], rows[:, 1], rows[:, 2]].numpy()
    l = lse.cpu().reshape(w.batch, -1, w.heads)[rows[:, 0], rows[:, 1], rows[:, 2]].numpy()
    assert np.abs(o - ro).max() <= O_MAX and np.abs(o - ro).mean() <= O_MEAN
    assert np.abs(l - rl).max() <= LSE_TOL
