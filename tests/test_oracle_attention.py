"""Pins for the oracle's attention arithmetic (§2.2; LSE P:615-616).

Reductions to library routines on special cases (dense SDPA, blocked SDPA,
causal sliding window) plus a general masked-softmax check where the mask is
built pair by pair (is_attended) while the oracle enumerates neighbourhoods.
"""
import itertools

import numpy as np
import pytest
import torch

import oracle as O
from gna_inputs import as_f32_numpy, make_qkv


def _masked_sdpa(q, k, v, mask, scale):
    """fp64 torch reference: q,k,v [N, D] float64, mask [N, N] bool."""
    qt, kt, vt = (torch.from_numpy(x).double() for x in (q, k, v))
    z = (qt @ kt.T) * scale
    z = z.masked_fill(~torch.from_numpy(mask), float("-inf"))
    lse = torch.logsumexp(z, dim=-1)
    out = torch.softmax(z, dim=-1) @ vt
    return out.numpy(), lse.numpy()


def _run_case(spatial, window, stride, dilation=None, causal=None, B=2, H=2, D=16, disc=False):
    p = O.Params(spatial, window, stride, dilation, causal)
    q, k, v = make_qkv(B, spatial, H, D, discriminating=disc)
    qn, kn, vn = as_f32_numpy(q), as_f32_numpy(k), as_f32_numpy(v)
    out, lse = O.forward(qn, kn, vn, p)
    return p, (qn, kn, vn), out, lse


def _per_head(x, b, h):
    B = x.shape[0]
    N = int(np.prod(x.shape[1:-2]))
    return x.reshape(B, N, x.shape[-2], x.shape[-1])[b, :, h, :].astype(np.float64)


def _check_against_mask(p, qkv, out, lse, mask, D):
    B, H = qkv[0].shape[0], qkv[0].shape[-2]
    N = p.n_tokens
    o = out.reshape(B, N, H, D)
    l = lse.reshape(B, N, H)
    for b in range(B):
        for h in range(H):
            ro, rl = _masked_sdpa(*(_per_head(x, b, h) for x in qkv), mask, 1.0 / np.sqrt(D))
            np.testing.assert_allclose(o[b, :, h], ro, rtol=0, atol=1e-12)
            np.testing.assert_allclose(l[b, :, h], rl, rtol=0, atol=1e-12)


@pytest.mark.parametrize("spatial,stride", [((37,), (5,)), ((7, 9), (2, 3)), ((3, 4, 5), (1, 2, 3))])
def test_window_equals_extent_matches_dense_sdpa(spatial, stride):
    """window = input size numerically matches self attention."""
    p, qkv, out, lse = _run_case(spatial, spatial, stride)
    _check_against_mask(p, qkv, out, lse, np.ones((p.n_tokens,) * 2, dtype=bool), 16)


def test_blocked_matches_per_block_sdpa():
    """stride = window (w | L) is blocked attention: each block of w
    tokens is an independent dense SDPA (computed here block by block)."""
    spatial, w = (12, 8), (4, 4)
    p, qkv, out, lse = _run_case(spatial, w, w)
    B, H, D = 2, 2, 16
    o = out.reshape(B, 12, 8, H, D)
    l = lse.reshape(B, 12, 8, H)
    for b, h in itertools.product(range(B), range(H)):
        for bi, bj in itertools.product(range(3), range(2)):
            sl = (slice(4 * bi, 4 * bi + 4), slice(4 * bj, 4 * bj + 4))
            blk = [x.reshape(B, 12, 8, H, D)[b][sl][..., h, :].reshape(16, D).astype(np.float64)
                   for x in qkv]
            qt, kt, vt = (torch.from_numpy(x) for x in blk)
            ref = torch.nn.functional.scaled_dot_product_attention(qt[None], kt[None], vt[None])[0]
            np.testing.assert_allclose(o[b][sl][..., h, :].reshape(16, D), ref.numpy(), atol=1e-12)
            rl = torch.logsumexp((qt @ kt.T) / np.sqrt(D), -1).numpy()
            np.testing.assert_allclose(l[b][sl][..., h].reshape(16), rl, atol=1e-12)


def test_causal_sliding_window_matches_sdpa_mask():
    """Reading R4 limit: s=1 causal is the textbook causal sliding window."""
    L, w = 40, 7
    p, qkv, out, lse = _run_case((L,), (w,), (1,), causal=(True,))
    i = np.arange(L)
    mask = (i[None, :] <= i[:, None]) & (i[None, :] >= i[:, None] - w + 1)
    _check_against_mask(p, qkv, out, lse, mask, 16)


def test_na_1d_matches_textbook_clamped_window():
    """s=1 non-causal: standard NA with a mask built from the
    nearest-centered-interval characterisation."""
    L, w = 33, 8
    p, qkv, out, lse = _run_case((L,), (w,), (1,))
    mask = np.zeros((L, L), dtype=bool)
    for i in range(L):
        best = min(range(0, L - w + 1), key=lambda t: (abs(t + w // 2 - i), t))
        mask[i, best:best + w] = True
    _check_against_mask(p, qkv, out, lse, mask, 16)


@pytest.mark.parametrize("case", [
    ((9, 11), (3, 5), (2, 3), (1, 2), (False, True)),
    ((6, 5, 7), (3, 2, 4), (3, 1, 2), (2, 1, 1), (True, False, False)),
    ((24,), (6,), (4,), (3,), (False,)),
    ((10, 12), (5, 4), (5, 4), (2, 3), (False, False)),
])
def test_general_matches_pairwise_mask(case):
    """Enumerated-neighbourhood forward == masked softmax with the brute-force
    pairwise mask, discriminating inputs (peaky softmax)."""
    p, qkv, out, lse = _run_case(*case, disc=True)
    _check_against_mask(p, qkv, out, lse, O.mask(p), 16)


def test_dilation_is_independent_na_per_class():
    """Reading R6 (cited only): dilation d = independent GNA on each
    interleaved class sub-grid [c::d], computed here by slicing."""
    spatial, w, s, d = (13, 10), (3, 4), (2, 3), (3, 2)
    p, qkv, out, lse = _run_case(spatial, w, s, d, (False, True), D=8)
    B, H, D = 2, 2, 8
    o = out.reshape(B, 13, 10, H, D)
    l = lse.reshape(B, 13, 10, H)
    q5 = [x.reshape(B, 13, 10, H, D) for x in qkv]
    for c0 in range(3):
        for c1 in range(2):
            sub = [np.ascontiguousarray(x[:, c0::3, c1::2]) for x in q5]
            sp = sub[0].shape[1:3]
            so, sl = O.forward(*sub, O.Params(sp, w, s, causal=(False, True)), scale=1 / np.sqrt(D))
            np.testing.assert_allclose(o[:, c0::3, c1::2], so, atol=1e-12)
            np.testing.assert_allclose(l[:, c0::3, c1::2], sl, atol=1e-12)


def test_single_key_lse_is_logit():
    """w = 1: out = v of the key, LSE = the scaled logit (natural log)."""
    p, qkv, out, lse = _run_case((5, 6), (1, 1), (1, 1), D=8)
    q, k, v = qkv
    np.testing.assert_allclose(out, v.astype(np.float64), atol=1e-12)
    np.testing.assert_allclose(lse, (q.astype(np.float64) * k).sum(-1) / np.sqrt(8), atol=1e-12)


def test_forward_rows_equals_full():
    p, qkv, out, lse = _run_case((6, 7, 5), (3, 4, 3), (2, 2, 1), (1, 1, 1), (False, False, True), D=8)
    rows = np.array([[0, 0, 0], [1, 209, 1], [0, 100, 1], [1, 5, 0]], dtype=np.int64)
    ro, rl, pairs = O.forward_rows(*qkv, p, rows)
    B, H, D, N = 2, 2, 8, 210
    o = out.reshape(B, N, H, D)
    l = lse.reshape(B, N, H)
    for r, (b, n, h) in enumerate(rows):
        np.testing.assert_array_equal(ro[r], o[b, n, h])
        assert rl[r] == l[b, n, h]
    assert pairs > 0


def test_rows_are_convex_combinations():
    """softmax weights are a probability vector: each output lies inside the
    per-dimension min/max of V over the whole grid."""
    p, qkv, out, lse = _run_case((9, 9), (3, 5), (1, 2), disc=True)
    v = qkv[2]
    vmin = v.min(axis=(1, 2), keepdims=True)
    vmax = v.max(axis=(1, 2), keepdims=True)
    assert (out >= vmin - 1e-12).all() and (out <= vmax + 1e-12).all()


def _extra_kv(B, T, H, D, seed):
    g = torch.Generator("cpu").manual_seed(seed)
    ek = torch.randn((B, T, H, D), generator=g).to(torch.bfloat16).float().numpy()
    ev = torch.randn((B, T, H, D), generator=g).to(torch.bfloat16).float().numpy()
    return ek, ev


def test_extra_kv_is_masked_softmax_with_dense_columns():
    """P:613-618 / SPEC gna_attention(extra_kv): extra (text) keys are attended by every
    query in the same softmax -- the mask extended by all-true columns."""
    spatial, w, s = (6, 7), (3, 4), (2, 3)
    B, H, D, T = 2, 2, 16, 5
    p, qkv, _, _ = _run_case(spatial, w, s, B=B, H=H, D=D, disc=True)
    ek, ev = _extra_kv(B, T, H, D, 5)
    out, lse = O.forward(*qkv, p, extra_k=ek, extra_v=ev)
    N = p.n_tokens
    mask = np.concatenate([O.mask(p), np.ones((N, T), dtype=bool)], axis=1)
    o = out.reshape(B, N, H, D)
    l = lse.reshape(B, N, H)
    for b in range(B):
        for h in range(H):
            q_, k_, v_ = (_per_head(x, b, h) for x in qkv)
            k_ = np.concatenate([k_, ek[b, :, h].astype(np.float64)])
            v_ = np.concatenate([v_, ev[b, :, h].astype(np.float64)])
            ro, rl = _masked_sdpa(q_, k_, v_, mask, 1.0 / np.sqrt(D))
            np.testing.assert_allclose(o[b, :, h], ro, atol=1e-12)
            np.testing.assert_allclose(l[b, :, h], rl, atol=1e-12)


def test_extra_kv_equals_lse_merge_of_partials():
    """attention over (neighbourhood + extra keys) equals the logsumexp merge
    of the GNA-only partial and a dense attention over the extra keys alone."""
    spatial, w, s = (5, 4, 6), (3, 2, 3), (1, 2, 3)
    B, H, D, T = 1, 3, 8, 7
    p, qkv, out0, lse0 = _run_case(spatial, w, s, B=B, H=H, D=D)
    ek, ev = _extra_kv(B, T, H, D, 9)
    out, lse = O.forward(*qkv, p, extra_k=ek, extra_v=ev)
    N = p.n_tokens
    qt = torch.from_numpy(qkv[0].reshape(B, N, H, D).astype(np.float64)).permute(0, 2, 1, 3)
    kt = torch.from_numpy(ek.astype(np.float64)).permute(0, 2, 1, 3)
    vt = torch.from_numpy(ev.astype(np.float64)).permute(0, 2, 1, 3)
    z = qt @ kt.transpose(-1, -2) / np.sqrt(D)
    lse_e = torch.logsumexp(z, -1).permute(0, 2, 1).numpy()
    out_e = (torch.softmax(z, -1) @ vt).permute(0, 2, 1, 3).numpy()
    la, lb = lse0.reshape(B, N, H), lse_e
    m = np.maximum(la, lb)
    wa, wb = np.exp(la - m), np.exp(lb - m)
    merged = (wa[..., None] * out0.reshape(B, N, H, D) + wb[..., None] * out_e) / (wa + wb)[..., None]
    np.testing.assert_allclose(out.reshape(B, N, H, D), merged, atol=1e-12)
    np.testing.assert_allclose(lse.reshape(B, N, H), m + np.log(wa + wb), atol=1e-12)
