"""Pins for the oracle's neighbourhood definition (§2.1, §3.1).

Each test checks the oracle against something other than its own formula:
paper-printed examples, characterisations stated in words by the paper,
brute force, or closed forms.
"""
import itertools
import json
import os

import numpy as np
import pytest

import oracle as O

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_values.json")))


def test_window_split_even_w8():
    """P:414-416 §3.1: w=8 -> 4 left, self, 3 right for a non-corner token."""
    g = GOLD["window_split_w8"]
    for L in (10, 16, 33):
        for i in range(g["w"], L - g["w"]):
            _, st, en = O.axis_window(i, L, g["w"])
            assert en - st == g["w"]
            assert i - st == g["left"] and en - 1 - i == g["right"]


def test_window_odd_is_centered():
    """NA is defined on odd windows with the query perfectly centered."""
    for w in (3, 5, 7, 9):
        for i in range(w, 30 - w):
            _, st, en = O.axis_window(i, 30, w)
            assert i - st == en - 1 - i == w // 2


def test_na_is_nearest_centered_interval():
    """P:222-226 §2.1: every query attends exactly w tokens; the window is the
    length-w interval inside the sequence that is as centered on the query as
    possible (shifted inward at borders).  Characterised by argmin, not by the
    clamp formula."""
    for L in (1, 2, 5, 8, 13, 31):
        for w in range(1, L + 1):
            for i in range(L):
                _, st, en = O.axis_window(i, L, w)
                best = min(range(0, L - w + 1), key=lambda t: (abs(t + w // 2 - i), t))
                assert (st, en) == (best, best + w), (L, w, i)


@pytest.mark.parametrize("s", [1, 2, 3, 4, 5, 8])
def test_stride_group_shares_leader_window(s):
    """a stride group attends the neighbourhood of its leader, the
    center-most member (right-biased for even s): member windows equal the
    stride-1 window of query floor(i/s)*s + floor(s/2) (clamped to L-1 for a
    partial last group: the clamped and unclamped choices coincide, R3)."""
    L, w = 29, 9
    if s > w:
        pytest.skip("s <= w only")
    for i in range(L):
        g0 = (i // s) * s
        members = list(range(g0, min(g0 + s, L)))
        if len(members) == s:
            # center-most member; of the two middle members of an even group, the right one
            leader = members[len(members) // 2]
        else:
            leader = min(g0 + s // 2, L - 1)
        assert O.axis_window(i, L, w, s)[1:] == O.axis_window(leader, L, w, 1)[1:]


def test_partial_last_group_irrelevant_noncausal():
    """Reading R3: for non-causal axes the last partial group's window is the same
    whether its leader is clamped to L-1 or is the partial group's own center."""
    for L in range(4, 40):
        for w in range(1, L + 1):
            for s in range(1, w + 1):
                g0 = ((L - 1) // s) * s
                own_center = g0 + (L - g0) // 2
                for i in range(g0, L):
                    assert O.axis_window(i, L, w, s)[1:] == O.axis_window(own_center, L, w, 1)[1:]


def _blocked_mask(L, w):
    idx = np.arange(L)
    return (idx[:, None] // w) == (idx[None, :] // w)


@pytest.mark.parametrize("L,w", [(8, 4), (12, 3), (16, 8), (9, 9)])
def test_stride_equals_window_is_blocked(L, w):
    """P:129-131 Fig.2: stride = window is (fully) blocked attention (WSA)
    when w divides L (reading R10)."""
    m = O.mask(O.Params((L,), (w,), (w,)))
    assert (m == _blocked_mask(L, w)).all()


def test_stride_equals_window_nondividing_overlaps():
    """Reading R10: L=30, w=18, s=18 -> the last block is clamped to [12, 30)."""
    assert O.axis_window(20, 30, 18, 18)[1:] == (12, 30)
    assert O.axis_window(5, 30, 18, 18)[1:] == (0, 18)


@pytest.mark.parametrize("spatial,stride", [((8,), (3,)), ((6, 5), (2, 4)), ((4, 3, 5), (1, 3, 2))])
def test_window_equals_extent_is_self_attention(spatial, stride):
    """P:226 and Fig.2: window = input size is self attention, any stride."""
    m = O.mask(O.Params(spatial, spatial, stride))
    assert m.all()


def test_blocked_2d_product():
    """Blocked attention in 2-D is the product of per-axis blocks (WSA)."""
    p = O.Params((8, 6), (4, 3), (4, 3))
    m = O.mask(p)
    ii = np.array(list(itertools.product(range(8), range(6))))
    ref = ((ii[:, None, 0] // 4) == (ii[None, :, 0] // 4)) & ((ii[:, None, 1] // 3) == (ii[None, :, 1] // 3))
    assert (m == ref).all()


def _grid_cases():
    rng = np.random.default_rng(7)
    cases = []
    for _ in range(60):
        n = int(rng.integers(1, 4))
        spatial, window, stride, dil, causal = [], [], [], [], []
        for _a in range(n):
            L = int(rng.integers(1, 12))
            d = int(rng.integers(1, 3)) if L >= 2 else 1
            w = int(rng.integers(1, L // d + 1))
            s = int(rng.integers(1, w + 1))
            spatial.append(L); window.append(w); stride.append(s); dil.append(d)
            causal.append(bool(rng.integers(0, 2)))
        if np.prod(spatial) <= 600:
            cases.append((tuple(spatial), tuple(window), tuple(stride), tuple(dil), tuple(causal)))
    return cases


@pytest.mark.parametrize("case", _grid_cases())
def test_mask_properties_bruteforce(case):
    """Brute force over every (q, k) pair of tiny grids:
    - enumerated windows (ora_windows) reproduce the pairwise mask,
    - fixed count prod(w) for all-non-causal queries,
    - no holes for s <= w: every key is attended by some query,
    - monotone grouping: same leader tuple -> identical rows,
    - queries attend only keys of their own dilation class,
    - causal axes never attend the future and always attend self (R4)."""
    spatial, window, stride, dil, causal = case
    p = O.Params(spatial, window, stride, dil, causal)
    m = O.mask(p)
    n = p.n_tokens
    win = O.windows(p)
    L = p.spatial
    coords = np.array(list(itertools.product(range(L[0]), range(L[1]), range(L[2]))))
    # windows -> mask
    for qi in range(n):
        ok = np.ones(n, dtype=bool)
        for a in range(3):
            c, st, en = win[qi, a]
            kc = coords[:, a]
            j = kc // p.dilation[a]
            ok &= (kc % p.dilation[a] == c) & (j >= st) & (j < en)
        assert (ok == m[qi]).all()
    cnt = m.sum(1)
    if not any(p.causal):
        assert (cnt == np.prod(p.window)).all()
    assert m.any(0).all(), "holes"
    for a in range(3):
        same_cls = (coords[:, None, a] % p.dilation[a]) == (coords[None, :, a] % p.dilation[a])
        assert not (m & ~same_cls).any()
        if p.causal[a]:
            assert not (m & (coords[None, :, a] > coords[:, None, a])).any()
    assert m[np.arange(n), np.arange(n)].all(), "self not attended"
    # monotone grouping on non-causal axes
    if not any(p.causal):
        key = []
        for qi in range(n):
            kk = []
            for a in range(3):
                i = coords[qi, a]
                d, s = p.dilation[a], p.stride[a]
                kk.append((i % d, (i // d) // s))
            key.append(tuple(kk))
        groups = {}
        for qi, kk in enumerate(key):
            groups.setdefault(kk, []).append(qi)
        for members in groups.values():
            for qi in members[1:]:
                assert (m[qi] == m[members[0]]).all()


def test_count_pairs_separable_closed_form():
    """Kept pairs = prod_a sum_i count_a(i) (the mask is a product over axes);
    SURVEY App.A vectors: 15390, 1600, 40 (re-derived by brute force here too)."""
    cases = [
        (((6, 7, 9), (3, 4, 5), (2, 3, 5), (1, 1, 1), (False, True, False)), 15390),
        (((12, 10), (5, 4), (5, 2), (2, 2), (True, False)), 1600),
        (((16,), (4,), (4,), (1,), (True,)), 40),
    ]
    for args, expect in cases:
        p = O.Params(*args)
        tot, _ = O.count_pairs(p)
        assert tot == expect
        per_axis = []
        for a in range(3):
            per_axis.append(sum(en - st for (_, st, en) in
                                (O.axis_window(i, p.spatial[a], p.window[a], p.stride[a],
                                               p.dilation[a], p.causal[a]) for i in range(p.spatial[a]))))
        assert np.prod(per_axis) == tot
        if p.n_tokens <= 4096:
            assert O.mask(p).sum() == tot


def test_causal_stride1_is_sliding_window():
    """Reading R4 limit (i): s=1 causal = textbook causal sliding window [i-w+1, i]."""
    for L in (5, 9, 16):
        for w in range(1, L + 1):
            m = O.mask(O.Params((L,), (w,), (1,), causal=(True,)))
            i = np.arange(L)
            ref = (i[None, :] <= i[:, None]) & (i[None, :] >= i[:, None] - w + 1)
            assert (m == ref).all()


def test_causal_stride_window_is_block_causal():
    """Reading R4 limit (ii): s=w (w | L) causal = block-causal attention."""
    for L, w in ((8, 4), (12, 3), (16, 16)):
        m = O.mask(O.Params((L,), (w,), (w,), causal=(True,)))
        i = np.arange(L)
        ref = ((i[:, None] // w) == (i[None, :] // w)) & (i[None, :] <= i[:, None])
        assert (m == ref).all()


def test_sparsity_values_printed_in_paper():
    """P:377 (~91%), P:903 (~56.4%), P:986 (90.2%) and the x10.2 FLUX op-level
    FLOP-wise speedup, from the closed-form pair counts."""
    g = GOLD["sparsity"]
    for c in g["cases"]:
        p = O.Params(c["spatial"], c["window"], [1] * len(c["spatial"]))
        n = p.n_tokens
        kept = int(np.prod(p.window)) * n   # fixed count per query
        tot, _ = O.count_pairs(p)
        assert tot == kept
        pct = 100.0 * (1 - kept / (n * n))
        assert abs(pct - c["pct_1dp"]) <= c["tol"], (c, pct)
    p = O.Params((256, 256), (80, 80), (16, 16))
    assert round((256 * 256) / (80 * 80), 1) == g["flux_flopwise_1dp"]
