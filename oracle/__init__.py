"""fp64 CPU oracle for the GNA forward (arXiv 2504.16922).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  It shares no code with the CUDA product path
(``paper_2504_16922_b200``) and never imports it.

The arithmetic lives in ``gna_oracle.c`` (plain C, fp64, OpenMP over rows);
this module only marshals numpy arrays through ctypes.  Each wrapper names
the PAPER.md passage its C function follows (see the C file header).

Parity pins: every function here is pinned by ``tests/test_oracle_*.py``
against paper-printed values (Fig.4, Tab.3, Tab.4, P:414-416 window split),
closed forms, library routines on special cases (dense SDPA, blocked SDPA,
causal sliding window) and brute force on tiny grids.  The causal+stride
reading (R4) for s >= 3 is "parity unpinned" by the paper: it is
pinned only by its two limits (s=1 causal sliding window, s=w block-causal).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "gna_oracle.c")
_LIB = os.path.join(_HERE, "libgna_oracle.so")
_lock = threading.Lock()
_lib = None


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (-O2 -fopenmp, fp64, no fast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=c11",
                               "-fno-fast-math", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    with _lock:
        if _lib is None:
            build()
            lib = ctypes.CDLL(_LIB)
            lp = ctypes.POINTER(ctypes.c_long)
            ip = ctypes.POINTER(ctypes.c_int)
            vp = ctypes.c_void_p
            lib.ora_axis_window.argtypes = [ctypes.c_long] * 5 + [ctypes.c_int, lp, lp, lp]
            lib.ora_windows.argtypes = [lp, lp, lp, lp, ip, vp]
            lib.ora_is_attended.argtypes = [lp, lp, lp, lp, lp, lp, ip]
            lib.ora_is_attended.restype = ctypes.c_int
            lib.ora_mask.argtypes = [lp, lp, lp, lp, ip, vp]
            lib.ora_count_pairs.argtypes = [lp, lp, lp, lp, ip, vp]
            lib.ora_count_pairs.restype = ctypes.c_longlong
            lib.ora_forward.argtypes = [vp, vp, vp, vp, vp, ctypes.c_long, vp, vp, ctypes.c_long,
                                        ctypes.c_long, ctypes.c_long, lp, lp, lp, lp, ip, ctypes.c_double]
            lib.ora_forward.restype = ctypes.c_longlong
            lib.ora_forward_rows.argtypes = [vp, vp, vp, vp, vp, ctypes.c_long, vp, ctypes.c_long,
                                             vp, vp, ctypes.c_long, ctypes.c_long, ctypes.c_long,
                                             lp, lp, lp, lp, ip, ctypes.c_double]
            lib.ora_forward_rows.restype = ctypes.c_longlong
            lib.ora_num_threads.restype = ctypes.c_int
            lib.ora_visits_bruteforce.argtypes = [lp, lp, lp, lp, ip, lp, lp, ctypes.c_long, vp]
            lib.ora_full_bruteforce.argtypes = [lp, lp, lp, lp, ip, lp, lp, ctypes.c_long, vp, vp]
            lib.ora_sim.argtypes = [lp, lp, lp, ip, lp, lp, vp]
            _lib = lib
    return _lib


def _l3(x, fill=1):
    x = list(x) + [fill] * (3 - len(x))
    return (ctypes.c_long * 3)(*[int(v) for v in x])


def _i3(x):
    x = [int(bool(v)) for v in x] + [0] * (3 - len(x))
    return (ctypes.c_int * 3)(*x)


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


class Params:
    """GNA parameters over a 1-3 axis layout; unused axes are trivial."""

    def __init__(self, spatial, window, stride=None, dilation=None, causal=None):
        n = len(spatial)
        self.spatial = list(spatial) + [1] * (3 - n)
        self.window = list(window) + [1] * (3 - n)
        self.stride = (list(stride) if stride is not None else [1] * n) + [1] * (3 - n)
        self.dilation = (list(dilation) if dilation is not None else [1] * n) + [1] * (3 - n)
        self.causal = [bool(c) for c in (causal if causal is not None else [False] * n)] + [False] * (3 - n)

    @property
    def n_tokens(self) -> int:
        return int(np.prod(self.spatial))

    def c(self):
        return (_l3(self.spatial), _l3(self.window), _l3(self.stride), _l3(self.dilation),
                _i3(self.causal))


def axis_window(i, L, w, s=1, d=1, causal=False):
    """(class, start, end) of query coordinate i on one axis (class-local sub-indices)."""
    lib = _load()
    c, st, en = ctypes.c_long(), ctypes.c_long(), ctypes.c_long()
    lib.ora_axis_window(i, L, w, s, d, int(causal), ctypes.byref(c), ctypes.byref(st),
                        ctypes.byref(en))
    return c.value, st.value, en.value


def windows(p: Params) -> np.ndarray:
    """int32 [N, 3, 3]: per token, per axis {class, start, end}."""
    out = np.zeros((p.n_tokens, 3, 3), dtype=np.int32)
    _load().ora_windows(*p.c(), _ptr(out))
    return out


def is_attended(p: Params, q, kv) -> bool:
    L, w, s, d, c = p.c()
    return bool(_load().ora_is_attended(_l3(q, 0), _l3(kv, 0), L, w, s, d, c))


def mask(p: Params) -> np.ndarray:
    """Dense bool [N, N] mask, pair by pair from is_attended (tiny grids only)."""
    n = p.n_tokens
    if n > 8192:
        raise ValueError("mask(): grid too large for a dense mask")
    m = np.zeros((n, n), dtype=np.uint8)
    _load().ora_mask(*p.c(), _ptr(m))
    return m.astype(bool)


def count_pairs(p: Params):
    """(total attended pairs, int32 per-query neighbourhood sizes)."""
    per = np.zeros(p.n_tokens, dtype=np.int32)
    tot = _load().ora_count_pairs(*p.c(), _ptr(per))
    return int(tot), per


def _extra(extra_k, extra_v, q):
    if extra_k is None:
        return None, None, 0, None
    ek = np.ascontiguousarray(extra_k, dtype=np.float32)
    ev = np.ascontiguousarray(extra_v, dtype=np.float32)
    assert ek.shape == ev.shape and ek.shape[0] == q.shape[0] and ek.shape[2:] == q.shape[-2:]
    return ek, ev, ek.shape[1], (ek, ev)


def forward(q: np.ndarray, k: np.ndarray, v: np.ndarray, p: Params, scale=None, extra_k=None, extra_v=None):
    """fp64 GNA forward. q,k,v: float32 [B, *spatial, H, D] (bf16-exact values);
    optional extra (text) keys/values [B, T, H, D] attended by every query.

    Returns (out float64 [B,*spatial,H,D], lse float64 [B,*spatial,H])."""
    B, H, D = q.shape[0], q.shape[-2], q.shape[-1]
    q = np.ascontiguousarray(q, dtype=np.float32)
    k = np.ascontiguousarray(k, dtype=np.float32)
    v = np.ascontiguousarray(v, dtype=np.float32)
    ek, ev, T, _keep = _extra(extra_k, extra_v, q)
    if scale is None or scale <= 0:
        scale = 1.0 / np.sqrt(D)
    out = np.zeros(q.shape, dtype=np.float64)
    lse = np.zeros(q.shape[:-1], dtype=np.float64)
    _load().ora_forward(_ptr(q), _ptr(k), _ptr(v), _ptr(ek) if T else None, _ptr(ev) if T else None, T,
                        _ptr(out), _ptr(lse), B, H, D, *p.c(), float(scale))
    return out, lse


def forward_rows(q, k, v, p: Params, rows: np.ndarray, scale=None, extra_k=None, extra_v=None):
    """fp64 forward of selected rows. rows: int64 [R, 3] = (b, token index, h)."""
    B, H, D = q.shape[0], q.shape[-2], q.shape[-1]
    q = np.ascontiguousarray(q, dtype=np.float32)
    k = np.ascontiguousarray(k, dtype=np.float32)
    v = np.ascontiguousarray(v, dtype=np.float32)
    ek, ev, T, _keep = _extra(extra_k, extra_v, q)
    rows = np.ascontiguousarray(rows, dtype=np.int64)
    if scale is None or scale <= 0:
        scale = 1.0 / np.sqrt(D)
    out = np.zeros((rows.shape[0], D), dtype=np.float64)
    lse = np.zeros(rows.shape[0], dtype=np.float64)
    pairs = _load().ora_forward_rows(_ptr(q), _ptr(k), _ptr(v), _ptr(ek) if T else None,
                                     _ptr(ev) if T else None, T, _ptr(rows), rows.shape[0],
                                     _ptr(out), _ptr(lse), B, H, D, *p.c(), float(scale))
    return out, lse, int(pairs)


def num_threads() -> int:
    return int(_load().ora_num_threads())


def class_extents(p: Params, cls):
    c = [cls // (p.dilation[1] * p.dilation[2]), (cls // p.dilation[2]) % p.dilation[1],
         cls % p.dilation[2]]
    return [-(-(p.spatial[a] - c[a]) // p.dilation[a]) for a in range(3)]


def visits_bruteforce(p: Params, tq, tk, cls=0) -> np.ndarray:
    """uint8 [nQtiles, nKVtiles] visited matrix for dilation class `cls`."""
    tq = list(tq) + [1] * (3 - len(tq))
    tk = list(tk) + [1] * (3 - len(tk))
    Lc = class_extents(p, cls)
    nq = int(np.prod([-(-Lc[a] // tq[a]) for a in range(3)]))
    nk = int(np.prod([-(-Lc[a] // tk[a]) for a in range(3)]))
    vis = np.zeros((nq, nk), dtype=np.uint8)
    _load().ora_visits_bruteforce(*p.c(), _l3(tq), _l3(tk), cls, _ptr(vis))
    return vis


def full_bruteforce(p: Params, tq, tk, visited: np.ndarray, cls=0) -> np.ndarray:
    tq = list(tq) + [1] * (3 - len(tq))
    tk = list(tk) + [1] * (3 - len(tk))
    visited = np.ascontiguousarray(visited, dtype=np.uint8)
    full = np.zeros_like(visited)
    _load().ora_full_bruteforce(*p.c(), _l3(tq), _l3(tk), cls, _ptr(visited), _ptr(full))
    return full


def sim(p: Params, tq, tk) -> dict:
    """NATTENSim (static multi-D KV tiling, dilation 1)."""
    if any(d != 1 for d in p.dilation):
        raise ValueError("sim(): dilation must be 1")
    tq = list(tq) + [1] * (3 - len(tq))
    tk = list(tk) + [1] * (3 - len(tk))
    rep = np.zeros(5, dtype=np.int64)
    L, w, s, _d, c = p.c()
    _load().ora_sim(L, w, s, c, _l3(tq), _l3(tk), _ptr(rep))
    dense, vmax, vsum, nqt, pbs = (int(x) for x in rep)
    return {"dense_tiles": dense, "visited_max": vmax, "visited_mean": vsum / nqt,
            "bound": dense / vmax, "bound_mean": dense * nqt / vsum,
            "perfectly_block_sparse": bool(pbs)}
