"""NATTENSim (§3.2) through the C ABI: gna_sim, gna_sim_sweep, gna_sim_e2e.

    python -m paper_2504_16922_b200.sim --spatial 30 48 80 --window 18 24 24 --stride 16 8 8 \
        --q-tile 4 8 8 --kv-tile 2 8 8 [--tiling static|dynamic|1d] [--sweep]
"""
from __future__ import annotations

import argparse
import ctypes
import json

from .gna import GnaError, load

_I3 = ctypes.c_int * 3
TILINGS = {"static": 0, "dynamic": 1, "1d": 2}


class SimArgs(ctypes.Structure):
    _fields_ = [("spatial", _I3), ("window", _I3), ("stride", _I3), ("causal", _I3), ("q_tile", _I3),
                ("kv_tile", _I3), ("tiling", ctypes.c_int), ("n_extra", ctypes.c_int)]


class SimReport(ctypes.Structure):
    _fields_ = [("dense_tiles", ctypes.c_longlong), ("visited_max", ctypes.c_longlong),
                ("visited_mean", ctypes.c_double), ("n_q_tiles", ctypes.c_longlong), ("bound", ctypes.c_double),
                ("bound_mean", ctypes.c_double), ("flopwise", ctypes.c_double),
                ("perfectly_block_sparse", ctypes.c_int), ("kept_pairs", ctypes.c_double),
                ("computed_pairs", ctypes.c_double), ("masked_fraction", ctypes.c_double)]


def _pad(x, fill=1):
    x = list(x)
    return _I3(*(x + [fill] * (3 - len(x))))


def _args(spatial, window, stride, q_tile, kv_tile, causal=None, tiling="static", n_extra=0):
    a = SimArgs()
    a.spatial, a.window, a.stride = _pad(spatial), _pad(window), _pad(stride)
    a.causal = _pad([int(bool(c)) for c in (causal or [])], 0)
    a.q_tile, a.kv_tile = _pad(q_tile), _pad(kv_tile)
    a.tiling = TILINGS[tiling]
    a.n_extra = int(n_extra)
    return a


def _lib():
    lib = load()
    if not getattr(lib, "_sim_ready", False):
        lib.gna_sim.argtypes = [ctypes.POINTER(SimArgs), ctypes.POINTER(SimReport)]
        lib.gna_sim_sweep.argtypes = [ctypes.POINTER(SimArgs), ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int,
                                      ctypes.POINTER(ctypes.c_int)]
        lib.gna_sim_e2e.argtypes = [ctypes.c_double, ctypes.c_int, ctypes.c_int, ctypes.c_double]
        lib.gna_sim_e2e.restype = ctypes.c_double
        lib._sim_ready = True
    return lib


def _rep(r: SimReport) -> dict:
    return {f: getattr(r, f) for f, _ in SimReport._fields_}


def simulate(spatial, window, stride, q_tile, kv_tile, causal=None, tiling="static", n_extra=0) -> dict:
    a = _args(spatial, window, stride, q_tile, kv_tile, causal, tiling, n_extra)
    r = SimReport()
    if _lib().gna_sim(ctypes.byref(a), ctypes.byref(r)) != 0:
        raise GnaError("gna_sim: invalid arguments (need 1 <= stride <= window <= extent, tiles >= 1)")
    return _rep(r)


def sweep(spatial, window, q_tile, kv_tile, causal=None, tiling="static", n_extra=0) -> list:
    a = _args(spatial, window, [1, 1, 1], q_tile, kv_tile, causal, tiling, n_extra)
    n = ctypes.c_int()
    lib = _lib()
    if lib.gna_sim_sweep(ctypes.byref(a), None, None, 0, ctypes.byref(n)) != 0:
        raise GnaError("gna_sim_sweep: invalid arguments")
    strides = (ctypes.c_int32 * (3 * n.value))()
    reps = (SimReport * n.value)()
    lib.gna_sim_sweep(ctypes.byref(a), strides, reps, n.value, ctypes.byref(n))
    return [dict(stride=[strides[3 * i], strides[3 * i + 1], strides[3 * i + 2]], **_rep(reps[i]))
            for i in range(n.value)]


def e2e(sa_share, steps, sa_steps, op_speedup) -> float:
    return float(_lib().gna_sim_e2e(sa_share, steps, sa_steps, op_speedup))


def main():
    ap = argparse.ArgumentParser(description=__doc__)
    ap.add_argument("--spatial", type=int, nargs="+", required=True)
    ap.add_argument("--window", type=int, nargs="+", required=True)
    ap.add_argument("--stride", type=int, nargs="+")
    ap.add_argument("--causal", type=int, nargs="+")
    ap.add_argument("--q-tile", type=int, nargs="+", required=True)
    ap.add_argument("--kv-tile", type=int, nargs="+", required=True)
    ap.add_argument("--tiling", default="static", choices=sorted(TILINGS))
    ap.add_argument("--n-extra", type=int, default=0)
    ap.add_argument("--sweep", action="store_true")
    a = ap.parse_args()
    if a.sweep:
        for r in sweep(a.spatial, a.window, a.q_tile, a.kv_tile, a.causal, a.tiling, a.n_extra):
            print(json.dumps({k: r[k] for k in ("stride", "bound", "flopwise", "perfectly_block_sparse")}))
    else:
        print(json.dumps(simulate(a.spatial, a.window, a.stride or [1] * len(a.window), a.q_tile, a.kv_tile,
                                  a.causal, a.tiling, a.n_extra)))


if __name__ == "__main__":
    main()
