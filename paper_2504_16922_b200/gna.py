"""ctypes binding of libgna_b200.so (include/gna.h).  Argument marshalling only:
every step of the GNA forward runs in the library's sm_100a kernels; there is
no Python or CPU fallback -- a missing library or device raises.

Names follow the C ABI: forward (gna_forward_ex), permute, attention_permuted,
unpermute, workspace_size, plan_info, debug_windows, debug_visits,
debug_worklist, release_workspace.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("GNA_LIB_PATH") or os.path.join(_HERE, "libgna_b200.so")

GNA_OK, GNA_EINVAL, GNA_EUNSUPPORTED, GNA_ECUDA, GNA_ENOMEM = range(5)
GNA_DTYPE_BF16 = 0
GNA_DTYPE_FP16 = 1
GNA_DTYPE_FP8_E4M3 = 2
GNA_FLAG_SYNC_CHECK = 1
GNA_FLAG_UNFUSED_EPILOGUE = 2
GNA_FLAG_PERMUTED = 4
GNA_FLAG_WORK_RANGE = 8

_I3 = ctypes.c_int * 3


class GnaArgs(ctypes.Structure):
    _fields_ = [
        ("q", ctypes.c_void_p), ("k", ctypes.c_void_p), ("v", ctypes.c_void_p),
        ("out", ctypes.c_void_p), ("lse", ctypes.c_void_p),
        ("batch", ctypes.c_int), ("heads", ctypes.c_int), ("head_dim", ctypes.c_int),
        ("spatial", _I3), ("window", _I3), ("stride", _I3), ("dilation", _I3), ("causal", _I3),
        ("scale", ctypes.c_float), ("dtype", ctypes.c_int),
        ("stream", ctypes.c_void_p), ("workspace", ctypes.c_void_p), ("workspace_bytes", ctypes.c_size_t),
        ("box", _I3), ("work_begin", ctypes.c_longlong), ("work_end", ctypes.c_longlong),
        ("flags", ctypes.c_int),
        ("extra_k", ctypes.c_void_p), ("extra_v", ctypes.c_void_p), ("n_extra", ctypes.c_int),
        ("q_scale", ctypes.c_float), ("k_scale", ctypes.c_float), ("v_scale", ctypes.c_float),
    ]


class GnaPlanInfo(ctypes.Structure):
    _fields_ = [
        ("box", _I3), ("q_sub", _I3), ("box_vol", ctypes.c_int), ("padded_head_dim", ctypes.c_int),
        ("n_classes", ctypes.c_int), ("n_boxes_per_class", ctypes.c_int),
        ("n_items", ctypes.c_longlong), ("n_work", ctypes.c_longlong), ("n_paired", ctypes.c_longlong),
        ("kv_stages_total", ctypes.c_longlong), ("subtile_stages", ctypes.c_longlong),
        ("visited_max", ctypes.c_longlong),
        ("dense_boxes", ctypes.c_longlong), ("bound", ctypes.c_double), ("kept_pairs", ctypes.c_longlong),
        ("workspace_bytes", ctypes.c_size_t),
    ]


EXPORTS = [
    "gna_forward", "gna_forward_ex", "gna_permute", "gna_attention_permuted", "gna_unpermute",
    "gna_workspace_size", "gna_plan_info", "gna_debug_windows", "gna_debug_visits", "gna_debug_worklist",
    "gna_release_workspace", "gna_last_error", "gna_device_supported", "gna_version",
    "gna_sim", "gna_sim_sweep", "gna_sim_e2e",
]

_lib = None


class GnaError(RuntimeError):
    pass


def load():
    """Load the in-tree library; raises if it is missing (no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise GnaError(f"{LIB_PATH} missing: run __graft_entry__.build() (there is no CPU fallback)")
        lib = ctypes.CDLL(LIB_PATH)
        pa = ctypes.POINTER(GnaArgs)
        for name in ("gna_forward_ex", "gna_permute", "gna_attention_permuted", "gna_unpermute"):
            getattr(lib, name).argtypes = [pa]
            getattr(lib, name).restype = ctypes.c_int
        lib.gna_workspace_size.argtypes = [pa, ctypes.POINTER(ctypes.c_size_t)]
        lib.gna_plan_info.argtypes = [pa, ctypes.POINTER(GnaPlanInfo)]
        lib.gna_debug_windows.argtypes = [pa, ctypes.c_void_p]
        lib.gna_debug_visits.argtypes = [pa, ctypes.c_void_p, ctypes.POINTER(ctypes.c_longlong)]
        lib.gna_debug_worklist.argtypes = [pa, ctypes.c_void_p, ctypes.POINTER(ctypes.c_longlong)]
        lib.gna_last_error.restype = ctypes.c_char_p
        lib.gna_version.restype = ctypes.c_char_p
        _lib = lib
    return _lib


def _check(rc):
    if rc != GNA_OK:
        raise GnaError(f"gna error {rc}: {load().gna_last_error().decode()}")


def _pad3(x, fill):
    x = list(x)
    return x + [fill] * (3 - len(x))


def make_args(batch, heads, head_dim, spatial, window, stride=None, dilation=None, causal=None,
              scale=0.0, q=None, k=None, v=None, out=None, lse=None, stream=None, box=None,
              work_range=None, workspace=None, workspace_bytes=0, flags=0, extra_k=None, extra_v=None,
              n_extra=0, dtype=GNA_DTYPE_BF16, scales=(0.0, 0.0, 0.0)) -> GnaArgs:
    n = len(spatial)
    a = GnaArgs()
    a.q, a.k, a.v, a.out, a.lse = q, k, v, out, lse
    a.batch, a.heads, a.head_dim = int(batch), int(heads), int(head_dim)
    a.spatial = _I3(*_pad3(spatial, 1))
    a.window = _I3(*_pad3(window, 1))
    a.stride = _I3(*_pad3(stride if stride is not None else [1] * n, 1))
    a.dilation = _I3(*_pad3(dilation if dilation is not None else [1] * n, 1))
    a.causal = _I3(*[int(bool(c)) for c in _pad3(causal if causal is not None else [0] * n, 0)])
    a.scale = float(scale or 0.0)
    a.dtype = int(dtype)
    a.q_scale, a.k_scale, a.v_scale = (float(x) for x in scales)
    a.stream = stream
    a.workspace = workspace
    a.workspace_bytes = int(workspace_bytes)
    a.box = _I3(*(_pad3(box, 1) if box else [0, 0, 0]))
    a.work_begin, a.work_end = (work_range if work_range is not None else (0, 0))
    # an explicit range is taken literally (an empty share launches nothing)
    a.flags = int(flags) | (GNA_FLAG_WORK_RANGE if work_range is not None else 0)
    a.extra_k, a.extra_v, a.n_extra = extra_k, extra_v, int(n_extra)
    return a


def _tensor_args(q, k, v, out, lse, window, stride, dilation, causal, scale, box, work_range, stream, flags,
                 workspace=None, extra_k=None, extra_v=None, scales=None):
    import torch

    fp8 = q.dtype == torch.float8_e4m3fn
    fp16 = q.dtype == torch.float16
    t16 = torch.float16 if fp16 else torch.bfloat16  # O (and extra K/V) dtype
    for name, t in (("q", q), ("k", k), ("v", v), ("out", out)):
        if not t.is_cuda:
            raise GnaError(f"{name} must be a CUDA tensor (no CPU fallback)")
        want = torch.float8_e4m3fn if (fp8 and name != "out") else t16
        if t.dtype != want:
            raise GnaError(f"{name} must be {want} (q, k, v, out all bfloat16 or all float16, or q, k, v "
                           f"float8_e4m3fn with a bfloat16 out)")
        if not t.is_contiguous():
            raise GnaError(f"{name} must be contiguous")
    if lse is not None and (lse.dtype != torch.float32 or not lse.is_contiguous() or not lse.is_cuda):
        raise GnaError("lse must be a contiguous CUDA float32 tensor")
    # the kernels index k, v, out and lse with q's geometry: any mismatch would read or write
    # out of bounds, so it is rejected here (nothing is launched)
    if not 4 <= q.dim() <= 6:
        raise GnaError("q must be [B, *spatial (1-3 axes), H, D]")
    for name, t in (("k", k), ("v", v), ("out", out)):
        if tuple(t.shape) != tuple(q.shape):
            raise GnaError(f"{name} shape {tuple(t.shape)} != q shape {tuple(q.shape)}")
    if lse is not None and tuple(lse.shape) != tuple(q.shape[:-1]):
        raise GnaError(f"lse shape {tuple(lse.shape)} != {tuple(q.shape[:-1])}")
    devs = {t.device for t in (q, k, v, out) + ((lse,) if lse is not None else ())}
    if len(devs) != 1:
        raise GnaError(f"all tensors must be on one CUDA device, got {sorted(map(str, devs))}")
    batch, heads, head_dim = q.shape[0], q.shape[-2], q.shape[-1]
    spatial = list(q.shape[1:-2])
    if stream is None:
        stream = torch.cuda.current_stream(q.device).cuda_stream
    ws_ptr, ws_bytes = None, 0
    if workspace is not None:
        if not workspace.is_cuda or not workspace.is_contiguous():
            raise GnaError("workspace must be a contiguous CUDA tensor")
        ws_ptr, ws_bytes = workspace.data_ptr(), workspace.numel() * workspace.element_size()
    ek = ev = None
    n_extra = 0
    if extra_k is not None:
        for name, t in (("extra_k", extra_k), ("extra_v", extra_v)):
            want = torch.float8_e4m3fn if fp8 else t16
            if t is None or not t.is_cuda or t.dtype != want or not t.is_contiguous():
                raise GnaError(f"{name} must be a contiguous CUDA {want} tensor [B, T, H, D]")
        if extra_k.shape != extra_v.shape or extra_k.dim() != 4 or extra_k.shape[0] != batch or \
                tuple(extra_k.shape[2:]) != (heads, head_dim):
            raise GnaError("extra_k/extra_v must be [B, T, H, D] matching q")
        if extra_k.device != q.device or extra_v.device != q.device:
            raise GnaError("extra_k/extra_v must be on q's device")
        ek, ev, n_extra = extra_k.data_ptr(), extra_v.data_ptr(), extra_k.shape[1]
    return make_args(batch, heads, head_dim, spatial, window, stride, dilation, causal, scale,
                     q=q.data_ptr(), k=k.data_ptr(), v=v.data_ptr(), out=out.data_ptr(),
                     lse=(lse.data_ptr() if lse is not None else None), stream=stream, box=box,
                     work_range=work_range, flags=flags, workspace=ws_ptr, workspace_bytes=ws_bytes,
                     extra_k=ek, extra_v=ev, n_extra=n_extra,
                     dtype=GNA_DTYPE_FP8_E4M3 if fp8 else (GNA_DTYPE_FP16 if fp16 else GNA_DTYPE_BF16),
                     scales=tuple(scales) if scales is not None else (0.0, 0.0, 0.0))


def forward(q, k, v, window, stride=None, dilation=None, causal=None, scale=None, out=None, lse=None,
            box=None, work_range=None, stream=None, return_lse=True, flags=0, workspace=None, extra_k=None,
            extra_v=None, scales=None):
    """GNA forward on CUDA bf16 (or fp16) tensors [B, *spatial, H, D] (heads-last); optional extra
    (text) keys/values [B, T, H, D] attended densely by every query.  q, k, v may instead be
    torch.float8_e4m3fn with per-tensor dequantisation scales=(q_scale, k_scale, v_scale)
    (GNA_DTYPE_FP8_E4M3, head_dim 128); out stays bfloat16.

    Returns (out, lse) -- lse fp32 [B, *spatial, H] (natural log)."""
    import torch

    if out is None:
        out = torch.empty(q.shape, dtype=torch.float16 if q.dtype == torch.float16 else torch.bfloat16,
                          device=q.device)
    if lse is None and return_lse:
        lse = torch.empty(q.shape[:-1], dtype=torch.float32, device=q.device)
    a = _tensor_args(q, k, v, out, lse, window, stride, dilation, causal, scale, box, work_range, stream, flags,
                     workspace, extra_k, extra_v, scales)
    with torch.cuda.device(q.device):
        _check(load().gna_forward_ex(ctypes.byref(a)))
    return out, lse


def _stage(fn_name, q, k, v, out, lse, window, stride, dilation, causal, scale, box, stream, flags,
           workspace=None, work_range=None, extra_k=None, extra_v=None):
    import torch

    a = _tensor_args(q, k, v, out, lse, window, stride, dilation, causal, scale, box, work_range, stream, flags,
                     workspace, extra_k, extra_v)
    with torch.cuda.device(q.device):
        _check(getattr(load(), fn_name)(ctypes.byref(a)))


def permute(q, k, v, out, window, stride=None, dilation=None, causal=None, box=None, stream=None, workspace=None):
    _stage("gna_permute", q, k, v, out, None, window, stride, dilation, causal, None, box, stream, 0, workspace)


def attention_permuted(q, k, v, out, window, stride=None, dilation=None, causal=None, scale=None, box=None,
                       stream=None, workspace=None, work_range=None, extra_k=None, extra_v=None):
    _stage("gna_attention_permuted", q, k, v, out, None, window, stride, dilation, causal, scale, box, stream, 0,
           workspace, work_range, extra_k, extra_v)


def unpermute(q, k, v, out, lse, window, stride=None, dilation=None, causal=None, box=None, stream=None,
              workspace=None):
    _stage("gna_unpermute", q, k, v, out, lse, window, stride, dilation, causal, None, box, stream, 0, workspace)


def plan_info(batch, heads, head_dim, spatial, window, stride=None, dilation=None, causal=None, box=None,
              n_extra=0) -> dict:
    a = make_args(batch, heads, head_dim, spatial, window, stride, dilation, causal, box=box, n_extra=n_extra)
    info = GnaPlanInfo()
    _check(load().gna_plan_info(ctypes.byref(a), ctypes.byref(info)))
    d = {f: getattr(info, f) for f, _ in GnaPlanInfo._fields_}
    for key in ("box", "q_sub"):
        d[key] = list(d[key])
    return d


def workspace_size(batch, heads, head_dim, spatial, window, stride=None, dilation=None, causal=None, box=None):
    a = make_args(batch, heads, head_dim, spatial, window, stride, dilation, causal, box=box)
    n = ctypes.c_size_t()
    _check(load().gna_workspace_size(ctypes.byref(a), ctypes.byref(n)))
    return n.value


def debug_windows(spatial, window, stride=None, dilation=None, causal=None, head_dim=128):
    """int32 [N, 3, 3] per token, per axis {class, start, end} computed on the GPU."""
    a = make_args(1, 1, head_dim, spatial, window, stride, dilation, causal)
    n = int(np.prod(spatial))
    out = np.zeros((n, 3, 3), dtype=np.int32)
    _check(load().gna_debug_windows(ctypes.byref(a), out.ctypes.data_as(ctypes.c_void_p)))
    return out


def debug_visits(spatial, window, stride=None, dilation=None, causal=None, box=None, head_dim=128):
    """int32 [n_classes * n_sub, 10] = {class, sub, lo0,hi0, lo1,hi1, lo2,hi2, n_full, nonempty}."""
    a = make_args(1, 1, head_dim, spatial, window, stride, dilation, causal, box=box)
    n = ctypes.c_longlong()
    _check(load().gna_debug_visits(ctypes.byref(a), None, ctypes.byref(n)))
    out = np.zeros((n.value, 10), dtype=np.int32)
    _check(load().gna_debug_visits(ctypes.byref(a), out.ctypes.data_as(ctypes.c_void_p), ctypes.byref(n)))
    return out


def debug_worklist(spatial, window, stride=None, dilation=None, causal=None, box=None, head_dim=128):
    a = make_args(1, 1, head_dim, spatial, window, stride, dilation, causal, box=box)
    n = ctypes.c_longlong()
    _check(load().gna_debug_worklist(ctypes.byref(a), None, ctypes.byref(n)))
    out = np.zeros((n.value, 4), dtype=np.int32)
    _check(load().gna_debug_worklist(ctypes.byref(a), out.ctypes.data_as(ctypes.c_void_p), ctypes.byref(n)))
    return out


def release_workspace():
    _check(load().gna_release_workspace())


def device_supported() -> bool:
    return bool(load().gna_device_supported())


def version() -> str:
    return load().gna_version().decode()
