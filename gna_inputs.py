"""Seeded synthetic inputs and the named workloads (BASELINE.json configs).

Shared by the tests, bench.py and smoke(): it holds NO GNA arithmetic, only
shapes and random numbers, so the oracle and the CUDA path can both consume
the same bf16 values without sharing any of the method's code.

Recipe: q, k, v i.i.d. N(0,1) drawn in fp32 from
``torch.Generator('cpu').manual_seed(16922 + t)`` (t = 0, 1, 2 for q, k, v),
then rounded to nearest-even bf16.  The "discriminating" set multiplies q by
3 and draws v ~ U(-1, 1) (seed + 10) so softmax is peaky and a wrong
neighbourhood moves O well past tolerance.  Layout is heads-last
[B, s0, (s1, (s2)), H, D].
"""
from __future__ import annotations

import dataclasses

import numpy as np
import torch

SEED = 16922


@dataclasses.dataclass(frozen=True)
class Workload:
    name: str
    spatial: tuple
    window: tuple
    stride: tuple
    dilation: tuple = None
    causal: tuple = None
    batch: int = 1
    heads: int = 1
    head_dim: int = 128
    note: str = ""

    def full(self):
        n = len(self.spatial)
        return dict(spatial=tuple(self.spatial), window=tuple(self.window), stride=tuple(self.stride),
                    dilation=tuple(self.dilation or (1,) * n),
                    causal=tuple(bool(c) for c in (self.causal or (False,) * n)))

    @property
    def n_tokens(self):
        return int(np.prod(self.spatial))


# BASELINE.json configs.  B=1 unless stated.
WORKLOADS = {w.name: w for w in [
    Workload("c1_tiny1d", (256,), (32,), (8,), heads=1, head_dim=32,
             note="configs[0]: 1-D tiny, D=32, fp32 inputs rounded once to bf16"),
    Workload("c2a_flux64_s8", (64, 64), (32, 32), (8, 8), heads=24,
             note="configs[1]: FLUX-like 64x64, stride 8x8"),
    Workload("c2b_flux64_s16", (64, 64), (32, 32), (16, 16), heads=24,
             note="configs[1]: FLUX-like 64x64, stride 16x16 (perfectly block-sparse)"),
    Workload("c3_cosmos", (16, 44, 80), (16, 32, 48), (1, 8, 16), heads=32,
             note="configs[2]: Cosmos-7B-like video (perfectly block-sparse)"),
    Workload("c4a_hunyuan_blocked", (30, 48, 80), (18, 24, 24), (18, 24, 24), heads=24,
             note="configs[3]: HunyuanVideo-like, stride = window (blocked)"),
    Workload("c4b_hunyuan_na", (30, 48, 80), (18, 24, 24), (1, 1, 1), heads=24,
             note="configs[3]: HunyuanVideo-like, stride 1 (pure NA)"),
    Workload("x1_hunyuan_s16", (30, 48, 80), (18, 24, 24), (16, 8, 8), heads=24,
             note="paper headline (Fig.4, P:383-384), perfectly block-sparse"),
    Workload("x2_flux4k", (256, 256), (80, 80), (16, 16), heads=24,
             note="paper FLUX 4K shape (P:986-989)"),
    Workload("x3_cosmos89", (16, 44, 80), (16, 24, 16), (1, 8, 16), heads=32,
             note="paper Cosmos-7B 89% sparsity shape (Fig.5 P:519, Tab.2 P:674-717), perfectly block-sparse"),
    Workload("s1_sweep1d", (8192,), (1024,), (1,), dilation=(2,), causal=(True,), batch=8, heads=16,
             note="configs[4] sweep 1-D, dilation 2, causal"),
    Workload("s2_sweep2d", (128, 128), (32, 32), (8, 8), dilation=(2, 2), batch=8, heads=16,
             note="configs[4] sweep 2-D, dilation 2"),
    Workload("s2c_sweep2d_causal", (128, 128), (32, 32), (8, 8), dilation=(2, 2), causal=(True, False),
             batch=8, heads=16, note="configs[4] sweep 2-D, dilation 2, causal axis 0"),
    Workload("s3_sweep3d", (16, 64, 64), (8, 16, 16), (2, 8, 8), dilation=(1, 2, 2),
             causal=(True, False, False), batch=8, heads=16,
             note="configs[4] sweep 3-D, dilation (1,2,2), causal axis 0"),
]}


def _normal(shape, seed):
    g = torch.Generator("cpu").manual_seed(seed)
    return torch.randn(shape, generator=g, dtype=torch.float32)


def _uniform(shape, seed):
    g = torch.Generator("cpu").manual_seed(seed)
    return torch.rand(shape, generator=g, dtype=torch.float32) * 2.0 - 1.0


def make_qkv(batch, spatial, heads, head_dim, discriminating=False, seed=SEED,
             dtype=torch.bfloat16):
    """Host (CPU) q, k, v in `dtype`, heads-last [B, *spatial, H, D]."""
    shape = (batch, *spatial, heads, head_dim)
    # each tensor is drawn from its own seeded generator and cast right away (same values as
    # drawing all three first; peak host memory is one fp32 tensor)
    if not discriminating:
        q = _normal(shape, seed + 0).to(dtype)
        k = _normal(shape, seed + 1).to(dtype)
        v = _normal(shape, seed + 2).to(dtype)
    else:
        q = (_normal(shape, seed + 10) * 3.0).to(dtype)
        k = _normal(shape, seed + 11).to(dtype)
        v = _uniform(shape, seed + 12).to(dtype)
    return q, k, v


def as_f32_numpy(t: torch.Tensor) -> np.ndarray:
    """Exact promotion of bf16/fp16 values to float32 numpy (for the oracle)."""
    return t.detach().to("cpu").to(torch.float32).contiguous().numpy()


def sample_rows(batch, spatial, heads, n_uniform, seed=SEED + 99, extra_tokens=()):
    """int64 [R, 3] rows (b, token, h) for sampled parity / cpu baseline:
    `n_uniform` uniform rows plus every head of each token in extra_tokens."""
    N = int(np.prod(spatial))
    rng = np.random.default_rng(seed)
    rows = np.stack([rng.integers(0, batch, n_uniform), rng.integers(0, N, n_uniform),
                     rng.integers(0, heads, n_uniform)], axis=1)
    ext = [(b, t, h) for t in extra_tokens for b in range(batch) for h in range(heads)]
    if ext:
        rows = np.concatenate([rows, np.asarray(ext, dtype=np.int64)], axis=0)
    return np.ascontiguousarray(rows, dtype=np.int64)


def quantize_e4m3(t: torch.Tensor):
    """Per-tensor E4M3 quantisation of an input tensor (SURVEY NEXT-3 inputs): scale =
    amax / 448 (E4M3's largest finite value), values rounded to nearest by torch's cast.
    Returns (e4m3 tensor, scale, dequantised fp32 tensor = e4m3 * scale) -- the exact values
    the FP8 kernel consumes, which is what the oracle is run on."""
    x = t.to(torch.float32)
    scale = float(x.abs().max().clamp_min(1e-30)) / 448.0
    t8 = (x / scale).to(torch.float8_e4m3fn)
    return t8, scale, t8.to(torch.float32) * scale
