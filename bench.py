#!/usr/bin/env python
"""bench.py -- GNA forward on B200: effective TFLOP/s (kept-pair FLOPs only),
speedup over the same kernel run densely, against the NATTENSim bound.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload NAME] [--dtype bf16|fp16|fp8]
                  [--partition auto|heads|batch|qtile] [--impl ours|reference]

A step = one pass of the hot path over one batch of the workload: the fused GNA forward
(analytic tile ranges, tcgen05 mainloop, O+LSE epilogue that scatters straight into the
user layout -- one kernel on the permute-free route), inputs resident in HBM, L2 flushed
(256 MiB write) between timed steps outside the events.  Default workload: the largest
single-GPU BASELINE.json config, C4a (HunyuanVideo-like 30x48x80, 24 heads, blocked).

Multi-GPU (one process per GPU; `--gpus N` spawns torchrun itself when WORLD_SIZE is
unset): strong scaling of ONE problem, partitioned by batch x heads (shard.partition:
heads, else batch, else Q-tile work ranges for single-sample video); no collective on the
data path; times are the max over ranks.  After timing, an NCCL all_gather of the O / LSE
shards feeds a rank-0 check: bit-exact against the 1-GPU launch and sampled rows against
the fp64 oracle.

Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import platform
import socket
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from gna_inputs import SEED, WORKLOADS, make_qkv, sample_rows  # noqa: E402

DEFAULT_WORKLOAD = "c4a_hunyuan_blocked"
METRIC = "GNA fwd effective TFLOP/s (bf16) and speedup vs dense FMHA vs simulator bound"
TRAFFIC_FILE = os.path.join(ROOT, "profiles", "r02_ncu_traffic.json")


def _peaks():
    try:
        mp = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        return mp.get("bf16_tflops", 1590.0), mp.get("bf16_tflops_sustained", 1400.0), mp.get("hbm_gbs", 6650.0), \
            "measured (MEASURED_PEAKS.json)"
    except Exception:
        return 1590.0, 1400.0, 6650.0, "fallback (B200_PROFILING.md)"


def _cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return platform.processor() or "unknown"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 100 ms in the background."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons, pw = [], None, set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            try:
                pw.append(float(f[3]))
            except ValueError:
                pass
            for n, val in zip(names, f[5:9]):
                if val.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm),
                "power_w": statistics.median(pw) if pw else None}


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _spawn_ranks(n):
    """--gpus N without a launcher: re-run this script under torchrun (one rank per GPU)."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def _dist():
    import torch
    import torch.distributed as dist

    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if ws > 1 and not dist.is_initialized():
        if torch.cuda.is_available():
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
    return ws, rank, local


def _max_over_ranks(vals, ws, device):
    """Element-wise max over ranks (device-measured times); identity at N=1."""
    if ws == 1:
        return list(vals)
    import torch
    import torch.distributed as dist

    t = torch.tensor(vals, dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.tolist()


def cpu_oracle_sample(w, budget_s, seed_offset=0, inputs=None):
    """Time the fp64 oracle (as it stands) on a bounded random row sample of the
    workload; returns (TFLOP/s, seconds, rows, cores)."""
    import numpy as np

    import oracle as O
    from gna_inputs import as_f32_numpy

    f = w.full()
    p = O.Params(f["spatial"], f["window"], f["stride"], f["dilation"], f["causal"])
    if inputs is None:
        inputs = make_qkv(w.batch, w.spatial, w.heads, w.head_dim, seed=SEED + seed_offset)
    qn, kn, vn = (t if isinstance(t, np.ndarray) else as_f32_numpy(t) for t in inputs)
    cores = O.num_threads()
    n = max(cores, 8)
    total_pairs, total_t, total_rows = 0, 0.0, 0
    rng_seed = SEED + 7
    while total_t < budget_s:
        rows = sample_rows(w.batch, w.spatial, w.heads, n, seed=rng_seed)
        rng_seed += 1
        t0 = time.perf_counter()
        _, _, pairs = O.forward_rows(qn, kn, vn, p, rows)
        dt = time.perf_counter() - t0
        total_pairs += pairs
        total_t += dt
        total_rows += n
        if dt < budget_s / 8:
            n *= 2
    tflops = 4.0 * w.head_dim * total_pairs / total_t / 1e12
    return tflops, total_t, total_rows, cores


def run_reference(args, ws, rank):
    """--impl reference: the fp64 CPU oracle on the host cores (bounded samples); rank 0 only."""
    if rank != 0:
        return
    w = WORKLOADS[args.workload]
    budget = max(2.0, min(20.0, 150.0 / max(1, args.steps + args.warmup)))
    from gna_inputs import as_f32_numpy

    inputs = tuple(as_f32_numpy(t) for t in make_qkv(w.batch, w.spatial, w.heads, w.head_dim, seed=SEED))
    for _ in range(args.warmup):
        cpu_oracle_sample(w, budget / 4, inputs=inputs)
    vals, secs, rows_tot = [], 0.0, 0
    cores = 1
    for _ in range(args.steps):
        v, t, r, cores = cpu_oracle_sample(w, budget, inputs=inputs)
        vals.append(v)
        secs += t
        rows_tot += r
    value = statistics.mean(vals)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 * secs / max(1, args.steps),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": _config(w, args, 1),
        "cpu_baseline": {"value": value, "unit": "TFLOP/s", "cores": cores, "kind": "oracle",
                         "cpu_model": _cpu_model(),
                         "sample": f"{rows_tot} random (b, token, h) rows of {w.name}, fp64, ~{budget:.0f} s per step"},
        "e2e": {"value": value, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def _config(w, args, ws, shard=None):
    f = w.full()
    c = {"workload": w.name, "spatial": list(w.spatial), "window": list(w.window), "stride": list(w.stride),
         "dilation": list(f["dilation"]), "causal": [int(x) for x in f["causal"]], "heads": w.heads,
         "head_dim": w.head_dim, "global_batch": w.batch,
         "l2": "flushed (256 MiB write) between timed steps; inputs > L2"}
    if shard is not None:
        c["parallelism"] = f"{shard.mode} x{ws}" if ws > 1 else "single GPU"
    return c


def _traffic(workload, dtype, launches_share=1.0):
    """DRAM bytes per launch of the dominant kernel from the committed ncu --set full capture
    (profiles/r02_ncu_traffic.json, written by scripts/ncu_traffic.py for this build)."""
    try:
        d = json.load(open(TRAFFIC_FILE))
        e = d[f"{workload}:{dtype}"]
        return e["dram_bytes_per_launch"] * launches_share, e.get("source")
    except Exception:
        return None, None


def run_nodevice(args, ws, rank):
    """No CUDA device (CPU CI): there is no CPU fallback, so nothing is timed.  The host side
    of the multi-rank path still runs over gloo -- plan, partition, and a check that the
    ranks' shards cover every (unit, work item) exactly once -- and rank 0 reports it."""
    import torch.distributed as dist

    import paper_2504_16922_b200 as gna
    from paper_2504_16922_b200.shard import partition

    w = WORKLOADS[args.workload]
    f = w.full()
    B, H, D = w.batch, w.heads, w.head_dim
    info = gna.plan_info(B, H, D, **f)
    sh = partition(B, H, ws, rank, info["n_items"], args.partition)
    mine = set()
    for u in sh.units(H):
        lo, hi = u * info["n_items"], (u + 1) * info["n_items"]
        if sh.work is not None:
            lo, hi = max(lo, sh.work[0]), min(hi, sh.work[1])
        mine.update(range(lo, hi))
    got = [None] * ws
    if ws > 1:
        dist.all_gather_object(got, (sh.mode, sorted(mine)))
    else:
        got = [(sh.mode, sorted(mine))]
    if rank != 0:
        return
    allw = sorted(x for _, m in got for x in m)
    ok = allw == list(range(info["n_work"]))
    line = {"metric": METRIC, "value": None, "unit": "TFLOP/s", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "higher_is_better": True, "scaling": "strong",
            "unavailable": "no CUDA device on this host: the sm_100a kernels were not run (no CPU fallback)",
            "config": _config(w, args, ws, sh), "partition": {"mode": sh.mode, "n_work": info["n_work"],
                                                              "covers_every_item_once": ok}}
    print(json.dumps(line), flush=True)


def run_ours(args, ws, rank, local):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2504_16922_b200 as gna
    from paper_2504_16922_b200.shard import partition

    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    w = WORKLOADS[args.workload]
    f = w.full()
    B, H, D = w.batch, w.heads, w.head_dim
    win, st, dil, cau = f["window"], f["stride"], f["dilation"], f["causal"]
    fp8, fp16 = args.dtype == "fp8", args.dtype == "fp16"
    info = gna.plan_info(B, H, D, **f)
    sh = partition(B, H, ws, rank, info["n_items"], args.partition)
    eff_flops = 4.0 * D * info["kept_pairs"] * B * H  # the whole problem (all ranks)

    # ---- host inputs (seeded, identical on every rank), this rank's shard pinned
    scales = None
    if fp8:  # E4M3 inputs with per-tensor scales, quantised on the host
        from gna_inputs import quantize_e4m3
        full = make_qkv(B, w.spatial, H, D, seed=SEED, dtype=torch.float32)
        q8 = [quantize_e4m3(t) for t in full]
        del full
        full = tuple(t[0] for t in q8)
        scales = tuple(t[1] for t in q8)
        del q8
    else:
        full = make_qkv(B, w.spatial, H, D, seed=SEED, dtype=torch.float16 if fp16 else torch.bfloat16)

    def take(t):
        if sh.mode == "heads":
            return t[..., sh.heads[0]:sh.heads[1], :].contiguous()
        if sh.mode == "batch":
            return t[sh.batch[0]:sh.batch[1]].contiguous()
        return t

    qh, kh, vh = (take(t).pin_memory() for t in full)
    if rank != 0:
        full = None  # rank 0 keeps the global inputs for the verification
    q, k, v = (t.to(dev) for t in (qh, kh, vh))
    odt = torch.float16 if fp16 else torch.bfloat16
    out = torch.empty(q.shape, dtype=odt, device=dev)
    lse = torch.empty(q.shape[:-1], dtype=torch.float32, device=dev)
    shard_flops = eff_flops * (sh.shard_batch * sh.shard_heads) / (B * H) if sh.work is None else \
        eff_flops * (sh.work[1] - sh.work[0]) / max(1, info["n_work"])
    wr = sh.work
    stream = torch.cuda.current_stream(dev)
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)

    def fwd(o=out, l=lse):
        gna.forward(q, k, v, win, st, dil, cau, out=o, lse=l, scales=scales, work_range=wr)

    def timed(fn, steps):
        ts = []
        for _ in range(steps):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            fn()
            e1.record(stream)
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        return ts

    for _ in range(max(3, args.warmup)):
        fwd()
    torch.cuda.synchronize()
    # The timed step is the gna_forward_ex launch replayed from a CUDA graph (the library call is
    # stream-ordered and host-sync free, so it captures): the ~25 us of Python/ctypes marshalling per
    # call stays out of the device time.  e2e below still goes through the public API every step.
    step_fn, launch_kind = fwd, "gna_forward_ex per step"
    try:
        graph = torch.cuda.CUDAGraph()
        side = torch.cuda.Stream(dev)
        side.wait_stream(stream)
        with torch.cuda.stream(side):
            fwd()
            side.synchronize()
            with torch.cuda.graph(graph, stream=side):
                fwd()
        torch.cuda.synchronize()
        graph.replay()
        torch.cuda.synchronize()
        step_fn, launch_kind = graph.replay, "CUDA graph replay of one gna_forward_ex"
    except Exception as exc:  # capture unsupported: time the direct calls
        print(f"bench: CUDA graph capture failed ({exc}); timing direct calls", file=sys.stderr)

    # ---- timed region: K full steps (value), clocks sampled around it
    with ClockSampler(local) as clk:
        t_soak = time.time()
        while time.time() - t_soak < 0.4:
            fwd()
        torch.cuda.synchronize()
        if ws > 1:
            dist.barrier()
        torch.cuda.synchronize()
        step_ms = timed(step_fn, args.steps)
        torch.cuda.synchronize()
        if ws > 1:
            dist.barrier()
        t_soak = time.time()
        while time.time() - t_soak < 0.3:
            fwd()
        torch.cuda.synchronize()
    total_ms = sum(step_ms)

    # ---- per-stage times of the permuted pipeline (same stream, events between the three
    #      launches), warmed up first; 16-bit types only (E4M3 is permute-free only)
    stage = {"permute": [], "attention": [], "unpermute": []}
    o2 = torch.empty_like(out)
    l2 = torch.empty_like(lse)
    if not fp8:
        for _ in range(2):
            gna.permute(q, k, v, o2, win, st, dil, cau)
            gna.attention_permuted(q, k, v, o2, win, st, dil, cau, work_range=wr)
            gna.unpermute(q, k, v, o2, l2, win, st, dil, cau)
        torch.cuda.synchronize()
        for _ in range(min(args.steps, 10)):
            flush.zero_()
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
            ev[0].record(stream)
            gna.permute(q, k, v, o2, win, st, dil, cau)
            ev[1].record(stream)
            gna.attention_permuted(q, k, v, o2, win, st, dil, cau, work_range=wr)
            ev[2].record(stream)
            gna.unpermute(q, k, v, o2, l2, win, st, dil, cau)
            ev[3].record(stream)
            ev[3].synchronize()
            for i, kname in enumerate(stage):
                stage[kname].append(ev[i].elapsed_time(ev[i + 1]))

    # ---- dense baseline: the same kernel on the same shard, window = extent, same box (a6)
    dense_win = tuple(w.spatial)
    ones = tuple(1 for _ in w.spatial)
    dinfo = gna.plan_info(B, H, D, w.spatial, dense_win, ones, box=info["box"])
    dense_wr = None
    if wr is not None:  # same fraction of the dense work list
        n_d = dinfo["n_work"]
        dense_wr = (wr[0] * n_d // info["n_work"], wr[1] * n_d // info["n_work"])

    def dense():
        gna.forward(q, k, v, dense_win, ones, None, None, out=o2, lse=l2, box=info["box"], scales=scales,
                    work_range=dense_wr)

    dense()
    torch.cuda.synchronize()
    dense_ms = timed(dense, max(3, min(args.steps, 10)))

    # ---- end to end through the public API with host buffers (pinned): H2D of this rank's
    #      inputs, the forward, D2H of its O and LSE, every step
    out_h = torch.empty(out.shape, dtype=out.dtype, pin_memory=True)
    lse_h = torch.empty(lse.shape, dtype=lse.dtype, pin_memory=True)
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    e2e_ms = []
    for _ in range(args.steps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        q.copy_(qh, non_blocking=True)
        k.copy_(kh, non_blocking=True)
        v.copy_(vh, non_blocking=True)
        fwd()
        out_h.copy_(out, non_blocking=True)
        lse_h.copy_(lse, non_blocking=True)
        e1.record(stream)
        e1.synchronize()
        e2e_ms.append(e0.elapsed_time(e1))
    h2d = sum(t.numel() * t.element_size() for t in (qh, kh, vh))
    d2h = out_h.numel() * out_h.element_size() + lse_h.numel() * lse_h.element_size()

    att_ms = statistics.mean(stage["attention"]) if stage["attention"] else statistics.mean(step_ms)
    vals = _max_over_ranks([total_ms, sum(e2e_ms), att_ms, statistics.mean(dense_ms), float(h2d), float(d2h)],
                           ws, dev)
    total_ms_max, e2e_total, att_ms_max, dense_max = vals[:4]
    if ws > 1:
        tb = torch.tensor([float(h2d), float(d2h)], dtype=torch.float64, device=dev)
        dist.all_reduce(tb)
        h2d_all, d2h_all = tb.tolist()
    else:
        h2d_all, d2h_all = float(h2d), float(d2h)

    # ---- verification (untimed): gather every rank's O / LSE to rank 0; bit-exact against the
    #      one-GPU launch (N > 1) and sampled rows against the fp64 oracle
    verify = _verify(args, w, f, sh, ws, rank, dev, q, k, v, out, lse, full, scales, fp8)

    if rank != 0:
        return
    peak_burst, peak_sus, hbm, peak_kind = _peaks()
    if fp8:  # E4M3 dense peak = measured bf16 peak x the nominal ratio (4.5 / 2.25 PFLOP/s)
        peak_burst, peak_sus, peak_kind = 2.0 * peak_burst, 2.0 * peak_sus, f"{peak_kind}, bf16 x2 (nominal e4m3:bf16)"
    else:
        peak_kind = f"{peak_kind}, bf16 burst (fp16 dense rate = bf16 on B200)"
    ms_per_step = total_ms_max / args.steps
    value = eff_flops / (ms_per_step * 1e-3) / 1e12
    e2e_value = eff_flops / (e2e_total / args.steps * 1e-3) / 1e12
    # dominant kernel = the one launch of the step (permute-free route); rank 0's launch
    direct = launch_is_direct(D, info, f)
    kernel_ms = statistics.mean(step_ms) if direct else statistics.mean(stage["attention"])
    achieved = shard_flops / (kernel_ms * 1e-3) / 1e12
    mma_flops = 4.0 * info["padded_head_dim"] * 128 * 128 * info["subtile_stages"] * B * H  # issued (both GEMMs)
    n_tok = w.n_tokens
    ebytes = 1 if fp8 else 2
    nat_bytes = B * n_tok * H * D * 2
    perm_bytes = 6 * nat_bytes  # read q,k,v + write permuted q,k,v (algorithmic, no padding)
    unperm_bytes = 2 * nat_bytes + 2 * B * n_tok * H * 4
    attn_bytes = B * n_tok * H * D * (3 * ebytes + 2) + B * n_tok * H * 4  # q,k,v,o once + lse
    traffic, traffic_src = (None, None)
    if ws == 1:
        traffic, traffic_src = _traffic(w.name, args.dtype)
    cpu = None
    if ws == 1 and not args.no_cpu_baseline:
        cv, ct, cr, cores = cpu_oracle_sample(w, args.cpu_budget, inputs=(qh, kh, vh) if not fp8 else None)
        cpu = {"value": cv, "unit": "TFLOP/s", "cores": cores, "kind": "oracle", "cpu_model": _cpu_model(),
               "sample": f"{cr} random (b, token, h) rows of {w.name} (fp64 oracle on the same inputs, {ct:.1f} s)"}
    cfg = _config(w, args, ws, sh)
    cfg.update({"launch": launch_kind, "box": info["box"], "q_sub": info["q_sub"],
                "shard": {"mode": sh.mode, "batch": list(sh.batch), "heads": list(sh.heads),
                          "work": list(sh.work) if sh.work else None, "rank": 0}})
    line = {
        "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": {"bf16": "bf16", "fp16": "fp16", "fp8": "e4m3"}[args.dtype],
        "data": "synthetic (seeded N(0,1), gna_inputs.py)", "config": cfg,
        "speedup_vs_dense": dense_max / att_ms_max if direct else dense_max / att_ms_max,
        "bound": info["bound"],
        "speedup_frac_of_bound": (dense_max / att_ms_max) / info["bound"],
        "flopwise_speedup": float(n_tok * n_tok) / info["kept_pairs"] if not any(f["causal"]) else None,
        "stages_ms": {k2: statistics.mean(v2) for k2, v2 in stage.items()} if stage["attention"] else None,
        "dense_attention_ms": statistics.mean(dense_ms),
        "dense_effective_tflops": 4.0 * D * n_tok * n_tok * B * H * (shard_flops / eff_flops)
        / (statistics.mean(dense_ms) * 1e-3) / 1e12,
        "permute_gbs": perm_bytes * (shard_flops / eff_flops) / (statistics.mean(stage["permute"]) * 1e-3) / 1e9
        if stage["permute"] else None,
        "unpermute_gbs": unperm_bytes * (shard_flops / eff_flops) / (statistics.mean(stage["unpermute"]) * 1e-3) / 1e9
        if stage["unpermute"] else None,
        "mma_issued_tflops": mma_flops * (shard_flops / eff_flops) / (kernel_ms * 1e-3) / 1e12,
        "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak_burst, "unit": "TFLOP/s",
                     "frac": achieved / peak_burst, "traffic": traffic,
                     "traffic_source": traffic_src, "algorithmic_bytes": attn_bytes * (shard_flops / eff_flops),
                     "kernel": "gna_attn_sm100 (permute-free, one launch per step)" if direct else "gna_attn_sm100",
                     "peak_kind": peak_kind, "frac_of_sustained": achieved / peak_sus},
        "e2e": {"value": e2e_value, "unit": "TFLOP/s", "h2d_bytes_per_step": int(h2d_all),
                "d2h_bytes_per_step": int(d2h_all)},
        "gpu_launches": args.steps * (1 if direct else 2),
        "clocks": clk.summary(),
        "cpu_baseline": cpu,
        "verify": verify,
        "context": {"paper_gna_pflops_fp16": 1.3, "paper_e2e_speedups": "28%-46% (P:72)"},
    }
    print(json.dumps(line), flush=True)


def launch_is_direct(D, info, f):
    """The default forward is one permute-free kernel when the direct path applies."""
    dil = list(f["dilation"]) + [1] * 3
    return D >= 64 and all(b * d <= 256 and d <= 8 for b, d in zip(info["box"], dil))


def _verify(args, w, f, sh, ws, rank, dev, q, k, v, out, lse, full, scales, fp8):
    """Untimed: gather every rank's O / LSE to rank 0 over NCCL (all_gather_into_tensor of the
    heads / batch shards, padded to equal size; a SUM reduce of zero-filled buffers for Q-tile
    ranges), compare bit for bit with the one-GPU launch of the whole problem (N > 1) and
    sampled rows (borders included) with the fp64 oracle."""
    import numpy as np
    import torch
    import torch.distributed as dist

    import oracle as O
    import paper_2504_16922_b200 as gna

    if args.no_verify:
        return None
    B, H, D = w.batch, w.heads, w.head_dim
    win, st, dil, cau = f["window"], f["stride"], f["dilation"], f["causal"]
    o_full, l_full = out, lse
    if ws > 1:
        if sh.mode == "qtile":
            o_z, l_z = torch.zeros_like(out), torch.zeros_like(lse)
            gna.forward(q, k, v, win, st, dil, cau, out=o_z, lse=l_z, scales=scales, work_range=sh.work)
            dist.reduce(o_z, dst=0, op=dist.ReduceOp.SUM)  # disjoint items over zeros: x + 0 == x
            dist.reduce(l_z, dst=0, op=dist.ReduceOp.SUM)
            o_full, l_full = o_z, l_z
        else:
            dim = -2 if sh.mode == "heads" else 0  # heads axis of O (LSE: its last axis)
            ldim = -1 if sh.mode == "heads" else 0
            total = H if sh.mode == "heads" else B
            sizes = [len(range(*_bal(total, ws, r))) for r in range(ws)]
            mx = max(sizes)

            def gather(t, d):
                pad = list(t.shape)
                pad[d] = mx
                buf = torch.zeros(pad, dtype=t.dtype, device=dev)
                buf.narrow(d, 0, t.shape[d]).copy_(t)
                allb = torch.empty((ws, *pad), dtype=t.dtype, device=dev)
                dist.all_gather_into_tensor(allb, buf)
                return torch.cat([allb[r].narrow(d, 0, sizes[r]) for r in range(ws)], dim=d)

            o_full, l_full = gather(out, dim), gather(lse, ldim)
    if rank != 0:
        return None
    res = {"gathered_from_ranks": ws, "mode": sh.mode}
    qf, kf, vf = full
    if ws > 1:
        # the same problem in one launch on rank 0's GPU
        qd, kd, vd = (t.to(dev) for t in full)
        o_ref, l_ref = gna.forward(qd, kd, vd, win, st, dil, cau, scales=scales)
        torch.cuda.synchronize()
        res["bitwise_vs_1gpu"] = bool(torch.equal(o_ref, o_full) and torch.equal(l_ref, l_full))
        del qd, kd, vd, o_ref, l_ref
    L = list(w.spatial) + [1] * (3 - len(w.spatial))
    corners = [0, L[1] * L[2] - 1, w.n_tokens - 1, (L[0] // 2) * L[1] * L[2] + (L[1] // 2) * L[2] + L[2] // 2]
    rows = sample_rows(B, w.spatial, H, 32, extra_tokens=corners)
    if fp8:
        qn, kn, vn = (t.to(torch.float32).numpy() * s for t, s in zip(full, scales))
    else:
        qn, kn, vn = (t.to(torch.float32).numpy() for t in full)
    p = O.Params(f["spatial"], f["window"], f["stride"], f["dilation"], f["causal"])
    ro, rl, _ = O.forward_rows(qn, kn, vn, p, rows)
    oo = o_full.float().cpu().reshape(B, -1, H, D)[rows[:, 0], rows[:, 1], rows[:, 2]].numpy()
    ll = l_full.cpu().reshape(B, -1, H)[rows[:, 0], rows[:, 1], rows[:, 2]].numpy()
    err, lerr = np.abs(oo - ro), np.abs(ll - rl)
    res.update({"oracle_rows": int(len(rows)), "o_max_abs": float(err.max()), "o_mean_abs": float(err.mean()),
                "lse_max_abs": float(lerr.max())})
    if fp8:  # per-element bound of tests/test_gpu_fp8.py
        ra, _, _ = O.forward_rows(qn, kn, np.abs(vn), p, rows)
        ok = bool((err <= 2.0 ** -4 * ra + 2.0 ** -8 * np.abs(ro) + 4e-3).all() and lerr.max() <= 1e-3)
    else:
        ok = bool(err.max() <= 2e-2 and err.mean() <= 2e-3 and lerr.max() <= 1e-3)
    res["oracle_pass"] = ok
    return res


def _bal(total, world, rank):
    from paper_2504_16922_b200.shard import balanced_range

    return balanced_range(total, world, rank)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--workload", default=DEFAULT_WORKLOAD, choices=sorted(WORKLOADS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-budget", type=float, default=12.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-verify", action="store_true", help="skip the untimed gather + oracle check")
    ap.add_argument("--dtype", default="bf16", choices=["bf16", "fp16", "fp8"],
                    help="bf16 (default), fp16, or fp8: E4M3 Q/K/V with per-tensor scales (permute-free path)")
    ap.add_argument("--partition", default="auto", choices=["auto", "heads", "batch", "qtile"],
                    help="multi-GPU split of the one problem (paper_2504_16922_b200/shard.py)")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(_spawn_ranks(args.gpus))
    ws, rank, local = _dist()
    import torch

    if args.impl == "reference":
        run_reference(args, ws, rank)
    elif not torch.cuda.is_available():
        run_nodevice(args, ws, rank)
    else:
        run_ours(args, ws, rank, local)
    if ws > 1:
        import torch.distributed as dist

        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
