"""Quick timing: bf16 vs E4M3 forward (direct path) on a workload; effective TFLOP/s."""
import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2504_16922_b200 as gna
from gna_inputs import WORKLOADS, make_qkv, quantize_e4m3
for name in sys.argv[1:]:
    w = WORKLOADS[name]
    f = w.full()
    q, k, v = make_qkv(w.batch, w.spatial, w.heads, w.head_dim, dtype=torch.float32)
    qb, kb, vb = (t.to(torch.bfloat16).cuda() for t in (q, k, v))
    (q8, qs, _), (k8, ks, _), (v8, vs, _) = (quantize_e4m3(t) for t in (q, k, v))
    q8, k8, v8 = q8.cuda(), k8.cuda(), v8.cuda()
    info = gna.plan_info(w.batch, w.heads, w.head_dim, **f)
    flops = 4.0 * w.head_dim * info["kept_pairs"] * w.batch * w.heads
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for label, args, kw in (("bf16", (qb, kb, vb), {}), ("e4m3", (q8, k8, v8), {"scales": (qs, ks, vs)})):
        for _ in range(3):
            gna.forward(*args, f["window"], f["stride"], f["dilation"], f["causal"], **kw)
        ts = []
        for _ in range(10):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            gna.forward(*args, f["window"], f["stride"], f["dilation"], f["causal"], **kw)
            e1.record()
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        ts.sort()
        print(f"{name:22s} {label}: {ts[len(ts)//2]:.3f} ms  {flops / (ts[len(ts)//2] * 1e-3) / 1e12:.0f} TF/s effective")
