"""Per-CTA timeline of the attention kernel (trace build): wave structure, per-CTA phase
durations and SM idle time.

usage: python scripts/timeline.py WORKLOAD [--direct]   (run on the GPU box)
Events (globaltimer ns): 0 CTA start, 1 first K issued, 2 first S ready (softmax A),
3 last P stored, 4 epilogue stores done, 5 TMEM released (CTA end); 7 = SM id."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2504_16922_b200 import build
import paper_2504_16922_b200.gna as G
G.LIB_PATH = os.environ.get("TRACE_LIB") or build.build(trace=True)
import numpy as np, torch
import paper_2504_16922_b200 as gna
from gna_inputs import WORKLOADS, make_qkv

w = WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "c2b_flux64_s16"]
f = w.full()
q, k, v = (t.cuda() for t in make_qkv(w.batch, w.spatial, w.heads, w.head_dim))
lib = gna.load()
V4 = False  # the v4 kernel was removed in round 2
if V4:
    lib.gna_debug_trace_reset = lib.gna_debug_timeline_v4_reset
    lib.gna_debug_timeline = lib.gna_debug_timeline_v4
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for it in range(4):
    flush.zero_()
    lib.gna_debug_trace_reset()
    torch.cuda.synchronize()
    gna.forward(q, k, v, f["window"], f["stride"], f["dilation"], f["causal"],
                flags=4 if os.environ.get("TRACE_PERMUTED") == "1" else 0)
    torch.cuda.synchronize()
buf = np.zeros((8192, 16) if not V4 else (8192, 8), dtype=np.uint64)
assert lib.gna_debug_timeline(buf.ctypes.data_as(ctypes.c_void_p), ctypes.c_size_t(buf.nbytes)) == 0
if V4:
    # per task: 0 softmax setup start, 2 first S ready, 3 last P / stats, 4 epilogue done, 7 SM id
    idx = np.where(buf[:, 0] > 0)[0]
    t = buf[idx, :5].astype(np.int64)
    sm = buf[idx, 7].astype(np.int64)
    t0 = t[:, 0].min()
    rel = (t - t0) / 1000.0
    span = rel[:, 4].max()
    print(f"{sys.argv[1]} (v4): {len(idx)} tasks, span {span:.1f} us (first task start -> last epilogue)")
    rows = []
    for s_ in np.unique(sm):
        ii = np.where(sm == s_)[0]
        ii = ii[np.argsort(rel[ii, 0])]
        for a, b in zip(ii[:-1], ii[1:]):
            rows.append((rel[a, 2] - rel[a, 0], rel[a, 3] - rel[a, 2], rel[a, 4] - rel[a, 3], rel[b, 2] - rel[a, 3]))
    r = np.array(rows)
    print("median setup->S0 %.2f  mainloop %.2f  lastP->epi done %.2f  softmax bubble between tasks %.2f us" %
          tuple(np.median(r, 0)))
    per_sm = np.bincount(sm)
    first = np.array([rel[sm == s_, 0].min() for s_ in np.unique(sm)])
    last = np.array([rel[sm == s_, 4].max() for s_ in np.unique(sm)])
    print(f"tasks per SM min {per_sm[per_sm>0].min()} max {per_sm.max()}; SM first start max {first.max():.1f} us; "
          f"SM end min {last.min():.1f} max {last.max():.1f} us")
    ml = rel[:, 3] - rel[:, 2]
    print("mainloop per task: p10 %.1f  median %.1f  p90 %.1f  max %.1f us" % tuple(np.percentile(ml, [10, 50, 90, 100])))
    bysm = {int(s_): np.median(ml[sm == s_]) for s_ in np.unique(sm)}
    v = np.array(sorted(bysm.values()))
    print("per-SM median mainloop: min %.1f  median %.1f  max %.1f us" % (v.min(), np.median(v), v.max()))
    print("first task: setup->S0 %.2f us" % np.median(rel[np.argsort(rel[:, 0])[:148], 2] - rel[np.argsort(rel[:, 0])[:148], 0]))
    sys.exit(0)
n = int((buf[:, 0] > 0).sum())
t = buf[:n, :6].astype(np.int64)
sm = buf[:n, 7].astype(np.int64)
t0 = t[:, 0].min()
rel = (t - t0) / 1000.0  # us
span = rel[:, 5].max()
print(f"{sys.argv[1]}: {n} CTAs, kernel span {span:.1f} us (first CTA start -> last CTA end)")
names = ["start->K issued", "K issued->S0 ready", "S0 ready->last P", "last P->epi done", "epi done->end", "total"]
d = np.stack([rel[:, 1] - rel[:, 0], rel[:, 2] - rel[:, 1], rel[:, 3] - rel[:, 2], rel[:, 4] - rel[:, 3],
              rel[:, 5] - rel[:, 4], rel[:, 5] - rel[:, 0]], 1)
order = np.argsort(rel[:, 0])
waves = [order[i:i + 148] for i in range(0, n, 148)]
print("wave  ctas  start(us) min..max   " + " | ".join(f"{x:>18s}" for x in names))
for wi, idx in enumerate(waves):
    med = np.median(d[idx], 0)
    print(f"{wi:4d} {len(idx):5d}  {rel[idx,0].min():7.1f}..{rel[idx,0].max():7.1f}  " +
          " | ".join(f"{m:18.2f}" for m in med))
busy = np.zeros(int(sm.max()) + 1)
for i in range(n):
    busy[sm[i]] += rel[i, 5] - rel[i, 0]
print(f"SMs used {len(np.unique(sm))}; mean SM busy {busy[busy>0].mean():.1f} us of span {span:.1f} "
      f"({busy[busy>0].mean()/span:.2f}); mainloop share of CTA time {d[:,2].sum()/d[:,5].sum():.2f}")
if buf.shape[1] == 16:
    e = buf[:n].astype(np.int64)
    def med(a, b):
        m = (e[:, a] > 0) & (e[:, b] > 0)
        return np.median((e[m, b] - e[m, a]) / 1000.0) if m.any() else float("nan")
    print("producer (median us): decoded->producer start %.2f, ->expect_tx %.2f, ->first Q TMA issued %.2f, "
          "->all Q issued %.2f" % (med(9, 12), med(12, 13), med(13, 14), med(14, 10)))
    print("prologue (median us): start->syncthreads %.2f, ->decoded %.2f, producer decoded->Q issued %.2f, "
          "Q issued->K issued %.2f, K issued->MMA Q ready %.2f, MMA Q ready->S0 ready %.2f" %
          (med(0, 8), med(8, 9), med(9, 10), med(10, 1), med(1, 11), med(11, 2)))
gaps = []
for s_ in np.unique(sm):
    idx = np.where(sm == s_)[0]
    idx = idx[np.argsort(rel[idx, 0])]
    for a, b in zip(idx[:-1], idx[1:]):
        gaps.append(rel[b, 0] - rel[a, 5])
if gaps:
    print(f"gap between consecutive CTAs on one SM: median {np.median(gaps):.2f} us, max {np.max(gaps):.2f} us")
if os.environ.get("GNA_PERSISTENT") == "1":
    # per-item events in the persistent kernel: 0 claimed, 1 Q issued, 2 first S ready (softmax A),
    # 3 last P (softmax A), 4 epilogue done, 5 last PV committed by the MMA
    print("persistent: per-SM item chains (us): claim->Q issue, Q->S0, S0->lastP (mainloop), lastP->epi, "
          "bubble = next item's S0 ready - this item's last P")
    rows = []
    for s_ in np.unique(sm):
        idx = np.where(sm == s_)[0]
        idx = idx[np.argsort(rel[idx, 0])]
        for a, b in zip(idx[:-1], idx[1:]):
            rows.append((rel[a, 1] - rel[a, 0], rel[a, 2] - rel[a, 1], rel[a, 3] - rel[a, 2], rel[a, 4] - rel[a, 3],
                         rel[b, 2] - rel[a, 3]))
    r = np.array(rows)
    print("median", np.round(np.median(r, 0), 2), " max", np.round(r.max(0), 2))
    per_sm = np.bincount(sm)
    print("items per SM: min", per_sm[per_sm > 0].min(), "max", per_sm.max())
