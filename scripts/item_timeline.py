"""Per-item timeline of the persistent attention kernel (trace build, GNA_TRACE): for each SM
the chain of work items it ran, with the phases of each item and the gaps between them.

usage (GPU box): python scripts/item_timeline.py WORKLOAD [N_SMS_TO_PRINT]
Events (globaltimer ns, per item t): 0 Q loads issued, 1 first K issued, 6 first QK^T issued,
2 / 8 first S ready in softmax A / B, 3 last P of A stored, 4 / 5 epilogue A / B done, 7 SM id."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2504_16922_b200 import build
import paper_2504_16922_b200.gna as G
G.LIB_PATH = os.environ.get("TRACE_LIB") or build.build(trace=True)
import numpy as np, torch
import paper_2504_16922_b200 as gna
from gna_inputs import WORKLOADS, make_qkv

w = WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "c2b_flux64_s16"]
nprint = int(sys.argv[2]) if len(sys.argv) > 2 else 4
f = w.full()
q, k, v = (t.cuda() for t in make_qkv(w.batch, w.spatial, w.heads, w.head_dim))
lib = gna.load()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for it in range(4):
    flush.zero_()
    lib.gna_debug_trace_reset()
    torch.cuda.synchronize()
    gna.forward(q, k, v, f["window"], f["stride"], f["dilation"], f["causal"])
    torch.cuda.synchronize()
buf = np.zeros((8192, 16), dtype=np.uint64)
assert lib.gna_debug_items(buf.ctypes.data_as(ctypes.c_void_p), ctypes.c_size_t(buf.nbytes)) == 0
idx = np.where(buf[:, 0] > 0)[0]
ev = buf[idx].astype(np.int64)
t0 = ev[:, 0].min()
rel = lambda x: (x - t0) / 1000.0
sm = ev[:, 7]
end = np.maximum(ev[:, 4], ev[:, 5])
print(f"{w.name}: {len(idx)} items, span {rel(end.max()):.1f} us (first Q issue -> last epilogue)")
per_sm = {}
for n, t in enumerate(idx):
    per_sm.setdefault(int(sm[n]), []).append(n)
loads = sorted(len(v) for v in per_sm.values())
print(f"SMs used {len(per_sm)}, items per SM min {loads[0]} max {loads[-1]}")
dur = (end - ev[:, 2]) / 1000.0
print(f"item S0->epilogue: mean {dur.mean():.2f} us  min {dur.min():.2f}  max {dur.max():.2f}")
q2s = (ev[:, 2] - ev[:, 0]) / 1000.0
print(f"item Q issue -> S0 ready: mean {q2s.mean():.2f} us  max {q2s.max():.2f}")
last_ep = (ev[:, 4] - ev[:, 3]) / 1000.0
print(f"last P(A) -> epilogue A done: mean {last_ep.mean():.2f} us")
has = ev[:, 12] > 0
if has.any():
    e = ev[has]
    d = lambda a, b: ((e[:, b] - e[:, a]) / 1000.0).mean()
    print(f"epilogue A phases (us): lastP->O full {d(3, 9):.2f}  O drain {d(9, 10):.2f}  staging+bar {d(10, 11):.2f}  "
          f"TMA issue+read {d(11, 12):.2f}  ->done {d(12, 4):.2f}")
gaps = []
for s_, ns in per_sm.items():
    ns = sorted(ns, key=lambda n: ev[n, 2])
    for a, b in zip(ns[:-1], ns[1:]):
        gaps.append((ev[b, 2] - ev[a, 3]) / 1000.0)  # last P(A) of item a -> first S(A) of item b
if gaps:
    g = np.array(gaps)
    print(f"between items on one SM, last P(A) -> next S(A) ready: mean {g.mean():.2f} us  max {g.max():.2f}")
for s_ in sorted(per_sm)[:nprint]:
    print(f"SM {s_}:")
    for n in sorted(per_sm[s_], key=lambda n: ev[n, 0]):
        e = ev[n]
        print("   item %5d  Q %7.2f  K %7.2f  QK %7.2f  S0a %7.2f  S0b %7.2f  lastPa %7.2f  epiA %7.2f  epiB %7.2f" %
              (idx[n], rel(e[0]), rel(e[1]), rel(e[6]), rel(e[2]), rel(e[8]) if e[8] else -1, rel(e[3]), rel(e[4]),
               rel(e[5]) if e[5] else -1))
