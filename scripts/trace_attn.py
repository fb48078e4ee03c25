"""Cycle trace of the attention pipeline (trace build of the library).

usage: python scripts/trace_attn.py WORKLOAD   (run on the GPU box)
Prints per-stage event times (clock64 cycles, relative to CTA start) for CTA 0."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2504_16922_b200 import build
import paper_2504_16922_b200.gna as G
G.LIB_PATH = os.environ.get("TRACE_LIB") or build.build(trace=True)
import numpy as np, torch
import paper_2504_16922_b200 as gna
from gna_inputs import WORKLOADS, make_qkv

w = WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "c4a_hunyuan_blocked"]
f = w.full()
q, k, v = (t.cuda() for t in make_qkv(w.batch, w.spatial, w.heads, w.head_dim))
lib = gna.load()
for it in range(3):
    lib.gna_debug_trace_reset()
    gna.forward(q, k, v, f["window"], f["stride"], f["dilation"], f["causal"],
                flags=4 if os.environ.get("TRACE_PERMUTED") == "1" else 0)
    torch.cuda.synchronize()
buf = np.zeros((4, 256, 16), dtype=np.uint64)
if False:  # the v4 kernel was removed in round 2
    assert lib.gna_debug_trace_v4(buf.ctypes.data_as(ctypes.c_void_p), ctypes.c_size_t(buf.nbytes)) == 0
    names = ["smWait", "smS", "smXchg", "smExp", "smSt", "smP", "Sbeg", "h1S", "Sdone", "PVp0", "PVp1", "h1P",
             "SKrdy", "PVbeg", "PVend", "prodK"]
    for cta in range(2):
        rows = buf[cta].astype(np.int64)
        t0 = rows[rows > 0].min()
        print(f"CTA {cta} (v4; cycles from the first event)")
        print("  t  " + " ".join(f"{n:>7}" for n in names))
        for t in range(256):
            if rows[t].max() == 0:
                break
            if t < 24 or t % 10 == 0:
                print(f"{t:3d}  " + " ".join(f"{int(x) - t0 if x else -1:7d}" for x in rows[t]))
        v = rows[:, 1]
        v = v[v > 0]
        if len(v) > 10:
            d = np.diff(v[4:])
            print("  period (h0 S ready) median", int(np.median(d)))
    sys.exit(0)
assert lib.gna_debug_trace(buf.ctypes.data_as(ctypes.c_void_p), ctypes.c_size_t(buf.nbytes)) == 0
names = {0: "S0rdy", 1: "S0ld", 2: "S0max", 3: "P0st", 4: "S1rdy", 5: "S1ld", 6: "S1max", 7: "P1st",
         8: "Vrdy", 9: "P0rdy", 10: "P1rdy", 11: "Knext", 12: "prodK", 13: "prodV"}
for cta in range(2):
    t0 = int(buf[cta, 0, 15])
    print(f"CTA {cta}")
    print("  j  " + " ".join(f"{names[e]:>7}" for e in range(14)))
    prev = None
    for j in range(256):
        row = buf[cta, j, :14].astype(np.int64)
        if row.max() == 0:
            break
        rel = [int(x) - t0 if x else -1 for x in row]
        if j < 12 or j % 10 == 0:
            print(f"{j:3d}  " + " ".join(f"{x:7d}" for x in rel))
    # steady-state period (median diff of S0rdy over stages 5..)
    s0 = buf[cta, :, 0].astype(np.int64)
    s0 = s0[s0 > 0]
    if len(s0) > 8:
        d = np.diff(s0[4:])
        med = lambda a, b: int(np.median((buf[cta, 4:len(s0), b] - buf[cta, 4:len(s0), a]).astype(np.int64)))
        print("  chunk0: max->st issue", med(2, 14), "st wait", med(14, 15), "-> P0st", med(15, 3),
              "; P0st->P0rdy", med(3, 9), "P0rdy->Knext", med(9, 11), "S1rdy-S0rdy", med(0, 4))
        print("  S0 period median", int(np.median(d)), "cycles;  softmax0 ld", int(np.median((buf[cta,4:len(s0),1]-buf[cta,4:len(s0),0]).astype(np.int64))),
              "max", int(np.median((buf[cta,4:len(s0),2]-buf[cta,4:len(s0),1]).astype(np.int64))),
              "exp+st", int(np.median((buf[cta,4:len(s0),3]-buf[cta,4:len(s0),2]).astype(np.int64))))
