"""Host-side cost of one gna.forward call (python binding + C ABI + launch) vs the GPU time,
and the same step replayed from a CUDA graph."""
import os, sys, time, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2504_16922_b200 as gna
from gna_inputs import WORKLOADS, make_qkv
w = WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "c2b_flux64_s16"]
f = w.full()
q, k, v = (t.cuda() for t in make_qkv(w.batch, w.spatial, w.heads, w.head_dim))
out = torch.empty_like(q); lse = torch.empty(q.shape[:-1], dtype=torch.float32, device="cuda")
fwd = lambda: gna.forward(q, k, v, f["window"], f["stride"], f["dilation"], f["causal"], out=out, lse=lse)
for _ in range(5): fwd()
torch.cuda.synchronize()
n = 200
t0 = time.perf_counter()
for _ in range(n): fwd()
t1 = time.perf_counter()
torch.cuda.synchronize(); t2 = time.perf_counter()
print(f"host enqueue per call {1e6*(t1-t0)/n:.1f} us; wall per call incl. GPU {1e6*(t2-t0)/n:.1f} us")
# GPU time per launch back to back (events around n launches)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(n): fwd()
e1.record(); e1.synchronize()
print(f"events around {n} back-to-back calls: {1e3*e0.elapsed_time(e1)/n:.1f} us per call")
g = torch.cuda.CUDAGraph()
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    fwd()
    torch.cuda.synchronize()
    with torch.cuda.graph(g, stream=s):
        fwd()
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(n): g.replay()
t1 = time.perf_counter(); torch.cuda.synchronize()
print(f"graph replay host per call {1e6*(t1-t0)/n:.1f} us")
e0.record()
for _ in range(n): g.replay()
e1.record(); e1.synchronize()
print(f"events around {n} graph replays: {1e3*e0.elapsed_time(e1)/n:.1f} us per step")
