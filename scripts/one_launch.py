"""One gna_forward_ex launch of a workload (the bench's launch configuration), for ncu.

usage: python scripts/one_launch.py WORKLOAD [bf16|fp16|fp8] [n_launches]
Warm-up launches are made first (plan cache, tensor maps); ncu selects the last launch of the
attention kernel with --launch-skip."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2504_16922_b200 as gna
from gna_inputs import WORKLOADS, make_qkv, quantize_e4m3

w = WORKLOADS[sys.argv[1]]
dtype = sys.argv[2] if len(sys.argv) > 2 else "bf16"
n = int(sys.argv[3]) if len(sys.argv) > 3 else 2
f = w.full()
q, k, v = make_qkv(w.batch, f["spatial"], w.heads, w.head_dim)
kw = {}
if dtype == "fp16":
    q, k, v = q.half(), k.half(), v.half()
elif dtype == "fp8":
    (q, sq), (k, sk), (v, sv) = quantize_e4m3(q), quantize_e4m3(k), quantize_e4m3(v)
    kw["scales"] = (sq, sk, sv)
q, k, v = q.cuda(), k.cuda(), v.cuda()
for _ in range(n):
    gna.forward(q, k, v, f["window"], f["stride"], f["dilation"], f["causal"], **kw)
torch.cuda.synchronize()
print("ok", w.name, dtype, n)
