"""Profiling driver: N SALE prefills (and optionally the dense run) of the
bench workload, for ncu. Not a benchmark (numbers under ncu are not bench
values)."""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_24179_b200 import sale  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--tokens", type=int, default=131072)
p.add_argument("--iters", type=int, default=2)
p.add_argument("--tau", type=float, default=0.004)
p.add_argument("--dense", action="store_true")
a = p.parse_args()
q16, k16, v16 = sale.workload_gqa("sink_local", 7, 1, a.tokens, 32, 8, 128)
dev = lambda x: torch.from_numpy(x.view(np.int16)).view(torch.bfloat16).cuda()
q, k, v = dev(q16), dev(k16), dev(v16)
for _ in range(a.iters):
    sale.prefill(q, k, v, a.tau)
    if a.dense:
        sale.block_sparse_attention(q, k, v, None)
torch.cuda.synchronize()
print("done")
