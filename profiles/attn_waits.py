"""Attention-kernel cycle breakdown (sale_b200_attention_profile) at the bench
workload, sparse (tau 0.004 mask) and dense: where the softmax warps and the
MMA issuer spend their cycles per tile."""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_24179_b200 import sale  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 131072
q16, k16, v16 = sale.workload_gqa("sink_local", 7, 1, N, 32, 8, 128)
dev = lambda x: torch.from_numpy(x.view(np.int16)).view(torch.bfloat16).cuda()
q, k, v = dev(q16), dev(k16), dev(v16)
nq, nk, nw = sale.grid(N)
mask = torch.empty((1, 32, nq, nw), dtype=torch.int32, device="cuda")
sale.prefill(q, k, v, 0.004, mask_out=mask)
ctx = sale.context()
lib = ctx.lib
lib.sale_b200_attention_profile.argtypes = [C.c_void_p, C.c_int, C.c_void_p]
for name, m in (("sparse", mask), ("dense", None)):
    cnt = (C.c_uint64 * 16)()
    lib.sale_b200_attention_profile(ctx.handle, 1, None)
    sale.block_sparse_attention(q, k, v, m)
    lib.sale_b200_attention_profile(ctx.handle, 0, cnt)
    c = list(cnt)
    t = max(c[3], 1)
    print(f"[{name}] tiles/CTA {c[3]/max(c[8],1):.0f}; softmax warp per tile: loop {c[0]/t:.0f} cyc, "
          f"S wait {c[1]/t:.0f}, softmax_part {c[2]/t:.0f}; MMA per tile: loop {c[4]/t:.0f}, "
          f"K wait {c[5]/t:.0f}, P wait {c[6]/t:.0f}, V wait {c[7]/t:.0f}; epilogue/CTA "
          f"{c[10]/max(c[8],1):.0f} cyc")
    if c[12]:
        print(f"   chain: P_(j-2) seen by the MMA issuer -> S_j seen by warp 3: {c[11]/c[12]:.0f} cyc")
