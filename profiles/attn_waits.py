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
mask64 = None
if len(sys.argv) > 2:  # a second tau: its mask as a third case
    mask64 = torch.empty_like(mask)
    sale.prefill(q, k, v, float(sys.argv[2]), mask_out=mask64)
cases = [("sparse", mask), ("dense", None)] + ([("sparse tau " + sys.argv[2], mask64)] if mask64 is not None else [])
for name, m in cases:
    cnt = (C.c_uint64 * 16)()
    lib.sale_b200_attention_profile(ctx.handle, 1, None)
    sale.block_sparse_attention(q, k, v, m)
    lib.sale_b200_attention_profile(ctx.handle, 0, cnt)
    c = list(cnt)
    t = max(c[3], 1)
    print(f"[{name}] tiles/CTA {c[3]/max(c[8],1):.0f}; softmax warp per tile: loop {c[0]/t:.0f} cyc, "
          f"S wait {c[1]/t:.0f}, softmax_part {c[2]/t:.0f}; MMA per tile: loop {c[4]/t:.0f}, "
          f"K wait {c[5]/t:.0f}, P wait {c[6]/t:.0f}, V wait {c[7]/t:.0f}; epilogue/CTA "
          f"{c[10]/max(c[8],1):.0f} cyc; prologue/CTA {c[9]/max(c[8],1):.0f} cyc "
          f"(list warp start {c[12]/max(c[8],1):.0f}, TMEM alloc done {c[13]/max(c[8],1):.0f}, tile list done {c[14]/max(c[8],1):.0f}, "
          f"barrier init + ones done {c[15]/max(c[8],1):.0f})")

