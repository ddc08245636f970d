"""Estimator wait-time breakdown (sale_b200_estimator_profile) at the bench
workload: where the MMA issuer and the epilogue spend their cycles."""
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
qc, qs, kc, ks = sale.quantize_qk(q, k)
ctx = sale.context()
lib = ctx.lib
lib.sale_b200_estimator_profile.argtypes = [C.c_void_p, C.c_int, C.c_void_p]
sale.selection_pass(q, k, qc, qs, kc, ks, 0.004)
cnt = (C.c_uint64 * 16)()
lib.sale_b200_estimator_profile(ctx.handle, 1, None)
sale.selection_pass(q, k, qc, qs, kc, ks, 0.004)
lib.sale_b200_estimator_profile(ctx.handle, 0, cnt)
c = list(cnt)
loop, wa, wf, we, stages, eloop, ew = c[:7]
print(f"MMA issuer: loop {loop/stages:.0f} cyc/stage; A wait {wa/loop*100:.1f}%, "
      f"K-stage wait {wf/loop*100:.1f}%, accumulator wait {we/loop*100:.1f}% "
      f"(ideal MMA time 1024 cyc/stage)")
print(f"epilogue (warp 4): loop {eloop/stages:.0f} cyc/stage; accumulator-full wait "
      f"{ew/eloop*100:.1f}%")
st = c[8:16]
if st[7]:
    names = ["staging", "dots", "logit store", "block max", "running max", "exp sums", "combine"]
    tot = sum(st[:7])
    print("stats kernel (thread 0, per CTA): " + ", ".join(
        f"{n} {v / st[7]:.0f} cyc ({100 * v / tot:.0f}%)" for n, v in zip(names, st[:7])))
# mode 2: epilogue skips its TMEM loads and math (MMA / TMA side alone)
lib.sale_b200_estimator_profile(ctx.handle, 2, None)
sale.selection_pass(q, k, qc, qs, kc, ks, 0.004)
lib.sale_b200_estimator_profile(ctx.handle, 0, cnt)
c = list(cnt)
print(f"[epilogue work skipped] MMA issuer loop {c[0]/c[4]:.0f} cyc/stage; K-stage wait "
      f"{c[2]/c[0]*100:.1f}%, accumulator wait {c[3]/c[0]*100:.1f}%")
