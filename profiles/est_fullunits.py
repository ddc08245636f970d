import ctypes as C, os, sys
import numpy as np, torch
sys.path.insert(0, '/root/repo')
from paper_2505_24179_b200 import sale
N = 131072
q16, k16, v16 = sale.workload_gqa("sink_local", 7, 1, N, 32, 8, 128)
dev = lambda x: torch.from_numpy(x.view(np.int16)).view(torch.bfloat16).cuda()
q, k, v = dev(q16), dev(k16), dev(v16)
qc, qs, kc, ks = sale.quantize_qk(q, k)
ctx = sale.context(); lib = ctx.lib
lib.sale_b200_estimator_profile.argtypes = [C.c_void_p, C.c_int, C.c_void_p]
sale.selection_pass(q, k, qc, qs, kc, ks, 0.004)
for mode in (1, 2, 3, 5):
    cnt = (C.c_uint64 * 16)()
    lib.sale_b200_estimator_profile(ctx.handle, mode, None)
    sale.selection_pass(q, k, qc, qs, kc, ks, 0.004)
    lib.sale_b200_estimator_profile(ctx.handle, 0, cnt)
    c = list(cnt)
    print(f"mode {mode}: all units {c[0]/c[4]:.0f} cyc/stage; full 64-stage units {c[1]/max(c[7],1):.0f} cyc/stage "
          f"({c[7]/c[4]*100:.0f}% of stages); others {(c[0]-c[1])/max(c[4]-c[7],1):.0f}")
