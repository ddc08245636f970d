"""Does the i8 estimator's MMA rate depend on the operand values? Profile
modes 2 (epilogue work skipped) and 1 on the bench workload, on
all-zero inputs, and on i.i.d. Gaussian inputs."""
import ctypes as C, os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_24179_b200 import sale
N = 131072
ctx = sale.context(); lib = ctx.lib
lib.sale_b200_estimator_profile.argtypes = [C.c_void_p, C.c_int, C.c_void_p]
q16, k16, v16 = sale.workload_gqa("sink_local", 7, 1, N, 32, 8, 128)
dev = lambda x: torch.from_numpy(x.view(np.int16)).view(torch.bfloat16).cuda()
cases = {"sink_local": (dev(q16), dev(k16)),
         "zeros": (torch.zeros(1, N, 32, 128, dtype=torch.bfloat16, device="cuda"),
                   torch.zeros(1, N, 8, 128, dtype=torch.bfloat16, device="cuda")),
         "gaussian": (torch.randn(1, N, 32, 128, device="cuda").bfloat16(),
                      torch.randn(1, N, 8, 128, device="cuda").bfloat16())}
for name, (q, k) in cases.items():
    qc, qs, kc, ks = sale.quantize_qk(q, k)
    sale.selection_pass(q, k, qc, qs, kc, ks, 0.004)
    for mode in (2, 1):
        cnt = (C.c_uint64 * 16)()
        lib.sale_b200_estimator_profile(ctx.handle, mode, None)
        sale.selection_pass(q, k, qc, qs, kc, ks, 0.004)
        lib.sale_b200_estimator_profile(ctx.handle, 0, cnt)
        c = list(cnt)
        print(f"{name:10s} mode {mode}: {c[0]/c[4]:.0f} cyc/stage")
