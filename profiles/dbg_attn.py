import sys, os, numpy as np, torch
sys.path.insert(0, os.getcwd())
from paper_2505_24179_b200 import sale
N = int(sys.argv[1]) if len(sys.argv) > 1 else 256
q16, k16, v16 = sale.workload_gqa("sink_local", 7, 1, N, 2, 1, 128)
t = lambda a: torch.from_numpy(a.view(np.int16)).view(torch.bfloat16).cuda()
q, k, v = t(q16), t(k16), t(v16)
out = sale.block_sparse_attention(q, k, v, None)
torch.cuda.synchronize()
print("ok", out.float().abs().mean().item())
