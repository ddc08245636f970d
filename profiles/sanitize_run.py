"""Drives every kernel of the library once at a small shape for
compute-sanitizer (profiles/sanitize.sh): quantizer, base mask, sink-local
statistics, i8 estimator (production and parity-debug instances), sparse and
dense attention with coverage, flop accounting, the chunked host pipeline,
query-block ranges, and the run_pipeline / l1 reductions. Checks the mask
against the oracle so a sanitizer-clean run is also a correct one."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import torch  # noqa: E402

from helpers import Inputs, O  # noqa: E402
from paper_2505_24179_b200 import sale  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
Hq, Hkv = 8, 2
torch.cuda.set_device(0)
inp = Inputs("sink_local", 7, 1, N, Hq, Hkv)
q, k, v = inp.torch()
nq, nk, nw = sale.grid(N)
qc, qs, kc, ks = sale.quantize_qk(q, k)
mask, dbg = sale.selection_pass(q, k, qc, qs, kc, ks, 0.004, debug=True)
mask2 = sale.selection_pass(q, k, qc, qs, kc, ks, 0.004)
out, cov = sale.block_sparse_attention(q, k, v, mask, coverage=True)
dense = sale.full_attention(q, k, v)
counts = sale.flop_accounting(mask, N)
pm = torch.empty_like(mask)
pre = sale.prefill(q, k, v, 0.004, mask_out=pm)
rng = sale.query_block_split(nq, 2)
for r in rng:
    sale.prefill(q, k, v, 0.004, mask_out=pm, q_blocks=r)
host = np.empty_like(inp.q16)
sale.prefill_host(inp.q16, inp.k16, inp.v16, [0.004] * Hq, host)
rep = sale.run_pipeline(q, k, v, [0.004] * Hq)
torch.cuda.synchronize()
cells = sale.unpack_mask(mask.cpu().numpy(), N)
for h in range(Hq):
    qh, kh = inp.qh(0, h), inp.kh(0, h // (Hq // Hkv))
    a, b = O.quantize(qh, 1)
    c, d = O.quantize(kh, 32)
    assert np.array_equal(cells[0, h], O.selection_pass(qh, kh, a, b, c, d)), h
assert torch.equal(mask, mask2) and torch.equal(mask, pm)
assert np.array_equal(host, pre.cpu().view(torch.int16).numpy().view(np.uint16))
computed = int(counts[..., 0].sum())
sale.context().close()  # free the ctx workspace (memcheck --leak-check)
del q, k, v, qc, qs, kc, ks, mask, mask2, dbg, out, cov, dense, counts, pm, pre
torch.cuda.empty_cache()
print(f"sanitize_run N={N}: ok (masks bit-exact, {computed} computed blocks)")
