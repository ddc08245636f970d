"""Shared test plumbing: B200-layout inputs, per-head oracle runs, comparisons.

The oracle (oracle/oracle.py) is the checker; the GPU path under test is
paper_2505_24179_b200.sale over the C ABI.
"""
from __future__ import annotations

import numpy as np

from oracle import oracle as O
from paper_2505_24179_b200 import sale

LLAMA = dict(q_heads=32, kv_heads=8)
QWEN = dict(q_heads=28, kv_heads=4)


class Inputs:
    """bf16 Q/K/V of the GQA sink-local (or gaussian) workload, as host bit
    patterns plus fp32 per-head views for the oracle."""

    def __init__(self, kind, seed, batch, tokens, q_heads, kv_heads, head_dim=128):
        self.kind, self.seed = kind, seed
        self.B, self.N, self.Hq, self.Hkv, self.d = batch, tokens, q_heads, kv_heads, head_dim
        self.G = q_heads // kv_heads
        self.q16, self.k16, self.v16 = sale.workload_gqa(kind, seed, batch, tokens, q_heads,
                                                         kv_heads, head_dim)

    def head(self, x16, b, h):
        return np.ascontiguousarray(sale.bf16_bits_to_f32(x16[b, :, h, :self.d]))

    def qh(self, b, h):
        return self.head(self.q16, b, h)

    def kh(self, b, g):
        return self.head(self.k16, b, g)

    def vh(self, b, g):
        return self.head(self.v16, b, g)

    def torch(self):
        import torch
        t = lambda a: torch.from_numpy(a.view(np.int16)).view(torch.bfloat16).cuda()
        return t(self.q16), t(self.k16), t(self.v16)

    def heads(self):
        return [(b, h) for b in range(self.B) for h in range(self.Hq)]


def oracle_quant(inp: Inputs):
    """Per-head oracle quantization: dicts keyed (b, h) / (b, g)."""
    qq = {(b, h): O.quantize(inp.qh(b, h), 1) for b in range(inp.B) for h in range(inp.Hq)}
    kq = {(b, g): O.quantize(inp.kh(b, g), 32) for b in range(inp.B) for g in range(inp.Hkv)}
    return qq, kq


def oracle_select(inp: Inputs, taus, qq=None, kq=None, debug=False, heads=None):
    qq, kq = (qq, kq) if qq is not None else oracle_quant(inp)
    taus = np.broadcast_to(np.asarray(taus, np.float64), (inp.Hq,))
    heads = heads or inp.heads()

    def one(i):
        b, h = heads[i]
        g = h // inp.G
        return O.selection_pass(inp.qh(b, h), inp.kh(b, g), *qq[(b, h)], *kq[(b, g)],
                                c=O.cfg(tau=float(taus[h])), debug=debug)

    res = O.map_heads(one, len(heads))
    return dict(zip(heads, res))


def mean_abs(a, b):
    return float(np.mean(np.abs(np.asarray(a, np.float64) - np.asarray(b, np.float64))))


def max_abs(a, b):
    return float(np.max(np.abs(np.asarray(a, np.float64) - np.asarray(b, np.float64))))
