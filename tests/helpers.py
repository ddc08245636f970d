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


def oracle_select(inp: Inputs, taus, qq=None, kq=None, debug=False, heads=None, geom=None):
    qq, kq = (qq, kq) if qq is not None else oracle_quant(inp)
    taus = np.broadcast_to(np.asarray(taus, np.float64), (inp.Hq,))
    heads = heads or inp.heads()

    def one(i):
        b, h = heads[i]
        g = h // inp.G
        sink, local, seg = geom or (32, 128, 4)
        return O.selection_pass(inp.qh(b, h), inp.kh(b, g), *qq[(b, h)], *kq[(b, g)],
                                c=O.cfg(tau=float(taus[h]), sink_tokens=sink, local_tokens_min=local,
                                        segment_size=seg), debug=debug)

    res = O.map_heads(one, len(heads))
    return dict(zip(heads, res))


def mean_abs(a, b):
    return float(np.mean(np.abs(np.asarray(a, np.float64) - np.asarray(b, np.float64))))


def max_abs(a, b):
    return float(np.max(np.abs(np.asarray(a, np.float64) - np.asarray(b, np.float64))))


# ------------------------------------------------ BLAS-exact Selection-Pass

def blas_selection(qc, qs, kc, ks, bound, tokens, c=None, i_lo=0, i_hi=None, chunk=8,
                   want_block_max=False):
    """The middle-block part of selection_pass (selection.hpp:253-271, with
    approx_weight_block / max_then_dequantize, quant.hpp:136-179) for one
    head, restated with exact integer products from an fp32 GEMM: every
    partial sum of 128 products of codes in [-7, 7] is an integer of magnitude
    <= 6272 < 2^24, so the float GEMM of the codes is exact whatever its
    summation order. `bound` are the oracle's per-row double bounds
    (oracle_selection_stats). The sink / local blocks and the segment rule come
    from the C oracle (sink_local_index_set, segment_aggregate).

    Returns (mask uint8 [nq, nk], report) where report holds the decision
    margins: for every estimated block the decision is
    max_r (est_r - bound_r) >= 0, and its margin |max_r (est_r - bound_r)| is
    how far the deciding estimate is from flipping; "min_cmp" is the smallest
    |est - bound| over every (row, block) comparison. With want_block_max the
    report also holds {i: int32 [rows, me-1]} block maxima per query block."""
    c = c or O.cfg()
    bq, bk = c.block_q, c.block_k
    nq, nk = -(-tokens // bq), -(-tokens // bk)
    i_hi = nq if i_hi is None else i_hi
    inv = np.float32(1.0) / np.sqrt(np.float32(qc.shape[1]))
    sink_blocks = -(-min(c.sink_tokens, tokens) // bk)
    mask = np.zeros((nq, nk), np.uint8)
    rep = dict(min_decision=np.inf, min_decision_rel=np.inf, min_cmp=np.inf, near_ties=0,
               decisions=0, comparisons=0, block_max={})
    me = {}
    for i in range(i_lo, i_hi):
        sl = O.sink_local_index_set(i, tokens, c)
        mask[i, sl] = 1
        after = [j for j in sl if j >= sink_blocks]
        me[i] = max(sink_blocks, after[0]) if after else sink_blocks
    for i0 in range(i_lo, i_hi, chunk):
        blocks = [i for i in range(i0, min(i0 + chunk, i_hi)) if me[i] > sink_blocks]
        if not blocks:
            continue
        mmax = max(me[i] for i in blocks)
        r0, r1 = bq * blocks[0], min(bq * (blocks[-1] + 1), tokens)
        k0, k1 = bk * sink_blocks, bk * mmax
        prods = qc[r0:r1].astype(np.float32) @ kc[k0:k1].astype(np.float32).T
        bm = prods.reshape(r1 - r0, mmax - sink_blocks, bk).max(-1).astype(np.int32)
        rs = (qs[r0:r1, None] * ks[None, sink_blocks:mmax]) * inv       # fp32, left to right
        est = (rs * bm.astype(np.float32)).astype(np.float32)           # max_then_dequantize
        diff = est.astype(np.float64) - bound[r0:r1, None]
        for i in blocks:
            a, b = bq * i - r0, min(bq * (i + 1), tokens) - r0
            nb = me[i] - sink_blocks
            d = diff[a:b, :nb]
            best = d.max(0)
            raw = (best >= 0).astype(np.uint8)
            O.C_LIB.oracle_segment_aggregate(raw, nb, c.segment_size)
            mask[i, sink_blocks:me[i]] = raw
            arg = d.argmax(0)
            bnd = np.abs(bound[r0 + a + arg])
            rep["min_decision"] = min(rep["min_decision"], float(np.abs(best).min()))
            rep["min_decision_rel"] = min(rep["min_decision_rel"],
                                          float((np.abs(best) / np.maximum(bnd, 1e-300)).min()))
            rep["min_cmp"] = min(rep["min_cmp"], float(np.abs(d).min()))
            rep["near_ties"] += int((np.abs(best) <= 1e-9 * np.maximum(bnd, 1.0)).sum())
            rep["decisions"] += nb
            rep["comparisons"] += d.size
            if want_block_max:
                rep["block_max"][i] = bm[a:b, :nb]
    return mask, rep
