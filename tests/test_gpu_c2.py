"""The C2 parity gate (BASELINE.json configs[1]): Llama-3.1-8B attention shape
(32 Q / 8 KV heads, d = 128), 32K tokens, one B200 — every head, every query
block — and its extension to 128K (configs[2]) for four heads.

Checked against the oracle (oracle/sale_oracle.c, pinned bit-for-bit to the
unmodified reference in tests/test_oracle.py) on the identical bf16 inputs:
* q / k codes and scales, bit-exact, all heads (quant.hpp:95-119);
* masks, bit-exact, all 32 heads x all 512 query blocks at 32K
  (selection.hpp:211-274): sink / local sets, bounds and the segment rule from
  the C oracle, middle-block estimates restated with exact BLAS products
  (helpers.blas_selection, itself checked against oracle_selection_pass here);
* running max bit-exact, exp_sum within 2 ulp (K2a's table exp vs glibc),
  bounds, and the integer block maxima of every estimated block, bit-exact,
  for 8 heads (two KV groups);
* every output row of 4 heads within 2e-2 max-abs / 1e-3 mean-abs of the
  oracle's block_sparse_attention on the same mask (sparse_attention.hpp:37-97);
* the decision margin report of SURVEY.md Appendix A.3: the smallest
  |max_r(est_r - bound_r)| over every estimated block, and the near-tie count
  — the l~ difference (<= 2 ulp, ~1e-16 relative in the bound) could flip a
  block only if a margin came within ~1e-15 of zero.
"""
import json
import os
import warnings

import numpy as np
import pytest

from helpers import Inputs, O, blas_selection
from paper_2505_24179_b200 import sale

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

ATOL_MAX, ATOL_MEAN = 2e-2, 1e-3
ULP_TOL = 2


@pytest.fixture(scope="module")
def torch():
    import torch as t
    assert t.cuda.is_available()
    return t


_INPUTS = {}


def _inputs(hq, hkv):
    """32K-token GQA sink-local inputs (seed 7), cached per shape."""
    if (hq, hkv) not in _INPUTS:
        _INPUTS.clear()
        _INPUTS[(hq, hkv)] = Inputs("sink_local", 7, 1, 32768, hq, hkv)
    return _INPUTS[(hq, hkv)]


def _np(t):
    return t.detach().cpu().numpy()


def _ulp_diff(a, b):
    a = np.asarray(a, np.float64).view(np.int64)
    b = np.asarray(b, np.float64).view(np.int64)
    return np.abs(a - b)


def _report(name, rep):
    """Margin report: a pytest warning (shown in the -q summary) and a JSON
    file next to the GPU run's other outputs."""
    rep = {k: (v.item() if hasattr(v, "item") else v) for k, v in rep.items()}
    warnings.warn(f"{name}: {json.dumps(rep)}", UserWarning)
    out = os.environ.get("SALE_REPORT_DIR", "gpurun_out")
    if os.path.isdir(out):
        with open(os.path.join(out, f"margin_{name}.json"), "w") as f:
            json.dump(rep, f, indent=1)


def _merge(reps):
    m = dict(min_decision=np.inf, min_decision_rel=np.inf, min_cmp=np.inf, near_ties=0,
             decisions=0, comparisons=0)
    for r in reps:
        for k in ("min_decision", "min_decision_rel", "min_cmp"):
            m[k] = min(m[k], r[k])
        for k in ("near_ties", "decisions", "comparisons"):
            m[k] += r[k]
    return m


def _oracle_head(inp, b, h, tau, want_block_max=False):
    """Oracle quantization, statistics and the (BLAS-exact) mask of one head."""
    g = h // inp.G
    qh, kh = inp.qh(b, h), inp.kh(b, g)
    qc, qs = O.quantize(qh, 1)
    kc, ks = O.quantize(kh, 32)
    c = O.cfg(tau=tau)
    m, l, bound = O.selection_stats(qh, kh, c)
    mask, rep = blas_selection(qc, qs, kc, ks, bound, inp.N, c, want_block_max=want_block_max)
    return dict(qc=qc, qs=qs, kc=kc, ks=ks, m=m, l=l, bound=bound, mask=mask, rep=rep)


@pytest.mark.parametrize("model,hq,hkv,tau", [("llama", 32, 8, 0.004), ("llama", 32, 8, 0.064),
                                              ("qwen", 28, 4, 0.004)])
def test_c2_gate_32k_all_heads(torch, model, hq, hkv, tau):
    """Llama-3.1-8B (configs[1]) and the Qwen2.5-7B shape (G = 7, configs[3]'s
    head layout) at 32K: every head, every query block."""
    inp = _inputs(hq, hkv)
    N, Hq, Hkv = inp.N, inp.Hq, inp.Hkv
    q, k, v = inp.torch()
    nq, nk, nw = sale.grid(N)
    # ---- the B200 path: quantization, Selection-Pass, prefill
    qc, qs, kc, ks = sale.quantize_qk(q, k)
    mask = sale.selection_pass(q, k, qc, qs, kc, ks, tau)
    pmask = torch.empty_like(mask)
    out = sale.prefill(q, k, v, tau, mask_out=pmask)
    assert torch.equal(mask, pmask), "prefill's mask differs from the stage-wise Selection-Pass"
    qc, qs, kc, ks = (_np(x) for x in (qc, qs, kc, ks))
    cells = sale.unpack_mask(_np(mask), N)
    # ---- debug instance for two KV groups (8 q heads): stats + block maxima
    dbg_groups = (0, Hkv - 1)
    dbg = {}
    for g in dbg_groups:
        hs = slice(g * inp.G, (g + 1) * inp.G)
        qg, kg = q[:, :, hs].contiguous(), k[:, :, g:g + 1].contiguous()
        a, b_, c_, d_ = sale.quantize_qk(qg, kg)
        mg, dg = sale.selection_pass(qg, kg, a, b_, c_, d_, tau, debug=True)
        assert torch.equal(mg, mask[:, hs]), f"group {g}: debug instance mask differs"
        dbg[g] = dg

    # ---- oracle, every head (threads: the C oracle and BLAS release the GIL)
    want_bm = {g * inp.G + r for g in dbg_groups for r in range(inp.G)}
    orc = O.map_heads(lambda h: _oracle_head(inp, 0, h, tau, h in want_bm), Hq,
                      threads=min(8, os.cpu_count() or 1))
    for g in range(Hkv):
        o = orc[g * inp.G]
        np.testing.assert_array_equal(kc[0, :, g], o["kc"], err_msg=f"k codes g={g}")
        np.testing.assert_array_equal(ks[0, g], o["ks"], err_msg=f"k scales g={g}")
    for h in range(Hq):
        o = orc[h]
        np.testing.assert_array_equal(qc[0, :, h], o["qc"], err_msg=f"q codes h={h}")
        np.testing.assert_array_equal(qs[0, h], o["qs"], err_msg=f"q scales h={h}")
        bad = np.argwhere(cells[0, h] != o["mask"])
        assert bad.size == 0, f"mask h={h}: {len(bad)} cells differ, first (i, j) = {bad[:4]}"
    # ---- statistics, bounds and block maxima of the debug heads
    for g in dbg_groups:
        dg = dbg[g]
        rm, es, bd = (_np(x)[0] for x in (dg.running_max, dg.exp_sum, dg.bound))
        bmax = _np(dg.block_max)[0]
        for r in range(inp.G):
            h = g * inp.G + r
            o = orc[h]
            valid = ~np.isnan(o["m"])
            assert valid.sum() == 64 * (nq - 3)
            np.testing.assert_array_equal(rm[r][valid], o["m"][valid], err_msg=f"m h={h}")
            assert _ulp_diff(es[r][valid], o["l"][valid]).max() <= ULP_TOL, f"l h={h}"
            np.testing.assert_allclose(bd[r][valid], o["bound"][valid], rtol=1e-15, atol=1e-15)
            for i, bm in o["rep"]["block_max"].items():
                est_blocks = 4 * ((2 * i - 5) // 4)  # full segments (the GPU skips the forced run)
                np.testing.assert_array_equal(
                    bmax[r, 64 * i:64 * i + 64, 1:1 + est_blocks], bm[:, :est_blocks],
                    err_msg=f"block max h={h} i={i}")
    # ---- the BLAS restatement itself against oracle_selection_pass (2 heads)
    for h in (0, Hq - 1):
        qh, kh = inp.qh(0, h), inp.kh(0, h // inp.G)
        o = orc[h]
        ref = O.selection_pass(qh, kh, o["qc"], o["qs"], o["kc"], o["ks"], c=O.cfg(tau=tau))
        np.testing.assert_array_equal(ref, o["mask"], err_msg=f"BLAS restatement h={h}")
    # ---- every output row of four heads
    outf = _np(out.float())

    def attn(h):
        g = h // inp.G
        ref, _, st = O.block_sparse_attention(inp.qh(0, h), inp.kh(0, g), inp.vh(0, g), cells[0, h])
        assert st == 0
        err = np.abs(outf[0, :, h, :128].astype(np.float64) - ref)
        return float(err.max()), float(err.mean())

    out_heads = (0, 9, Hq - 10, Hq - 1)
    errs = O.map_heads(lambda x: attn(out_heads[x]), 4, threads=4)
    for (mx, mn), h in zip(errs, out_heads):
        assert mx < ATOL_MAX and mn < ATOL_MEAN, (h, mx, mn)
    rep = _merge([o["rep"] for o in orc])
    rep.update(tokens=N, heads=Hq, tau=tau, max_abs_err=max(e[0] for e in errs),
               mean_abs_err=max(e[1] for e in errs),
               density=float(cells[0].sum() / (Hq * sum(2 * i + 2 for i in range(nq)))))
    assert rep["near_ties"] == 0 and rep["min_decision_rel"] > 1e-12, rep
    _report(f"c2_32k_{model}_tau{tau}", rep)


@pytest.mark.parametrize("model,hq,hkv,heads", [("llama", 32, 8, (0, 9, 18, 27)),
                                                 ("qwen", 28, 4, (0, 9, 17, 26))])
def test_c2_extension_128k_four_heads_all_query_blocks(torch, model, hq, hkv, heads):
    """configs[2] / configs[3] size: masks of every query block, statistics and
    bounds of four heads (spread over the KV groups) against the oracle."""
    N, tau = 131072, 0.004
    inp = Inputs("sink_local", 7, 1, N, hq, hkv)
    q, k, v = inp.torch()
    nq, nk, nw = sale.grid(N)
    mask = torch.empty((1, hq, nq, nw), dtype=torch.int32, device="cuda")
    sale.prefill(q, k, v, tau, mask_out=mask)
    cells = sale.unpack_mask(_np(mask), N)
    dbg = {}
    for h in heads:  # the debug instance on the head's own (1 q / 1 kv) problem
        g = h // inp.G
        qg, kg = q[:, :, h:h + 1].contiguous(), k[:, :, g:g + 1].contiguous()
        a, b_, c_, d_ = sale.quantize_qk(qg, kg)
        mg, dg = sale.selection_pass(qg, kg, a, b_, c_, d_, tau, debug=True)
        assert torch.equal(mg[0, 0], mask[0, h])
        dbg[h] = (_np(dg.running_max)[0, 0], _np(dg.exp_sum)[0, 0])
        del dg
    orc = O.map_heads(lambda x: _oracle_head(inp, 0, heads[x], tau), len(heads), threads=4)
    for h, o in zip(heads, orc):
        bad = np.argwhere(cells[0, h] != o["mask"])
        assert bad.size == 0, f"mask h={h}: {len(bad)} cells differ, first (i, j) = {bad[:4]}"
        valid = ~np.isnan(o["m"])
        np.testing.assert_array_equal(dbg[h][0][valid], o["m"][valid], err_msg=f"m h={h}")
        assert _ulp_diff(dbg[h][1][valid], o["l"][valid]).max() <= ULP_TOL, f"l h={h}"
    rep = _merge([o["rep"] for o in orc])
    rep.update(tokens=N, heads=list(heads), tau=tau)
    assert rep["near_ties"] == 0 and rep["min_decision_rel"] > 1e-12, rep
    _report("c3_128k_tau0.004" if model == "llama" else f"c4_128k_{model}_tau0.004", rep)
