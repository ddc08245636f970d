"""Parity at the BASELINE.json sizes (configs[1]: 32K, configs[2]: 128K,
Llama-3.1-8B attention shape) where the full CPU oracle would take hours:

* masks of sampled query blocks against the oracle restated per block
  (oracle C stats + exact integer products via fp32 BLAS: |p| <= 6272 < 2^24,
  so float matmul of the int codes is exact) + segment aggregation;
* attention outputs of sampled rows against a float64 evaluation of
  sparse_attention.hpp:37-97 restricted to the GPU mask;
* size-independent properties: tau monotonicity (selection_pass's bound is
  monotone in tau), the all-ones mask equals the dense run bit-for-bit,
  coverage = sum over selected causal blocks.
"""
import numpy as np
import pytest

from helpers import O, Inputs
from paper_2505_24179_b200 import sale

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


@pytest.fixture(scope="module")
def torch():
    import torch as t
    assert t.cuda.is_available()
    return t


def _np(t):
    return t.detach().cpu().numpy()


def oracle_mask_row(q, k, qc, qs, kc, ks, i, tau, n):
    """selection.hpp:224-271 for one query block i (default geometry)."""
    nk = (n + 31) // 32
    row = np.zeros(nk, np.uint8)
    sl = O.sink_local_index_set(i, n)
    row[sl] = 1
    me = 2 * i - 4
    if i < 3 or me <= 1:
        return row
    q0, q1 = 64 * i, min(64 * i + 64, n)
    m = np.empty(q1 - q0)
    l = np.empty(q1 - q0)
    O.C_LIB.oracle_sink_local_stats(q, k, n, q.shape[1], 64, 32, i, sl, len(sl), m, l)
    bounds = np.array([O.threshold_bound(tau, a, b) for a, b in zip(m, l)])
    prods = qc[q0:q1].astype(np.float32) @ kc[32:32 * me].astype(np.float32).T  # exact ints
    bm = prods.reshape(q1 - q0, me - 1, 32).max(-1)                          # [rows, blocks]
    inv = np.float32(1.0) / np.sqrt(np.float32(q.shape[1]))
    rs = (qs[q0:q1, None] * ks[None, 1:me]) * inv                             # fp32, left to right
    est = (rs * bm.astype(np.float32)).astype(np.float32)
    raw = (est.astype(np.float64) >= bounds[:, None]).any(0).astype(np.uint8)
    O.C_LIB.oracle_segment_aggregate(raw, len(raw), 4)
    row[1:me] = raw
    return row


def sampled_attention(q, k, v, cells, rows):
    """float64 sparse_attention.hpp semantics for selected rows."""
    d = q.shape[1]
    out = np.empty((len(rows), d))
    for n_, g in enumerate(rows):
        i = g // 64
        keys = np.arange(g + 1)
        keep = cells[i, keys // 32] > 0
        kk = keys[keep]
        s = (k[kk].astype(np.float64) @ q[g].astype(np.float64)) / np.sqrt(d)
        w = np.exp(s - s.max())
        out[n_] = (w / w.sum()) @ v[kk].astype(np.float64)
    return out


@pytest.mark.parametrize("N,tau", [(32768, 0.004), (131072, 0.004), (131072, 0.064)])
def test_sampled_parity_llama(torch, N, tau):
    inp = Inputs("sink_local", 7, 1, N, 32, 8)
    q, k, v = inp.torch()
    nq, nk, nw = sale.grid(N)
    mask = torch.empty((1, 32, nq, nw), dtype=torch.int32, device="cuda")
    out = sale.prefill(q, k, v, tau, mask_out=mask)
    cells = sale.unpack_mask(_np(mask), N)
    outf = _np(out.float())
    rng = np.random.default_rng(N)
    for h in (0, 5, 18, 31):
        g = h // 4
        qh, kh, vh = inp.qh(0, h), inp.kh(0, g), inp.vh(0, g)
        qc, qs = O.quantize(qh, 1)
        kc, ks = O.quantize(kh, 32)
        blocks = sorted(set([3, 4, nq - 1, nq - 2] + list(rng.integers(3, nq, 6))))
        for i in blocks:
            ref = oracle_mask_row(qh, kh, qc, qs, kc, ks, int(i), tau, N)
            np.testing.assert_array_equal(cells[0, h, i], ref, err_msg=f"h={h} i={i}")
        rows = sorted(set([0, 63, 64, N - 1] + list(rng.integers(0, N, 24))))
        ref = sampled_attention(qh, kh, vh, cells[0, h], rows)
        got = outf[0, rows, h, :128]
        err = np.abs(got - ref)
        assert err.max() < 2e-2 and err.mean() < 1e-3, (h, err.max(), err.mean())


def test_tau_monotone_and_dense_identity_128k(torch):
    N = 131072
    inp = Inputs("sink_local", 11, 1, N, 32, 8)
    q, k, v = inp.torch()
    qc, qs, kc, ks = sale.quantize_qk(q, k)
    prev = None
    for tau in (0.064, 0.016, 0.004, 0.001):
        m = _np(sale.selection_pass(q, k, qc, qs, kc, ks, tau)).view(np.uint32)
        if prev is not None:  # smaller tau selects a superset (test_selection.cpp:282-302)
            assert ((prev & ~m) == 0).all()
        prev = m
    # coverage of the selected mask == sum over selected causal blocks
    mask = sale.selection_pass(q, k, qc, qs, kc, ks, 0.004)
    _, cov = sale.block_sparse_attention(q, k, v, mask, coverage=True)
    cells = sale.unpack_mask(_np(mask), N)
    nq, nk, nw = sale.grid(N)
    for h in (0, 13, 31):
        for i in (0, 5, 1000, nq - 1):
            rows = np.arange(64 * i, min(64 * i + 64, N))
            sel = np.flatnonzero(cells[0, h, i])
            want = [sum(min(32 * j + 32, g + 1) - 32 * j for j in sel if 32 * j <= g) for g in rows]
            np.testing.assert_array_equal(_np(cov)[0, h, rows], want)
    # the all-ones mask through the sparse path == the dense (mask = NULL) run
    ones = torch.full((1, 32, nq, nw), -1, dtype=torch.int32, device="cuda")
    a = sale.block_sparse_attention(q, k, v, ones)
    b = sale.block_sparse_attention(q, k, v, None)
    assert torch.equal(a, b)


def test_long_sequence_300k_sampled(torch):
    """Beyond 256K tokens the attention kernel's tile lists take several
    build rounds (> 2048 key tiles per query block) and the estimator several
    units per query tile: sampled masks and rows against the oracle, and the
    all-ones mask against the dense run bit for bit."""
    N, tau = 300032, 0.016
    inp = Inputs("sink_local", 5, 1, N, 2, 1)
    q, k, v = inp.torch()
    nq, nk, nw = sale.grid(N)
    mask = torch.empty((1, 2, nq, nw), dtype=torch.int32, device="cuda")
    out = sale.prefill(q, k, v, tau, mask_out=mask)
    cells = sale.unpack_mask(_np(mask), N)
    outf = _np(out.float())
    rng = np.random.default_rng(3)
    for h in (0, 1):
        qh, kh, vh = inp.qh(0, h), inp.kh(0, 0), inp.vh(0, 0)
        qc, qs = O.quantize(qh, 1)
        kc, ks = O.quantize(kh, 32)
        for i in sorted(set([3, nq - 1] + list(rng.integers(3, nq, 3)))):
            ref = oracle_mask_row(qh, kh, qc, qs, kc, ks, int(i), tau, N)
            np.testing.assert_array_equal(cells[0, h, i], ref, err_msg=f"h={h} i={i}")
        rows = sorted(set([0, N - 1] + list(rng.integers(N // 2, N, 10))))
        ref = sampled_attention(qh, kh, vh, cells[0, h], rows)
        err = np.abs(outf[0, rows, h, :128] - ref)
        assert err.max() < 2e-2 and err.mean() < 1e-3, (h, err.max(), err.mean())
    ones = torch.full_like(mask, -1)
    dense = sale.block_sparse_attention(q, k, v, None)
    assert torch.equal(sale.block_sparse_attention(q, k, v, ones), dense)
