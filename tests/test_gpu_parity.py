"""GPU parity: every stage of the B200 path through the C ABI against the
oracle on identical bf16 inputs.

Bars (BASELINE.json north_star): codes, scales, integer block maxima and
masks bit-exact; running max bit-exact; exp_sum within 2 ulp (CUDA vs glibc
double exp); attention output within 2e-2 max-abs and 1e-3 mean-abs of the
oracle's block_sparse_attention on the same mask (bf16 MMA, fp32 accumulate).
"""
import numpy as np
import pytest

from helpers import Inputs, O, max_abs, mean_abs, oracle_quant, oracle_select
from paper_2505_24179_b200 import sale

pytestmark = pytest.mark.gpu

ATOL_MAX = 2e-2
ATOL_MEAN = 1e-3


@pytest.fixture(scope="module")
def torch():
    import torch as t
    assert t.cuda.is_available(), "GPU tests need a B200"
    return t


def _to_np(t):
    return t.detach().cpu().numpy()


# ------------------------------------------------------ golden (reference)

def test_golden_reference_fixture(torch):
    """tests/golden/ref_gqa_640.npz was produced by the unmodified reference
    (tests/golden/make_golden.py); no oracle involved."""
    import os
    g = np.load(os.path.join(os.path.dirname(__file__), "golden", "ref_gqa_640.npz"))
    t = lambda a: torch.from_numpy(a.view(np.int16)).view(torch.bfloat16).cuda()
    q, k, v = t(g["q16"]), t(g["k16"]), t(g["v16"])
    N = q.shape[1]
    qc, qs, kc, ks = (_to_np(x) for x in sale.quantize_qk(q, k))
    np.testing.assert_array_equal(kc[0, :, 0], g["k_codes"])
    np.testing.assert_array_equal(ks[0, 0], g["k_scales"])
    qct, qst, kct, kst = sale.quantize_qk(q, k)
    for tau in (0.004, 0.05):
        mask = sale.selection_pass(q, k, qct, qst, kct, kst, tau)
        cells = sale.unpack_mask(_to_np(mask), N)
        for h in range(q.shape[2]):
            np.testing.assert_array_equal(cells[0, h], g[f"mask_{h}_{tau}"])
    mask = sale.selection_pass(q, k, qct, qst, kct, kst, 0.004)
    out, cov = sale.block_sparse_attention(q, k, v, mask, coverage=True)
    full = sale.full_attention(q, k, v)
    out, cov, full = _to_np(out.float()), _to_np(cov), _to_np(full.float())
    for h in range(q.shape[2]):
        np.testing.assert_array_equal(qc[0, :, h], g[f"q_codes_{h}"])
        np.testing.assert_array_equal(qs[0, h], g[f"q_scales_{h}"])
        np.testing.assert_array_equal(cov[0, h], g[f"coverage_{h}"])
        for got, ref in ((out[0, :, h], g[f"sparse_out_{h}"]), (full[0, :, h], g[f"full_out_{h}"])):
            assert max_abs(got, ref) < ATOL_MAX and mean_abs(got, ref) < ATOL_MEAN


# ------------------------------------------------------------------ stage 1

@pytest.mark.parametrize("kind,N,Hq,Hkv,d", [("sink_local", 1000, 4, 2, 128),
                                              ("gaussian", 517, 8, 8, 128),
                                              ("sink_local", 300, 4, 1, 64),
                                              ("gaussian", 33, 2, 1, 16)])
def test_quantize_bit_exact(torch, kind, N, Hq, Hkv, d):
    inp = Inputs(kind, 11, 2, N, Hq, Hkv, d)
    q, k, _ = inp.torch()
    qc, qs, kc, ks = (_to_np(x) for x in sale.quantize_qk(q, k, d))
    qq, kq = oracle_quant(inp)
    for b in range(inp.B):
        for h in range(Hq):
            np.testing.assert_array_equal(qc[b, :, h, :d], qq[(b, h)][0])
            assert (qc[b, :, h, d:] == 0).all()
            np.testing.assert_array_equal(qs[b, h], qq[(b, h)][1])
        for g in range(Hkv):
            np.testing.assert_array_equal(kc[b, :, g, :d], kq[(b, g)][0])
            np.testing.assert_array_equal(ks[b, g], kq[(b, g)][1])
    # the standalone entry points agree with the fused launch
    qc2, qs2 = sale.quantize_per_token(q)
    kc2, ks2 = sale.quantize_per_key_block(k)
    np.testing.assert_array_equal(_to_np(qc2), qc)
    np.testing.assert_array_equal(_to_np(ks2), ks)


def test_quantize_hand_rows(torch):
    # test_quant.cpp:16-33: [7,-7,3.5,0] -> codes [7,-7,4,0] (half away from
    # zero), scale 1; an all-zero row gets scale 1 and zero codes.
    x = np.zeros((1, 2, 1, 128), np.float32)
    x[0, 0, 0, :4] = [7.0, -7.0, 3.5, 0.0]
    xt = torch.from_numpy(x).to(torch.bfloat16).cuda()
    codes, scales = sale.quantize_per_token(xt)
    codes, scales = _to_np(codes), _to_np(scales)
    assert list(codes[0, 0, 0, :4]) == [7, -7, 4, 0]
    assert scales[0, 0, 0] == 1.0 and scales[0, 0, 1] == 1.0
    assert (codes[0, 1] == 0).all()


# ------------------------------------------------------------------ stage 2

def _check_selection(inp, taus, dbg_check=True, geom=None):
    """geom = (sink_tokens, local_tokens_min, segment_size) with blocks 64/32,
    or None for the default SelectionConfig."""
    import torch
    q, k, _ = inp.torch()
    sink, local, seg = geom or (32, 128, 4)
    cfg = sale.SelectionConfig(sink, local, seg, 64, 32)
    qc, qs, kc, ks = sale.quantize_qk(q, k, inp.d)
    mask, dbg = sale.selection_pass(q, k, qc, qs, kc, ks, taus, inp.d, config=cfg, debug=True)
    torch.cuda.synchronize()
    cells = sale.unpack_mask(_to_np(mask), inp.N)
    ref = oracle_select(inp, taus, debug=True, geom=geom)
    m, l, bound, bmax = (_to_np(x) for x in (dbg.running_max, dbg.exp_sum, dbg.bound,
                                             dbg.block_max))
    # the B200 path estimates the full segments only: the trailing partial run
    # is forced on by segment_aggregate (selection.hpp:188) whatever its
    # estimate, so its products are never needed.
    nq, nk, _ = sale.grid(inp.N)
    sb = -(-min(sink, inp.N) // 32)
    nl = -(-local // 32)
    i = np.arange(inp.N) // 64
    lo = np.maximum(2 * i - nl, 0)
    E = np.where(lo > sb, seg * ((lo - sb) // seg), 0)
    j = np.arange(nk)[None, :]
    est_blocks = (j >= sb) & (j < sb + E[:, None])
    for (b, h), (rmask, rdbg) in ref.items():
        np.testing.assert_array_equal(cells[b, h], rmask, err_msg=f"mask b={b} h={h} geom={geom}")
        if not dbg_check:
            continue
        est = ~np.isnan(rdbg["m"])
        np.testing.assert_array_equal(m[b, h][est], rdbg["m"][est])
        # exp_sum: table-driven double exp (~0.5 ulp) vs glibc -> allow 2 ulp
        np.testing.assert_allclose(l[b, h][est], rdbg["l"][est], rtol=4.5e-16, atol=0)
        np.testing.assert_allclose(bound[b, h][est], rdbg["bound"][est], rtol=1e-15, atol=1e-15)
        ok = (rdbg["block_max"] != np.iinfo(np.int32).min) & est_blocks
        assert ok.sum() == est_blocks.sum()
        np.testing.assert_array_equal(bmax[b, h][ok], rdbg["block_max"][ok])
    return cells, ref


@pytest.mark.parametrize("geom,N,seed", [((1, 32, 1), 1000, 1), ((40, 95, 5), 2048, 2),
                                         ((64, 128, 4), 1536, 3), ((300, 700, 9), 4096, 4),
                                         ((33, 256, 2), 3000, 5), ((1, 33, 3), 777, 6),
                                         ((200, 64, 7), 2500, 7), ((32, 128, 1), 2048, 8)])
def test_selection_general_geometry(torch, geom, N, seed):
    """Non-default sink_tokens / local_tokens_min / segment_size with the
    64/32 blocks (selection.hpp:18-38, :92-123, :182-195): masks, statistics
    and estimated block maxima against the oracle; then the sparse pass, the
    one-shot prefill, query-block ranges and the chunked host pipeline on
    the same geometry."""
    inp = Inputs("sink_local" if seed % 2 else "gaussian", 40 + seed, 1, N, 4, 2)
    taus = [0.004, 0.05, 0.0005, 0.02]
    cells, _ = _check_selection(inp, taus, geom=geom)
    q, k, v = inp.torch()
    cfg = sale.SelectionConfig(*geom, 64, 32)
    nq, nk, nw = sale.grid(N)
    pm = torch.empty((1, 4, nq, nw), dtype=torch.int32, device="cuda")
    out = sale.prefill(q, k, v, taus, mask_out=pm, config=cfg)
    np.testing.assert_array_equal(sale.unpack_mask(_to_np(pm), N), cells)
    ref = _oracle_attention(inp, cells, inp.heads())
    outf = _to_np(out.float())
    for (b, h), (o, rcov, st) in ref.items():
        assert st == 0
        got = outf[b, :, h, :inp.d]
        assert max_abs(got, o) < ATOL_MAX and mean_abs(got, o) < ATOL_MEAN
    for r in sale.query_block_split(nq, 2):
        part = torch.zeros_like(pm)
        po = sale.prefill(q, k, v, taus, mask_out=part, config=cfg, q_blocks=r)
        assert torch.equal(part[:, :, r[0]:r[1]], pm[:, :, r[0]:r[1]])
        t0, t1 = 64 * r[0], min(64 * r[1], N)
        assert torch.equal(po[:, t0:t1].view(torch.int16), out[:, t0:t1].view(torch.int16))
    host = np.empty_like(inp.q16)
    sale.prefill_host(inp.q16, inp.k16, inp.v16, taus, host, config=cfg)
    assert np.array_equal(host, out.cpu().view(torch.int16).numpy().view(np.uint16))


@pytest.mark.parametrize("N", [2048, 1000, 200])
def test_selection_bit_exact_small(torch, N):
    inp = Inputs("sink_local", 7, 1, N, 8, 2)
    _check_selection(inp, [0.004, 0.05, 0.004, 1e-9, 0.5, 0.004, 0.016, 0.1])


def test_selection_llama_4k(torch):
    """configs[0]: Llama-3.1-8B shape (32 Q / 8 KV heads), seq 4K, tau 0.004."""
    inp = Inputs("sink_local", 7, 1, 4096, 32, 8)
    _check_selection(inp, 0.004)


def test_selection_qwen_group_of_seven(torch):
    """configs[3] shape family: Qwen2.5-7B has 28 Q / 4 KV heads (G = 7, not a
    multiple of the estimator's 4-head CTAs or the attention's head pairs)."""
    inp = Inputs("sink_local", 13, 1, 1536, 14, 2)
    cells, _ = _check_selection(inp, [0.004, 0.016] * 7)
    q, k, v = inp.torch()
    mask = torch.from_numpy(sale.pack_mask(cells, inp.N).view(np.int32)).cuda()
    out, cov = sale.block_sparse_attention(q, k, v, mask, coverage=True)
    ref = _oracle_attention(inp, cells, inp.heads())
    out, cov = _to_np(out.float()), _to_np(cov)
    for (b, h), (o, rcov, st) in ref.items():
        got = out[b, :, h, :inp.d]
        assert max_abs(got, o) < ATOL_MAX and mean_abs(got, o) < ATOL_MEAN
        np.testing.assert_array_equal(cov[b, h], rcov)


def test_selection_gaussian_batch(torch):
    inp = Inputs("gaussian", 3, 2, 1536, 4, 1)
    _check_selection(inp, 0.004)


# ------------------------------------------------------------------ stage 3

def _oracle_attention(inp, cells, heads):
    def one(i):
        b, h = heads[i]
        g = h // inp.G
        m = cells[b, h] if cells is not None else None
        if m is None:
            return O.full_attention(inp.qh(b, h), inp.kh(b, g), inp.vh(b, g)), None, 0
        return O.block_sparse_attention(inp.qh(b, h), inp.kh(b, g), inp.vh(b, g), m)
    return dict(zip(heads, O.map_heads(one, len(heads))))


@pytest.mark.parametrize("kind,N,Hq,Hkv", [("gaussian", 1024, 4, 1), ("sink_local", 777, 2, 2),
                                           ("sink_local", 64, 2, 1), ("gaussian", 129, 2, 1)])
def test_dense_attention(torch, kind, N, Hq, Hkv):
    inp = Inputs(kind, 5, 1, N, Hq, Hkv)
    q, k, v = inp.torch()
    out, cov = sale.block_sparse_attention(q, k, v, None, inp.d, coverage=True)
    out = _to_np(out.float())
    cov = _to_np(cov)
    ref = _oracle_attention(inp, None, inp.heads())
    for (b, h), (o, _, _) in ref.items():
        got = out[b, :, h, :inp.d]
        assert max_abs(got, o) < ATOL_MAX, (b, h, max_abs(got, o))
        assert mean_abs(got, o) < ATOL_MEAN, (b, h, mean_abs(got, o))
        np.testing.assert_array_equal(cov[b, h], np.arange(1, N + 1))


def test_sparse_attention_selected_mask(torch):
    inp = Inputs("sink_local", 7, 1, 2048, 8, 2)
    q, k, v = inp.torch()
    qc, qs, kc, ks = sale.quantize_qk(q, k)
    mask = sale.selection_pass(q, k, qc, qs, kc, ks, 0.004)
    out, cov = sale.block_sparse_attention(q, k, v, mask, coverage=True)
    cells = sale.unpack_mask(_to_np(mask), inp.N)
    ref = _oracle_attention(inp, cells, inp.heads())
    out, cov = _to_np(out.float()), _to_np(cov)
    for (b, h), (o, rcov, st) in ref.items():
        assert st == 0
        got = out[b, :, h, :inp.d]
        assert max_abs(got, o) < ATOL_MAX
        assert mean_abs(got, o) < ATOL_MEAN
        np.testing.assert_array_equal(cov[b, h], rcov)


def test_sparse_attention_random_masks(torch):
    """test_sparse_exec.cpp:24-38 random_valid_mask: anchors on block 0 and the
    overlapping blocks, others kept with probability p; plus future bits set
    (sparse_attention.hpp ignores them)."""
    rng = np.random.default_rng(220)
    inp = Inputs("gaussian", 9, 1, 1000, 4, 2)
    q, k, v = inp.torch()
    nq, nk, _ = sale.grid(inp.N)
    cells = np.zeros((1, inp.Hq, nq, nk), np.uint8)
    for h in range(inp.Hq):
        p = 0.2 + 0.2 * h
        for i in range(nq):
            for j in range(nk):
                kb, qe = 32 * j, min(64 * i + 64, inp.N)
                future = kb >= qe
                overl = not future and 32 * j + 32 > 64 * i
                cells[0, h, i, j] = 1 if (j == 0 or overl or rng.random() < p) else 0
                if future and h == 3:
                    cells[0, h, i, j] = 1
    words = torch.from_numpy(sale.pack_mask(cells, inp.N).view(np.int32)).cuda()
    out, cov = sale.block_sparse_attention(q, k, v, words, coverage=True)
    ref = _oracle_attention(inp, cells, inp.heads())
    out, cov = _to_np(out.float()), _to_np(cov)
    for (b, h), (o, rcov, st) in ref.items():
        got = out[b, :, h, :inp.d]
        assert max_abs(got, o) < ATOL_MAX
        assert mean_abs(got, o) < ATOL_MEAN
        np.testing.assert_array_equal(cov[b, h], rcov)


@pytest.mark.parametrize("N,Hq,Hkv", [(1, 2, 1), (31, 3, 1), (65, 2, 2), (191, 4, 1), (193, 3, 1)])
def test_tiny_and_ragged_lengths(torch, N, Hq, Hkv):
    """Whole prefill at lengths around the block edges (one token, a partial
    sink block, a ragged second query block, the first query block with a
    middle region) and odd group sizes (a head pair with one head): masks
    bit-exact, output and coverage against the oracle on the same mask."""
    inp = Inputs("sink_local", 21, 1, N, Hq, Hkv)
    cells, _ = _check_selection(inp, [0.004 + 0.01 * h for h in range(Hq)])
    q, k, v = inp.torch()
    mask = torch.from_numpy(sale.pack_mask(cells, inp.N).view(np.int32)).cuda()
    out, cov = sale.block_sparse_attention(q, k, v, mask, coverage=True)
    ref = _oracle_attention(inp, cells, inp.heads())
    out, cov = _to_np(out.float()), _to_np(cov)
    for (b, h), (o, rcov, st) in ref.items():
        got = out[b, :, h, :inp.d]
        assert max_abs(got, o) < ATOL_MAX and mean_abs(got, o) < ATOL_MEAN
        np.testing.assert_array_equal(cov[b, h], rcov)
    taus = [0.004 + 0.01 * h for h in range(Hq)]
    np.testing.assert_array_equal(_to_np(sale.prefill(q, k, v, taus).view(torch.int16)),
                                  _to_np(sale.block_sparse_attention(q, k, v, mask).view(torch.int16)))


# ------------------------------------------------------------- accounting

def test_flop_count(torch):
    inp = Inputs("sink_local", 7, 2, 1500, 4, 2)
    q, k, _ = inp.torch()
    qc, qs, kc, ks = sale.quantize_qk(q, k)
    mask = sale.selection_pass(q, k, qc, qs, kc, ks, [0.004, 0.01, 0.05, 0.3])
    counts = _to_np(sale.flop_accounting(mask, inp.N))
    cells = sale.unpack_mask(_to_np(mask), inp.N)
    for b in range(inp.B):
        for h in range(inp.Hq):
            r = O.flop_accounting(cells[b, h], inp.N)
            assert tuple(counts[b, h]) == (r["computed"], r["skipped"], r["total"])


def test_quantize_ties_and_tiny_groups(torch):
    """Exact half-away ties ((k + 1/2) * scale with scale a power of two) and
    groups whose scale is subnormal (the kernel's exact 2^64 rescaling path),
    per token (Q) and per 32-token block (K), against the C oracle."""
    rng = np.random.default_rng(3)
    N = 64
    x = np.zeros((1, N, 2, 128), np.float32)
    for n in range(N):
        for h in range(2):
            e = [-3, -131, 5, -126][(n + h) % 4]
            ties = (rng.integers(-7, 7, 128) + 0.5) * 2.0 ** e
            row = np.where(rng.random(128) < 0.5, ties, rng.normal(0, 4, 128) * 2.0 ** e)
            row[0] = 7 * 2.0 ** e                          # peak -> scale 2^e exactly
            x[0, n, h] = np.clip(row, -7 * 2.0 ** e, 7 * 2.0 ** e)
    xt = torch.from_numpy(x).to(torch.bfloat16)
    xb = xt.float().numpy()                                # the bf16 values the kernel sees
    qc, qs = (_to_np(t) for t in sale.quantize_per_token(xt.cuda()))
    kc, ks = (_to_np(t) for t in sale.quantize_per_key_block(xt.cuda()))
    for h in range(2):
        codes, scales = O.quantize(np.ascontiguousarray(xb[0, :, h]), 1)
        np.testing.assert_array_equal(qc[0, :, h], codes)
        np.testing.assert_array_equal(qs[0, h], scales)
        codes, scales = O.quantize(np.ascontiguousarray(xb[0, :, h]), 32)
        np.testing.assert_array_equal(kc[0, :, h], codes)
        np.testing.assert_array_equal(ks[0, h], scales)


# -------------------------------------------------------------- pipeline

def test_prefill_matches_stages_and_host_path(torch):
    inp = Inputs("sink_local", 7, 1, 2048, 8, 2)
    q, k, v = inp.torch()
    taus = [0.004] * 4 + [0.02] * 4
    nq, nk, nw = sale.grid(inp.N)
    mask_out = torch.empty((1, inp.Hq, nq, nw), dtype=torch.int32, device="cuda")
    out = sale.prefill(q, k, v, taus, mask_out=mask_out)
    qc, qs, kc, ks = sale.quantize_qk(q, k)
    mask = sale.selection_pass(q, k, qc, qs, kc, ks, taus)
    out2 = sale.block_sparse_attention(q, k, v, mask)
    assert torch.equal(mask, mask_out)
    assert torch.equal(out, out2)
    host_out = np.empty_like(inp.q16)
    sale.prefill_host(inp.q16, inp.k16, inp.v16, taus, host_out)
    np.testing.assert_array_equal(host_out, _to_np(out.view(torch.int16)).view(np.uint16))


@pytest.mark.parametrize("B,N,Hq,Hkv", [(1, 16384, 8, 2), (2, 20000, 4, 1), (3, 3000, 7, 1), (1, 65600, 4, 1)])
def test_chunked_host_pipeline_bit_identical(torch, B, N, Hq, Hkv):
    """sale_b200_prefill_host streams token chunks through three streams (H2D /
    kernels / D2H overlap; 15 uneven chunks at >= 64K tokens, 8 at >= 16K, 4 at >= 2K); every stage
    reads only its own and earlier chunks, so the output equals the one-shot
    device prefill bit for bit (batch > 1 exercises the strided 2-D copies)."""
    inp = Inputs("sink_local", 9, B, N, Hq, Hkv)
    q, k, v = inp.torch()
    taus = [0.004 * (1 + h % 3) for h in range(Hq)]
    out = sale.prefill(q, k, v, taus)
    host_out = torch.empty(q.shape, dtype=torch.bfloat16).pin_memory()
    pin = lambda a: torch.from_numpy(a.view(np.int16)).view(torch.bfloat16).pin_memory()
    sale.prefill_host(pin(inp.q16), pin(inp.k16), pin(inp.v16), taus, host_out)
    assert torch.equal(host_out.view(torch.int16), out.cpu().view(torch.int16))


@pytest.mark.parametrize("B,N,Hq,Hkv,parts", [(1, 20000, 4, 1, 3), (2, 4100, 7, 1, 2)])
def test_query_block_ranges_compose_to_the_full_prefill(torch, B, N, Hq, Hkv, parts):
    """a (batch, KV group) unit split across GPUs by query-block
    ranges (K/V replicated): the ranges' masks and outputs equal the one-shot
    prefill bit for bit; the dense-mask attention likewise."""
    inp = Inputs("sink_local", 17, B, N, Hq, Hkv)
    q, k, v = inp.torch()
    taus = [0.004 * (1 + h % 3) for h in range(Hq)]
    nq, nk, nw = sale.grid(N)
    full_mask = torch.zeros((B, Hq, nq, nw), dtype=torch.int32, device="cuda")
    full = sale.prefill(q, k, v, taus, mask_out=full_mask)
    dense = sale.block_sparse_attention(q, k, v, None)
    mask = torch.zeros_like(full_mask)
    for i0, i1 in sale.query_block_split(nq, parts):
        part = sale.prefill(q, k, v, taus, mask_out=mask, q_blocks=(i0, i1))
        t0, t1 = 64 * i0, min(64 * i1, N)
        assert torch.equal(part[:, t0:t1].view(torch.int16), full[:, t0:t1].view(torch.int16))
        dpart = sale.block_sparse_attention(q, k, v, None, q_blocks=(i0, i1))
        assert torch.equal(dpart[:, t0:t1].view(torch.int16), dense[:, t0:t1].view(torch.int16))
    assert torch.equal(mask, full_mask)
    with pytest.raises(ValueError):
        sale.prefill(q, k, v, taus, q_blocks=(2, nq))  # even inner boundary


def test_invalid_arguments(torch):
    inp = Inputs("gaussian", 1, 1, 256, 4, 2)
    q, k, v = inp.torch()
    qc, qs, kc, ks = sale.quantize_qk(q, k)
    with pytest.raises(ValueError):
        sale.selection_pass(q, k, qc, qs, kc, ks, 0.0)
    with pytest.raises(ValueError):
        sale.selection_pass(q, k, qc, qs, kc, ks, 1.0)
    cfg = sale.default_config()
    cfg.segment_size = 0
    with pytest.raises(ValueError):
        sale.selection_pass(q, k, qc, qs, kc, ks, 0.004, config=cfg)
    cfg = sale.default_config()
    cfg.block_q = 32  # only the 64 / 32 blocks are implemented
    with pytest.raises(NotImplementedError):
        sale.selection_pass(q, k, qc, qs, kc, ks, 0.004, config=cfg)
