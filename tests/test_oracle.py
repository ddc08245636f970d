"""The oracle pinned: the C restatement (oracle/sale_oracle.c) against
(a) the reference's own golden values (proj/tests/*.cpp, acceptance.cpp) and
(b) the unmodified reference headers compiled into oracle/_ref, bit-for-bit,
on seeded inputs. CPU only."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2505_24179_b200 import sale

needs_ref = pytest.mark.skipif(O.REF is None, reason="oracle/_ref not built")


def head(kind, seed, n, d, h=0):
    return sale.workload_head_f32(kind, seed, n, d, h)


def bf16(x):
    return sale.bf16_bits_to_f32(sale.f32_to_bf16_bits(x))


# ----------------------------------------------------------- golden values

def test_quant_hand_rows():
    # test_quant.cpp:16-33
    c, s = O.quantize(np.array([[0, 0, 0, 0]], np.float32), 1)
    assert s[0] == 1.0 and (c == 0).all()
    c, s = O.quantize(np.array([[7.0, -7.0, 3.5, 0.0]], np.float32), 1)
    assert s[0] == 1.0 and list(c[0]) == [7, -7, 4, 0]


def test_scalar_products_and_argmax():
    # test_quant.cpp:114-126: q=3 -> code 7 (scale 3/7); k = 2, -2 -> codes 7, -7
    qc, qs = O.quantize(np.array([[3.0]], np.float32), 1)
    kc, ks = O.quantize(np.array([[2.0], [-2.0]], np.float32), 2)
    prods = np.empty(2, np.int32)
    rs = np.empty(1, np.float32)
    O.C_LIB.oracle_approx_weight_block(qc, qs, 1, 0, 1, kc, ks, 2, 0, 2, 1, prods, rs)
    assert list(prods) == [49, -49]
    # test_quant.cpp:159-170: ties resolve to the lowest index
    import ctypes as C
    v, col = C.c_float(), C.c_int64()
    O.C_LIB.oracle_max_then_dequantize(np.array([4, 4, 4], np.int32), 3, 2.0, C.byref(v),
                                       C.byref(col))
    assert col.value == 0 and v.value == 8.0
    O.C_LIB.oracle_max_then_dequantize(np.array([6, -6], np.int32), 2, 0.5, C.byref(v),
                                       C.byref(col))
    assert v.value == 3.0 and col.value == 0


def test_threshold_bound_closed_form():
    # test_selection.cpp:131-144
    assert O.threshold_bound(0.25, 3.5, 4.0) == pytest.approx(3.5)
    assert O.threshold_bound(0.004, 0.0, 10.0) == pytest.approx(-3.2188758248682006, rel=1e-12)
    assert np.isfinite(O.threshold_bound(1e-300, 0.0, 1e-60))


def test_sink_local_geometry():
    # test_selection.cpp:51-81
    assert list(O.sink_local_index_set(0, 512)) == [0, 1]
    assert list(O.sink_local_index_set(7, 512)) == [0, 10, 11, 12, 13, 14, 15]
    assert list(O.sink_local_index_set(0, 64)) == [0, 1]
    s = O.sink_local_index_set(4, 300)
    assert s[0] == 0 and s[-1] == (300 + 31) // 32 - 1
    with pytest.raises(IndexError):
        O.sink_local_index_set(2, 128)


def test_segment_aggregate_cases():
    # test_selection.cpp:170-204
    def agg(row, seg):
        a = np.array(row, np.uint8)
        O.C_LIB.oracle_segment_aggregate(a, len(a), seg)
        return list(a)
    assert agg([1, 0, 1, 0, 0], 1) == [1, 0, 1, 0, 0]
    assert agg([1, 0, 0, 0, 0, 0, 0, 0], 4) == [1, 1, 1, 1, 0, 0, 0, 0]
    assert agg([0, 0, 0, 0, 0], 4) == [0, 0, 0, 0, 1]


def test_acceptance_sparsity_pins():
    # acceptance.cpp:319-346: sink_local seed 9900, d 64, tau 0.004 ->
    # sparsity 0.058824 (N=1024) and 0.286538 (N=4096), printed to 6 digits
    for n, want in ((1024, 0.058824), (4096, 0.286538)):
        q, k, _ = head("sink_local", 9900, n, 64)
        qc, qs = O.quantize(q, 1)
        kc, ks = O.quantize(k, 32)
        m = O.selection_pass(q, k, qc, qs, kc, ks)
        c = O.flop_accounting(m, n)
        assert round(c["skipped"] / c["total"], 6) == want


def test_frozen_full_attention():
    # test_core.cpp:83-96: gaussian_head(42, 4, 2), frozen float64 oracle values
    q, k, v = head("gaussian", 42, 4, 2)
    expected = np.array([-0.45516559481620789, 1.2834087610244751, -0.20167922986371103,
                         -0.24234179398790157, -0.26102200377751661, -0.097599191509265104,
                         0.018673329263568073, -1.1848281022247265]).reshape(4, 2)
    assert np.abs(O.full_attention(q, k, v) - expected).max() < 1e-6


def test_sparse_accepts_all_true_and_rejects_empty():
    # test_sparse_exec.cpp:43-56 and :116-121
    q, k, v = head("gaussian", 200, 257, 16)
    nq, nk = 5, 9
    out, cov, st = O.block_sparse_attention(q, k, v, np.ones((nq, nk), np.uint8))
    assert st == 0 and (cov == np.arange(1, 258)).all()
    assert np.abs(out - O.full_attention(q, k, v)).max() < 1e-5
    q, k, v = head("gaussian", 250, 64, 8)
    _, _, st = O.block_sparse_attention(q, k, v, np.zeros((1, 2), np.uint8), 32, 32)
    assert st == 2  # domain_error


# ----------------------------------------------- C restatement == reference

GEOMETRIES = [(512, 16, 64, 32, 4), (300, 32, 64, 32, 4), (257, 8, 64, 32, 4),
              (640, 64, 64, 32, 4), (500, 16, 32, 32, 4), (480, 16, 16, 32, 2),
              (512, 16, 64, 16, 1), (2048, 128, 64, 32, 4)]


@needs_ref
@pytest.mark.parametrize("n,d,bq,bk,seg", GEOMETRIES)
@pytest.mark.parametrize("kind", ["sink_local", "gaussian"])
@pytest.mark.parametrize("round_bf16", [False, True])
def test_c_oracle_matches_reference(n, d, bq, bk, seg, kind, round_bf16):
    q, k, v = head(kind, 71 + n, n, d)
    if round_bf16:  # the B200 parity inputs: exact .5 ties in the quantizer occur
        q, k, v = bf16(q), bf16(k), bf16(v)
    qc, qs = O.quantize(q, 1)
    kc, ks = O.quantize(k, bk)
    rqc, rqs = np.empty_like(qc), np.empty_like(qs)
    rkc, rks = np.empty_like(kc), np.empty_like(ks)
    assert O.REF.ref_quantize_per_token(q, n, d, rqc, rqs) == 0
    assert O.REF.ref_quantize_per_key_block(k, n, d, bq, bk, rkc, rks) == 0
    np.testing.assert_array_equal(qc, rqc)
    np.testing.assert_array_equal(qs, rqs)
    np.testing.assert_array_equal(kc, rkc)
    np.testing.assert_array_equal(ks, rks)
    for tau in (0.004, 0.05):
        c = O.cfg(tau=tau, block_q=bq, block_k=bk, segment_size=seg)
        mask = O.selection_pass(q, k, qc, qs, kc, ks, c)
        rmask = np.empty_like(mask)
        assert O.REF.ref_selection_pass(q, k, n, d, qc, qs, kc, ks, tau, 32, 128, seg, bq, bk,
                                        rmask) == 0
        np.testing.assert_array_equal(mask, rmask)
        # the debug (no early exit) path cannot change the mask
        mask2, dbg = O.selection_pass(q, k, qc, qs, kc, ks, c, debug=True)
        np.testing.assert_array_equal(mask2, rmask)
    out, cov, st = O.block_sparse_attention(q, k, v, mask, bq, bk)
    rout, rcov = np.empty_like(out), np.empty_like(cov)
    assert O.REF.ref_block_sparse_attention(q, k, v, n, d, mask, bq, bk, rout, rcov) == st
    np.testing.assert_array_equal(out, rout)
    np.testing.assert_array_equal(cov, rcov)
    counts = np.empty(3, np.int64)
    O.REF.ref_flop_accounting(mask, n, bq, bk, counts)
    r = O.flop_accounting(mask, n, bq, bk)
    assert (r["computed"], r["skipped"], r["total"]) == tuple(counts)


@needs_ref
@pytest.mark.parametrize("n,d", [(320, 16), (1000, 128), (2048, 64)])
def test_c_oracle_stats_match_reference(n, d):
    q, k, _ = head("sink_local", 3, n, d)
    q, k = bf16(q), bf16(k)
    nq = (n + 63) // 64
    for i in range(nq):
        blocks = O.sink_local_index_set(i, n)
        rows = min(64, n - 64 * i)
        m, l = np.empty(rows), np.empty(rows)
        rm, rl = np.empty(rows), np.empty(rows)
        O.C_LIB.oracle_sink_local_stats(q, k, n, d, 64, 32, i, blocks, len(blocks), m, l)
        O.REF.ref_sink_local_stats(q, k, n, d, 64, 32, i, blocks, len(blocks), rm, rl)
        np.testing.assert_array_equal(m, rm)
        np.testing.assert_array_equal(l, rl)


@needs_ref
def test_full_attention_matches_reference():
    q, k, v = head("gaussian", 104, 96, 128)
    out = O.full_attention(q, k, v)
    rout = np.empty_like(out)
    O.REF.ref_full_attention(q, k, v, 96, 128, rout)
    np.testing.assert_array_equal(out, rout)


@needs_ref
def test_random_geometries_match_reference():
    """test_selection.cpp:297-346: random grids, windows and segment sizes."""
    rng = np.random.default_rng(700)
    for trial in range(20):
        n = int(33 + rng.integers(288))
        d = int(4 + rng.integers(13))
        bq, bk = int(1 + rng.integers(70)), int(1 + rng.integers(40))
        sink, seg = int(1 + rng.integers(40)), int(1 + rng.integers(5))
        local = bk + int(rng.integers(64))
        tau = float(2.0 ** (-3.0 - rng.random() * 10.0))
        q, k, v = head("sink_local" if trial % 2 else "gaussian", 710 + trial, n, d)
        qc, qs = O.quantize(q, 1)
        kc, ks = O.quantize(k, bk)
        c = O.Cfg(tau, sink, local, seg, bq, bk)
        mask = O.selection_pass(q, k, qc, qs, kc, ks, c)
        rmask = np.empty_like(mask)
        assert O.REF.ref_selection_pass(q, k, n, d, qc, qs, kc, ks, tau, sink, local, seg, bq, bk,
                                        rmask) == 0
        np.testing.assert_array_equal(mask, rmask)
