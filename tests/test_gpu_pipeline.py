"""GPU: the orchestration layer (csrc/pipeline.cu) against the unmodified
reference (oracle/_ref): run_pipeline's RunReport, sweep_thresholds and the
calibration ladder, on identical bf16-valued inputs (MHA heads of the
reference generator). Counts, sparsity and coverage statistics are exact
(they follow from bit-exact masks); l1 errors agree within the attention
tolerance (bf16 outputs vs the reference's fp32 / double arithmetic)."""
import ctypes as C

import numpy as np
import pytest

from helpers import Inputs, O
from paper_2505_24179_b200 import sale

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(O.REF is None, reason="oracle/_ref not built")]


@pytest.fixture(scope="module")
def torch():
    import torch as t
    assert t.cuda.is_available(), "GPU tests need a B200"
    return t


def _ref_heads(inp):
    f = lambda x16: np.ascontiguousarray(np.stack([inp.head(x16, 0, h) for h in range(inp.Hq)]))
    return f(inp.q16).ravel(), f(inp.k16).ravel(), f(inp.v16).ravel()


def _err_close(ours, ref):
    return abs(ours - ref) <= 0.03 * ref + 2e-3


@pytest.mark.parametrize("n,h,d", [(1024, 4, 64), (1337, 3, 128)])
def test_run_pipeline_matches_reference(torch, n, h, d):
    inp = Inputs("sink_local", 7, 1, n, h, h, d)
    q, k, v = inp.torch()
    taus = [0.004, 0.02, 0.001, 0.05, 0.3][:h]
    rep = sale.run_pipeline(q, k, v, taus, head_dim=d)
    out = np.zeros(10 * h)
    assert O.REF.ref_run_report(*_ref_heads(inp), h, n, d, np.asarray(taus, np.float64), 0,
                                4, out) == 0
    assert rep["kind"] == "run_report" and rep["tokens"] == n and rep["heads"] == h
    t = rep["timing"]
    assert abs(t["overhead_ratio"] - (t["quantization_ms"] + t["selection_ms"]) / t["dense_ms"]) < 1e-12
    for i, hr in enumerate(rep["head_reports"]):
        r = out[10 * i:10 * i + 10]
        assert hr["head"] == i and hr["tau"] == taus[i]
        assert (hr["computed_blocks"], hr["skipped_blocks"], hr["total_blocks"]) == tuple(int(x) for x in r[2:5])
        assert hr["sparsity"] == r[0]
        assert (hr["coverage"]["min"], hr["coverage"]["max"]) == (int(r[5]), int(r[6]))
        assert hr["coverage"]["mean"] == pytest.approx(r[7], rel=1e-12)
        assert _err_close(hr["err"], r[1]), (i, hr["err"], r[1])


def test_run_pipeline_dense_mask(torch):
    inp = Inputs("sink_local", 11, 1, 700, 2, 2, 64)
    q, k, v = inp.torch()
    rep = sale.run_pipeline(q, k, v, [0.004, 0.004], dense_mask=True, head_dim=64)
    out = np.zeros(20)
    assert O.REF.ref_run_report(*_ref_heads(inp), 2, 700, 64, np.full(2, 0.004), 1, 2, out) == 0
    for i, hr in enumerate(rep["head_reports"]):
        assert hr["sparsity"] == 0.0 and hr["skipped_blocks"] == 0
        assert hr["total_blocks"] == int(out[10 * i + 4])
        assert hr["err"] == 0.0 and out[10 * i + 1] == 0.0  # same kernel, all-true mask
        assert hr["coverage"]["max"] == 700 and hr["coverage"]["min"] == 1


def test_sweep_thresholds_matches_reference(torch):
    inp = Inputs("sink_local", 5, 1, 1024, 3, 3, 64)
    q, k, v = inp.torch()
    taus = [0.001, 0.004, 0.016, 0.064]
    rows = sale.sweep_thresholds(q, k, v, taus, head_dim=64)
    ref = np.zeros(3 * len(taus))
    assert O.REF.ref_sweep(*_ref_heads(inp), 3, 1024, 64, np.asarray(taus), len(taus), 4, ref) == 0
    for t, row in enumerate(rows):
        assert row["tau"] == taus[t]
        assert row["sparsity"] == pytest.approx(ref[3 * t + 1], abs=1e-15)
        assert _err_close(row["err"], ref[3 * t + 2]), (t, row["err"], ref[3 * t + 2])
    assert all(a["sparsity"] <= b["sparsity"] for a, b in zip(rows, rows[1:]))


@pytest.mark.parametrize("theta", [0.4, 0.15])
def test_calibration_ladder_matches_reference(torch, theta):
    """calibrate_model on the device (every head's ladder in the same
    launches) vs the reference calibrate_head per head: same tau, flag and
    halvings (errors are checked away from theta so the last-digit
    difference between bf16 and fp32 outputs cannot flip a rung)."""
    n, h, d = 1024, 3, 64
    samples = [Inputs("sink_local", s, 1, n, h, h, d) for s in (7, 8)]
    prof = sale.calibrate_model([s.torch() for s in samples], theta=theta, tau0=0.008,
                                max_halvings=12, head_dim=d, sample_names=["seed7", "seed8"])
    assert prof["theta"] == theta and prof["samples"] == ["seed7", "seed8"]
    for hh in range(h):
        qs = np.concatenate([s.head(s.q16, 0, hh).ravel() for s in samples])
        ks = np.concatenate([s.head(s.k16, 0, hh).ravel() for s in samples])
        vs = np.concatenate([s.head(s.v16, 0, hh).ravel() for s in samples])
        tau, flag, halv = np.zeros(1), C.c_int32(), np.zeros(1, np.int64)
        assert O.REF.ref_calibrate_head(qs, ks, vs, 2, n, d, theta, 0.008, 12, tau,
                                        C.byref(flag), halv) == 0
        got = prof["heads"][hh]
        assert got["head"] == hh and got["layer"] == 0
        assert (got["tau"], got["halvings"]) == (tau[0], int(halv[0])), (hh, got, tau, halv)
        assert got["flag"] == ("converged" if flag.value == 0 else "floor-reached")
        assert got["tau"] == 0.008 / 2 ** got["halvings"]


def test_l1_error_matches_oracle(torch):
    inp = Inputs("gaussian", 3, 2, 300, 2, 1, 96)
    q, k, v = inp.torch()
    dense = sale.full_attention(q, k, v, head_dim=96)
    mask = sale.selection_pass(q, k, *sale.quantize_qk(q, k, head_dim=96), 0.05, head_dim=96)
    sparse = sale.block_sparse_attention(q, k, v, mask, head_dim=96)
    got = sale.l1_error(dense, sparse, head_dim=96)
    f = lambda t, b, hh: t[b, :, hh, :96].float().cpu().numpy()
    for b in range(2):
        for hh in range(2):
            assert got[b, hh] == pytest.approx(O.l1_error(f(dense, b, hh), f(sparse, b, hh)), rel=1e-9)
