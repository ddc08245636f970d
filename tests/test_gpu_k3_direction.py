"""K3 walks the key tiles of alternate waves of query blocks in opposite
directions (L2 reuse of K / V, attention.cu). On the bench sizes the reversed
CTAs only appear past the first wave (74 query blocks for Llama on 148 SMs),
so these tests shrink the group to one query block (SALE_B200_K3_WAVE_QB,
read once per process: a subprocess) and check, on sequences short enough for
the oracle, that every other query block computed back to front still matches
block_sparse_attention (sparse_attention.hpp:37-97): the sink tile, with the
largest logits of the sink_local workload, then comes last and moves the
running reference (the O rescale path), the diagonal tile comes first."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))

CHECK = r"""
import sys
import numpy as np
import torch
sys.path.insert(0, {here!r})
from helpers import Inputs, O, max_abs, mean_abs
from paper_2505_24179_b200 import sale

inp = Inputs({kind!r}, {seed}, {B}, {N}, {Hq}, {Hkv})
q, k, v = inp.torch()
if {dense}:
    cells = None
    out, cov = sale.block_sparse_attention(q, k, v, None, coverage=True)
else:
    qc, qs, kc, ks = sale.quantize_qk(q, k)
    mask = sale.selection_pass(q, k, qc, qs, kc, ks, 0.004)
    out, cov = sale.block_sparse_attention(q, k, v, mask, coverage=True)
    cells = sale.unpack_mask(mask.cpu().numpy(), inp.N)
out = out.float().cpu().numpy()
cov = cov.cpu().numpy()
worst = 0.0
for b, h in inp.heads():
    g = h // inp.G
    if cells is None:
        o = O.full_attention(inp.qh(b, h), inp.kh(b, g), inp.vh(b, g))
        rcov = np.arange(1, inp.N + 1)
    else:
        o, rcov, st = O.block_sparse_attention(inp.qh(b, h), inp.kh(b, g), inp.vh(b, g), cells[b, h])
        assert st == 0
    got = out[b, :, h, :inp.d]
    assert max_abs(got, o) < 2e-2 and mean_abs(got, o) < 1e-3, (b, h, max_abs(got, o), mean_abs(got, o))
    np.testing.assert_array_equal(cov[b, h], rcov)
    worst = max(worst, max_abs(got, o))
print("ok", worst)
"""


def _run(wave, **kw):
    env = dict(os.environ, SALE_B200_K3_WAVE_QB=str(wave))
    code = CHECK.format(here=HERE, **kw)
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                       cwd=os.path.dirname(HERE), timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    assert r.stdout.strip().splitlines()[-1].startswith("ok")


@pytest.mark.parametrize("wave", [1, 3])
def test_reversed_tile_order_sparse(wave):
    _run(wave, kind="sink_local", seed=13, B=1, N=2048, Hq=4, Hkv=1, dense=False)


def test_reversed_tile_order_dense_ragged_batch():
    _run(1, kind="gaussian", seed=17, B=2, N=1000, Hq=3, Hkv=1, dense=True)
