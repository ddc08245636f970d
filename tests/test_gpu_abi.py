"""GPU: behaviour of the C ABI around the kernels — the reference's error
classes, input validation of the Python mirror, several contexts / streams
in one process, and the chunked host pipeline's isolation from stale device
memory.

Reference behaviour mirrored:
* block_sparse_attention throws std::domain_error("... query row g attends no
  tokens") for the first empty row (sparse_attention.hpp:88-90);
* HeadInput::validate rejects mismatched shapes (matrix.hpp:66-72);
* the functions are pure and thread-safe (run_pipeline calls them
  concurrently, runner.hpp:57) — results do not depend on which thread /
  stream / context computes them (acceptance.cpp:381-419).
"""
import threading

import numpy as np
import pytest

from helpers import Inputs
from paper_2505_24179_b200 import sale

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch():
    import torch as t
    assert t.cuda.is_available(), "GPU tests need a B200"
    return t


# ------------------------------------------------------------ domain error

@pytest.mark.parametrize("use_range", [False, True])
def test_empty_row_raises_domain_error(torch, use_range):
    """A mask whose query block 3 keeps only its diagonal block 7: rows
    192..223 (tokens before key block 7) attend nothing."""
    N, Hq, Hkv = 512, 2, 1
    inp = Inputs("gaussian", 3, 1, N, Hq, Hkv)
    q, k, v = inp.torch()
    nq, nk, nw = sale.grid(N)
    cells = np.zeros((1, Hq, nq, nk), np.uint8)
    for i in range(nq):
        cells[0, :, i, : 2 * i + 2] = 1  # all causal blocks
    cells[0, 1, 3, :] = 0
    cells[0, 1, 3, 7] = 1                 # head 1, query block 3: the diagonal block only
    mask = torch.from_numpy(sale.pack_mask(cells, N).view(np.int32)).cuda()
    with pytest.raises(ArithmeticError, match=r"query row 192 attends no tokens \(batch 0, head 1\)"):
        if use_range:
            sale.block_sparse_attention(q, k, v, mask, q_blocks=(3, nq))
        else:
            sale.block_sparse_attention(q, k, v, mask)
    # the same mask with the sink block restored is fine
    cells[0, 1, 3, 0] = 1
    mask = torch.from_numpy(sale.pack_mask(cells, N).view(np.int32)).cuda()
    _, cov = sale.block_sparse_attention(q, k, v, mask, coverage=True)
    assert int(cov.min()) >= 1
    # a range that does not contain the empty rows does not raise
    cells[0, 1, 3, 0] = 0
    mask = torch.from_numpy(sale.pack_mask(cells, N).view(np.int32)).cuda()
    sale.block_sparse_attention(q, k, v, mask, q_blocks=(5, nq))


def test_single_head_message_is_the_reference_message(torch):
    N = 256
    inp = Inputs("gaussian", 4, 1, N, 1, 1)
    q, k, v = inp.torch()
    mask = torch.zeros((1, 1, 4, 1), dtype=torch.int32, device="cuda")
    with pytest.raises(ArithmeticError) as e:
        sale.block_sparse_attention(q, k, v, mask)
    assert str(e.value) == "block_sparse_attention: query row 0 attends no tokens"


# -------------------------------------------------------- input validation

def test_python_mirror_rejects_malformed_tensors(torch):
    inp = Inputs("gaussian", 5, 1, 256, 4, 2)
    q, k, v = inp.torch()
    with pytest.raises(ValueError, match="contiguous"):
        qkv = torch.cat([q, q], dim=2)
        sale.prefill(qkv[:, :, :4], k, v, 0.004)          # head slice of a fused tensor
    with pytest.raises(ValueError, match="CUDA"):
        sale.prefill(q.cpu(), k, v, 0.004)
    with pytest.raises(ValueError, match="bfloat16"):
        sale.prefill(q.float(), k, v, 0.004)
    with pytest.raises(ValueError, match="value shape"):
        sale.prefill(q, k, v[:, :128].contiguous(), 0.004)
    with pytest.raises(ValueError, match="key rows"):
        sale.block_sparse_attention(q, k[:, :128].contiguous(), v[:, :128].contiguous())
    with pytest.raises(ValueError, match="mask"):
        sale.block_sparse_attention(q, k, v, torch.zeros((1, 4, 2, 1), dtype=torch.int32,
                                                         device="cuda"))
    qc, qs, kc, ks = sale.quantize_qk(q, k)
    with pytest.raises(ValueError, match="k_scales"):
        sale.selection_pass(q, k, qc, qs, kc, ks[:, :, :4].contiguous(), 0.004)
    with pytest.raises(ValueError, match="shape differs"):
        sale.calibrate_model([(q, k, v), (q[:, :128].contiguous(), k[:, :128].contiguous(),
                                          v[:, :128].contiguous())])


# ------------------------------------------- contexts, streams, threads

def test_two_contexts_two_threads_two_streams(torch):
    """Two ctxs (one per host thread, each on its own stream) run prefills
    concurrently; every result is bit-identical to the single-context one."""
    inp_a = Inputs("sink_local", 7, 1, 2048, 8, 2)
    inp_b = Inputs("sink_local", 8, 2, 1024, 4, 1)
    tensors = [inp_a.torch(), inp_b.torch()]
    want = [sale.prefill(*t, 0.004) for t in tensors]
    torch.cuda.synchronize()
    ctxs = [sale.Context(0), sale.Context(0)]
    got = [[None] * 3 for _ in range(2)]
    errors = []

    def worker(w):
        try:
            stream = torch.cuda.Stream()
            with torch.cuda.stream(stream):
                for r in range(3):
                    got[w][r] = sale.prefill(*tensors[w], 0.004, ctx=ctxs[w])
            stream.synchronize()
        except Exception as e:  # surfaced below
            errors.append(e)

    th = [threading.Thread(target=worker, args=(w,)) for w in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errors, errors
    for w in range(2):
        for r in range(3):
            assert torch.equal(got[w][r].view(torch.int16), want[w].view(torch.int16))
    for c in ctxs:
        c.close()


def test_workspace_handoff_between_streams(torch):
    """Back-to-back calls of one ctx on two streams with no host sync: the
    second waits for the first's workspace use (ws event), so both masks and
    outputs equal the serial results."""
    inp = Inputs("sink_local", 9, 1, 4096, 8, 2)
    q, k, v = inp.torch()
    nq, nk, nw = sale.grid(4096)
    m_ref = [torch.empty((1, 8, nq, nw), dtype=torch.int32, device="cuda") for _ in range(2)]
    o_ref = [sale.prefill(q, k, v, t, mask_out=m) for t, m in zip((0.004, 0.05), m_ref)]
    torch.cuda.synchronize()
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    m = [torch.zeros_like(x) for x in m_ref]
    with torch.cuda.stream(s1):
        o1 = sale.prefill(q, k, v, 0.004, mask_out=m[0])
    with torch.cuda.stream(s2):
        o2 = sale.prefill(q, k, v, 0.05, mask_out=m[1])
    torch.cuda.synchronize()
    assert torch.equal(m[0], m_ref[0]) and torch.equal(m[1], m_ref[1])
    assert torch.equal(o1.view(torch.int16), o_ref[0].view(torch.int16))
    assert torch.equal(o2.view(torch.int16), o_ref[1].view(torch.int16))


def test_entry_points_keep_the_callers_device(torch):
    if torch.cuda.device_count() < 2:
        inp = Inputs("gaussian", 2, 1, 256, 2, 1)
        q, k, v = inp.torch()
        before = torch.cuda.current_device()
        sale.prefill(q, k, v, 0.01)
        assert torch.cuda.current_device() == before
        return
    # two devices: a ctx on cuda:1 driven while cuda:0 is current
    inp = Inputs("sink_local", 2, 1, 1024, 4, 1)
    with torch.cuda.device(1):
        t1 = [torch.from_numpy(x.view(np.int16)).view(torch.bfloat16).to("cuda:1")
              for x in (inp.q16, inp.k16, inp.v16)]
    ctx1 = sale.Context(1)
    torch.cuda.set_device(0)
    with torch.cuda.device(1):
        o1 = sale.prefill(*t1, 0.004, ctx=ctx1)
    assert torch.cuda.current_device() == 0
    o0 = sale.prefill(*inp.torch(), 0.004)
    assert torch.equal(o1.cpu().view(torch.int16), o0.cpu().view(torch.int16))
    ctx1.close()


# ------------------------------------------- chunked host pipeline

def test_chunked_host_pipeline_ignores_stale_device_rows(torch):
    """A first prefill_host leaves NaN K / V in the ctx's device buffers; the
    second call's chunk c must not read chunk c+1's rows before they arrive
    (the diagonal K / V tile extends past the chunk end): its output is finite
    and bit-identical to the device prefill."""
    B, N, Hq, Hkv = 1, 16384, 4, 1
    ctx = sale.Context(0)
    nan16 = np.full((B, N, Hkv, 128), 0x7FC0, np.uint16)   # bf16 NaN
    q16 = np.zeros((B, N, Hq, 128), np.uint16)
    out = np.empty((B, N, Hq, 128), np.uint16)
    sale.prefill_host(q16, nan16, nan16, [0.004] * Hq, out, ctx=ctx)
    inp = Inputs("sink_local", 12, B, N, Hq, Hkv)
    sale.prefill_host(inp.q16, inp.k16, inp.v16, [0.004] * Hq, out, ctx=ctx)
    want = sale.prefill(*inp.torch(), 0.004).cpu().view(torch.int16).numpy().view(np.uint16)
    assert np.array_equal(out, want)
    ctx.close()
