"""CPU-side checks of the product: the C-ABI library loads and exports every
symbol include/sale_b200.h declares, fails loudly without a GPU, and its host
logic (workload generator, mask packing, default-geometry formulas, sharding)
matches the reference / oracle. No GPU compute here."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from oracle import oracle as O
from paper_2505_24179_b200 import sale

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "sale_b200.h")).read()
    return sorted(set(re.findall(r"\b(sale_b200_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = sale.load_library()
    syms = declared_symbols()
    assert len(syms) >= 16
    for s in syms:
        assert hasattr(lib, s), f"{s} not exported"
    assert lib.sale_b200_version() == 1


def test_library_is_sm100a_native():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", sale.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
    for mnemonic in ("UTCIMMA", "UTCHMMA", "UTMALDG", "LDTM", "STTM", "FFMA2"):
        assert mnemonic in out, mnemonic


def test_ctx_create_fails_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(RuntimeError):
        sale.Context(0)


def test_default_config():
    c = sale.SelectionConfig()
    sale.load_library().sale_b200_default_config(C.byref(c))
    assert (c.sink_tokens, c.local_tokens_min, c.segment_size, c.block_q, c.block_k) == \
        (32, 128, 4, 64, 32)


@pytest.mark.skipif(O.REF is None, reason="oracle/_ref not built")
@pytest.mark.parametrize("kind,seed,n,d,h", [("sink_local", 7, 300, 32, 2), ("gaussian", 42, 4, 2, 0),
                                             ("sink_local", 9900, 1024, 64, 0),
                                             ("sink_local", 5, 777, 128, 3)])
def test_workload_generator_matches_reference(kind, seed, n, d, h):
    q, k, v = sale.workload_head_f32(kind, seed, n, d, h)
    rq, rk, rv = (np.empty((n, d), np.float32) for _ in range(3))
    assert O.REF.ref_workload_head(1 if kind == "sink_local" else 0, seed, n, d, h, rq, rk, rv) == 0
    np.testing.assert_array_equal(q, rq)
    np.testing.assert_array_equal(k, rk)
    np.testing.assert_array_equal(v, rv)


def test_gqa_workload_extends_reference_heads():
    """KV head g and query head 0 of its group are the reference head g
    (bf16-rounded); other query heads share the planted terms."""
    q16, k16, v16 = sale.workload_gqa("sink_local", 7, 2, 333, 8, 2, 64)
    for b in range(2):
        for g in range(2):
            rq, rk, rv = sale.workload_head_f32("sink_local", 7 + b, 333, 64, g)
            np.testing.assert_array_equal(k16[b, :, g, :64], sale.f32_to_bf16_bits(rk))
            np.testing.assert_array_equal(v16[b, :, g, :64], sale.f32_to_bf16_bits(rv))
            np.testing.assert_array_equal(q16[b, :, 4 * g, :64], sale.f32_to_bf16_bits(rq))
            assert not np.array_equal(q16[b, :, 4 * g + 1], q16[b, :, 4 * g])
    assert (q16[..., 64:] == 0).all() and (k16[..., 64:] == 0).all()


@pytest.mark.parametrize("kind,n,d,hq,hkv", [("sink_local", 300, 128, 8, 2), ("gaussian", 97, 64, 7, 1),
                                              ("sink_local", 129, 32, 4, 4)])
def test_gqa_workload_equals_reference_built_generator(kind, n, d, hq, hkv):
    """The product's GQA generator (workload.cpp) == the same extension built
    from the reference's own Rng / generators in oracle/_ref
    (ref_workload_gqa_heads), bit for bit: bench.py's reference arm builds its
    inputs there without loading the product library."""
    q16, k16, v16 = sale.workload_gqa(kind, 7, 1, n, hq, hkv, d)
    q, k, v = (np.empty((hq, n, d), np.float32) for _ in range(3))
    assert O.REF.ref_workload_gqa_heads(1 if kind == "sink_local" else 0, 7, n, d, hq, hkv, 1, 2,
                                        q, k, v) == 0
    f = sale.bf16_bits_to_f32
    G = hq // hkv
    for h in range(hq):
        np.testing.assert_array_equal(q[h], f(q16[0, :, h, :d]))
        np.testing.assert_array_equal(k[h], f(k16[0, :, h // G, :d]))
        np.testing.assert_array_equal(v[h], f(v16[0, :, h // G, :d]))


def test_sharded_generation_equals_full():
    full = sale.workload_gqa("sink_local", 3, 1, 500, 8, 4, 128)
    for rank in range(2):
        part = sale.workload_gqa("sink_local", 3, 1, 500, 4, 2, 128, kv_begin=2 * rank)
        np.testing.assert_array_equal(part[0], full[0][:, :, 4 * rank:4 * rank + 4])
        np.testing.assert_array_equal(part[1], full[1][:, :, 2 * rank:2 * rank + 2])
        np.testing.assert_array_equal(part[2], full[2][:, :, 2 * rank:2 * rank + 2])


def test_mask_pack_roundtrip():
    rng = np.random.default_rng(1)
    for n in (1, 63, 64, 1000, 2080):
        nq, nk, nw = sale.grid(n)
        cells = (rng.random((2, 3, nq, nk)) < 0.3).astype(np.uint8)
        words = sale.pack_mask(cells, n)
        assert words.shape == (2, 3, nq, nw)
        np.testing.assert_array_equal(sale.unpack_mask(words, n), cells)


def base_mask_formula(n):
    """Python mirror of the device closed form (common.cuh frontier_block /
    full_segments, stats.cu base_mask_kernel)."""
    nq, nk, _ = sale.grid(n)
    out = np.zeros((nq, nk), np.uint8)
    for i in range(nq):
        fr = min((min(64 * i + 64, n) - 1) // 32, nk - 1)
        lo = 1 + 4 * ((2 * i - 5) // 4) if i >= 3 else 0
        for j in range(nk):
            out[i, j] = j == 0 or lo <= j <= fr
    return out


@pytest.mark.parametrize("n", [1, 64, 100, 191, 192, 256, 1000, 2049])
def test_base_mask_and_segment_geometry_match_oracle(n):
    """The kernels' closed-form geometry equals the reference algorithm: with
    tau -> 0 every middle block is selected, with an impossible-to-pass
    threshold only I_SL and the forced trailing run remain."""
    q, k, _ = sale.workload_head_f32("gaussian", 1, n, 16, 0)
    qc, qs = O.quantize(q, 1)
    kc, ks = O.quantize(k, 32)
    # zero query codes -> every estimate is 0, far below any bound at tau 0.5
    zero = np.zeros_like(qc)
    base = O.selection_pass(q * 0 + 1e-30, k, zero, qs, kc, ks, O.cfg(tau=0.999999))
    np.testing.assert_array_equal(base, base_mask_formula(n))
    allc = O.selection_pass(q, k, qc, qs, kc, ks, O.cfg(tau=1e-300))
    nq, nk, _ = sale.grid(n)
    causal = (32 * np.arange(nk)[None, :]) < np.minimum(64 * (np.arange(nq)[:, None] + 1), n)
    np.testing.assert_array_equal(allc, causal.astype(np.uint8))


def _gloo_worker(rank, world, port, q):
    import torch.distributed as dist
    import torch
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    hkv = 8 // world
    part = sale.workload_gqa("sink_local", 7, 1, 256, 4 * hkv, hkv, 128, threads=2,
                             kv_begin=rank * hkv)
    digest = torch.tensor([float(np.int64(part[1].astype(np.int64).sum()))], dtype=torch.float64)
    ms = torch.tensor([10.0 + rank], dtype=torch.float64)
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)  # bench.py: job time = max over ranks
    gathered = [torch.zeros(1, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(gathered, digest)
    if rank == 0:
        q.put((float(ms[0]), [float(x[0]) for x in gathered]))
    dist.destroy_process_group()


def _gather_worker(rank, world, port, q):
    import torch.distributed as dist
    import torch
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    g = torch.Generator().manual_seed(3)
    full = torch.randn(2, 64, 8, 16, generator=g)       # [B, N, Hq, d]
    shard = full[:, :, 4 * rank:4 * rank + 4].clone()   # this rank's query heads
    got = sale.gather_heads(shard)
    q.put((rank, bool(torch.equal(got, full))))
    dist.destroy_process_group()


def test_output_gather_two_ranks_gloo():
    """The optional output gather (sale.gather_heads): head-sliced shards of O
    concatenate back to the full [B, N, Hq, d] on every rank."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 30500 + os.getpid() % 1000
    procs = [ctx.Process(target=_gather_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    res = sorted(q.get(timeout=10) for _ in range(2))
    assert res == [(0, True), (1, True)]


def test_kv_group_sharding_two_ranks_gloo():
    """bench.py's N>1 host path: each rank generates and owns a disjoint KV-group
    shard (no data-path collective); only timings are reduced (max)."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + os.getpid() % 1000
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    ms, digests = q.get(timeout=10)
    assert ms == 11.0
    full = sale.workload_gqa("sink_local", 7, 1, 256, 32, 8, 128, threads=2)
    want = [float(full[1][:, :, 4 * r:4 * r + 4].astype(np.int64).sum()) for r in range(2)]
    assert digests == want


def test_query_block_split_balanced():
    """a unit split across GPUs gets contiguous query-block
    ranges with odd inner boundaries and about equal causal work (~ i^2)."""
    for nq, parts in ((3, 3), (4, 4), (8, 8), (1, 2)):
        with pytest.raises(ValueError):
            sale.query_block_split(nq, parts)
    for nq in (5, 17, 64, 1000, 2048, 4096):
        for parts in (1, 2, 3, 4, 8):
            if parts - 1 > nq // 2:  # odd inner boundaries available in (0, nq)
                continue
            r = sale.query_block_split(nq, parts)
            assert r[0][0] == 0 and r[-1][1] == nq
            assert all(a < b for a, b in r) and all(r[k][1] == r[k + 1][0] for k in range(len(r) - 1))
            assert all(b % 2 == 1 for _, b in r[:-1])
            assert len(r) == parts
            if nq >= 1000:
                work = [(b * b - a * a) / (nq * nq) for a, b in r]
                assert max(work) - min(work) < 0.02, (nq, parts, work)
