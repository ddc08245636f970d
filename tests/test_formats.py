"""The reference's file formats on this path (no GPU): .tns tensor files and
RLE mask dumps written / read by libsale_b200 (csrc/formats.cpp) against the
unmodified reference's own writer and reader (oracle/_ref): byte-identical
files, identical values, identical error messages and offsets."""
import ctypes as C
import os
import struct

import numpy as np
import pytest

from oracle import oracle as O
from paper_2505_24179_b200 import sale

pytestmark = pytest.mark.skipif(O.REF is None, reason="oracle/_ref not built")


def _heads_f32(h, n, d, seed):
    """bf16-representable fp32 heads [h][n][d] (q, k, v)."""
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(3):
        x = rng.standard_normal((h, n, d)).astype(np.float32)
        out.append(sale.bf16_bits_to_f32(sale.f32_to_bf16_bits(x)))
    return out


def _to_layout(x):
    """[h][n][d] fp32 -> bf16 bits [1][n][h][128] (zero padded)."""
    h, n, d = x.shape
    out = np.zeros((1, n, h, 128), np.uint16)
    out[0, :, :, :d] = sale.f32_to_bf16_bits(np.ascontiguousarray(x.transpose(1, 0, 2)))
    return out


@pytest.mark.parametrize("h,n,d", [(1, 1, 1), (3, 17, 64), (2, 130, 128)])
def test_tensor_file_reference_written_read_by_b200(tmp_path, h, n, d):
    q, k, v = _heads_f32(h, n, d, seed=h * 1000 + n)
    path = str(tmp_path / "ref.tns")
    assert O.REF.ref_write_tensor_file(path.encode(), q.ravel(), k.ravel(), v.ravel(), h, n, d) == 0
    gq, gk, gv, dim = sale.read_tensor_file(path)
    assert dim == d
    for got, want in ((gq, q), (gk, k), (gv, v)):
        np.testing.assert_array_equal(got, _to_layout(want))


@pytest.mark.parametrize("h,n,d", [(1, 5, 3), (4, 64, 128)])
def test_tensor_file_b200_written_byte_identical_and_bf16_tag(tmp_path, h, n, d):
    q, k, v = _heads_f32(h, n, d, seed=7)
    ref_path, our_path, bf_path = (str(tmp_path / f) for f in ("r.tns", "o.tns", "b.tns"))
    assert O.REF.ref_write_tensor_file(ref_path.encode(), q.ravel(), k.ravel(), v.ravel(), h, n, d) == 0
    sale.write_tensor_file(our_path, _to_layout(q), _to_layout(k), _to_layout(v), d, dtype="f32")
    assert open(ref_path, "rb").read() == open(our_path, "rb").read()
    # the reference reads what we wrote
    rq, rk, rv = (np.empty(h * n * d, np.float32) for _ in range(3))
    msg = C.create_string_buffer(256)
    assert O.REF.ref_read_tensor_file(our_path.encode(), rq, rk, rv, msg, 256) == 0
    np.testing.assert_array_equal(rq.reshape(h, n, d), q)
    # bf16 payload tag (this path's extension): half the bytes, same values
    sale.write_tensor_file(bf_path, _to_layout(q), _to_layout(k), _to_layout(v), d, dtype="bf16")
    assert os.path.getsize(bf_path) == 28 + 3 * h * n * d * 2
    gq, gk, gv, dim = sale.read_tensor_file(bf_path)
    np.testing.assert_array_equal(gq, _to_layout(q))
    np.testing.assert_array_equal(gv, _to_layout(v))


def _corrupt_cases(good: bytes):
    hdr = bytearray(good)
    yield "bad magic", b"XALETNSR" + good[8:]
    yield "truncated magic", good[:5]
    yield "version", good[:8] + struct.pack("<I", 2) + good[12:]
    yield "dtype", good[:12] + struct.pack("<I", 9) + good[16:]
    yield "zero heads", good[:16] + struct.pack("<I", 0) + good[20:]
    yield "zero tokens", good[:20] + struct.pack("<I", 0) + good[24:]
    yield "zero dim", good[:24] + struct.pack("<I", 0) + good[28:]
    yield "truncated header", good[:22]
    yield "truncated payload", good[:-6]
    yield "trailing", good + b"\x00"
    nan = bytearray(hdr)
    nan[28 + 4 * 5:28 + 4 * 6] = struct.pack("<f", float("nan"))
    yield "non-finite", bytes(nan)
    inf = bytearray(hdr)
    inf[-4:] = struct.pack("<f", float("-inf"))
    yield "non-finite last", bytes(inf)


def test_tensor_file_errors_match_reference(tmp_path):
    h, n, d = 2, 6, 4
    q, k, v = _heads_f32(h, n, d, seed=3)
    good_path = str(tmp_path / "g.tns")
    assert O.REF.ref_write_tensor_file(good_path.encode(), q.ravel(), k.ravel(), v.ravel(), h, n, d) == 0
    good = open(good_path, "rb").read()
    for name, blob in _corrupt_cases(good):
        path = str(tmp_path / "bad.tns")
        open(path, "wb").write(blob)
        buf = [np.empty(64 * 64, np.float32) for _ in range(3)]
        msg = C.create_string_buffer(512)
        st = O.REF.ref_read_tensor_file(path.encode(), *buf, msg, 512)
        assert st == 6, name
        with pytest.raises(sale.TensorFileError) as e:
            sale.read_tensor_file(path)
        assert str(e.value) == msg.value.decode(), name
    with pytest.raises(OSError):
        sale.read_tensor_file(str(tmp_path / "missing.tns"))


def _masks(n, records, seed):
    """Random causal masks (uint8 cells [r][nq][nk]) shaped like selection output."""
    nq, nk, _ = sale.grid(n)
    rng = np.random.default_rng(seed)
    causal = (32 * np.arange(nk)[None, :]) < np.minimum(64 * (np.arange(nq)[:, None] + 1), n)
    cells = (rng.random((records, nq, nk)) < 0.4) & causal[None]
    cells[:, :, 0] = causal[:, 0]
    return cells.astype(np.uint8)


@pytest.mark.parametrize("n,b,h", [(64, 1, 1), (1000, 1, 3), (4096, 2, 2)])
def test_mask_dump_byte_identical_and_round_trip(tmp_path, n, b, h):
    cells = _masks(n, b * h, seed=n + h)
    nq, nk, _ = sale.grid(n)
    words = np.stack([sale.pack_mask(c, n) for c in cells]).reshape(b, h, nq, -1)
    taus = (np.arange(b * h, dtype=np.float32) + 1) * np.float32(0.001)
    ref_path, our_path = str(tmp_path / "r.mask"), str(tmp_path / "o.mask")
    heads = np.arange(b * h, dtype=np.uint32)
    assert O.REF.ref_write_mask_dump(ref_path.encode(), np.ascontiguousarray(cells),
                                     heads.ctypes.data_as(C.POINTER(C.c_uint32)), taus,
                                     b * h, nq, nk) == 0
    sale.write_mask_dump(our_path, words, n, taus)
    assert open(ref_path, "rb").read() == open(our_path, "rb").read()
    got, gh, gt = sale.read_mask_dump(ref_path)
    np.testing.assert_array_equal(got, words.reshape(b * h, nq, -1))
    np.testing.assert_array_equal(gh, heads)
    np.testing.assert_array_equal(gt, taus)


def test_mask_dump_errors(tmp_path):
    p = str(tmp_path / "x.mask")
    open(p, "wb").write(b"SALEMASK" + struct.pack("<II", 1, 1) + struct.pack("<IIIf", 0, 1, 2, 0.5)
                        + b"\x01" + struct.pack("<II", 2, 1) + struct.pack("<I", 0))
    with pytest.raises(sale.TensorFileError, match="zero-length run"):
        sale.read_mask_dump(p)
    open(p, "wb").write(b"SALEMASK" + struct.pack("<II", 1, 1) + struct.pack("<IIIf", 0, 1, 2, 0.5)
                        + b"\x01" + struct.pack("<II", 1, 1))
    with pytest.raises(sale.TensorFileError, match="runs cover 1 of 2 cells"):
        sale.read_mask_dump(p)
    open(p, "wb").write(b"NOTAMASK")
    with pytest.raises(sale.TensorFileError, match="bad mask dump magic"):
        sale.read_mask_dump(p)
