"""ctypes bindings for the two CPU checkers — TEST INFRASTRUCTURE ONLY.

* ``C``   : oracle/lib/libsale_oracle.so — the plain-C restatement
           (oracle/sale_oracle.c), each function citing the reference file:line.
* ``REF`` : oracle/_ref/libsale_ref.so — the UNMODIFIED reference headers behind
           a flat C ABI (oracle/ref_capi.cpp); None when it was never built.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference legs import this module. The product package never does.
All functions take one head at a time: fp32 numpy arrays [tokens, dim].
"""
from __future__ import annotations

import ctypes as C
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_C_PATH = os.path.join(_HERE, "lib", "libsale_oracle.so")
_REF_PATH = os.path.join(_HERE, "_ref", "libsale_ref.so")

f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
i8p = np.ctypeslib.ndpointer(np.int8, flags="C_CONTIGUOUS")
u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
i64 = C.c_int64


class Cfg(C.Structure):
    """Mirror of sale::SelectionConfig (selection.hpp:18-24)."""

    _fields_ = [("tau", C.c_double), ("sink_tokens", i64), ("local_tokens_min", i64),
                ("segment_size", i64), ("block_q", i64), ("block_k", i64)]


def cfg(tau=0.004, sink_tokens=32, local_tokens_min=128, segment_size=4, block_q=64, block_k=32):
    return Cfg(tau, sink_tokens, local_tokens_min, segment_size, block_q, block_k)


def build():
    """Builds both checkers with oracle/Makefile (the _ref part only when the
    reference tree is present)."""
    import subprocess
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


def _load_c():
    if not os.path.exists(_C_PATH):
        build()
    lib = C.CDLL(_C_PATH)
    lib.oracle_quantize.argtypes = [f32p, i64, i64, i64, i8p, f32p]
    lib.oracle_sink_local_index_set.argtypes = [i64, i64, C.POINTER(Cfg), i64p]
    lib.oracle_sink_local_index_set.restype = i64
    lib.oracle_sink_local_stats.argtypes = [f32p, f32p, i64, i64, i64, i64, i64, i64p, i64,
                                            f64p, f64p]
    lib.oracle_threshold_bound.argtypes = [C.c_double] * 3
    lib.oracle_threshold_bound.restype = C.c_double
    lib.oracle_segment_aggregate.argtypes = [u8p, i64, i64]
    lib.oracle_max_then_dequantize.argtypes = [i32p, i64, C.c_float, C.POINTER(C.c_float),
                                               C.POINTER(i64)]
    lib.oracle_approx_weight_block.argtypes = [i8p, f32p, i64, i64, i64, i8p, f32p, i64, i64,
                                               i64, i64, i32p, f32p]
    lib.oracle_selection_pass.argtypes = [f32p, f32p, i64, i64, i8p, f32p, i8p, f32p,
                                          C.POINTER(Cfg), u8p, C.c_void_p, C.c_void_p,
                                          C.c_void_p, C.c_void_p]
    lib.oracle_selection_stats.argtypes = [f32p, f32p, i64, i64, C.POINTER(Cfg), i64, i64, f64p,
                                           f64p, f64p]
    lib.oracle_block_sparse_attention.argtypes = [f32p, f32p, f32p, i64, i64, u8p, i64, i64,
                                                  f32p, i64p]
    lib.oracle_full_attention.argtypes = [f32p, f32p, f32p, i64, i64, f32p]
    lib.oracle_flop_accounting.argtypes = [u8p, i64, i64, i64, i64p]
    lib.oracle_l1_error.argtypes = [f32p, f32p, i64, i64]
    lib.oracle_l1_error.restype = C.c_double
    return lib


def _load_ref():
    if not os.path.exists(_REF_PATH):
        return None
    lib = C.CDLL(_REF_PATH)
    lib.ref_quantize_per_token.argtypes = [f32p, i64, i64, i8p, f32p]
    lib.ref_quantize_per_key_block.argtypes = [f32p, i64, i64, i64, i64, i8p, f32p]
    lib.ref_sink_local_index_set.argtypes = [i64] * 7 + [i64p]
    lib.ref_sink_local_index_set.restype = i64
    lib.ref_sink_local_stats.argtypes = [f32p, f32p, i64, i64, i64, i64, i64, i64p, i64, f64p, f64p]
    lib.ref_threshold_bound.argtypes = [C.c_double] * 3
    lib.ref_threshold_bound.restype = C.c_double
    lib.ref_selection_pass.argtypes = [f32p, f32p, i64, i64, i8p, f32p, i8p, f32p, C.c_double,
                                       i64, i64, i64, i64, i64, u8p]
    lib.ref_block_sparse_attention.argtypes = [f32p, f32p, f32p, i64, i64, u8p, i64, i64, f32p,
                                               i64p]
    lib.ref_full_attention.argtypes = [f32p, f32p, f32p, i64, i64, f32p]
    lib.ref_flop_accounting.argtypes = [u8p, i64, i64, i64, i64p]
    lib.ref_workload_head.argtypes = [C.c_int, C.c_uint64, i64, i64, i64, f32p, f32p, f32p]
    lib.ref_run_pipeline.argtypes = [f32p, f32p, f32p, i64, i64, i64, C.c_double, i64, f64p,
                                     f64p, f64p]
    lib.ref_workload_gqa_heads.argtypes = [C.c_int, C.c_uint64, i64, i64, i64, i64, C.c_int, i64,
                                           f32p, f32p, f32p]
    lib.ref_sale_heads.argtypes = [f32p, f32p, f32p, i64, i64, i64, C.c_double, i64, f64p, f64p]
    lib.ref_run_report.argtypes = [f32p, f32p, f32p, i64, i64, i64, f64p, C.c_int, i64, f64p]
    lib.ref_sweep.argtypes = [f32p, f32p, f32p, i64, i64, i64, f64p, i64, i64, f64p]
    lib.ref_calibrate_head.argtypes = [f32p, f32p, f32p, i64, i64, i64, C.c_double, C.c_double, i64,
                                       f64p, C.POINTER(C.c_int32), i64p]
    lib.ref_write_tensor_file.argtypes = [C.c_char_p, f32p, f32p, f32p, i64, i64, i64]
    lib.ref_read_tensor_file.argtypes = [C.c_char_p, f32p, f32p, f32p, C.c_char_p, i64]
    lib.ref_write_mask_dump.argtypes = [C.c_char_p, u8p, C.POINTER(C.c_uint32), f32p, i64, i64, i64]
    return lib


C_LIB = _load_c()
REF = _load_ref()

# ----------------------------------------------------------------- wrappers


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def quantize(x, group_rows):
    """quant.hpp:95-119 — returns (codes int8 [rows, d], scales f32 [groups])."""
    x = _f32(x)
    rows, d = x.shape
    codes = np.empty((rows, d), np.int8)
    scales = np.empty(((rows + group_rows - 1) // group_rows,), np.float32)
    st = C_LIB.oracle_quantize(x, rows, d, group_rows, codes, scales)
    assert st == 0
    return codes, scales


def sink_local_index_set(i, tokens, c=None):
    c = c or cfg()
    out = np.empty(((tokens + c.block_k - 1) // c.block_k,), np.int64)
    n = C_LIB.oracle_sink_local_index_set(i, tokens, C.byref(c), out)
    if n < 0:
        raise IndexError("sink_local_index_set: query block out of range")
    return out[:n].copy()


def threshold_bound(tau, m, l):
    return C_LIB.oracle_threshold_bound(tau, m, l)


def selection_pass(q, k, qcodes, qscales, kcodes, kscales, c=None, debug=False):
    """selection.hpp:211-274. Returns mask uint8 [nq, nk] (and, with debug,
    dict(m, l, bound [tokens] f64, block_max int32 [tokens, nk]))."""
    c = c or cfg()
    q, k = _f32(q), _f32(k)
    n, d = q.shape
    nq, nk = (n + c.block_q - 1) // c.block_q, (n + c.block_k - 1) // c.block_k
    mask = np.empty((nq, nk), np.uint8)
    dbg = None
    ptrs = [None] * 4
    if debug:
        dbg = dict(m=np.empty(n, np.float64), l=np.empty(n, np.float64),
                   bound=np.empty(n, np.float64), block_max=np.empty((n, nk), np.int32))
        ptrs = [dbg[x].ctypes.data for x in ("m", "l", "bound", "block_max")]
    st = C_LIB.oracle_selection_pass(q, k, n, d, np.ascontiguousarray(qcodes), _f32(qscales),
                                     np.ascontiguousarray(kcodes), _f32(kscales), C.byref(c), mask,
                                     *ptrs)
    if st:
        raise ValueError(f"selection_pass: status {st}")
    return (mask, dbg) if debug else mask


def selection_stats(q, k, c=None, i_lo=0, i_hi=-1):
    """The statistics of selection_pass (selection.hpp:224-251): (m, l, bound)
    float64 [tokens], NaN for rows whose query block has an empty middle."""
    c = c or cfg()
    q, k = _f32(q), _f32(k)
    n, d = q.shape
    m, l, b = (np.full(n, np.nan) for _ in range(3))
    st = C_LIB.oracle_selection_stats(q, k, n, d, C.byref(c), i_lo, i_hi, m, l, b)
    if st:
        raise ValueError(f"selection_stats: status {st}")
    return m, l, b


def block_sparse_attention(q, k, v, mask, block_q=64, block_k=32):
    """sparse_attention.hpp:37-97 -> (out f32 [n, d], coverage int64 [n], status)."""
    q, k, v = _f32(q), _f32(k), _f32(v)
    n, d = q.shape
    out = np.empty((n, d), np.float32)
    cov = np.empty((n,), np.int64)
    st = C_LIB.oracle_block_sparse_attention(q, k, v, n, d, np.ascontiguousarray(mask, np.uint8),
                                             block_q, block_k, out, cov)
    return out, cov, st


def full_attention(q, k, v):
    q, k, v = _f32(q), _f32(k), _f32(v)
    n, d = q.shape
    out = np.empty((n, d), np.float32)
    assert C_LIB.oracle_full_attention(q, k, v, n, d, out) == 0
    return out


def flop_accounting(mask, tokens, block_q=64, block_k=32):
    counts = np.empty(3, np.int64)
    C_LIB.oracle_flop_accounting(np.ascontiguousarray(mask, np.uint8), tokens, block_q, block_k,
                                 counts)
    return dict(computed=int(counts[0]), skipped=int(counts[1]), total=int(counts[2]))


def l1_error(a, b):
    a, b = _f32(a), _f32(b)
    return C_LIB.oracle_l1_error(a, b, a.shape[0], a.shape[1])


def map_heads(fn, n_items, threads=None):
    """Runs fn(h) for h in range(n_items) on a thread pool. ctypes releases
    the GIL, so per-head oracle calls run in parallel on the host cores."""
    threads = threads or os.cpu_count() or 1
    with ThreadPoolExecutor(max_workers=threads) as ex:
        return list(ex.map(fn, range(n_items)))
