"""Python host mirror of the reference's hot-path API over the C ABI.

Same names and argument meaning as the reference's `namespace sale`
(/root/reference/proj/include/sale), lifted from one head of fp32 to the
B200 layout: bf16 torch tensors [B, N, H, 128] on the GPU (rows zero-padded
past head_dim). Every call goes through lib/libsale_b200.so (include/sale_b200.h);
there is no CPU fallback — a missing library or a non-sm_100 device raises.

Error classes follow the reference: ValueError for std::invalid_argument,
ArithmeticError for std::domain_error, IndexError for std::out_of_range,
RuntimeError for CUDA failures and NotImplementedError for configurations the
B200 path does not implement.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SALE_B200_LIB") or os.path.join(_HERE, "lib", "libsale_b200.so")

BLOCK_Q, BLOCK_K, SEGMENT, HEAD_PITCH = 64, 32, 4, 128

i64 = C.c_int64
vp = C.c_void_p


class Shape(C.Structure):
    _fields_ = [("batch", i64), ("tokens", i64), ("q_heads", i64), ("kv_heads", i64),
                ("head_dim", i64)]


class SelectionConfig(C.Structure):
    """sale::SelectionConfig (selection.hpp:18-24) minus tau (per head)."""

    _fields_ = [("sink_tokens", i64), ("local_tokens_min", i64), ("segment_size", i64),
                ("block_q", i64), ("block_k", i64)]


def default_config() -> SelectionConfig:
    return SelectionConfig(32, 128, 4, 64, 32)


class SelectDebug(C.Structure):
    _fields_ = [("running_max", vp), ("exp_sum", vp), ("bound", vp), ("block_max", vp)]


class TensorFileError(RuntimeError):
    """sale::TensorFileError (tensor_file.hpp:22-33): format error; `offset` is
    the byte offset the message names."""

    def __init__(self, message: str):
        super().__init__(message)
        import re
        m = re.search(r"\(offset (\d+)\)$", message)
        self.offset = int(m.group(1)) if m else None


class HeadReport(C.Structure):
    """sale::HeadReport (report.hpp:12-23) of one (batch, q head)."""

    _fields_ = [("head", i64), ("tau", C.c_double), ("sparsity", C.c_double), ("err", C.c_double),
                ("computed_blocks", i64), ("skipped_blocks", i64), ("total_blocks", i64),
                ("coverage_min", i64), ("coverage_max", i64), ("coverage_mean", C.c_double)]


class StageTiming(C.Structure):
    _fields_ = [("quantization_ms", C.c_double), ("selection_ms", C.c_double),
                ("computation_ms", C.c_double), ("dense_ms", C.c_double)]


class SweepRow(C.Structure):
    _fields_ = [("tau", C.c_double), ("sparsity", C.c_double), ("err", C.c_double)]


class CalibrationSettings(C.Structure):
    """sale::CalibrationSettings (calibrate.hpp:56-68) minus the geometry."""

    _fields_ = [("theta", C.c_double), ("tau0", C.c_double), ("max_halvings", i64)]


class HeadCalibration(C.Structure):
    _fields_ = [("layer", i64), ("head", i64), ("tau", C.c_double), ("flag", C.c_int32),
                ("halvings", i64)]


_ERRORS = {1: ValueError, 2: ArithmeticError, 3: IndexError, 4: RuntimeError,
           5: NotImplementedError, 6: TensorFileError, 7: OSError}

_lib = None


def load_library() -> C.CDLL:
    """Loads lib/libsale_b200.so (built by `make -C paper_2505_24179_b200`)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} missing: build it with __graft_entry__.build() "
                          "(there is no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    P = C.POINTER
    sig = {
        "sale_b200_ctx_create": (C.c_int, [C.c_int, P(vp)]),
        "sale_b200_ctx_destroy": (None, [vp]),
        "sale_b200_last_error": (C.c_char_p, [vp]),
        "sale_b200_version": (C.c_int, []),
        "sale_b200_default_config": (None, [P(SelectionConfig)]),
        "sale_b200_quantize": (C.c_int, [vp, vp, i64, i64, i64, i64, vp, vp, vp]),
        "sale_b200_quantize_qk": (C.c_int, [vp, vp, vp, P(Shape), vp, vp, vp, vp, vp]),
        "sale_b200_select": (C.c_int, [vp, vp, vp, vp, vp, vp, vp, P(Shape), P(C.c_double),
                                       P(SelectionConfig), vp, P(SelectDebug), vp]),
        "sale_b200_sparse_attention": (C.c_int, [vp, vp, vp, vp, P(Shape), vp, vp, vp, vp]),
        "sale_b200_flop_count": (C.c_int, [vp, vp, i64, i64, i64, vp, vp]),
        "sale_b200_prefill": (C.c_int, [vp, vp, vp, vp, P(Shape), P(C.c_double),
                                        P(SelectionConfig), vp, vp, vp]),
        "sale_b200_prefill_host": (C.c_int, [vp, vp, vp, vp, P(Shape), P(C.c_double),
                                             P(SelectionConfig), vp]),
        "sale_b200_prefill_range": (C.c_int, [vp, vp, vp, vp, P(Shape), P(C.c_double),
                                              P(SelectionConfig), i64, i64, vp, vp, vp]),
        "sale_b200_sparse_attention_range": (C.c_int, [vp, vp, vp, vp, P(Shape), vp, i64, i64,
                                                       vp, vp, vp]),
        "sale_b200_workload_head_f32": (C.c_int, [C.c_int, C.c_uint64, i64, i64, i64, vp, vp, vp]),
        "sale_b200_workload_gqa_bf16": (C.c_int, [C.c_int, C.c_uint64, P(Shape), vp, vp, vp,
                                                  C.c_int]),
        "sale_b200_workload_gqa_shard_bf16": (C.c_int, [C.c_int, C.c_uint64, P(Shape), i64, vp,
                                                        vp, vp, C.c_int]),
        "sale_b200_set_timing": (C.c_int, [vp, C.c_int]),
        "sale_b200_l1_error": (C.c_int, [vp, vp, vp, P(Shape), vp]),
        "sale_b200_run_pipeline": (C.c_int, [vp, vp, vp, vp, P(Shape), P(C.c_double),
                                             P(SelectionConfig), C.c_int, P(HeadReport),
                                             P(StageTiming)]),
        "sale_b200_sweep_thresholds": (C.c_int, [vp, vp, vp, vp, P(Shape), P(C.c_double), i64,
                                                 P(SelectionConfig), P(SweepRow)]),
        "sale_b200_calibrate": (C.c_int, [vp, P(vp), P(vp), P(vp), i64, P(Shape),
                                          P(CalibrationSettings), P(SelectionConfig),
                                          P(HeadCalibration)]),
        "sale_b200_tensor_file_info": (C.c_int, [C.c_char_p, vp, vp, vp, vp]),
        "sale_b200_tensor_file_read_bf16": (C.c_int, [C.c_char_p, vp, vp, vp]),
        "sale_b200_tensor_file_write": (C.c_int, [C.c_char_p, vp, vp, vp, C.c_uint32, C.c_uint32,
                                                  C.c_uint32, C.c_uint32]),
        "sale_b200_mask_dump_write": (C.c_int, [C.c_char_p, vp, i64, i64, i64, vp]),
        "sale_b200_mask_dump_read": (C.c_int, [C.c_char_p, vp, vp, vp, vp, vp, vp]),
        "sale_b200_stage_times": (C.c_int, [vp, P(C.c_float)]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def _ptr(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def _stream():
    import torch
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


class Context:
    """sale_b200_ctx on one device (one stream at a time)."""

    def __init__(self, device: int = 0):
        self.lib = load_library()
        self.handle = vp()
        self.device = device
        self._check(self.lib.sale_b200_ctx_create(device, C.byref(self.handle)), create=True)

    def _check(self, status, create=False):
        if status:
            msg = self.lib.sale_b200_last_error(None if create else self.handle)
            raise _ERRORS.get(status, RuntimeError)((msg or b"").decode())

    def close(self):
        if self.handle:
            self.lib.sale_b200_ctx_destroy(self.handle)
            self.handle = vp()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_ctx: Context | None = None


def context() -> Context:
    global _ctx
    if _ctx is None:
        import torch
        _ctx = Context(torch.cuda.current_device())
    return _ctx


# ------------------------------------------------------------------ geometry

def grid(tokens: int):
    nq = -(-tokens // BLOCK_Q)
    nk = -(-tokens // BLOCK_K)
    return nq, nk, -(-nk // 32)


def unpack_mask(words, tokens: int) -> np.ndarray:
    """Packed mask words (any leading dims, last = words) -> uint8 [..., Nq, Nk]
    (the sale::BlockMask cell layout, selection.hpp:84)."""
    w = np.ascontiguousarray(np.asarray(words).astype(np.uint32))
    nq, nk, nw = grid(tokens)
    bits = np.unpackbits(w.view(np.uint8).reshape(*w.shape[:-1], nw * 4), axis=-1,
                         bitorder="little")
    return bits[..., :nk].astype(np.uint8)


def pack_mask(cells: np.ndarray, tokens: int) -> np.ndarray:
    """uint8 [..., Nq, Nk] -> uint32 words [..., Nq, W] (inverse of unpack_mask)."""
    nq, nk, nw = grid(tokens)
    cells = np.asarray(cells, np.uint8)
    pad = np.zeros((*cells.shape[:-1], nw * 32), np.uint8)
    pad[..., :nk] = cells != 0
    return np.packbits(pad, axis=-1, bitorder="little").view(np.uint32)


# ---------------------------------------------------------- stage wrappers

def _check_tensor(name, t, dtype, device=None, ndim=4):
    """The C ABI takes raw pointers: anything but a contiguous tensor of the
    expected dtype on the context's device would be read out of bounds or
    misinterpreted, so it is rejected here (ValueError, like the reference's
    std::invalid_argument for malformed inputs)."""
    import torch
    if not isinstance(t, torch.Tensor):
        raise ValueError(f"{name} must be a torch tensor")
    if t.dtype != dtype:
        raise ValueError(f"{name} must be {dtype}, got {t.dtype}")
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor")
    if device is not None and t.device.index != device:
        raise ValueError(f"{name} is on cuda:{t.device.index}, the context on cuda:{device}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous (e.g. not a head slice of a fused QKV)")
    if t.dim() != ndim:
        raise ValueError(f"{name} must have {ndim} dimensions, got {t.dim()}")


def _shape_of(q, k, head_dim, v=None, ctx=None):
    """Validated Shape of q [B,N,Hq,128], k (and v) [B,N,Hkv,128] (bf16,
    contiguous, on the context's device) — HeadInput::validate
    (matrix.hpp:66-72) lifted to the batched layout."""
    import torch
    dev = (ctx or context()).device
    for name, t in (("q", q), ("k", k)) + ((("v", v),) if v is not None else ()):
        _check_tensor(name, t, torch.bfloat16, dev)
    B, N, Hq, P = q.shape
    if P != HEAD_PITCH or k.shape[3] != HEAD_PITCH:
        raise ValueError("rows must be padded to 128 elements")
    if tuple(k.shape[:2]) != (B, N):
        raise ValueError("HeadInput: key rows must match query rows (batch, tokens)")
    if v is not None and tuple(v.shape) != tuple(k.shape):
        raise ValueError("HeadInput: value shape must match key shape")
    if not 1 <= head_dim <= HEAD_PITCH:
        raise ValueError("head_dim must be in [1, 128]")
    return Shape(B, N, Hq, k.shape[2], head_dim)


def _check_mask(mask, s, ctx=None):
    import torch
    if mask is None:
        return
    _check_tensor("mask", mask, torch.int32, (ctx or context()).device)
    nq, _, nw = grid(s.tokens)
    if tuple(mask.shape) != (s.batch, s.q_heads, nq, nw):
        raise ValueError(f"mask must be [B, Hq, Nq, W] = {(s.batch, s.q_heads, nq, nw)}, "
                         f"got {tuple(mask.shape)}")


def quantize_qk(q, k, head_dim=128):
    """quantize_per_token(Q) + quantize_per_key_block(K) (quant.hpp:95/107), fused.
    Returns (q_codes int8 [B,N,Hq,128], q_scales f32 [B,Hq,N],
             k_codes int8 [B,N,Hkv,128], k_scales f32 [B,Hkv,Nk])."""
    import torch
    ctx = context()
    s = _shape_of(q, k, head_dim)
    _, nk, _ = grid(s.tokens)
    qc = torch.empty(q.shape, dtype=torch.int8, device=q.device)
    kc = torch.empty(k.shape, dtype=torch.int8, device=k.device)
    qs = torch.empty((s.batch, s.q_heads, s.tokens), dtype=torch.float32, device=q.device)
    ks = torch.empty((s.batch, s.kv_heads, nk), dtype=torch.float32, device=q.device)
    ctx._check(ctx.lib.sale_b200_quantize_qk(ctx.handle, _ptr(q), _ptr(k), C.byref(s), _ptr(qc),
                                             _ptr(qs), _ptr(kc), _ptr(ks), _stream()))
    return qc, qs, kc, ks


def quantize_per_token(x):
    """quant.hpp:95 for every (batch, head) of x [B,N,H,128]."""
    import torch
    ctx = context()
    _check_tensor("x", x, torch.bfloat16, ctx.device)
    if x.shape[3] != HEAD_PITCH:
        raise ValueError("rows must be padded to 128 elements")
    B, N, H, _ = x.shape
    codes = torch.empty(x.shape, dtype=torch.int8, device=x.device)
    scales = torch.empty((B, H, N), dtype=torch.float32, device=x.device)
    ctx._check(ctx.lib.sale_b200_quantize(ctx.handle, _ptr(x), B, N, H, 1, _ptr(codes),
                                          _ptr(scales), _stream()))
    return codes, scales


def quantize_per_key_block(x):
    """quant.hpp:107 (block_k = 32) for every (batch, head) of x [B,N,H,128]."""
    import torch
    ctx = context()
    _check_tensor("x", x, torch.bfloat16, ctx.device)
    if x.shape[3] != HEAD_PITCH:
        raise ValueError("rows must be padded to 128 elements")
    B, N, H, _ = x.shape
    codes = torch.empty(x.shape, dtype=torch.int8, device=x.device)
    scales = torch.empty((B, H, grid(N)[1]), dtype=torch.float32, device=x.device)
    ctx._check(ctx.lib.sale_b200_quantize(ctx.handle, _ptr(x), B, N, H, BLOCK_K, _ptr(codes),
                                          _ptr(scales), _stream()))
    return codes, scales


@dataclass
class SelectDebugOut:
    running_max: object
    exp_sum: object
    bound: object
    block_max: object


def selection_pass(q, k, q_codes, q_scales, k_codes, k_scales, taus, head_dim=128,
                   config: SelectionConfig | None = None, debug=False):
    """selection.hpp:211 for every (batch, q head). taus: one per q head.
    Returns packed mask words int32 [B,Hq,Nq,W] (and SelectDebugOut)."""
    import torch
    ctx = context()
    s = _shape_of(q, k, head_dim)
    nq, nk, nw = grid(s.tokens)
    for name, t, dt, shp in (("q_codes", q_codes, torch.int8, tuple(q.shape)),
                             ("k_codes", k_codes, torch.int8, tuple(k.shape)),
                             ("q_scales", q_scales, torch.float32, (s.batch, s.q_heads, s.tokens)),
                             ("k_scales", k_scales, torch.float32, (s.batch, s.kv_heads, nk))):
        _check_tensor(name, t, dt, ctx.device, len(shp))
        if tuple(t.shape) != shp:
            raise ValueError(f"{name} must have shape {shp}, got {tuple(t.shape)}")
    taus = np.ascontiguousarray(np.broadcast_to(np.asarray(taus, np.float64), (s.q_heads,)))
    mask = torch.empty((s.batch, s.q_heads, nq, nw), dtype=torch.int32, device=q.device)
    dbg_struct = None
    dbg = None
    if debug:
        f = dict(dtype=torch.float64, device=q.device)
        dbg = SelectDebugOut(torch.full((s.batch, s.q_heads, s.tokens), float("nan"), **f),
                             torch.full((s.batch, s.q_heads, s.tokens), float("nan"), **f),
                             torch.full((s.batch, s.q_heads, s.tokens), float("nan"), **f),
                             torch.full((s.batch, s.q_heads, s.tokens, nk), -2 ** 31,
                                        dtype=torch.int32, device=q.device))
        dbg_struct = SelectDebug(dbg.running_max.data_ptr(), dbg.exp_sum.data_ptr(),
                                 dbg.bound.data_ptr(), dbg.block_max.data_ptr())
    cfg = config if config is not None else default_config()
    ctx._check(ctx.lib.sale_b200_select(
        ctx.handle, _ptr(q), _ptr(k), _ptr(q_codes), _ptr(q_scales), _ptr(k_codes),
        _ptr(k_scales), C.byref(s), taus.ctypes.data_as(C.POINTER(C.c_double)), C.byref(cfg),
        _ptr(mask), C.byref(dbg_struct) if dbg_struct is not None else None, _stream()))
    return (mask, dbg) if debug else mask


def block_sparse_attention(q, k, v, mask=None, head_dim=128, coverage=False, q_blocks=None):
    """sparse_attention.hpp:37 (mask = packed words) or, with mask=None,
    full_attention (attention.hpp:18). Returns out bf16 [B,N,Hq,128]
    (and coverage int32 [B,Hq,N]). q_blocks=(i_lo, i_hi): only those query
    blocks' rows are computed (boundaries 0, nq or odd)."""
    import torch
    ctx = context()
    s = _shape_of(q, k, head_dim, v)
    _check_mask(mask, s)
    out = torch.empty(q.shape, dtype=torch.bfloat16, device=q.device)
    cov = (torch.empty((s.batch, s.q_heads, s.tokens), dtype=torch.int32, device=q.device)
           if coverage else None)
    if q_blocks is None:
        ctx._check(ctx.lib.sale_b200_sparse_attention(ctx.handle, _ptr(q), _ptr(k), _ptr(v),
                                                      C.byref(s), _ptr(mask), _ptr(out),
                                                      _ptr(cov), _stream()))
    else:
        ctx._check(ctx.lib.sale_b200_sparse_attention_range(
            ctx.handle, _ptr(q), _ptr(k), _ptr(v), C.byref(s), _ptr(mask), int(q_blocks[0]),
            int(q_blocks[1]), _ptr(out), _ptr(cov), _stream()))
    return (out, cov) if coverage else out


def full_attention(q, k, v, head_dim=128):
    return block_sparse_attention(q, k, v, None, head_dim)


def flop_accounting(mask, tokens):
    """sparse_attention.hpp:101 per (batch, head): int64 [B,Hq,3] =
    (computed, skipped, total) causal blocks."""
    import torch
    ctx = context()
    _check_tensor("mask", mask, torch.int32, ctx.device)
    B, H = mask.shape[0], mask.shape[1]
    if tuple(mask.shape[2:]) != grid(tokens)[::2]:
        raise ValueError(f"mask must be [B, Hq, Nq, W] for {tokens} tokens")
    counts = torch.empty((B, H, 3), dtype=torch.int64, device=mask.device)
    ctx._check(ctx.lib.sale_b200_flop_count(ctx.handle, _ptr(mask), B, H, tokens, _ptr(counts),
                                            _stream()))
    return counts


def prefill(q, k, v, taus, head_dim=128, mask_out=None, config=None, q_blocks=None, ctx=None):
    """run_pipeline's stage composition (runner.hpp:63-80) on device tensors:
    quantize -> selection -> block-sparse attention. Returns out bf16.
    q_blocks=(i_lo, i_hi): only that query-block range (one GPU's share of a
    split unit, K/V replicated); rows outside it are left untouched."""
    import torch
    ctx = ctx or context()
    s = _shape_of(q, k, head_dim, v, ctx)
    _check_mask(mask_out, s, ctx)
    taus = np.ascontiguousarray(np.broadcast_to(np.asarray(taus, np.float64), (s.q_heads,)))
    out = torch.empty(q.shape, dtype=torch.bfloat16, device=q.device)
    cfg = config if config is not None else default_config()
    tp = taus.ctypes.data_as(C.POINTER(C.c_double))
    if q_blocks is None:
        ctx._check(ctx.lib.sale_b200_prefill(ctx.handle, _ptr(q), _ptr(k), _ptr(v), C.byref(s), tp,
                                             C.byref(cfg), _ptr(out), _ptr(mask_out), _stream()))
    else:
        ctx._check(ctx.lib.sale_b200_prefill_range(ctx.handle, _ptr(q), _ptr(k), _ptr(v),
                                                   C.byref(s), tp, C.byref(cfg),
                                                   int(q_blocks[0]), int(q_blocks[1]), _ptr(out),
                                                   _ptr(mask_out), _stream()))
    return out


def query_block_split(nq, parts):
    """Query-block ranges of one (batch, KV group) unit split across `parts`
    GPUs (units < GPUs). The causal work of query block i
    grows like i, so the cumulative work like i^2: boundary p sits near
    nq * sqrt(p / parts), rounded to an odd block (the estimator pairs query
    blocks 2m+1, 2m+2). Returns [(i_lo, i_hi), ...] covering [0, nq)."""
    if parts < 1:
        raise ValueError("query_block_split: parts must be >= 1")
    bounds = [0]
    top = nq - 1 if (nq - 1) % 2 == 1 else nq - 2  # largest odd boundary < nq
    for p in range(1, parts):
        x = int(round(nq * (p / parts) ** 0.5)) | 1
        x = max(x, bounds[-1] + 2 if bounds[-1] > 0 else 1)  # strictly increasing, odd
        x = min(x, top - 2 * (parts - 1 - p))               # room for the later boundaries
        if bounds[-1] < x < nq:
            bounds.append(x)
    bounds.append(nq)
    if len(bounds) - 1 != parts:
        raise ValueError(f"query_block_split: {nq} query blocks cannot be split into {parts} "
                         "ranges with odd inner boundaries")
    return list(zip(bounds[:-1], bounds[1:]))


def prefill_host(q, k, v, taus, out, head_dim=128, config=None, ctx=None):
    """End to end from host buffers (numpy uint16 / pinned torch bf16 on CPU):
    H2D + the three stages + D2H of out, synchronous."""
    ctx = ctx or context()
    ptr = (lambda a: C.c_void_p(a.ctypes.data)) if isinstance(q, np.ndarray) else _ptr
    B, N, Hq, _ = q.shape
    s = Shape(B, N, Hq, k.shape[2], head_dim)
    taus = np.ascontiguousarray(np.broadcast_to(np.asarray(taus, np.float64), (Hq,)))
    cfg = config if config is not None else default_config()
    ctx._check(ctx.lib.sale_b200_prefill_host(ctx.handle, ptr(q), ptr(k), ptr(v), C.byref(s),
                                              taus.ctypes.data_as(C.POINTER(C.c_double)),
                                              C.byref(cfg), ptr(out)))
    return out


# --------------------------------------------------- orchestration (device)

TIMING_LABEL = "B200 (sm_100a)"


def l1_error(reference, approx, head_dim=128):
    """l1_error (calibrate.hpp:20-29) per (batch, q head) of two bf16 outputs
    [B, N, Hq, 128]: mean over tokens of the L1 distance. -> float64 [B, Hq]."""
    ctx = context()
    B, N, H, _ = reference.shape
    s = Shape(B, N, H, H, head_dim)
    out = np.empty((B, H), np.float64)
    ctx._check(ctx.lib.sale_b200_l1_error(ctx.handle, _ptr(reference), _ptr(approx), C.byref(s),
                                          out.ctypes.data))
    return out


def run_pipeline(q, k, v, taus, config=None, dense_mask=False, head_dim=128):
    """run_pipeline (runner.hpp:37-108) for every (batch, q head) of device
    tensors; returns the RunReport as report.hpp:51-87's to_json dict (head
    index b*Hq+h; "timing" holds device-event stage times of the whole batch,
    label TIMING_LABEL)."""
    ctx = context()
    s = _shape_of(q, k, head_dim, v)
    taus = np.ascontiguousarray(np.broadcast_to(np.asarray(taus, np.float64), (s.q_heads,)))
    cfg = config if config is not None else default_config()
    reps = (HeadReport * (s.batch * s.q_heads))()
    tm = StageTiming()
    ctx._check(ctx.lib.sale_b200_run_pipeline(ctx.handle, _ptr(q), _ptr(k), _ptr(v), C.byref(s),
                                              taus.ctypes.data_as(C.POINTER(C.c_double)),
                                              C.byref(cfg), int(bool(dense_mask)), reps,
                                              C.byref(tm)))
    heads = [{"head": r.head, "tau": r.tau, "sparsity": r.sparsity, "err": r.err,
              "computed_blocks": r.computed_blocks, "skipped_blocks": r.skipped_blocks,
              "total_blocks": r.total_blocks,
              "coverage": {"min": r.coverage_min, "max": r.coverage_max,
                           "mean": r.coverage_mean}} for r in reps]
    t = {"label": TIMING_LABEL, "quantization_ms": tm.quantization_ms,
         "selection_ms": tm.selection_ms, "computation_ms": tm.computation_ms,
         "dense_ms": tm.dense_ms}
    t["overhead_ratio"] = ((t["quantization_ms"] + t["selection_ms"]) / t["dense_ms"]
                           if t["dense_ms"] > 0 else 0.0)
    t["computation_speedup"] = t["dense_ms"] / t["computation_ms"] if t["computation_ms"] > 0 else 0.0
    return {"version": 1, "kind": "run_report", "tokens": s.tokens, "head_dim": s.head_dim,
            "heads": s.batch * s.q_heads,
            "selection": {"sink_tokens": cfg.sink_tokens, "local_tokens_min": cfg.local_tokens_min,
                          "segment_size": cfg.segment_size, "block_q": cfg.block_q,
                          "block_k": cfg.block_k},
            "head_reports": heads, "timing": t}


def strip_timing(report: dict) -> dict:
    """report.hpp:89-92: the report without wall-clock data, for diffs."""
    return {k: v for k, v in report.items() if k != "timing"}


def sweep_thresholds(q, k, v, taus, config=None, head_dim=128):
    """sweep_thresholds (runner.hpp:119-165): rows [{tau, sparsity (mean over
    heads), err (max over heads)}] in the given order."""
    ctx = context()
    s = _shape_of(q, k, head_dim, v)
    taus = np.ascontiguousarray(np.asarray(taus, np.float64).ravel())
    rows = (SweepRow * max(1, len(taus)))()
    cfg = config if config is not None else default_config()
    ctx._check(ctx.lib.sale_b200_sweep_thresholds(ctx.handle, _ptr(q), _ptr(k), _ptr(v), C.byref(s),
                                                  taus.ctypes.data_as(C.POINTER(C.c_double)),
                                                  len(taus), C.byref(cfg), rows))
    return [{"tau": r.tau, "sparsity": r.sparsity, "err": r.err} for r in rows[:len(taus)]]


def calibrate_model(samples, theta=0.4, tau0=0.008, max_halvings=30, config=None, head_dim=128,
                    sample_names=None):
    """calibrate_model (calibrate.hpp:149-175): samples = [(q, k, v), ...]
    device tensors [1, N, Hq, 128] / [1, N, Hkv, 128]; every q head runs the
    greedy halving ladder on the device. Returns the CalibrationProfile as
    profile_io.hpp:16-30's JSON dict."""
    ctx = context()
    if not samples:
        raise ValueError("calibrate_model: no samples")
    s = _shape_of(samples[0][0], samples[0][1], head_dim, samples[0][2])
    for j, smp in enumerate(samples):  # every sample shares the first one's shape
        if len(smp) != 3:
            raise ValueError(f"calibrate_model: sample {j} is not a (q, k, v) triple")
        sj = _shape_of(smp[0], smp[1], head_dim, smp[2])
        if (sj.batch, sj.tokens, sj.q_heads, sj.kv_heads) != (s.batch, s.tokens, s.q_heads,
                                                              s.kv_heads):
            raise ValueError(f"calibrate_model: sample {j} shape differs from sample 0")
    n = len(samples)
    arr = lambda i: (vp * n)(*[C.c_void_p(x[i].data_ptr()) for x in samples])
    st = CalibrationSettings(theta, tau0, max_halvings)
    out = (HeadCalibration * s.q_heads)()
    cfg = config if config is not None else default_config()
    ctx._check(ctx.lib.sale_b200_calibrate(ctx.handle, arr(0), arr(1), arr(2), n, C.byref(s),
                                           C.byref(st), C.byref(cfg), out))
    return {"version": 1, "tau0": tau0, "theta": theta,
            "samples": list(sample_names or []),
            "heads": [{"layer": h.layer, "head": h.head, "tau": h.tau,
                       "flag": "converged" if h.flag == 0 else "floor-reached",
                       "halvings": h.halvings} for h in out]}


# ------------------------------------------------------------ file formats

def _file_check(status):
    if status:
        lib = load_library()
        raise _ERRORS.get(status, RuntimeError)((lib.sale_b200_last_error(None) or b"").decode())


def read_tensor_file(path):
    """read_tensor_file (tensor_file.hpp:98-158) into this path's layout:
    (q, k, v) bf16 bit patterns uint16 [1, N, H, 128] (MHA) and the head dim."""
    lib = load_library()
    h, n, d, t = C.c_uint32(), C.c_uint32(), C.c_uint32(), C.c_uint32()
    _file_check(lib.sale_b200_tensor_file_info(path.encode(), C.byref(h), C.byref(n), C.byref(d),
                                               C.byref(t)))
    q, k, v = (np.empty((1, n.value, h.value, HEAD_PITCH), np.uint16) for _ in range(3))
    _file_check(lib.sale_b200_tensor_file_read_bf16(path.encode(), q.ctypes.data, k.ctypes.data,
                                                    v.ctypes.data))
    return q, k, v, d.value


def write_tensor_file(path, q, k, v, head_dim, dtype="f32"):
    """write_tensor_file (tensor_file.hpp:69-96) from bf16 bit patterns
    [1, N, H, 128]; dtype "f32" (the reference's tag 1) or "bf16" (tag 2)."""
    lib = load_library()
    _, n, h, _ = q.shape
    a = lambda x: np.ascontiguousarray(x, np.uint16)
    q, k, v = a(q), a(k), a(v)
    _file_check(lib.sale_b200_tensor_file_write(path.encode(), q.ctypes.data, k.ctypes.data,
                                                v.ctypes.data, h, n, head_dim,
                                                {"f32": 1, "bf16": 2}[dtype]))


def write_mask_dump(path, mask_words, tokens, taus):
    """write_mask_dump (mask_io.hpp:28-69) from packed mask words
    [B, Hq, nq, W] (host numpy or device tensor): one record per (b, h)."""
    lib = load_library()
    words = mask_words.cpu().numpy() if hasattr(mask_words, "cpu") else np.asarray(mask_words)
    words = np.ascontiguousarray(words.view(np.uint32))
    B, H = words.shape[:2]
    t = np.asarray(taus, np.float32).ravel()
    t = np.ascontiguousarray(np.resize(t, B * H) if t.size in (1, H) else t)
    if t.size != B * H:
        raise ValueError("write_mask_dump: taus must be scalar, per head or per record")
    _file_check(lib.sale_b200_mask_dump_write(path.encode(), words.ctypes.data, B, H, tokens,
                                              t.ctypes.data))


def read_mask_dump(path):
    """read_mask_dump (mask_io.hpp:71-125) -> (packed words [R, nq, W] uint32,
    head indices [R], taus float32 [R])."""
    lib = load_library()
    r, nq, nk = C.c_int64(), C.c_int64(), C.c_int64()
    _file_check(lib.sale_b200_mask_dump_read(path.encode(), C.byref(r), C.byref(nq), C.byref(nk),
                                             None, None, None))
    if r.value == 0:
        return np.zeros((0, 0, 0), np.uint32), np.zeros(0, np.uint32), np.zeros(0, np.float32)
    W = (nk.value + 31) // 32
    words = np.zeros((r.value, nq.value, W), np.uint32)
    heads = np.zeros(r.value, np.uint32)
    taus = np.zeros(r.value, np.float32)
    _file_check(lib.sale_b200_mask_dump_read(path.encode(), None, None, None, words.ctypes.data,
                                             heads.ctypes.data, taus.ctypes.data))
    return words, heads, taus


# ------------------------------------------------------------- multi-GPU

def gather_heads(out_shard, group=None):
    """The optional output gather of a KV-group-sharded prefill (SURVEY.md
    §8(e)): every rank holds O for its contiguous slice of query heads,
    [B, N, Hq/world, d]; all_gather (NCCL over NVLink on GPUs, gloo on CPU)
    and concatenate along the head axis -> [B, N, Hq, d] on every rank. Not on
    the critical path: the three SALE stages never exchange data."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    parts = [torch.empty_like(out_shard) for _ in range(world)]
    dist.all_gather(parts, out_shard.contiguous(), group=group)
    return torch.cat(parts, dim=2)


# ------------------------------------------------------------- workloads

def workload_head_f32(kind: str, seed: int, tokens: int, dim: int, head: int = 0):
    """workloads.hpp gaussian_head / sink_local_head: (q, k, v) fp32 [n, d]."""
    lib = load_library()
    q, k, v = (np.empty((tokens, dim), np.float32) for _ in range(3))
    st = lib.sale_b200_workload_head_f32({"gaussian": 0, "sink_local": 1}[kind], seed, tokens,
                                         dim, head, q.ctypes.data, k.ctypes.data, v.ctypes.data)
    if st:
        raise ValueError(f"workload_head_f32: status {st}")
    return q, k, v


def set_timing(enable: bool = True):
    ctx = context()
    ctx._check(ctx.lib.sale_b200_set_timing(ctx.handle, int(enable)))


def stage_times():
    """ms of the last timed prefill: quantize, base mask, stats, estimator, attention."""
    ctx = context()
    ms = (C.c_float * 5)()
    ctx._check(ctx.lib.sale_b200_stage_times(ctx.handle, ms))
    return dict(zip(("quantize", "base_mask", "stats", "estimate", "attention"), list(ms)))


def workload_gqa(kind: str, seed: int, batch: int, tokens: int, q_heads: int, kv_heads: int,
                 head_dim: int = 128, threads: int = 0, out=None, kv_begin: int = 0):
    """GQA extension of the reference generator as bf16 bit
    patterns: uint16 q [B,N,Hq,128], k, v [B,N,Hkv,128] (numpy, host).
    kv_begin > 0 generates the shard of KV heads [kv_begin, kv_begin+kv_heads)
    of a larger model (with their q heads)."""
    lib = load_library()
    if out is None:
        q = np.empty((batch, tokens, q_heads, HEAD_PITCH), np.uint16)
        k = np.empty((batch, tokens, kv_heads, HEAD_PITCH), np.uint16)
        v = np.empty((batch, tokens, kv_heads, HEAD_PITCH), np.uint16)
    else:
        q, k, v = out
    s = Shape(batch, tokens, q_heads, kv_heads, head_dim)
    st = lib.sale_b200_workload_gqa_shard_bf16({"gaussian": 0, "sink_local": 1}[kind], seed,
                                               C.byref(s), kv_begin, q.ctypes.data,
                                               k.ctypes.data, v.ctypes.data, threads)
    if st:
        raise ValueError(f"workload_gqa: status {st}")
    return q, k, v


def bf16_bits_to_f32(a: np.ndarray) -> np.ndarray:
    return (np.asarray(a, np.uint16).astype(np.uint32) << 16).view(np.float32)


def f32_to_bf16_bits(a: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even fp32 -> bf16 bit patterns (finite inputs)."""
    u = np.ascontiguousarray(a, np.float32).view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) >> 16
    return u.astype(np.uint16)
