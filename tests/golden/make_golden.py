"""Generates tests/golden/*.npz from the UNMODIFIED reference (oracle/_ref,
built from /root/reference/proj/include by oracle/Makefile). Run here, where
the reference tree exists; the fixtures are committed and used on the GPU box.

  python tests/golden/make_golden.py

Fixture ref_gqa_640.npz: GQA sink_local workload (seed 7, B=1, N=640,
Hq=2, Hkv=1, d=128, bf16 inputs), per q head: reference quantize_per_token /
quantize_per_key_block outputs, selection_pass masks at tau 0.004 and 0.05,
block_sparse_attention outputs + coverage at tau 0.004, full_attention output.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import oracle as O  # noqa: E402
from paper_2505_24179_b200 import sale  # noqa: E402


def main():
    assert O.REF is not None, "oracle/_ref/libsale_ref.so missing (make -C oracle)"
    N, Hq, Hkv, d = 640, 2, 1, 128
    q16, k16, v16 = sale.workload_gqa("sink_local", 7, 1, N, Hq, Hkv, d)
    f = sale.bf16_bits_to_f32
    out = dict(q16=q16, k16=k16, v16=v16)
    k = np.ascontiguousarray(f(k16[0, :, 0]))
    v = np.ascontiguousarray(f(v16[0, :, 0]))
    kc, ks = np.empty((N, d), np.int8), np.empty(((N + 31) // 32,), np.float32)
    assert O.REF.ref_quantize_per_key_block(k, N, d, 64, 32, kc, ks) == 0
    out.update(k_codes=kc, k_scales=ks)
    for h in range(Hq):
        q = np.ascontiguousarray(f(q16[0, :, h]))
        qc, qs = np.empty((N, d), np.int8), np.empty((N,), np.float32)
        assert O.REF.ref_quantize_per_token(q, N, d, qc, qs) == 0
        out[f"q_codes_{h}"], out[f"q_scales_{h}"] = qc, qs
        for tau in (0.004, 0.05):
            m = np.empty((10, 20), np.uint8)
            assert O.REF.ref_selection_pass(q, k, N, d, qc, qs, kc, ks, tau, 32, 128, 4, 64, 32,
                                            m) == 0
            out[f"mask_{h}_{tau}"] = m
        o, cov = np.empty((N, d), np.float32), np.empty((N,), np.int64)
        assert O.REF.ref_block_sparse_attention(q, k, v, N, d, out[f"mask_{h}_0.004"], 64, 32, o,
                                                cov) == 0
        out[f"sparse_out_{h}"], out[f"coverage_{h}"] = o, cov
        fo = np.empty((N, d), np.float32)
        assert O.REF.ref_full_attention(q, k, v, N, d, fo) == 0
        out[f"full_out_{h}"] = fo
    np.savez_compressed(os.path.join(HERE, "ref_gqa_640.npz"), **out)
    print("wrote", os.path.join(HERE, "ref_gqa_640.npz"))


if __name__ == "__main__":
    main()
