"""Tile-level statistics of the Selection-Pass masks at the bench workload:
block density (reference accounting, 64x32 blocks) vs the fraction of
128x128 attention tiles the K3 kernel must visit under different pairings."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_24179_b200 import sale  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 131072
for tau in (0.004, 0.016, 0.064):
    q16, k16, v16 = sale.workload_gqa("sink_local", 7, 1, N, 32, 8, 128)
    dev = lambda x: torch.from_numpy(x.view(np.int16)).view(torch.bfloat16).cuda()
    q, k, v = dev(q16), dev(k16), dev(v16)
    nq, nk, nw = sale.grid(N)
    mask = torch.empty((1, 32, nq, nw), dtype=torch.int32, device="cuda")
    sale.prefill(q, k, v, tau, mask_out=mask)
    cells = sale.unpack_mask(mask.cpu().numpy(), N)[0]  # [32, nq, nk]
    i = np.arange(nq)[:, None]; j = np.arange(nk)[None, :]
    causal = (32 * j < 64 * (i + 1))
    dens = cells[:, causal].mean()
    # segment-tile view: tile 0 = block 0, tile s+1 = blocks 1+4s..4+4s
    ns = (nk - 1 + 3) // 4
    seg = np.zeros((32, nq, ns + 1), bool)
    seg[:, :, 0] = cells[:, :, 0] > 0
    pad = np.zeros((32, nq, 4 * ns + 1), np.uint8); pad[:, :, :nk] = cells
    seg[:, :, 1:] = pad[:, :, 1:].reshape(32, nq, ns, 4).any(-1)
    qi = np.arange(nq)[:, None]; sj = np.arange(ns + 1)[None, :]
    key0 = np.where(sj == 0, 0, 32 + 128 * (sj - 1))
    seg_causal = key0 < 64 * (qi + 1)
    # pairing within head: tile t = q-blocks (2t-1, 2t)
    T = nq // 2 + 1
    pa = np.zeros((32, T, ns + 1), bool)
    for t in range(T):
        for qb in (2 * t - 1, 2 * t):
            if 0 <= qb < nq:
                pa[:, t] |= seg[:, qb]
    pair_tiles = pa.sum()
    single = seg.sum()  # tiles if every q-block had its own M=64 tile
    dense_pairs = sum(((np.where(np.arange(ns + 1) == 0, 0, 32 + 128 * (np.arange(ns + 1) - 1)) < 64 * (min(2 * t, nq - 1) + 1)).sum()) for t in range(T)) * 32
    # pairing across heads of a GQA group: (h, h+1) at the same q-block
    hp = (seg[0::2] | seg[1::2]).sum()
    # four heads of a group at the same q-block (M=256 as 2x128 pairs, union)
    h4 = (seg[0::4] | seg[1::4] | seg[2::4] | seg[3::4]).sum()
    print(f"N={N} tau={tau}: block density {dens:.4f}; segment-tile density (per q-block) "
          f"{single / (seg_causal.sum() * 32):.4f}; 128-row pair tiles {pair_tiles} = "
          f"{pair_tiles / dense_pairs:.4f} of dense pair tiles; q-block-pair overhead "
          f"{2 * pair_tiles / single:.3f}x; head-pair overhead {2 * hp / single:.3f}x; "
          f"4-head union overhead {4 * h4 / single:.3f}x")
    # best of the three head pairings of each GQA group of four, per q-block
    if seg.shape[0] % 4 == 0:
        best = 0
        for g in range(seg.shape[0] // 4):
            s4 = seg[4 * g:4 * g + 4]                       # [4, nq, ns+1]
            opts = []
            for (a, b), (c, d) in (((0, 1), (2, 3)), ((0, 2), (1, 3)), ((0, 3), (1, 2))):
                opts.append((s4[a] | s4[b]).sum(-1) + (s4[c] | s4[d]).sum(-1))  # per q-block
            best += np.minimum(np.minimum(opts[0], opts[1]), opts[2]).sum()
        print(f"   best-of-3 head pairing per q-block overhead {2 * best / single:.3f}x")
