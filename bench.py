#!/usr/bin/env python
"""bench.py — SALE prefill attention on B200 (BASELINE.json configs[2]).

One step = one full SALE prefill of one attention layer: fused 4-bit Q/K
quantization -> Selection-Pass (exact sink-local stats + tcgen05 i8
estimator) -> block-sparse tcgen05 flash attention, for Llama-3.1-8B's
attention shape (32 Q / 8 KV heads, d = 128), B = 1, 131072 tokens, causal,
on the GQA sink-local synthetic workload, tau = 0.004 (the reference's
SelectionConfig default, selection.hpp:19). Inputs (1.5 GiB) are resident in
HBM and larger than L2.

  python bench.py [--gpus N --steps K --warmup W]          # B200 arm
  python bench.py --impl reference [...]                   # reference CPU arm

Multi-GPU (torchrun): the 8 KV-head groups are sharded across ranks with no
collective on the data path (strong scaling, fixed total work); times are the
max over ranks. Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "prefill attention ms & speedup vs dense at 64K/128K; estimation overhead % of dense"
MODELS = {"llama": ("Llama-3.1-8B", dict(q_heads=32, kv_heads=8, head_dim=128)),
          "qwen": ("Qwen2.5-7B", dict(q_heads=28, kv_heads=4, head_dim=128))}
MODEL = dict(MODELS["llama"][1])  # the selected shape (parse() updates it)


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="b200", choices=["b200", "reference"])
    p.add_argument("--tokens", type=int, default=131072)
    p.add_argument("--batch", type=int, default=1)
    p.add_argument("--tau", type=float, default=0.004)
    p.add_argument("--sweep", default="0.004,0.016,0.064",
                   help="comma list of taus for the density/latency sweep ('' = off)")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--seed", type=int, default=7)
    p.add_argument("--model", default="llama", choices=sorted(MODELS),
                   help="attention shape: llama (32 Q / 8 KV heads) or qwen (28 / 4)")
    p.add_argument("--gather", action="store_true",
                   help="N>1: also time the optional NCCL all_gather of O (not on the critical path)")
    p.add_argument("--second-tokens", type=int, default=65536,
                   help="second sequence length reported beside the headline (0 = off)")
    a = p.parse_args()
    MODEL.clear()
    MODEL.update(MODELS[a.model][1])
    return a


def workload_name(a, tokens=None):
    name = MODELS[a.model][0]
    return (f"{name} attention layer ({MODEL['q_heads']} Q / {MODEL['kv_heads']} KV heads, d=128), "
            f"B={a.batch}, seq {tokens or a.tokens}, causal, GQA sink_local synthetic "
            f"(seed {a.seed}), tau={a.tau}")


def bench_config(a, N, B, world):
    """The config dict of a bench line; both arms print the same one for the
    same command (the driver compares them)."""
    Hq, Hkv, d = MODEL["q_heads"], MODEL["kv_heads"], MODEL["head_dim"]
    split = world // Hkv if world > Hkv and world % Hkv == 0 else 1
    return {"workload": workload_name(a), "tokens": N, "batch": B, "tau": a.tau,
            "q_heads": Hq, "kv_heads": Hkv, "head_dim": d,
            "parallelism": (f"kv-group sharded x{world}, no collective" if split == 1 else
                            f"{Hkv} kv groups x {split} query-block ranges (K/V "
                            "replicated), no collective"),
            "l2": f"inputs ({B * N * (Hq + 2 * Hkv) * d * 2 / 2**30:.2f} GiB) larger "
                  "than L2; no flush"}


def ncu_traffic(kernel):
    """DRAM bytes per launch of `kernel` from the committed ncu --set full
    capture summary (profiles/ncu_traffic.json), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            t = json.load(f)
        return t["kernels"][kernel]["dram_bytes_per_launch"]
    except (OSError, KeyError, ValueError):
        return None


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except OSError:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, \
            "fallback"


def measured_i8_peak():
    """Sustained tcgen05 kind::i8 rate measured on this pool's B200s by
    profiles/i8_peak.cu (profiles/i8_peak.json, TOP/s at the clocks the probe
    saw), else the datasheet dense int8 figure."""
    try:
        with open(os.path.join(ROOT, "profiles", "i8_peak.json")) as f:
            j = json.load(f)
        return float(j["sustained_tops"]), "measured kind::i8 sustained (profiles/i8_peak.json)"
    except (OSError, KeyError, ValueError):
        return 4500.0, "nominal int8 dense (datasheet)"


class ClockSampler:
    """nvidia-smi sampled every 200 ms during the timed region."""

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.path = f"/tmp/sale_clocks_{os.getpid()}.csv"

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={q}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            self.proc.wait()

    def summary(self):
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        sm, mx, reasons = [], [], set()
        try:
            for line in open(self.path):
                f = [x.strip() for x in line.split(",")]
                if len(f) < 6 or not f[0].isdigit():
                    continue
                sm.append(int(f[0]))
                mx.append(int(f[1]))
                for n, v in zip(names, f[2:6]):
                    if v.lower() == "active":
                        reasons.add(n)
        except OSError:
            pass
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": int(np.median(sm)), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


# ------------------------------------------------------------- reference arm
#
# The reference's own CPU hot path (oracle/_ref = the unmodified reference
# headers: quantize_per_token + quantize_per_key_block + selection_pass +
# block_sparse_attention per head under its parallel_for, runner.hpp:57-80
# without the dense baseline) on the box's host cores. Inputs are built in
# oracle/_ref too (ref_workload_gqa_heads: the GQA extension from the
# reference's own Rng / generators, bit-identical to the product generator),
# so this arm never loads the product library.

REF_SAMPLES = (4096, 8192)  # tokens per measured sample; 4096 is configs[0] (C1)


def ref_inputs(a, ns, threads):
    from oracle import oracle as O
    Hq, Hkv, d = MODEL["q_heads"], MODEL["kv_heads"], MODEL["head_dim"]
    q, k, v = (np.empty((Hq, ns, d), np.float32) for _ in range(3))
    st = O.REF.ref_workload_gqa_heads(1, a.seed, ns, d, Hq, Hkv, 1, threads, q, k, v)
    if st:
        raise RuntimeError(f"ref_workload_gqa_heads failed: {st}")
    return q, k, v


def ref_run(inputs, ns, a, threads):
    """One reference run at ns tokens: (wall ms, per-stage thread-time ms
    [quant, selection, computation] summed over heads, runner.hpp:101-106)."""
    from oracle import oracle as O
    wall, stage = np.zeros(1), np.zeros(3)
    st = O.REF.ref_sale_heads(*inputs, MODEL["q_heads"], ns, MODEL["head_dim"], a.tau, threads,
                              wall, stage)
    if st:
        raise RuntimeError(f"reference run failed: {st}")
    return float(wall[0]), stage


def ref_extrapolate(samples, N):
    """Extrapolates the measured wall time to N tokens stage by stage with a
    power law fitted through the two samples (exponent clamped to [1, 2]):
    quantization is linear in N, the selection pass ~quadratic, and the
    computation pass grows like density(N) * N^2 — density falls with N on
    this workload, which the fitted exponent (< 2) carries. Returns
    (ms, exponents)."""
    (n1, w1, s1), (n2, w2, s2) = samples
    alpha = np.clip(np.log(np.maximum(s2, 1e-9) / np.maximum(s1, 1e-9)) / np.log(n2 / n1), 1.0, 2.0)
    grown = s2 * (N / n2) ** alpha
    return float(w2 * grown.sum() / max(s2.sum(), 1e-9)), [float(x) for x in alpha]


def run_reference(a):
    world, rank, _ = dist_env()
    if rank != 0:
        return
    from oracle import oracle as O
    if O.REF is None:
        print(json.dumps({"impl": "reference",
                          "unavailable": "oracle/_ref/libsale_ref.so was not built"}))
        return
    threads = os.cpu_count() or 1
    sizes = [min(n, a.tokens) for n in REF_SAMPLES]
    inputs = {n: ref_inputs(a, n, threads) for n in sizes}
    for _ in range(a.warmup):  # untimed; the smaller sample only
        ref_run(inputs[sizes[0]], sizes[0], a, threads)
    vals, walls, c1 = [], [], []
    for _ in range(a.steps):
        samples = []
        for n in sizes:
            w, stage = ref_run(inputs[n], n, a, threads)
            samples.append((n, w, stage))
        vals.append(ref_extrapolate(samples, a.tokens)[0])
        walls.append(sum(x[1] for x in samples))
        c1.append(samples[0][1])
    _, alpha = ref_extrapolate(samples, a.tokens)
    value = float(np.mean(vals))
    sample = (f"reference quant + selection_pass + block_sparse_attention (runner.hpp:63-80, no "
              f"dense baseline) for all {MODEL['q_heads']} Q heads of the same GQA sink_local "
              f"workload (seed {a.seed}) at {sizes[0]} and {sizes[1]} tokens, {threads} threads, "
              f"measured every step; value extrapolated to {a.tokens} tokens per stage by a "
              f"power law through the two samples (exponents quant/selection/computation "
              f"{alpha[0]:.2f}/{alpha[1]:.2f}/{alpha[2]:.2f})")
    line = {"metric": METRIC, "value": value, "unit": "ms", "n_gpus": a.gpus, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": float(np.mean(walls)), "higher_is_better": False,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32/f64 (CPU reference)",
            "data": "synthetic", "impl": "reference",
            "value_is": f"extrapolated to {a.tokens} tokens from measured samples; ms_per_step is "
                        "the measured wall of one step (both samples)",
            "config": bench_config(a, a.tokens, a.batch, world),
            "cpu_baseline": {"value": value, "unit": "ms", "cores": threads, "kind": "reference",
                             "sample": sample, "extrapolated": True},
            "c1_measured": {"tokens": sizes[0], "q_heads": MODEL["q_heads"],
                            "kv_heads": MODEL["kv_heads"], "wall_ms": float(np.mean(c1)),
                            "threads": threads,
                            "what": "configs[0] (C1) measured, not extrapolated"},
            "e2e": {"value": value, "unit": "ms", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


def cpu_pair(a, threads):
    """The measured CPU-vs-B200 pair at configs[0] (C1: 32 Q / 8 KV heads x
    4096 tokens, tau 0.004) plus the extrapolated reference figure for the
    headline size (same model as the reference arm). The B200 side is the
    public host-buffer call sale_b200_prefill_host on the same inputs (the
    product generator is bit-identical to the reference-built one,
    tests/test_abi.py)."""
    import torch
    from paper_2505_24179_b200 import sale
    sizes = [min(n, a.tokens) for n in REF_SAMPLES]
    samples = []
    for n in sizes:
        w, stage = ref_run(ref_inputs(a, n, threads), n, a, threads)
        samples.append((n, w, stage))
    ext, alpha = ref_extrapolate(samples, a.tokens)
    n1 = sizes[0]
    q16, k16, v16 = sale.workload_gqa("sink_local", a.seed, 1, n1, MODEL["q_heads"],
                                      MODEL["kv_heads"], MODEL["head_dim"])
    pin = lambda x: torch.from_numpy(x).pin_memory()
    hq, hk, hv = pin(q16), pin(k16), pin(v16)
    hout = torch.empty_like(hq).pin_memory()
    taus = [a.tau] * MODEL["q_heads"]
    for _ in range(3):
        sale.prefill_host(hq, hk, hv, taus, hout)
    walls = []
    for _ in range(10):
        t0 = time.perf_counter()
        sale.prefill_host(hq, hk, hv, taus, hout)
        walls.append((time.perf_counter() - t0) * 1e3)
    gpu_ms = float(np.median(walls))
    return {"value": ext, "unit": "ms", "cores": threads, "kind": "reference", "extrapolated": True,
            "sample": f"reference quant + selection_pass + block_sparse_attention, all "
                      f"{MODEL['q_heads']} Q heads, measured at {sizes[0]} and {sizes[1]} tokens "
                      f"({samples[0][1]:.0f} / {samples[1][1]:.0f} ms wall, {threads} threads), "
                      f"extrapolated to {a.tokens} tokens (per-stage power law, exponents "
                      f"{alpha[0]:.2f}/{alpha[1]:.2f}/{alpha[2]:.2f})",
            "c1_pair": {"tokens": n1, "q_heads": MODEL["q_heads"], "kv_heads": MODEL["kv_heads"],
                        "tau": a.tau, "reference_wall_ms": samples[0][1],
                        "b200_e2e_ms": gpu_ms, "speedup": samples[0][1] / gpu_ms,
                        "b200_api": "sale_b200_prefill_host (pinned host buffers, copies timed)",
                        "reference_threads": threads}}


# ------------------------------------------------------------------ B200 arm

def run_b200(a):
    import torch
    world, rank, local = dist_env()
    if world > 1:
        import torch.distributed as dist
        # one GPU per rank; more ranks than GPUs (a functional check on a
        # single-GPU box) share devices round-robin
        torch.cuda.set_device(local % torch.cuda.device_count())
        # NCCL needs one GPU per rank; BENCH_DIST_BACKEND=gloo runs a functional
        # multi-rank check with several ranks on one GPU (timings not meaningful)
        dist.init_process_group(os.environ.get("BENCH_DIST_BACKEND", "nccl"))
    else:
        torch.cuda.set_device(0)
    from paper_2505_24179_b200 import sale
    sale.load_library()

    Hq, Hkv, d = MODEL["q_heads"], MODEL["kv_heads"], MODEL["head_dim"]
    # (batch, KV group) units sharded over ranks; with fewer groups than ranks
    # each group is split into query-block ranges over `split` ranks with K/V
    # replicated, balanced by causal work
    if Hkv % world == 0:
        split, hkv, kv_begin = 1, Hkv // world, rank * (Hkv // world)
    elif world % Hkv == 0:
        split, hkv, kv_begin = world // Hkv, 1, rank // (world // Hkv)
    else:
        raise SystemExit(f"--gpus {world} must divide or be a multiple of the {Hkv} KV heads")
    part = rank % split
    hq = hkv * (Hq // Hkv)
    B = a.batch
    threads = max(1, (os.cpu_count() or 1) // max(1, int(os.environ.get("LOCAL_WORLD_SIZE",
                                                                          world))))
    stream = torch.cuda.current_stream()
    dev = lambda x: torch.from_numpy(x.view(np.int16)).view(torch.bfloat16).cuda()

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
            torch.cuda.synchronize()

    def timed(fn, steps, warmup):
        for _ in range(warmup):
            fn()
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(steps):
            fn()
        e1.record(stream)
        barrier()
        return e0.elapsed_time(e1) / steps

    def measure(N, steps, warmup, headline):
        """One sequence length: prefill (headline: clocks, sweep, e2e), the
        dense-mask run, per-stage times, density, algorithmic work. Per-rank
        values; the caller reduces over ranks."""
        q16, k16, v16 = sale.workload_gqa("sink_local", a.seed, B, N, hq, hkv, d, threads=threads,
                                          kv_begin=kv_begin)
        q, k, v = dev(q16), dev(k16), dev(v16)
        taus = [a.tau] * hq
        nq, nk, nw = sale.grid(N)
        rng = sale.query_block_split(nq, split)[part] if split > 1 else None
        mask = torch.zeros((B, hq, nq, nw), dtype=torch.int32, device="cuda")
        prefill = lambda: sale.prefill(q, k, v, taus, mask_out=mask, q_blocks=rng)
        dense = lambda: sale.block_sparse_attention(q, k, v, None, q_blocks=rng)
        r = {"N": N}
        # ---- K full SALE prefills, device-timed (clocks sampled on the headline)
        if headline:
            with ClockSampler(local) as clocks:
                r["ms"] = timed(prefill, steps, warmup)
            r["clock"] = clocks.summary()
        else:
            r["ms"] = timed(prefill, steps, warmup)
        # ---- dense-mask run of the same attention kernel
        r["dense_ms"] = timed(dense, max(3, steps // 2), warmup)
        # ---- per-stage times (events between the kernels inside the ABI)
        sale.set_timing(True)
        stages = []
        for _ in range(max(3, steps // 2)):
            prefill()
            stages.append(sale.stage_times())
        sale.set_timing(False)
        r["stage_ms"] = {key: float(np.mean([st[key] for st in stages])) for key in stages[0]}
        # ---- density and algorithmic work (this rank's rows)
        i0, i1 = rng if rng is not None else (0, nq)
        r["computed"], r["total"] = rank_counts(mask, N, rng)
        _, cov = sale.block_sparse_attention(q, k, v, mask, coverage=True, q_blocks=rng)
        t0, t1 = 64 * i0, min(64 * i1, N)
        r["attended"] = int(cov[:, :, t0:t1].to(torch.int64).sum().item())
        f_i = np.arange(i0, i1)
        r["est_blocks"] = B * hq * int(np.where(f_i >= 3, 4 * ((2 * f_i - 5) // 4), 0).sum())
        if not headline:
            return r
        # ---- optional output gather over NCCL (timed separately, max over ranks)
        if a.gather and world > 1 and split == 1:
            out = prefill()
            r["gather_ms"] = timed(lambda: sale.gather_heads(out), 3, 1)
        # ---- tau sweep (density vs latency)
        r["sweep"] = []
        taus_sweep = [float(x) for x in a.sweep.split(",") if x.strip()] if a.sweep else []
        for t in taus_sweep:
            tt = [t] * hq
            ms_t = timed(lambda: sale.prefill(q, k, v, tt, mask_out=mask, q_blocks=rng), 3, warmup)
            comp, tot = rank_counts(mask, N, rng)
            r["sweep"].append({"tau": t, "computed": comp, "total": tot, "ms": ms_t})
        # ---- e2e through the public host API (pinned buffers, copies timed)
        r["e2e_ms"] = None
        if not a.no_e2e and split > 1:
            # one rank's share through the public API: pinned host -> device
            # copies of its Q rows and the replicated K / V, the range prefill,
            # the D2H of its output rows, all inside the timed region
            pin = lambda x: torch.from_numpy(x.view(np.int16)).pin_memory()
            t0_, t1_ = 64 * i0, min(64 * i1, N)
            hq16 = pin(np.ascontiguousarray(q16[:, t0_:t1_]))
            hk16, hv16 = pin(k16), pin(v16)
            hout = torch.empty_like(hq16).pin_memory()
            dq = torch.empty_like(q)

            def share():
                dq.view(torch.int16)[:, t0_:t1_].copy_(hq16, non_blocking=True)
                k.view(torch.int16).copy_(hk16, non_blocking=True)
                v.view(torch.int16).copy_(hv16, non_blocking=True)
                o = sale.prefill(dq, k, v, taus, mask_out=mask, q_blocks=rng)
                hout.copy_(o.view(torch.int16)[:, t0_:t1_], non_blocking=True)
                torch.cuda.current_stream().synchronize()
            for _ in range(2):
                share()
            barrier()
            walls = []
            for _ in range(max(3, steps // 2)):
                t0 = time.perf_counter()
                share()
                walls.append((time.perf_counter() - t0) * 1e3)
            r["e2e_ms"] = float(np.mean(walls))
            r["h2d"] = hq16.numel() * 2 + hk16.numel() * 2 + hv16.numel() * 2
            r["d2h"] = hout.numel() * 2
            r["e2e_api"] = "sale.prefill (q_blocks range) with pinned H2D / D2H copies, per rank"
        if not a.no_e2e and split == 1:
            del q, k, v
            pin = lambda x: torch.from_numpy(x).pin_memory()
            hq16, hk16, hv16 = pin(q16), pin(k16), pin(v16)
            hout = torch.empty_like(hq16).pin_memory()
            del q16, k16, v16
            for _ in range(2):
                sale.prefill_host(hq16, hk16, hv16, taus, hout)
            barrier()
            walls = []
            for _ in range(max(3, steps // 2)):
                t0 = time.perf_counter()
                sale.prefill_host(hq16, hk16, hv16, taus, hout)
                walls.append((time.perf_counter() - t0) * 1e3)
            r["e2e_ms"] = float(np.mean(walls))
            r["h2d"] = hq16.numel() * 2 + hk16.numel() * 2 + hv16.numel() * 2
            r["d2h"] = hout.numel() * 2
            r["e2e_api"] = "sale_b200_prefill_host (pinned host buffers)"
        return r

    def rank_counts(mask, N, rng):
        """(computed, total) causal blocks of this rank's query-block rows
        (flop_accounting restricted to [i0, i1), sparse_attention.hpp:101)."""
        if rng is None:
            counts = sale.flop_accounting(mask, N).cpu().numpy()
            return int(counts[..., 0].sum()), int(counts[..., 2].sum())
        i0, i1 = rng
        nq_, nk_, _ = sale.grid(N)
        cells = sale.unpack_mask(mask[:, :, i0:i1].cpu().numpy(), N)
        ii = np.arange(i0, i1)[:, None]
        causal = (32 * np.arange(nk_))[None, :] < np.minimum(64 * (ii + 1), N)
        return int((cells * causal).sum()), int(mask.shape[0] * mask.shape[1] * causal.sum())

    def gather_rows(vec):
        """[world, len(vec)] float64: every rank's vector (all_gather)."""
        if world == 1:
            return np.array([vec], np.float64)
        dev_ = "cuda" if torch.distributed.get_backend() == "nccl" else "cpu"
        t = torch.tensor(vec, dtype=torch.float64, device=dev_)
        parts = [torch.empty_like(t) for _ in range(world)]
        torch.distributed.all_gather(parts, t)
        return np.array([p_.cpu().tolist() for p_ in parts], np.float64)

    def reduce_ranks(r):
        """Times: max over ranks; counts: sum; plus the per-rank values (for
        the imbalance and the per-GPU roofline). Rank 0 gets the result."""
        keys = list(r["stage_ms"])
        mine = [r["ms"], r["dense_ms"], r.get("e2e_ms") or 0.0, r.get("gather_ms", 0.0),
                r["computed"], r["total"], r["attended"], r["est_blocks"]] + \
            [r["stage_ms"][k2] for k2 in keys]
        M = gather_rows(mine)
        if r.get("e2e_ms") is not None:
            r["h2d"], r["d2h"] = (float(x) for x in gather_rows([r["h2d"], r["d2h"]]).sum(0))
        if "sweep" in r:
            for e in r["sweep"]:
                S = gather_rows([e.pop("ms"), e.pop("computed"), e.pop("total")])
                e["ms"], e["density"] = float(S[:, 0].max()), float(S[:, 1].sum() / S[:, 2].sum())
        r["per_rank"] = M
        r["ms"], r["dense_ms"] = float(M[:, 0].max()), float(M[:, 1].max())
        if r.get("e2e_ms") is not None:
            r["e2e_ms"] = float(M[:, 2].max())
        if "gather_ms" in r:
            r["gather_ms"] = float(M[:, 3].max())
        r["computed"], r["total"], r["attended"], r["est_blocks"] = (float(x) for x in M[:, 4:8].sum(0))
        r["stage_ms"] = dict(zip(keys, [float(x) for x in M[:, 8:].max(0)]))
        r["stage_ms_rank"] = {k2: M[:, 8 + n_].tolist() for n_, k2 in enumerate(keys)}
        r["density"] = r["computed"] / r["total"]
        sel = r["stage_ms"]["base_mask"] + r["stage_ms"]["stats"] + r["stage_ms"]["estimate"]
        r["overhead"] = (r["stage_ms"]["quantize"] + sel) / r["dense_ms"]
        r["imbalance"] = {"ms_max_over_mean": float(M[:, 0].max() / M[:, 0].mean()),
                          "ms_per_rank": M[:, 0].tolist(),
                          "density_per_rank": (M[:, 4] / np.maximum(M[:, 5], 1)).tolist()}
        return r

    main_r = reduce_ranks(measure(a.tokens, a.steps, a.warmup, True))
    second = None
    if a.second_tokens and a.second_tokens != a.tokens:
        second = reduce_ranks(measure(a.second_tokens, max(3, a.steps // 2), a.warmup, False))
    if rank != 0:
        torch.distributed.destroy_process_group()
        return
    N = a.tokens
    ms_step, ms_dense, e2e_ms = main_r["ms"], main_r["dense_ms"], main_r.get("e2e_ms")
    stage_ms, density, overhead = main_r["stage_ms"], main_r["density"], main_r["overhead"]
    clock, sweep = main_r["clock"], main_r["sweep"]
    attn_flops = 4.0 * d * main_r["attended"]                # QK^T + PV, 2 flop per MAC
    dense_flops = 4.0 * d * B * Hq * N * (N + 1) / 2
    est_ops = 2.0 * 64 * 32 * 128 * main_r["est_blocks"]
    peaks, peak_src = measured_peaks()
    i8_peak, i8_src = measured_i8_peak()
    P = main_r["per_rank"]  # per-rank [.., computed, total, attended, est_blocks, stage ms...]
    sk = list(main_r["stage_ms"])
    col = lambda name: P[:, 8 + sk.index(name)]
    dom = max(("attention", "estimate", "stats", "quantize"), key=lambda s_: stage_ms[s_])
    # achieved = per-GPU algorithmic work / that GPU's kernel time, averaged
    # over ranks (each against ONE GPU's peak); min over ranks beside it
    if dom == "attention":
        per = 4.0 * d * P[:, 6] / (col("attention") * 1e-3) / 1e12
        roof = {"kernel": "sparse_attention_kernel (K3)", "bound": "tensor",
                "achieved": float(per.mean()), "peak": peaks["bf16_tflops_sustained"],
                "unit": "TFLOP/s", "peak_source": f"{peak_src} bf16 sustained",
                "algorithmic": f"4*d*sum(coverage) = {attn_flops:.4g} flop per launch (all ranks)"}
    elif dom == "estimate":
        per = 2.0 * 64 * 32 * 128 * P[:, 7] / (col("estimate") * 1e-3) / 1e12
        roof = {"kernel": "estimate_kernel (K2b)", "bound": "tensor", "achieved": float(per.mean()),
                "peak": i8_peak, "unit": "TOP/s", "peak_source": i8_src,
                "algorithmic": f"2*64*32*128 per estimated block = {est_ops:.4g} op per launch"}
    else:
        per = np.zeros(world)
        roof = {"kernel": dom, "bound": "compute", "achieved": 0.0, "peak": 1.0, "unit": "n/a"}
    roof["per_gpu"] = True
    roof["achieved_min_rank"] = float(per.min())
    roof["frac"] = roof["achieved"] / roof["peak"]
    kname = roof["kernel"].split()[0]
    tb = ncu_traffic(kname) if world == 1 and N == 131072 and B == 1 and a.model == "llama" else None
    roof["traffic"] = tb / 1e9 if tb else None
    if tb:
        roof["traffic_unit"] = "GB per launch (dram read+write, ncu --set full, profiles/ncu_traffic.json)"

    line = {"metric": METRIC, "value": ms_step, "unit": "ms", "n_gpus": world,
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": ms_step,
            "higher_is_better": False, "scaling": "strong", "vs_baseline": None,
            "dtype": "bf16 (attention) / int8 (estimator)", "data": "synthetic",
            "config": bench_config(a, N, B, world),
            "speedup_vs_dense": ms_dense / ms_step, "dense_ms": ms_dense,
            "estimation_overhead_pct": 100.0 * overhead, "density": density,
            "stage_ms": stage_ms, "effective_tflops": dense_flops / (ms_step * 1e-3) / 1e12,
            "tau_sweep": sweep, "roofline": roof, "clocks": clock,
            "gpu_launches": (5 if split == 1 else 6) * a.steps,
            "estimator_roofline": {
                "kernel": "estimate_kernel (K2b)", "bound": "tensor", "unit": "TOP/s",
                "achieved": float((2.0 * 64 * 32 * 128 * P[:, 7] / (col("estimate") * 1e-3) / 1e12).mean()),
                "peak": i8_peak, "peak_source": i8_src}}
    line["estimator_roofline"]["frac"] = line["estimator_roofline"]["achieved"] / i8_peak
    if world > 1:
        line["imbalance"] = main_r["imbalance"]
    if "gather_ms" in main_r:
        line["output_gather_ms"] = main_r["gather_ms"]
    if second is not None:
        line["at_%dk" % (second["N"] // 1024)] = {
            "tokens": second["N"], "ms": second["ms"], "dense_ms": second["dense_ms"],
            "speedup_vs_dense": second["dense_ms"] / second["ms"],
            "estimation_overhead_pct": 100.0 * second["overhead"], "density": second["density"],
            "stage_ms": second["stage_ms"]}
    if e2e_ms is not None:
        line["e2e"] = {"value": e2e_ms, "unit": "ms", "h2d_bytes_per_step": int(main_r["h2d"]),
                       "d2h_bytes_per_step": int(main_r["d2h"]), "api": main_r["e2e_api"],
                       "max_over_ranks": world > 1}
    if world == 1 and not a.no_cpu_baseline:
        try:
            line["cpu_baseline"] = cpu_pair(a, os.cpu_count() or 1)
        except Exception as e:  # the oracle is a reported baseline, never the product
            line["cpu_baseline"] = {"value": None, "unavailable": str(e)}
    print(json.dumps(line))
    if world > 1:
        torch.distributed.destroy_process_group()


def main():
    a = parse()
    if a.impl == "reference":
        run_reference(a)
    else:
        run_b200(a)


if __name__ == "__main__":
    main()
