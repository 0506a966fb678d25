"""GEMM-form prefill ring build at serving scale (development probe, not the bench).

Times mac_build_ring (BatchDecodeEngine.build_ring: the W-1 ring entries AS[1, t-r] under q_t
of a prompt, one tensor-core pass over the cache) against one forced-miss decode step (what
the step-based prefill pays per ring entry), on device-random K/V of the given context.

    python tools/prefill_probe.py [--batch 32] [--ctx 131072] [--reps 3]

Algorithmic work: rows x keys x (2 d for Q K^T + 2 d for P V) flops, rows = B * Hq * (W - 1);
the kernel issues twice that (Q and P split hi/lo into bf16 pairs for fp32-exact logits).
"""

from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=32)
    ap.add_argument("--ctx", type=int, default=131072)
    ap.add_argument("--hq", type=int, default=32)
    ap.add_argument("--hkv", type=int, default=8)
    ap.add_argument("--window", type=int, default=1024)
    ap.add_argument("--band", type=int, default=256)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--chunks", type=int, default=0)
    ap.add_argument("--variant", default="auto", choices=("auto", "mma", "tcgen05"))
    a = ap.parse_args()
    import torch

    from paper_2604_00235_b200 import BatchDecodeEngine, EngineConfig

    dev = torch.device("cuda", 0)
    cfg = EngineConfig(d=128, d_v=128, n_q_heads=a.hq, n_kv_heads=a.hkv, window=a.window, band=a.band,
                       storage="bf16")
    eng = BatchDecodeEngine(cfg, a.batch, a.ctx + 8, device=dev)
    g = torch.Generator(device=dev).manual_seed(3)
    for t in (eng.k_cache[0], eng.v_cache[0]):
        for i in range(0, t.shape[0], 4096):  # bf16 N(0,1) in slabs (no fp32 temporary of the whole cache)
            t[i:i + 4096].copy_(torch.randn(t[i:i + 4096].shape, device=dev, generator=g))
    eng.seq_lens[0].fill_(a.ctx)
    eng._len[0] = a.ctx
    rows = a.window - 1
    q = torch.randn(a.batch, rows, a.hq, 128, device=dev, generator=g).bfloat16()
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    times = []
    for _ in range(a.reps + 1):
        e0, e1 = ev(), ev()
        e0.record()
        eng.build_ring(0, q, n_chunks=a.chunks or None, variant=a.variant)
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1))
    ms = min(times[1:])
    # one forced-miss decode step on the same cache (the step-based prefill's cost per ring entry)
    qs = torch.randn(a.batch, a.hq, 128, device=dev, generator=g).bfloat16()
    ks = torch.randn(a.batch, a.hkv, 128, device=dev, generator=g).bfloat16()
    eng.reserve(a.ctx + 2)
    st = []
    for _ in range(3):
        eng.seq_lens[0].fill_(a.ctx)
        eng._len[0] = a.ctx
        e0, e1 = ev(), ev()
        e0.record()
        eng.decode_step(0, qs, ks, ks, force_miss=True)
        e1.record()
        torch.cuda.synchronize()
        st.append(e0.elapsed_time(e1))
    step_ms = min(st)
    keys = a.ctx - a.band  # per row, ~ (the last rows read up to ctx - r)
    flops = float(a.batch) * a.hq * rows * keys * 4 * 128
    print(json.dumps({"batch": a.batch, "ctx": a.ctx, "rows_per_request": rows, "build_ring_ms": round(ms, 3),
                      "algorithmic_tflops": round(flops / ms / 1e9, 1), "issued_tflops": round(2 * flops / ms / 1e9, 1),
                      "forced_miss_step_ms": round(step_ms, 3), "step_based_ms": round(step_ms * rows, 1),
                      "speedup_vs_steps": round(step_ms * rows / ms, 1), "n_chunks": a.chunks or "auto",
                      "variant": a.variant}))


if __name__ == "__main__":
    main()
