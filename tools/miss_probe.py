"""Miss-heavy decode step at a short context (development probe, not the bench).

C3's geometry (32Q/8KV, d=128, bf16, W=1024, r=256) at a short context with FRESH queries
(no near-repeat in the ring: every head misses, every ring row survives pass 1 of the
two-pass match): device time of the MAC step vs the full-attention decode on the same state,
L2 flushed as in bench.py.

    python tools/miss_probe.py [--ctx 4096] [--batch 32] [--steps 8]
"""

from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ctx", type=int, default=4096)
    ap.add_argument("--batch", type=int, default=32)
    ap.add_argument("--steps", type=int, default=8)
    ap.add_argument("--miss-frac", type=float, default=1.0, help="fraction of heads given a fresh query")
    ap.add_argument("--mode", default="adaptive", choices=("adaptive", "two_pass", "one_pass", "dense"))
    ap.add_argument("--max-chunks", type=int, default=0, help="splits of a full span per group (0: engine default)")
    ap.add_argument("--slot-cap", type=int, default=0, help="partial slots per group (0: engine default)")
    ap.add_argument("--min-chunk", type=int, default=128)
    a = ap.parse_args()
    import bench

    S = a.steps + 2
    n0 = a.ctx - 2 * S - 1
    states = bench.make_states(list(range(a.batch)), n0=n0, steps=S, hq=32, hkv=8, d=bench.D, dv=bench.D,
                               window=bench.WINDOW, band=bench.BAND)
    import torch

    from paper_2604_00235_b200 import BatchDecodeEngine, EngineConfig
    from paper_2604_00235_b200.synth import inject_into_engine

    dev = torch.device("cuda", 0)
    cfg = EngineConfig(d=bench.D, d_v=bench.D, n_q_heads=32, n_kv_heads=8, window=bench.WINDOW, band=bench.BAND,
                       tau=bench.TAU, storage="bf16")
    eng = BatchDecodeEngine(cfg, a.batch, a.ctx + 64, device=dev, max_chunks=a.max_chunks or None,
                           slot_cap=a.slot_cap or None, min_chunk=a.min_chunk)
    eng.match_mode = a.mode
    inject_into_engine(eng, 0, states, n0, bulk_seed=0)
    g = torch.Generator(device=dev).manual_seed(7)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    mac, full, miss = [], [], []
    q_rep = torch.from_numpy(np.stack([st.step_q for st in states], 1)).to(dev, torch.bfloat16)  # near-repeats
    for s in range(S):
        fresh = torch.randn(a.batch, 32, bench.D, device=dev, generator=g).bfloat16()
        pick = torch.rand(a.batch, 32, 1, device=dev, generator=g) < a.miss_frac
        q = torch.where(pick, fresh, q_rep[s])
        k = torch.randn(a.batch, 8, bench.D, device=dev, generator=g).bfloat16()
        v = torch.randn(a.batch, 8, bench.D, device=dev, generator=g).bfloat16()
        for fn, acc in ((lambda: eng.decode_step(0, q, k, v), mac), (lambda: eng.full_decode(0, q, k, v), full)):
            bench.l2_flush(flush)
            torch.cuda._sleep(200_000)
            e0, e1 = ev(), ev()
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            if s >= 2:
                acc.append(e0.elapsed_time(e1) * 1e3)
        miss.append(1.0 - float(eng.o_use.float().mean()))
    print(json.dumps({"ctx": a.ctx, "batch": a.batch, "mode": a.mode, "miss_frac": a.miss_frac,
                      "max_chunks": eng.max_chunks, "slot_cap": eng.slot_cap, "min_chunk": a.min_chunk, "amend_tma": os.environ.get("MAC_AMEND_TMA", ""),
                      "miss_rate": float(np.mean(miss)),
                      "mac_us": float(np.mean(mac)), "full_us": float(np.mean(full)),
                      "mac_us_median": float(np.median(mac)), "full_us_median": float(np.median(full))}))


if __name__ == "__main__":
    main()
