"""In-step kernel timeline of the C3 decode step (development tool).

Runs the C3 hit-path workload of bench.py through the MAC_TIMELINE build of the
library (lib/libmacattn_tl.so: every kernel stamps %globaltimer at entry, after its
grid-dependency wait, and at exit, min and max over CTAs) and prints, per kernel,
when its first / last CTA entered, got past the wait and left, relative to the
first scan CTA, averaged over the steps.

    MAC_TIMELINE=1 python -m paper_2604_00235_b200.build
    python tools/timeline.py [--steps 10] [--batch 32] [--ctx 131072]
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
os.environ["MACATTN_LIB"] = os.path.join(ROOT, "paper_2604_00235_b200", "lib", "libmacattn_tl.so")
sys.path.insert(0, ROOT)

SLOTS = ["scan_in", "scan_out", "verify_in", "verify_waited", "verify_out", "amend_in", "amend_waited",
         "amend_out", "complete_in", "complete_waited", "complete_out", "v_selected", "v_bound", "v_survived", "v_decided", "v_m",
         "dense_in", "dense_waited", "dense_out", "dense_task",
         "plan_in", "plan_alloc", "plan_out", "spare"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--batch", type=int, default=32)
    ap.add_argument("--ctx", type=int, default=131072)
    ap.add_argument("--no-flush", action="store_true")
    ap.add_argument("--max-chunks", type=int, default=0)
    ap.add_argument("--min-chunk", type=int, default=128)
    ap.add_argument("--slot-cap", type=int, default=0)
    ap.add_argument("--fresh", action="store_true", help="random queries: every head misses")
    ap.add_argument("--miss-frac", type=float, default=0.0, help="fraction of heads given a fresh query each step")
    ap.add_argument("--mode", default="adaptive", choices=("adaptive", "two_pass", "one_pass", "dense"))
    a = ap.parse_args()
    import bench

    S = a.steps + 2
    n0 = a.ctx - S - 1
    states = bench.make_states(list(range(a.batch)), n0=n0, steps=S, hq=32, hkv=8, d=bench.D, dv=bench.D,
                               window=bench.WINDOW, band=bench.BAND)
    import torch

    from paper_2604_00235_b200 import BatchDecodeEngine, EngineConfig, _lib
    from paper_2604_00235_b200.synth import inject_into_engine

    dev = torch.device("cuda", 0)
    cfg = EngineConfig(d=bench.D, d_v=bench.D, n_q_heads=32, n_kv_heads=8, window=bench.WINDOW, band=bench.BAND,
                       tau=bench.TAU, storage="bf16")
    eng = BatchDecodeEngine(cfg, a.batch, a.ctx + 64, device=dev, max_chunks=a.max_chunks or None,
                            min_chunk=a.min_chunk, slot_cap=a.slot_cap or None)
    eng.match_mode = a.mode
    inject_into_engine(eng, 0, states, n0, bulk_seed=0)
    lib = _lib.load()
    lib.mac_timeline_offset.restype = ctypes.c_size_t
    lib.mac_timeline_offset.argtypes = [ctypes.POINTER(_lib.MacDecodeParams)]
    bf = torch.bfloat16
    q_all = torch.from_numpy(np.stack([s.step_q for s in states], 1)).to(dev, bf)
    k_all = torch.from_numpy(np.stack([s.step_k for s in states], 1)).to(dev, bf)
    v_all = torch.from_numpy(np.stack([s.step_v for s in states], 1)).to(dev, bf)
    if a.fresh:
        gen = torch.Generator(device=dev).manual_seed(7)
        q_all = torch.randn(q_all.shape, device=dev, generator=gen).to(bf)
    elif a.miss_frac > 0:
        gen = torch.Generator(device=dev).manual_seed(7)
        fresh = torch.randn(q_all.shape, device=dev, generator=gen).to(bf)
        pick = torch.rand(q_all.shape[:3] + (1,), device=dev, generator=gen) < a.miss_frac
        q_all = torch.where(pick, fresh, q_all)
    P = eng._params(0, q_all[0], k_all[0], v_all[0], _lib.DT_BF16)
    off = int(lib.mac_timeline_offset(P))
    tl = eng.workspace[off:off + 16 * len(SLOTS)].view(torch.int64).view(len(SLOTS), 2)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    rows, amends = [], []
    lib.mac_timeline_amend.restype = ctypes.c_int
    lib.mac_timeline_amend.argtypes = [ctypes.c_void_p, ctypes.c_int]
    tr = np.zeros((4096, 8), np.uint64)
    for s in range(S):
        tl[:, 0] = torch.iinfo(torch.int64).max
        tl[:, 1] = 0
        if not a.no_flush:
            bench.l2_flush(flush)
        torch.cuda._sleep(200_000)
        eng.decode_step(0, q_all[s], k_all[s], v_all[s])
        torch.cuda.synchronize()
        t = tl.cpu().numpy().astype(np.float64)
        if s >= 2:
            rows.append(t)
            tr[:] = 0
            lib.mac_timeline_amend(tr.ctypes.data, 4096)
            amends.append((tr.copy(), t[0, 0]))
    t = np.stack(rows)  # [steps, 16, 2] ns
    base = t[:, 0, 0][:, None, None]
    rel = (t - base) / 1e3  # us
    out = {}
    for i, name in enumerate(SLOTS):
        first, last = rel[:, i, 0], rel[:, i, 1]
        ok = t[:, i, 1] > 0
        if ok.any():
            out[name] = (round(float(first[ok].mean()), 2), round(float(last[ok].mean()), 2))
    print(json.dumps({"batch": a.batch, "ctx": a.ctx, "miss_frac": a.miss_frac, "mode": a.mode, "max_chunks": eng.max_chunks, "slot_cap": eng.slot_cap, "min_chunk": a.min_chunk, "hit_rate": float(eng.o_use.float().mean()),
                      "first_last_us": out}))
    for name, (f, l) in out.items():
        print(f"{name:16s} first {f:8.2f}  last {l:8.2f}")
    if os.environ.get("MAC_AMEND_TC") == "1":  # the tcgen05 amend's per-CTA role counters
        lib.mac_timeline_amend_tc.restype = ctypes.c_int
        lib.mac_timeline_amend_tc.argtypes = [ctypes.c_void_p, ctypes.c_int]
        tc = np.zeros((1024, 16), np.uint64)
        lib.mac_timeline_amend_tc(tc.ctypes.data, 1024)
        live = tc[:, 1] > 0
        a = tc[live].astype(np.float64)
        dur = (a[:, 1] - a[:, 0]) / 1e3
        cyc = 1.965e3  # cycles per us
        q = lambda x: " ".join(f"{v:7.2f}" for v in np.percentile(x, [10, 50, 90]))
        print(f"tc amend CTAs {int(live.sum())}  items/CTA p10/50/90 {q(a[:, 7])}  blocks {q(a[:, 12])}  duration us {q(dur)}")
        for i, name in ((2, "softmax wait S"), (3, "softmax wait O"), (4, "softmax item start"),
                        (5, "producer wait stage"), (6, "mma wait data"), (8, "sm logits/masks"),
                        (9, "sm vote barrier"), (10, "sm rescale"), (11, "sm P write+fence"), (13, "sm finalize")):
            print(f"  {name:20s} us p10/50/90: {q(a[:, i] / cyc)}")
    # per-CTA amend trace: start/end spread, items and tokens per warp, first-item duration
    for tr, base in amends[-2:]:
        live = tr[:, 1] > 0
        if not live.any():  # (the per-CTA trace is the one-warp amend's; the TMA amend has none)
            continue
        a = tr[live].astype(np.float64)
        t0 = (a[:, 0] - base) / 1e3
        t1 = (a[:, 1] - base) / 1e3
        tf = (a[:, 4] - base) / 1e3
        items, toks = a[:, 2], a[:, 3]
        q = lambda x: " ".join(f"{v:7.2f}" for v in np.percentile(x, [0, 10, 50, 90, 100]))
        print(f"amend CTAs {int(live.sum())}  items total {int(items.sum())}  tokens total {int(toks.sum())}")
        tin = (a[:, 6] - base) / 1e3
        print(f"  entry  us p0/10/50/90/100: {q(tin)}")
        bnd = a[:, 7] > 0
        if bnd.any():
            tb = (a[bnd, 7] - base) / 1e3
            print(f"  band CTAs {int(bnd.sum())}: band end us p0/10/50/90/100: {q(tb)}  band dur us: {q(tb - tin[bnd])}")
        print(f"  start  us p0/10/50/90/100: {q(t0)}")
        print(f"  end    us p0/10/50/90/100: {q(t1)}")
        has = items > 0
        print(f"  first item dur us        : {q((tf - t0)[has])}  tokens {q(a[has, 5])}")
        print(f"  items/CTA hist: {np.bincount(items.astype(int)).tolist()}")
        busy = (t1 - t0)
        print(f"  busy us                  : {q(busy)}  -> tokens/us/warp {toks.sum() / busy.sum():.2f}")


if __name__ == "__main__":
    main()
