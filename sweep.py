"""Hit-rate / window sweep (BASELINE.json configs[4]).

    python sweep.py [--batch 16] [--seq-len 16384] [--windows 16,64,256] [--taus 0.3,0.45,0.6,0.75]
                    [--noise 0.05,0.4] [--out gpurun_out/sweep.jsonl]

Continuous generation from m = 1 for a batch of independent requests (the
reference generator's `redundant` preset, Llama-3-8B attention shape 32Q/8KV,
d = 128, bf16 storage) through `BatchDecodeEngine.decode_step`, for every
(window W, threshold tau, query noise) cell.  Per cell it reports the
reference's metrics (acceptance = hit rate, skip ratio, kv_fraction; engine.py:
226-243), the physical GQA KV bytes the hit path read (group spans from the
device decisions), the match bytes, and the decode latency per
step against this repo's full-attention decode on the same state, sampled at
fixed positions (device time: each sampled step is queued behind a GPU spin so
host launch overhead is not in it).  The threshold sweep also varies the query noise: on the
stock preset repeat distances (~noise*sqrt(d)) sit far inside every radius,
so tau alone is flat.

Traces come from `gen_synthetic` (byte-identical to the reference generator),
one seed per request, generated once per noise level in worker processes.
"""

from __future__ import annotations

import argparse
import json
import multiprocessing as mp
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


def _trace(args):
    seed, seq_len, noise = args
    from paper_2604_00235_b200 import PRESETS, SyntheticSpec, gen_synthetic

    kw = dict(PRESETS["redundant"])
    kw["noise_eps"] = noise
    tr = gen_synthetic(SyntheticSpec(seq_len=seq_len, d=128, d_v=128, n_q_heads=32, n_kv_heads=8, seed=seed, **kw))
    return tr.q_pre[:, 0], tr.k_pre[:, 0], tr.v[:, 0]


def _timed(fn, samples, m):
    """Device time of one step launched behind a GPU spin, so the host's launch overhead is
    hidden (the step's kernels run back to back)."""
    import torch

    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda._sleep(400_000)
    a.record()
    fn()
    b.record()
    samples.append((m, a, b))


def run_cell(traces, W, tau, batch, seq_len, sample_every, device):
    import torch

    from paper_2604_00235_b200 import BatchDecodeEngine, EngineConfig

    q_all, k_all, v_all = traces
    cfg = EngineConfig(d=128, d_v=128, n_q_heads=32, n_kv_heads=8, window=W, band=256, tau=tau, storage="bf16")
    eng = BatchDecodeEngine(cfg, batch, seq_len + 1, device=device)
    r, g, hq, hkv = 256, 4, 32, 8
    use_log = torch.empty(seq_len, batch, hq, dtype=torch.int32, device=device)
    pos_log = torch.empty(seq_len, batch, hq, dtype=torch.int32, device=device)
    mac = []
    for m in range(1, seq_len + 1):
        step = lambda: eng.decode_step(0, q_all[m - 1], k_all[m - 1], v_all[m - 1])  # noqa: E731
        if m % sample_every == 0:
            _timed(step, mac, m)
        else:
            step()
        use_log[m - 1].copy_(eng.o_use)
        pos_log[m - 1].copy_(eng.o_pos)
    torch.cuda.synchronize()
    # the reference's metrics (engine.py:188-243) from the logged device decisions
    mm = torch.arange(1, seq_len + 1, device=device, dtype=torch.int64).view(-1, 1, 1)
    use = use_log.bool()
    skipped = torch.where(use, (pos_log.long() - r).clamp(min=0), torch.zeros_like(mm))   # (p - r)+ on hits
    head_tok = (mm - skipped).sum()
    grp_tok = (mm.view(-1, 1, 1) - skipped.view(seq_len, batch, hkv, g).min(-1).values).sum()  # GQA spans
    decisions = seq_len * batch * hq
    full_tok = batch * hkv * seq_len * (seq_len + 1) // 2
    match_rows = batch * hq * sum(min(m - 1, W) for m in range(1, seq_len + 1))
    out = {
        "window": W, "tau": tau, "acceptance": float(use.sum()) / decisions,
        "skip_ratio": float((skipped.double() / mm).sum()) / decisions,
        "kv_fraction": float(head_tok) / (hq / hkv * full_tok),
        "group_kv_fraction": float(grp_tok) / full_tok,
        "kv_bytes_read": int(grp_tok) * 2 * 128 * 2,
        "kv_bytes_full": int(full_tok) * 2 * 128 * 2,
        "match_bytes": int(match_rows) * 128 * 2,
        "mac_ms_at": {str(m): a.elapsed_time(b) for m, a, b in mac},
    }
    # full-attention decode on a fresh engine (append + exact attention over [1, m]), same positions
    full = BatchDecodeEngine(cfg, batch, seq_len + 1, device=device)
    samples = []
    for m in range(1, seq_len + 1):
        step = lambda: full.full_decode(0, q_all[m - 1], k_all[m - 1], v_all[m - 1])  # noqa: E731
        if m % sample_every == 0:
            _timed(step, samples, m)
        else:
            step()
    torch.cuda.synchronize()
    out["full_ms_at"] = {str(m): a.elapsed_time(b) for m, a, b in samples}
    del eng, full
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=16)
    ap.add_argument("--seq-len", type=int, default=16384)
    ap.add_argument("--windows", default="16,64,256")
    ap.add_argument("--taus", default="0.3,0.45,0.6,0.75")
    ap.add_argument("--noise", default="0.05,0.4")
    ap.add_argument("--sample-every", type=int, default=2048)
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "sweep.jsonl"))
    a = ap.parse_args()
    windows = [int(x) for x in a.windows.split(",")]
    taus = [float(x) for x in a.taus.split(",")]
    noises = [float(x) for x in a.noise.split(",")]
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    results = []
    for noise in noises:
        t0 = time.time()
        with mp.get_context("fork").Pool(min(a.batch, os.cpu_count() or 1, 8)) as pool:
            per_req = pool.map(_trace, [(sd, a.seq_len, noise) for sd in range(a.batch)])
        import torch

        dev = torch.device("cuda", 0)
        traces = tuple(torch.from_numpy(np.stack([r[i] for r in per_req], 1)).to(dev, torch.bfloat16).contiguous()
                       for i in range(3))  # [L, B, H, d]
        del per_req
        gen_s = time.time() - t0
        for W in windows:
            for tau in taus:
                res = run_cell(traces, W, tau, a.batch, a.seq_len, a.sample_every, dev)
                res.update(noise_eps=noise, batch=a.batch, seq_len=a.seq_len, trace_gen_s=gen_s)
                print(json.dumps(res), flush=True)
                results.append(res)
                with open(a.out, "a") as fh:
                    fh.write(json.dumps(res) + "\n")
        del traces
    return results


if __name__ == "__main__":
    main()
