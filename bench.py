"""Benchmark of the MAC-Attention decode step on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--workload c3|c2]

One "step" = one decode step of one attention layer for every request of the
batch (append + match + amend + complete), i.e. one token per request.
Default workload is BASELINE configs[2] / SURVEY C3 (Llama-3-8B attention
shape 32Q/8KV, d=128, bf16, 128K context, batch 32 per GPU, W=1024, r=256,
tau=0.45), hit-path variant (every query repeats a recent one), started from
injected state (paper_2604_00235_b200/synth.py).

`value` is whole-job decode throughput (tokens/s over all ranks) with inputs
resident in HBM, timed with CUDA events per step, L2 flushed (256 MiB write)
between steps; `e2e` is the same through the public engine API with pinned
host inputs copied in and outputs copied out inside the timed region.
`--impl reference` times the reference algorithm's CPU implementation (the
numpy restatement in oracle/, the reference package being Python) on the
host cores on the same workload.
"""

from __future__ import annotations

import argparse
import json
import math
import multiprocessing as mp
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOADS = {
    # name: (context, batch per GPU, Hq, Hkv, description)
    "c3": dict(ctx=131072, batch=32, hq=32, hkv=8, desc="C3: Llama-3-8B attention 32Q/8KV d=128 bf16, 128K ctx, batch 32/GPU"),
    "c2": dict(ctx=32768, batch=8, hq=32, hkv=8, desc="C2: Llama-3-8B attention 32Q/8KV d=128 bf16, 32K ctx, batch 8/GPU"),
    # one 512K request, miss path, KV sequence-sharded over the ranks (sharded.py)
    "c4": dict(ctx=524288, batch=1, hq=64, hkv=8, desc="C4: Llama-3-70B attention 64Q/8KV d=128 bf16, 512K ctx, batch 1, "
                                                          "miss path, KV-sharded over the GPUs"),
}
D = 128
WINDOW, BAND, TAU = 1024, 256, 0.45


def measured_peak_gbs():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


FLUSH_MODE = "write+read"


def l2_flush(buf: torch.Tensor):
    """Evict L2 between timed steps: write a 256 MiB buffer (2x the 126 MB L2), then, in the
    default mode, read it back — the read evicts the write's dirty lines, so their write-back
    does not land inside the next timed step (a pure write flush leaves up to ~126 MB of dirty
    lines that the step's own misses must write back: measured ~2-4 us per C3 step).  Either
    way no input of the step is L2-resident when its timed region starts."""
    buf.zero_()
    if FLUSH_MODE == "write+read":
        buf.sum()


def ncu_traffic(stage: str):
    """Per-launch DRAM bytes (read + write) of a stage's kernel from the committed ncu --set full
    capture (profiles/r02/ncu_traffic.json, written by tools/ncu_traffic.py), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "r02", "ncu_traffic.json")) as fh:
            return float(json.load(fh)[stage]["traffic_bytes"])
    except Exception:
        return None


# ----------------------------------------------------------------------------
# clocks sampler (nvidia-smi during the timed region)
# ----------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index, self.proc, self.lines = index, None, []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, flag in zip(names, parts[2:6]):
                if flag.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


# ----------------------------------------------------------------------------
# algorithmic bytes
# ----------------------------------------------------------------------------
def step_bytes(use, pos, m, hq, hkv, d, window, band, s_kv=2, s_ring=2, two_pass=True):
    """Per-request algorithmic bytes of one MAC step, from the step's device decisions.

    use/pos: [B, Hq] arrays; m: [B] positions.  Returns dict of totals over the batch.
    Two-pass match (default): the scan streams dims 0..P-1 of every live ring row (the
    contiguous ring_qp plane, P = MAC_PLANAR_DIMS), writes a 4-byte partial per row and a
    16-byte summary per 64 rows; the verify reads the summaries and the other d - P dims of
    two candidate rows per head.  Rows that survive the bound (a few near-repeats on the hit path) are not counted
    (a lower bound: the GB/s derived from it cannot be overstated; ncu's DRAM bytes
    cross-check it in profiles/)."""
    from paper_2604_00235_b200._lib import PLANAR_DIMS as PD
    g = hq // hkv
    B = use.shape[0]
    match = verify = kv = summ = 0
    n_sum = -(-window // 64)
    for b in range(B):
        live = min(int(m[b]) - 1, window)
        if two_pass:
            match += hq * (live * PD * s_ring + window * 4 + n_sum * 16 + d * s_ring)
            verify += hq * (n_sum * 16 + 2 * (d - PD) * s_ring + d * s_ring)
        else:
            match += hq * live * d * s_ring + hq * d * s_ring
        for j in range(hkv):
            u = use[b, j * g:(j + 1) * g]
            p = pos[b, j * g:(j + 1) * g]
            lo = min((max(1, int(pp) - band + 1) if uu else 1) for uu, pp in zip(u, p))
            kv += (int(m[b]) - lo + 1) * 2 * d * s_kv
        summ += int(use[b].sum()) * (d * 4 + 4)
    ring_w = B * hq * (d * s_ring + PD * s_ring + d * 4 + 4)  # ring_q row, its ring_qp copy, summary
    out_w = B * hq * d * 4
    append = B * hkv * 2 * d * s_kv
    return {"match": match, "verify": verify, "amend": kv, "complete": summ + ring_w + out_w, "append": append,
            "total": match + verify + kv + summ + ring_w + out_w + append}


def full_bytes(m, hq, hkv, d, s_kv=2):
    return sum(int(x) * hkv * 2 * d * s_kv for x in m) + len(m) * hq * d * 4


# ----------------------------------------------------------------------------
# CPU reference leg (oracle restatement of the reference, one request per process)
# ----------------------------------------------------------------------------
def _cpu_worker(args):
    seed, n0, steps, warm = args
    from threadpoolctl import threadpool_limits

    threadpool_limits(1)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import mac_oracle as orc
    from paper_2604_00235_b200.synth import inject_into_oracle, request_state

    wl = _CPU_WL
    st = request_state(seed, n0=n0, steps=warm + steps, hq=wl["hq"], hkv=wl["hkv"], d=D, dv=D, window=WINDOW,
                       band=BAND)
    cfg = orc.OracleConfig(d=D, d_v=D, n_q_heads=wl["hq"], n_kv_heads=wl["hkv"], window=WINDOW, band=BAND, tau=TAU,
                           storage="bf16")
    eng = orc.OracleEngine(cfg, capacity=n0 + warm + steps + 64)
    inject_into_oracle(eng, 0, st, n0)
    times, outs, hits = [], [], 0
    for s in range(warm + steps):
        t0 = time.perf_counter()
        r = eng.decode_step(0, st.step_q[s], st.step_k[s], st.step_v[s], n0 + s + 1)
        dt = time.perf_counter() - t0
        if s >= warm:
            times.append(dt)
        outs.append(r.outputs)
        hits += int(r.use_hit.sum())
    return times, np.stack(outs), hits


_CPU_WL = None


def cpu_reference(wl, n0, steps, warm, procs, seeds):
    global _CPU_WL
    _CPU_WL = wl
    ctx = mp.get_context("fork")
    t0 = time.perf_counter()
    with ctx.Pool(procs) as pool:
        res = pool.map(_cpu_worker, [(sd, n0, steps, warm) for sd in seeds])
    wall = time.perf_counter() - t0
    per_step = [t for r in res for t in r[0]]
    return {
        "per_step_s_mean": float(np.mean(per_step)),
        "per_step_s_p50": float(np.median(per_step)),
        "tokens_per_s": len(seeds) / float(np.mean([sum(r[0]) / len(r[0]) for r in res])) if per_step else 0.0,
        "outputs": {sd: r[1] for sd, r in zip(seeds, res)},
        "hits": sum(r[2] for r in res),
        "wall_s": wall,
    }


def cpu_model():
    try:
        with open("/proc/cpuinfo") as fh:
            for ln in fh:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


REF_DIR = os.path.join(ROOT, "baseline", "_ref")


def reference_available() -> bool:
    return os.path.isdir(os.path.join(REF_DIR, "attnreuse"))


def _ref_worker(args):
    """One request through the UNMODIFIED reference package (baseline/_ref/attnreuse,
    DecodeEngine.decode_step, engine.py:410-539) on one host core.  The decode state at n0 is
    injected into the reference's own containers (KvStore head buffers, QueryRing,
    SummaryRing) before timing — the reference has no prefill, and replaying 128K steps per
    request is out of reach on a CPU — then every timed step is a stock decode_step call.
    Storage: the reference's f32 store (it has no bf16 mode) holding the same bf16-rounded
    keys/values the GPU reads, so both sides see identical values."""
    seed, n0, steps, warm = args
    from threadpoolctl import threadpool_limits

    threadpool_limits(1)
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    import attnreuse as ar
    from attnreuse import engine as ar_engine
    from attnreuse import kvstore as ar_kv
    from paper_2604_00235_b200.synth import request_state

    wl = _CPU_WL
    hq, hkv = wl["hq"], wl["hkv"]
    st = request_state(seed, n0=n0, steps=warm + steps, hq=hq, hkv=hkv, d=D, dv=D, window=WINDOW, band=BAND)
    cfg = ar.EngineConfig(d=D, d_v=D, n_layers=1, n_q_heads=hq, n_kv_heads=hkv, window=WINDOW, band=BAND,
                          tau=TAU, storage="f32")
    eng = ar.DecodeEngine(cfg)
    T = st.tail_k.shape[1]
    cap = n0 + warm + steps + 64
    for j in range(hkv):
        buf = ar_kv._HeadBuffer(D, D)
        buf.keys = np.zeros((cap, D))   # lazily mapped: only the tail pages are touched
        buf.values = np.zeros((cap, D))
        buf.keys[n0 - T:n0] = st.tail_k[j]
        buf.values[n0 - T:n0] = st.tail_v[j]
        buf.n = n0
        eng.store._heads[(0, j)] = buf
    pos = np.arange(n0 - WINDOW + 1, n0 + 1)
    slots = (pos - 1) % WINDOW
    for h in range(hq):
        qr, sr = eng.rings(0, h)
        qr._q[slots] = st.ring_q[h]
        qr._sqnorm[slots] = np.einsum("wd,wd->w", st.ring_q[h].astype(np.float64), st.ring_q[h].astype(np.float64))
        qr._pos[slots] = pos
        qr._count = n0
        for i, (p, sl) in enumerate(zip(pos, slots)):
            sr._items[sl] = ar_engine.AttentionSummary(acc=st.ring_acc[h, i].astype(np.float64),
                                                       lse=float(st.ring_lse[h, i]), count=max(0, int(p) - BAND))
        sr._pos[slots] = pos
        sr._count = n0
    times, outs, hits = [], [], 0
    for s in range(warm + steps):
        t0 = time.perf_counter()
        r = eng.decode_step(0, st.step_q[s], st.step_k[s], st.step_v[s], n0 + s + 1)
        dt = time.perf_counter() - t0
        if s >= warm:
            times.append(dt)
        outs.append(r.outputs)
        hits += sum(1 for c in r.cached_summaries if c is not None)
    return times, np.stack(outs), hits


def ref_reference(wl, n0, steps, warm, procs, seeds):
    global _CPU_WL
    _CPU_WL = wl
    t0 = time.perf_counter()
    with mp.get_context("fork").Pool(procs) as pool:
        res = pool.map(_ref_worker, [(sd, n0, steps, warm) for sd in seeds])
    wall = time.perf_counter() - t0
    per_step = [t for r in res for t in r[0]]
    return {
        "per_step_s_mean": float(np.mean(per_step)),
        "tokens_per_s": len(seeds) / float(np.mean([sum(r[0]) / len(r[0]) for r in res])),
        "hits": sum(r[2] for r in res), "wall_s": wall,
    }


def run_reference_arm(args, wl):
    """--impl reference: the reference's own CPU implementation of the path (the unmodified
    `attnreuse` package installed in baseline/_ref) on the host cores, one request per process,
    on this workload; the numpy restatement in oracle/ stands in only when baseline/_ref is
    absent (kind "port")."""
    cores = os.cpu_count() or 1
    procs = max(1, min(cores, args.cpu_procs or cores, wl["batch"]))
    n0 = wl["ctx"] - args.warmup - args.steps - 1
    seeds = list(range(procs))
    if reference_available():
        r = ref_reference(wl, n0, args.steps, args.warmup, procs, seeds)
        kind, what = "reference", "the unmodified reference package (baseline/_ref/attnreuse, DecodeEngine.decode_step, f32 store)"
        dtype = "f64 math / f32 store of bf16-rounded values"
    else:
        r = cpu_reference(wl, n0, args.steps, args.warmup, procs, seeds)
        kind, what = "port", "oracle/ numpy restatement (baseline/_ref absent)"
        dtype = "f64 math / bf16-rounded storage"
    val = r["tokens_per_s"]
    line = {
        "impl": "reference",
        "metric": "decode attention throughput (MAC hit path), tokens/s",
        "value": val,
        "unit": "tokens/s",
        "n_gpus": args.gpus,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": r["per_step_s_mean"] * 1e3,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": dtype,
        "data": "synthetic injected state (paper_2604_00235_b200/synth.py)",
        "config": {"workload": wl["desc"] + " — CPU sample", "requests_sampled": procs, "context": wl["ctx"],
                   "window": WINDOW, "band": BAND, "tau": TAU},
        "hit_rate": r["hits"] / max(1, procs * (args.steps + args.warmup) * wl["hq"]),
        "cpu_baseline": {"value": val, "unit": "tokens/s", "cores": procs, "kind": kind,
                         "sample": f"{procs} requests x {args.steps} timed steps (1 process each) of {what}, "
                                   f"model {cpu_model()}"},
        "e2e": {"value": val, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------
# GPU arm
# ----------------------------------------------------------------------------
def _state(a):
    from paper_2604_00235_b200.synth import request_state

    sd, kw = a
    return request_state(sd, **kw)


def make_states(seeds, **kw):
    # generated in forked workers before CUDA is initialised in this process
    with mp.get_context("fork").Pool(max(1, min(len(seeds), os.cpu_count() or 1))) as pool:
        return pool.map(_state, [(sd, kw) for sd in seeds])


def run_ours(args, wl):
    B, hq, hkv = wl["batch"], wl["hq"], wl["hkv"]
    rank = int(os.environ.get("RANK", "0"))
    S = args.warmup + args.steps
    n0 = wl["ctx"] - S - 1
    seeds = [rank * B + b for b in range(B)]
    states = make_states(seeds, n0=n0, steps=S, hq=hq, hkv=hkv, d=D, dv=D, window=WINDOW, band=BAND)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    sub = None
    if args.workload == "c3" and world == 1 and not args.no_sub:
        # the 32K point of the headline metric (C2), measured in the same run as a sub-record
        wl2 = WORKLOADS["c2"]
        S2 = args.warmup + min(args.steps, 20)
        n2 = wl2["ctx"] - S2 - 1
        sub = (wl2, n2, S2, make_states([10_000 + b for b in range(wl2["batch"])], n0=n2, steps=S2, hq=wl2["hq"],
                                        hkv=wl2["hkv"], d=D, dv=D, window=WINDOW, band=BAND))

    import torch
    import torch.distributed as dist

    from paper_2604_00235_b200 import BatchDecodeEngine, EngineConfig
    from paper_2604_00235_b200.synth import inject_into_engine

    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    nccl_ranks = 1
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
        nccl_ranks = dist.get_world_size()
        if rank == 0:
            print(f"bench: NCCL process group of {nccl_ranks} ranks (request-sharded, no data-path collective)",
                  file=sys.stderr, flush=True)

    W_, K = args.warmup, args.steps
    cfg = EngineConfig(d=D, d_v=D, n_q_heads=hq, n_kv_heads=hkv, window=WINDOW, band=BAND, tau=TAU, storage="bf16",
                       page_size=args.page_size)
    eng = BatchDecodeEngine(cfg, B, wl["ctx"] + args.full_steps + 64, device=dev, min_chunk=args.min_chunk,
                            max_chunks=args.max_chunks or None)
    inject_into_engine(eng, 0, states, n0, bulk_seed=rank)
    bf = torch.bfloat16
    q_all = torch.from_numpy(np.stack([s.step_q for s in states], 1)).to(dev, bf)  # [S, B, Hq, d]
    k_all = torch.from_numpy(np.stack([s.step_k for s in states], 1)).to(dev, bf)
    v_all = torch.from_numpy(np.stack([s.step_v for s in states], 1)).to(dev, bf)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream(dev)

    stages = ("mac_append_kv", "mac_match_scan", "mac_match_verify", "mac_amend", "mac_complete")
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(len(stages) + 1)] for _ in range(S)]
    use_log = torch.empty(S, B, hq, dtype=torch.int32, device=dev)
    pos_log = torch.empty(S, B, hq, dtype=torch.int32, device=dev)
    m_log = torch.empty(S, B, dtype=torch.int32, device=dev)
    cpu_procs = max(1, min(os.cpu_count() or 1, args.cpu_procs or (os.cpu_count() or 1), B))
    outs0 = torch.empty(S, cpu_procs, hq, D, dtype=torch.float32, device=dev)

    # pass 1 (the measurement): W warm-up + K timed decode steps, one engine call each
    # (3 kernels: front = append+match+plan, amend, complete), CUDA events around each
    # step on the launching stream, L2 flushed (256 MiB write) before every step
    sev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(S)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    with ClockSampler(local) as clk:
        for s in range(S):
            l2_flush(flush)
            torch.cuda._sleep(200_000)  # keep the host ahead of the device: no launch gaps inside the step
            sev[s][0].record(stream)
            eng.decode_step(0, q_all[s], k_all[s], v_all[s])
            sev[s][1].record(stream)
            use_log[s].copy_(eng.o_use)
            pos_log[s].copy_(eng.o_pos)
            m_log[s].copy_(eng.seq_lens[0])
            outs0[s].copy_(eng.o_out[: outs0.shape[1]])
        torch.cuda.synchronize(dev)
        # pass 2 (breakdown): the same steps again from the same state, one launch per stage
        inject_into_engine(eng, 0, states, n0, bulk_seed=rank)
        torch.cuda.synchronize(dev)
        for s in range(S):
            l2_flush(flush)
            torch.cuda._sleep(400_000)  # ~0.2 ms of GPU spin: the stage launches queue up behind it
            q, k, v = q_all[s], k_all[s], v_all[s]
            ev[s][0].record(stream)
            for i, name in enumerate(stages):
                eng.stage(name, 0, q, k, v)
                ev[s][i + 1].record(stream)
        torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    stage_ms = np.array([[ev[s][i].elapsed_time(ev[s][i + 1]) for i in range(len(stages))] for s in range(W_, S)])
    step_ms = np.array([sev[s][0].elapsed_time(sev[s][1]) for s in range(W_, S)])
    total_ms = float(step_ms.sum())
    if world > 1:
        t = torch.tensor([total_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    ms_per_step = total_ms / K

    use = use_log.cpu().numpy()
    pos = pos_log.cpu().numpy()
    mm = m_log.cpu().numpy()
    from paper_2604_00235_b200 import _lib as mac_lib

    two_pass = bool(eng.match_path() & mac_lib.PATH_TWO_PASS)  # the scan the timed steps ran
    byts = [step_bytes(use[s], pos[s], mm[s], hq, hkv, D, WINDOW, BAND, two_pass=two_pass) for s in range(W_, S)]
    hit_rate = float(use[W_:].mean())

    # full-attention decode baseline on the same state (runs after the MAC steps: it does not write rings)
    F = max(3, min(K, args.full_steps))
    fev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(F + 2)]
    fm = []
    for s in range(F + 2):
        l2_flush(flush)
        fev[s][0].record(stream)
        eng.full_decode(0, q_all[s % S], k_all[s % S], v_all[s % S])
        fev[s][1].record(stream)
        fm.append(eng.seq_lens[0].clone())
    torch.cuda.synchronize(dev)
    full_ms = float(np.mean([a.elapsed_time(b) for a, b in fev[2:]]))
    full_b = float(np.mean([full_bytes((x + 0).cpu().numpy(), hq, hkv, D) for x in fm[2:]]))

    # e2e: the public serving API (StepGraph: one CUDA-graph replay per step holding the H2D
    # copies of the step's inputs from pinned host memory, the step's kernels and the D2H copy
    # of its output); the host writes each step's inputs into the pinned staging buffers first
    from paper_2604_00235_b200 import StepGraph

    E = max(3, min(K, 20))
    e_q = q_all[:E].cpu()
    e_k = k_all[:E].cpu()
    e_v = v_all[:E].cpu()
    # rewind to a consistent state: re-inject so e2e steps are real MAC steps again
    inject_into_engine(eng, 0, states, n0, bulk_seed=rank)
    # serving output dtype: bf16 to the next layer; inputs read from the pinned buffer by the step
    sg = StepGraph(eng, 0, out_dtype=torch.bfloat16, host_inputs=not args.e2e_pull)
    torch.cuda.synchronize(dev)
    eev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(E)]
    e_out0 = []
    for s in range(E):
        sg.q_host.copy_(e_q[s])
        sg.k_host.copy_(e_k[s])
        sg.v_host.copy_(e_v[s])
        l2_flush(flush)
        torch.cuda._sleep(400_000)  # the replay is queued before the first event: device time only
        eev[s][0].record(stream)
        sg.replay()
        eev[s][1].record(stream)
        torch.cuda.synchronize(dev)  # the staging buffers are rewritten for the next step
        e_out0.append(sg.out_host[0].clone())
    e2e_ms = float(np.mean([a.elapsed_time(b) for a, b in eev[1:]]))
    if world > 1:
        t = torch.tensor([e2e_ms, full_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms, full_ms = float(t[0]), float(t[1])
    h2d, d2h = sg.h2d_bytes, sg.d2h_bytes
    # the graph path computes the same steps as the timed pass (same state, same inputs)
    e2e_vs_timed = max(float((e_out0[s].float() - outs0[s, 0].cpu()).abs().max() /
                             outs0[s, 0].abs().max().cpu()) for s in range(min(E, S)))

    peak, peak_kind = measured_peak_gbs()
    mean_b = {k_: float(np.mean([b[k_] for b in byts])) for k_ in byts[0]}
    stage_mean = stage_ms.mean(0)
    kern = {name: {"ms": float(stage_mean[i]), "bytes": mean_b[key],
                   "gbs": mean_b[key] / (stage_mean[i] * 1e-3) / 1e9}
            for i, (name, key) in enumerate(zip(stages, ("append", "match", "verify", "amend", "complete")))}
    dom = max(("mac_match_scan", "mac_amend"), key=lambda n: kern[n]["bytes"])
    step_gbs = mean_b["total"] / (ms_per_step * 1e-3) / 1e9

    sub_rec = mix_rec = None
    if sub is not None:
        del sg
        sub_rec = measure_sub(args, dev, *sub)
        mix_rec = measure_mix(args, dev)

    result = None
    if rank == 0:
        cpu = None
        if world == 1 and not args.no_cpu:
            procs = cpu_procs
            cpu = cpu_reference(wl, n0, args.cpu_steps, 1, procs, seeds[:procs])
            # parity of the timed GPU steps against the CPU reference on the sampled requests
            worst = 0.0
            o = outs0.cpu().numpy()
            for i, sd in enumerate(seeds[:procs]):
                ref = cpu["outputs"][sd]
                for s in range(min(ref.shape[0], S)):
                    for h in range(hq):
                        if use[s, i, h]:
                            den = np.linalg.norm(ref[s, h])
                            worst = max(worst, float(np.linalg.norm(o[s, i, h] - ref[s, h]) / den))
            cpu["parity_worst_rel"] = worst
        value = world * B / (ms_per_step * 1e-3)
        result = {
            "metric": "decode attention throughput (MAC hit path), tokens/s",
            "value": value,
            "unit": "tokens/s",
            "n_gpus": world,
            "steps": K,
            "warmup": W_,
            "ms_per_step": ms_per_step,
            "higher_is_better": True,
            "scaling": "weak",
            "vs_baseline": None,
            "dtype": "bf16",
            "data": "synthetic injected state + all-hit query trace (paper_2604_00235_b200/synth.py)",
            "config": {"workload": wl["desc"], "batch_per_gpu": B, "global_batch": B * world, "context": wl["ctx"],
                       "hq": hq, "hkv": hkv, "d": D, "window": WINDOW, "band": BAND, "tau": TAU,
                       "page_size": args.page_size, "variant": "hit path (rep_prob=1, noise 0.05, gap<=512)",
                       "l2": f"flushed (256 MiB {FLUSH_MODE}) between steps", "parallelism": f"request-sharded x{world}",
                       "nccl_ranks": nccl_ranks},
            "per_token_latency_us": ms_per_step * 1e3,
            "hit_rate": hit_rate,
            "kv_gbs": step_gbs,
            "kv_frac_of_peak": step_gbs / peak,
            "bytes_per_step": mean_b,
            "kernels": kern,
            "full_attention": {"ms_per_step": full_ms, "gbs": full_b / (full_ms * 1e-3) / 1e9,
                               "frac": full_b / (full_ms * 1e-3) / 1e9 / peak, "bytes_per_step": full_b},
            "speedup_vs_full_attention": full_ms / ms_per_step,
            "roofline": {"bound": "hbm", "achieved": kern[dom]["gbs"], "peak": peak, "peak_kind": peak_kind,
                         "unit": "GB/s", "frac": kern[dom]["gbs"] / peak, "traffic": ncu_traffic(dom),
                         "algorithmic_bytes": kern[dom]["bytes"], "kernel": dom,
                         "traffic_source": "profiles/r02/ncu_traffic.json (ncu --set full, DRAM read+write per launch)"},
            "e2e": {"value": world * B / (e2e_ms * 1e-3), "unit": "tokens/s", "ms_per_step": e2e_ms,
                    "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "path": ("StepGraph replay: pinned-host q/k/v pulled over PCIe by mac_io_copy (zero-copy kernel), the step "
                             "kernels, the complete kernel writing the bf16 output into the pinned host buffer (out_bf16)"
                             if args.e2e_pull else
                             "StepGraph replay: the step reads q/k/v from the pinned host buffer over PCIe itself (inputs_host: "
                             "the scan its 16 query dims, the append warps the rest, staging q for the later kernels), the "
                             "complete kernel writes the bf16 output into the pinned host buffer (out_bf16)"),
                    "output_dtype": "bf16",
                    "max_rel_diff_vs_timed_pass_fp32": e2e_vs_timed},
            # front (append + ring scan), verify, amend, complete with the two-pass match
            # (csrc/match_fast.cu launch_front_bf16: B*Hq >= 148 heads); the one-pass match has
            # no verify launch
            "gpu_launches": (4 if two_pass and B * hq >= 148 else 3) * K,
            "clocks": clk.summary(),
        }
        if sub_rec is not None:
            result["c2"] = sub_rec
        if mix_rec is not None:
            result["c3mix"] = mix_rec
        if cpu is not None:
            result["cpu_baseline"] = {"value": cpu["tokens_per_s"], "unit": "tokens/s", "cores": procs, "kind": "port",
                                      "sample": f"{procs} requests x {args.cpu_steps} steps of this workload "
                                                f"(oracle/ numpy restatement, 1 process each), {cpu_model()}",
                                      "per_step_ms": cpu["per_step_s_mean"] * 1e3,
                                      "parity_worst_rel_vs_gpu": cpu["parity_worst_rel"]}
        print(json.dumps(result), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return result


def measure_sub(args, dev, wl, n0, S, states):
    """A second workload's MAC step and full-attention baseline on this GPU (the C2 point of the
    headline metric: B = 8, 32K): same protocol as the main line (L2 flushed before every step,
    CUDA events on the launching stream), fewer steps."""
    import torch

    from paper_2604_00235_b200 import BatchDecodeEngine, EngineConfig
    from paper_2604_00235_b200.synth import inject_into_engine

    B, hq, hkv = wl["batch"], wl["hq"], wl["hkv"]
    cfg = EngineConfig(d=D, d_v=D, n_q_heads=hq, n_kv_heads=hkv, window=WINDOW, band=BAND, tau=TAU, storage="bf16",
                       page_size=args.page_size)
    eng = BatchDecodeEngine(cfg, B, wl["ctx"] + args.full_steps + 64, device=dev, min_chunk=args.min_chunk)
    inject_into_engine(eng, 0, states, n0, bulk_seed=77)
    bf = torch.bfloat16
    q_all = torch.from_numpy(np.stack([s.step_q for s in states], 1)).to(dev, bf)
    k_all = torch.from_numpy(np.stack([s.step_k for s in states], 1)).to(dev, bf)
    v_all = torch.from_numpy(np.stack([s.step_v for s in states], 1)).to(dev, bf)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream(dev)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(S)]
    use_log, pos_log, m_log = [], [], []
    torch.cuda.synchronize(dev)
    for s in range(S):
        l2_flush(flush)
        torch.cuda._sleep(200_000)
        ev[s][0].record(stream)
        eng.decode_step(0, q_all[s], k_all[s], v_all[s])
        ev[s][1].record(stream)
        use_log.append(eng.o_use.clone())
        pos_log.append(eng.o_pos.clone())
        m_log.append(eng.seq_lens[0].clone())
    torch.cuda.synchronize(dev)
    W_ = args.warmup
    ms = float(np.mean([a.elapsed_time(b) for a, b in ev[W_:]]))
    byts = [step_bytes(use_log[s].cpu().numpy(), pos_log[s].cpu().numpy(), m_log[s].cpu().numpy(), hq, hkv, D,
                       WINDOW, BAND)["total"] for s in range(W_, S)]
    F = max(3, min(S - W_, args.full_steps))
    fev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(F + 2)]
    fm = []
    for s in range(F + 2):
        l2_flush(flush)
        fev[s][0].record(stream)
        eng.full_decode(0, q_all[s % S], k_all[s % S], v_all[s % S])
        fev[s][1].record(stream)
        fm.append(eng.seq_lens[0].clone())
    torch.cuda.synchronize(dev)
    full_ms = float(np.mean([a.elapsed_time(b) for a, b in fev[2:]]))
    peak, peak_kind = measured_peak_gbs()
    gbs = float(np.mean(byts)) / (ms * 1e-3) / 1e9
    rec = {"workload": wl["desc"], "steps": S - W_, "ms_per_step": ms, "per_token_latency_us": ms * 1e3,
           "value": B / (ms * 1e-3), "unit": "tokens/s",
           "hit_rate": float(torch.stack(use_log[W_:]).float().mean()),
           "bytes_per_step": float(np.mean(byts)), "kv_gbs": gbs, "frac_of_peak": gbs / peak, "peak_kind": peak_kind,
           "full_attention_ms": full_ms, "speedup_vs_full_attention": full_ms / ms}
    del eng
    torch.cuda.empty_cache()
    return rec


def measure_mix(args, dev):
    """The mixed regime at the C3 geometry (B = 32, 32Q/8KV, W = 1024, r = 256) and a 16K context:
    a fraction of the heads gets a fresh query (no near-repeat: it misses, and its GQA group reads
    the whole context), the rest near-repeats.  The default (adaptive) engine's device time per
    step after it has adapted (the second half of each run) vs full-attention decode on the same
    state; L2 flushed before every step (tools/miss_probe.py protocol)."""
    import torch

    from paper_2604_00235_b200 import BatchDecodeEngine, EngineConfig
    from paper_2604_00235_b200.synth import inject_into_engine

    ctx, B, hq, hkv, S = 16384, 32, 32, 8, 32
    fracs = (0.005, 0.02, 0.1, 0.3)
    n0 = ctx - len(fracs) * S - 16
    states = make_states(list(range(20_000, 20_000 + B)), n0=n0, steps=S, hq=hq, hkv=hkv, d=D, dv=D, window=WINDOW,
                         band=BAND)
    cfg = EngineConfig(d=D, d_v=D, n_q_heads=hq, n_kv_heads=hkv, window=WINDOW, band=BAND, tau=TAU, storage="bf16")
    eng = BatchDecodeEngine(cfg, B, ctx + 64, device=dev)
    inject_into_engine(eng, 0, states, n0, bulk_seed=5)
    g = torch.Generator(device=dev).manual_seed(11)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream(dev)
    q_rep = torch.from_numpy(np.stack([st.step_q for st in states], 1)).to(dev, torch.bfloat16)
    out = {"workload": "C3 geometry (B=32, 32Q/8KV, W=1024, r=256), 16K context, a fraction of heads with fresh "
                       "queries; adaptive engine, steady state", "context": ctx}
    for frac in fracs:
        ts, miss, modes = [], [], []
        for s in range(S):
            fresh = torch.randn(B, hq, D, device=dev, generator=g).bfloat16()
            pick = torch.rand(B, hq, 1, device=dev, generator=g) < frac
            q = torch.where(pick, fresh, q_rep[s])
            k = torch.randn(B, hkv, D, device=dev, generator=g).bfloat16()
            v = torch.randn(B, hkv, D, device=dev, generator=g).bfloat16()
            l2_flush(flush)
            torch.cuda._sleep(200_000)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            eng.decode_step(0, q, k, v)
            e1.record(stream)
            torch.cuda.synchronize(dev)
            if s >= S - 12:  # the feedback is published every 8th step: measure after two rounds
                ts.append(e0.elapsed_time(e1) * 1e3)
                miss.append(1.0 - float(eng.o_use.float().mean()))
                modes.append(int(eng._step_mode))
        out[f"miss_{frac}"] = {"mac_us": float(np.mean(ts)), "miss_rate": float(np.mean(miss)),
                               "match_modes": sorted(set(modes))}
    fts = []
    for s in range(5):
        l2_flush(flush)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        eng.full_decode(0, q_rep[s], q_rep[s][:, :hkv].contiguous(), q_rep[s][:, :hkv].contiguous())
        e1.record(stream)
        torch.cuda.synchronize(dev)
        if s >= 2:
            fts.append(e0.elapsed_time(e1) * 1e3)
    out["full_attention_us"] = float(np.mean(fts))
    for frac in fracs:
        out[f"miss_{frac}"]["vs_full_attention"] = out[f"miss_{frac}"]["mac_us"] / out["full_attention_us"]
    del eng
    torch.cuda.empty_cache()
    return out


# ----------------------------------------------------------------------------
# C4: KV-sequence-sharded miss path for one very long request
# ----------------------------------------------------------------------------
def run_c4(args, wl):
    """One 512K-token request at the Llama-3-70B attention shape; every query is fresh (the
    miss path: exact attention over [1, m]); the KV sequence is split over the ranks
    (ShardLayout), each rank computes its shard's (piece, band) summaries, one NCCL
    all-gather exchanges them, every rank merges (sharded.py)."""
    import torch
    import torch.distributed as dist

    from paper_2604_00235_b200 import EngineConfig
    from paper_2604_00235_b200.sharded import ShardedDecodeEngine, ShardLayout
    from paper_2604_00235_b200.synth import request_state, tail_len

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    hq, hkv, ctx = wl["hq"], wl["hkv"], wl["ctx"]
    S = args.warmup + args.steps
    n0 = ctx - S - 1
    st = request_state(0, n0=n0, steps=S, hq=hq, hkv=hkv, d=D, dv=D, window=WINDOW, band=BAND, rep_prob=0.0)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    cfg = EngineConfig(d=D, d_v=D, n_q_heads=hq, n_kv_heads=hkv, window=WINDOW, band=BAND, tau=TAU, storage="bf16",
                       page_size=args.page_size)
    T = tail_len(WINDOW, BAND)
    layout = ShardLayout.for_context(ctx, world, min_tail=T + S + 1)
    eng = ShardedDecodeEngine(cfg, 1, layout, rank, ctx + 8, device=dev, min_chunk=args.min_chunk,
                              max_chunks=args.max_chunks or None)
    e = eng.engine
    lo, hi = layout.local_range(rank, n0)
    n_local = hi - lo + 1
    e.reserve(n_local + S + 1)
    gen = torch.Generator(device=dev).manual_seed(1000 + rank)
    e.k_cache[0].normal_(generator=gen)
    e.v_cache[0].normal_(generator=gen)
    if layout.owner(n0) == rank:  # the seeded tail (shared with any CPU check) lives on the tail shard
        pos = torch.arange(n0 - T, n0, device=dev) - layout.offset(rank)
        pages = e.page_table[0, pos // e.page_size].long()
        slots = pos % e.page_size
        for j in range(hkv):
            e.k_cache[0][pages, j, slots] = torch.from_numpy(st.tail_k[j]).to(dev, e.sdt)
            e.v_cache[0][pages, j, slots] = torch.from_numpy(st.tail_v[j]).to(dev, e.sdt)
    slots_r = (torch.arange(n0 - WINDOW + 1, n0 + 1, device=dev) - 1) % WINDOW
    e.ring_q[0][0][:, slots_r] = torch.from_numpy(st.ring_q).to(dev, e.sdt)
    e.ring_acc[0][0][:, slots_r] = torch.from_numpy(st.ring_acc).to(dev, e.sumdt)
    e.ring_lse[0][0][:, slots_r] = torch.from_numpy(st.ring_lse).to(dev, e.sumdt)
    e.sync_ring_qp(0)
    e.seq_lens[0].fill_(n0)
    bf = torch.bfloat16
    q_all = torch.from_numpy(st.step_q[:, None]).to(dev, bf)
    k_all = torch.from_numpy(st.step_k[:, None]).to(dev, bf)
    v_all = torch.from_numpy(st.step_v[:, None]).to(dev, bf)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream(dev)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(S)]
    miss = torch.zeros((), dtype=torch.int64, device=dev)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    with ClockSampler(local) as clk:
        for s in range(S):
            l2_flush(flush)
            torch.cuda._sleep(200_000)
            ev[s][0].record(stream)
            res = eng.decode_step(0, q_all[s], k_all[s], v_all[s])
            ev[s][1].record(stream)
            if s >= args.warmup:
                miss += (res.use_hit == 0).sum()
        torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    total_ms = float(sum(a.elapsed_time(b) for a, b in ev[args.warmup:]))
    if world > 1:
        t = torch.tensor([total_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    ms = total_ms / args.steps
    local_bytes = (n_local + S // 2) * hkv * 2 * D * 2
    peak, peak_kind = measured_peak_gbs()
    gbs = local_bytes / (ms * 1e-3) / 1e9
    if rank == 0:
        line = {
            "metric": "decode attention throughput, KV-sharded miss path (one 512K request), tokens/s",
            "value": 1.0 / (ms * 1e-3), "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic injected state, fresh queries (every head misses)",
            "config": {"workload": wl["desc"], "context": ctx, "hq": hq, "hkv": hkv, "d": D, "window": WINDOW,
                       "band": BAND, "shard_tokens": layout.shard_tokens, "parallelism": f"kv-sharded x{world}",
                       "l2": f"flushed (256 MiB {FLUSH_MODE}) between steps"},
            "miss_rate": float(miss) / (args.steps * hq),
            "per_rank_kv_bytes": local_bytes,
            "roofline": {"bound": "hbm", "achieved": gbs, "peak": peak, "peak_kind": peak_kind, "unit": "GB/s",
                         "frac": gbs / peak, "traffic": None, "kernel": "sharded step (rank 0 shard)"},
            "exchange_bytes_per_rank": hq * 2 * (D + 1) * 4,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=("ours", "reference"))
    ap.add_argument("--workload", default="c3", choices=sorted(WORKLOADS))
    ap.add_argument("--page-size", type=int, default=16)
    ap.add_argument("--min-chunk", type=int, default=128)
    ap.add_argument("--max-chunks", type=int, default=0, help="split-KV slots per group (0: engine default)")
    ap.add_argument("--full-steps", type=int, default=10)
    ap.add_argument("--cpu-procs", type=int, default=0, help="CPU reference processes (0: every host core, "
                    "at most one per request of the workload's batch)")
    ap.add_argument("--cpu-steps", type=int, default=12)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--flush", default="write+read", choices=("write+read", "write"),
                    help="L2 flush between timed steps (see l2_flush)")
    ap.add_argument("--no-sub", action="store_true", help="skip the C2 sub-record of the default c3 line")
    ap.add_argument("--e2e-pull", action="store_true", help="e2e: pull q/k/v with a zero-copy kernel first "
                    "instead of letting the step read them from pinned memory (inputs_host)")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl == "ours":
        # one process per GPU: re-launch this command under torchrun (the driver's own launch
        # sets WORLD_SIZE and lands below)
        import socket

        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
        sys.exit(subprocess.call(cmd))
    world_env = int(os.environ.get("WORLD_SIZE", "1"))
    if args.impl == "ours" and world_env != args.gpus:
        print(f"bench: --gpus {args.gpus} but WORLD_SIZE={world_env}; measuring {world_env} ranks", file=sys.stderr)
    global FLUSH_MODE
    FLUSH_MODE = args.flush
    wl = WORKLOADS[args.workload]
    if args.impl == "reference":
        if int(os.environ.get("RANK", "0")) != 0:
            return
        if args.workload == "c4":
            print(json.dumps({"impl": "reference", "unavailable": "the CPU reference's f64 KV store needs 8.6 GB and "
                              "~10 s per 512K miss step per process; use the default c3 workload"}), flush=True)
            return
        run_reference_arm(args, wl)
        return
    if args.workload == "c4":
        run_c4(args, wl)
        return
    run_ours(args, wl)


if __name__ == "__main__":
    main()
