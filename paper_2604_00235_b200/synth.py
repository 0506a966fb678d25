"""Injected decode state + step traces for long-context benchmarks (C2/C3/C4 shapes).

Replaying 128K decode steps to fill rings is infeasible on the CPU side
(SURVEY.md §7.3 item 7), so benchmarks start from an injected state:

* KV rows 1..n0 of every request: the tail [n0-T+1, n0] (T >= W + r, every
  row a hit can read) comes from a seeded per-request numpy stream and is
  identical for the GPU engine and the CPU reference; older rows are bulk
  random on the device (read only by misses).
* ring entries for positions n0-W+1..n0: queries on the sqrt(d) sphere,
  prefix summaries with random acc and lse.
* step s (position n0+s) queries: with probability rep_prob a repeat of a
  query in [m-gap_max, m-1] plus noise_eps Gaussian noise, re-projected to
  the sphere (the generator model of workload.py:148-198); else fresh.

All arrays are rounded through bf16 (kept as float32) when storage is bf16.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np


def _bf16(x: np.ndarray) -> np.ndarray:
    f = np.ascontiguousarray(x, dtype=np.float32)
    u = f.view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32)


@dataclass
class RequestState:
    ring_q: np.ndarray    # [Hq, W, d] positions n0-W+1..n0 (oldest first)
    ring_acc: np.ndarray  # [Hq, W, dv]
    ring_lse: np.ndarray  # [Hq, W]
    tail_k: np.ndarray    # [Hkv, T, d] post-RoPE keys at positions n0-T+1..n0
    tail_v: np.ndarray    # [Hkv, T, dv]
    step_q: np.ndarray    # [S, Hq, d] pre-RoPE queries of steps n0+1..n0+S
    step_k: np.ndarray    # [S, Hkv, d]
    step_v: np.ndarray    # [S, Hkv, dv]


def tail_len(window: int, band: int) -> int:
    return ((window + band + 64 + 63) // 64) * 64


def request_state(seed: int, *, n0: int, steps: int, hq: int, hkv: int, d: int, dv: int, window: int, band: int,
                  rep_prob: float = 1.0, noise_eps: float = 0.05, gap_max: int = 512, bf16: bool = True,
                  lse_mean: float = 12.0) -> RequestState:
    """Deterministic per-request state and step trace (numpy PCG64 stream `seed`)."""
    rng = np.random.default_rng(seed)
    W, T, S = window, tail_len(window, band), steps
    rnd = _bf16 if bf16 else (lambda a: np.asarray(a, dtype=np.float32))
    radius = math.sqrt(d)

    def sphere(x):
        return x * (radius / np.linalg.norm(x, axis=-1, keepdims=True))

    hist = np.empty((hq, W + S, d), dtype=np.float32)  # queries of positions n0-W+1 .. n0+S
    hist[:, :W] = rnd(sphere(rng.standard_normal((hq, W, d))))
    ring_acc = rng.standard_normal((hq, W, dv)).astype(np.float32)
    ring_lse = (lse_mean + rng.standard_normal((hq, W))).astype(np.float32)
    tail_k = rnd(rng.standard_normal((hkv, T, d)))
    tail_v = rnd(rng.standard_normal((hkv, T, dv)))
    step_k = np.empty((S, hkv, d), dtype=np.float32)
    step_v = np.empty((S, hkv, dv), dtype=np.float32)
    hidx = np.arange(hq)
    for s in range(S):
        # one child stream per step: the first s steps do not depend on the trace length
        sr = np.random.default_rng([seed, 1, s])
        step_k[s] = rnd(sr.standard_normal((hkv, d)))
        step_v[s] = rnd(sr.standard_normal((hkv, dv)))
        rep = sr.random(hq) < rep_prob
        gap = sr.integers(1, gap_max + 1, size=hq)
        noise = sr.standard_normal((hq, d))
        fresh = sphere(sr.standard_normal((hq, d)))
        i = W + s                     # hist index of position n0 + s + 1
        src = np.maximum(i - gap, 0)  # never older than the injected ring
        q = sphere(hist[hidx, src].astype(np.float64) + noise_eps * noise)
        hist[:, i] = rnd(np.where(rep[:, None], q, fresh))
    return RequestState(hist[:, :W].copy(), ring_acc, ring_lse, tail_k, tail_v,
                        np.ascontiguousarray(hist[:, W:].transpose(1, 0, 2)), step_k, step_v)


def inject_into_engine(eng, layer: int, states: list, n0: int, *, bulk_seed: int = 0):
    """Write injected state into a BatchDecodeEngine (device tensors, in place)."""
    import torch

    cfg = eng.cfg
    B, ps, W = eng.batch, eng.page_size, cfg.window
    T = states[0].tail_k.shape[1]
    eng.reserve(n0 + states[0].step_q.shape[0] + 1)
    gen = torch.Generator(device=eng.device).manual_seed(bulk_seed)
    eng.k_cache[layer].normal_(generator=gen)
    eng.v_cache[layer].normal_(generator=gen)
    dev = eng.device
    pos = torch.arange(n0 - T, n0, device=dev)  # 0-based rows of the tail
    for b, st in enumerate(states):
        pages = eng.page_table[b, pos // ps].long()
        slots = pos % ps
        for j in range(cfg.n_kv_heads):
            eng.k_cache[layer][pages, j, slots] = torch.from_numpy(st.tail_k[j]).to(dev, eng.sdt)
            eng.v_cache[layer][pages, j, slots] = torch.from_numpy(st.tail_v[j]).to(dev, eng.sdt)
        slots_r = (torch.arange(n0 - W + 1, n0 + 1, device=dev) - 1) % W
        eng.ring_q[layer][b][:, slots_r] = torch.from_numpy(st.ring_q).to(dev, eng.sdt)
        eng.ring_acc[layer][b][:, slots_r] = torch.from_numpy(st.ring_acc).to(dev, eng.sumdt)
        eng.ring_lse[layer][b][:, slots_r] = torch.from_numpy(st.ring_lse).to(dev, eng.sumdt)
    eng.sync_ring_qp(layer)
    eng.seq_lens[layer].fill_(n0)


def inject_into_oracle(oeng, layer: int, st: RequestState, n0: int):
    """Same state into a CPU OracleEngine (rows older than the tail stay zero, lazily allocated)."""
    T = st.tail_k.shape[1]
    oeng.inject_tail(layer, n0, st.tail_k.astype(np.float64), st.tail_v.astype(np.float64), n0 - T,
                     st.ring_q.astype(np.float64), st.ring_acc.astype(np.float64), st.ring_lse.astype(np.float64))
