"""Standalone query and summary rings with the reference API, matched on the device.

`QueryRing` / `match_query` (matching.py:67-175) and `SummaryRing`
(engine.py:284-320) as independent objects, for callers that build their own
decode loop from the reference's parts.  Ring rows live in device tensors
(f64, holding whatever rounding the caller pushed, as the reference does);
positions and counts are host bookkeeping.  `match_query` scans the device
ring in the CUDA library (`mac_match_rows`); `match_queries` matches many
rings in one launch.  The engine's own rings are the slot-aligned device
tensors of `BatchDecodeEngine` (`QueryRingView` / `SummaryRingView`).
"""

from __future__ import annotations

import ctypes as C
import math

import numpy as np
import torch

from . import _lib
from .config import MATCH_POST_ROPE, AttentionSummary, MatchConfig, MatchResult, threshold
from .summary import RopeTable, _device, _stream

__all__ = ["QueryRing", "SummaryRing", "match_query", "match_queries"]


class QueryRing:
    """Ring of the `capacity` most recent pre-RoPE queries with cached squared norms.
    Positions must increase; slot = pushes % capacity, so a position sits at
    (pos - 1) mod capacity when pushed once per decode step (matching.py:67-126)."""

    def __init__(self, capacity: int, d: int, *, device=None):
        if capacity < 1:
            raise ValueError("ring capacity must be >= 1")
        self.capacity = capacity
        self.d = d
        self.device = _device(device)
        self._qd = torch.zeros((capacity, d), dtype=torch.float64, device=self.device)
        self._nd = torch.zeros(capacity, dtype=torch.float64, device=self.device)
        self._pd = torch.zeros(capacity, dtype=torch.int64, device=self.device)
        # host mirror for view() / query_at() / evictions (d doubles per push)
        self._q = np.zeros((capacity, d), dtype=np.float64)
        self._sqnorm = np.zeros(capacity, dtype=np.float64)
        self._pos = np.zeros(capacity, dtype=np.int64)
        self._count = 0

    def __len__(self) -> int:
        return min(self._count, self.capacity)

    @property
    def last_position(self) -> int:
        return 0 if self._count == 0 else int(self._pos[(self._count - 1) % self.capacity])

    def push(self, pos: int, q):
        """Store q at `pos`; returns the evicted (pos, query, sq_norm) once full, else None."""
        if pos < 1:
            raise ValueError("positions are 1-based")
        if self._count and pos <= self.last_position:
            raise ValueError(f"ring positions must increase: got {pos} after {self.last_position}")
        q = np.asarray(q, dtype=np.float64)
        if q.shape != (self.d,):
            raise ValueError(f"expected query of dim {self.d}, got shape {q.shape}")
        slot = self._count % self.capacity
        evicted = None
        if self._count >= self.capacity:
            evicted = (int(self._pos[slot]), self._q[slot].copy(), float(self._sqnorm[slot]))
        self._q[slot] = q
        self._sqnorm[slot] = float(q @ q)
        self._pos[slot] = pos
        self._qd[slot].copy_(torch.from_numpy(self._q[slot]))
        self._nd[slot] = self._sqnorm[slot]
        self._pd[slot] = pos
        self._count += 1
        return evicted

    def view(self):
        """(queries, squared norms, positions) of the live entries."""
        n = len(self)
        return self._q[:n], self._sqnorm[:n], self._pos[:n]

    def slot_of(self, pos: int) -> int:
        slot = (pos - 1) % self.capacity
        if len(self) == 0 or self._pos[slot] != pos:
            raise KeyError(f"position {pos} is not in the ring")
        return slot

    def query_at(self, pos: int) -> np.ndarray:
        return self._q[self.slot_of(pos)]


def match_queries(qs, ms, rings: list[QueryRing], cfg: MatchConfig) -> list[MatchResult]:
    """match_query for many (query, position, ring) triples in one library launch.  Rings
    must share capacity, dim and device."""
    n = len(rings)
    if n == 0:
        return []
    r0 = rings[0]
    dev = r0.device
    for ring in rings:
        if ring.capacity != r0.capacity or ring.d != r0.d or ring.device != dev:
            raise ValueError("match_queries needs rings of one capacity, dim and device")
    qs = np.asarray(qs, dtype=np.float64).reshape(n, -1)
    if qs.shape[1] != r0.d:
        raise ValueError(f"expected query of dim {r0.d}, got shape {qs.shape[1:]}")
    for ring, m in zip(rings, ms):
        if len(ring) and ring.last_position >= m:
            raise ValueError("all ring entries must precede the current position")
    W, d = r0.capacity, r0.d
    ring_q = torch.stack([r._qd for r in rings]) if n > 1 else r0._qd[None]
    ring_n = torch.stack([r._nd for r in rings]) if n > 1 else r0._nd[None]
    ring_p = torch.stack([r._pd for r in rings]) if n > 1 else r0._pd[None]
    q = torch.from_numpy(qs).to(dev)
    live = torch.tensor([len(r) for r in rings], dtype=torch.int32, device=dev)
    mm = torch.tensor([int(m) for m in ms], dtype=torch.int32, device=dev)
    hit = torch.empty(n, dtype=torch.int32, device=dev)
    pos = torch.empty(n, dtype=torch.int32, device=dev)
    dist = torch.empty(n, dtype=torch.float64, device=dev)
    scanned = torch.empty(n, dtype=torch.int32, device=dev)
    post = cfg.space == MATCH_POST_ROPE
    freqs = torch.from_numpy(RopeTable(cfg.d, cfg.rope_base).freqs).to(dev) if post else None
    P = _lib.MacMatchRowsParams(
        n_rings=n, capacity=W, head_dim=d, delta_max=int(cfg.delta_max) if cfg.delta_max is not None else 0,
        post_rope=int(post), thr_sq=threshold(cfg.d, cfg.tau) ** 2,
        rope_freqs=freqs.data_ptr() if freqs is not None else None, q=q.data_ptr(), ring_q=ring_q.data_ptr(),
        ring_sqnorm=ring_n.data_ptr(), ring_pos=ring_p.data_ptr(), n_live=live.data_ptr(), m=mm.data_ptr(),
        out_hit=hit.data_ptr(), out_pos=pos.data_ptr(), out_dist=dist.data_ptr(), out_scanned=scanned.data_ptr())
    _lib.check(_lib.load().mac_match_rows(C.byref(P), C.c_void_p(_stream(dev))), "mac_match_rows")
    h, p, dd, s = (t.cpu().numpy() for t in (hit, pos, dist, scanned))
    return [MatchResult(bool(h[i]), int(p[i]) if h[i] else MatchResult.MISS_POS, float(dd[i]), int(s[i]))
            for i in range(n)]


def match_query(q, m: int, ring: QueryRing, cfg: MatchConfig) -> MatchResult:
    """Nearest stored query to `q` and the hit decision (matching.py:141-175): squared
    distance |q|^2 + |c|^2 - 2 q.c from the cached norms, clamped at 0, exact ties to the
    most recent position, hit iff strictly inside threshold(d, tau); Δmax filter and the
    post-RoPE frame change as configured."""
    q = np.asarray(q, dtype=np.float64)
    if q.shape != (ring.d,):
        raise ValueError(f"expected query of dim {ring.d}, got shape {q.shape}")
    if len(ring) and ring.last_position >= m:
        raise ValueError("all ring entries must precede the current position")
    if len(ring) == 0:
        return MatchResult(False, MatchResult.MISS_POS, math.inf, 0)
    return match_queries(q[None], [m], [ring], cfg)[0]


class SummaryRing:
    """Prefix summaries slot-aligned with a QueryRing (engine.py:284-320): acc rows in a device
    tensor, lse / count / position / dtype on the host."""

    def __init__(self, capacity: int, *, device=None):
        if capacity < 1:
            raise ValueError("ring capacity must be >= 1")
        self.capacity = capacity
        self.device = _device(device)
        self._acc = None  # [capacity, d_v] f64, allocated on the first push
        self._meta: list[tuple[float, int, np.dtype] | None] = [None] * capacity
        self._pos = np.zeros(capacity, dtype=np.int64)
        self._count = 0

    def __len__(self) -> int:
        return min(self._count, self.capacity)

    @property
    def last_position(self) -> int:
        return 0 if self._count == 0 else int(self._pos[(self._count - 1) % self.capacity])

    def push(self, pos: int, summary: AttentionSummary):
        if self._count and pos <= self.last_position:
            raise ValueError(f"ring positions must increase: got {pos} after {self.last_position}")
        slot = self._count % self.capacity
        evicted = None
        if self._count >= self.capacity:
            evicted = (int(self._pos[slot]), self._summary(slot))
        acc = np.asarray(summary.acc)
        if self._acc is None or self._acc.shape[1] != acc.shape[0]:
            if self._acc is not None and self._count:
                raise ValueError("summary value dim differs from the ring's")
            self._acc = torch.zeros((self.capacity, acc.shape[0]), dtype=torch.float64, device=self.device)
        self._acc[slot].copy_(torch.from_numpy(acc.astype(np.float64)))
        self._meta[slot] = (float(summary.lse), int(summary.count), acc.dtype)
        self._pos[slot] = pos
        self._count += 1
        return evicted

    def _summary(self, slot: int) -> AttentionSummary:
        lse, count, dt = self._meta[slot]
        return AttentionSummary(acc=self._acc[slot].cpu().numpy().astype(dt), lse=lse, count=count)

    def summary_at(self, pos: int) -> AttentionSummary:
        slot = (pos - 1) % self.capacity
        if len(self) == 0 or self._pos[slot] != pos or self._meta[slot] is None:
            raise KeyError(f"position {pos} is not in the ring")
        return self._summary(slot)

    def acc_device(self) -> torch.Tensor:
        """The [capacity, d_v] f64 device tensor of stored accumulators (slot order)."""
        return self._acc
