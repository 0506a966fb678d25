"""KV-sequence-sharded decode for single very long requests (BASELINE config 4).

One request's KV cache is split into G contiguous shards, one per GPU: rank r
holds positions ``r*S+1 .. (r+1)*S`` and the last rank holds everything from
``(G-1)*S+1`` on (it receives the appends).  The rings (query ring, summary
ring) are small (Hq·W·(d+d_v+1) values per request) and are *replicated* on
every rank, so every rank runs the identical match and reaches identical
decisions without any broadcast.

One decode step is two C-ABI calls around the path's only exchange
(SURVEY.md §8e):

1. ``mac_shard_partial``: append (stored only by the shard that owns position
   m), match, plan clamped to this shard's tokens, amend, and the per-head
   (piece, band) summaries of this shard — piece = tokens ``t <= m-r``, band =
   ``t > m-r`` (engine.py:404-408,469-470,484-493) — into ``shard_send``
   ``[B, Hq, 2, d_v+1]`` f32 (acc..., lse).
2. one ``all_gather_into_tensor`` of ``shard_send`` into ``shard_parts``
   ``[G, B, Hq, 2, d_v+1]`` over NCCL (NVLink 5 / NVSwitch); 64 heads · 2 ·
   129 · 4 B = 66 KB per rank at the Llama-3-70B shape.
3. ``mac_shard_complete``: every rank merges ``cached(p) ⊕ pieces`` and
   ``prefix ⊕ bands`` in rank order (attention.py:119-135), writes the output,
   ρ and the ring slot ``(m-1) mod W`` (engine.py:374-402), and advances
   ``seq_lens``.  The merge order is fixed, so the ring replicas stay
   bit-identical across ranks.

Hit heads read ``[p-r+1, m]`` — at most W+r tokens — which lies in the tail
shard when it holds at least W+r tokens; the other shards' plans for such a
group are empty and contribute empty summaries (lse = -inf, the merge
identity).  Misses read their share of ``[1, m]`` on every rank in parallel.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch

from . import _lib
from .engine import BatchDecodeEngine, BatchStepResult


@dataclass(frozen=True)
class ShardLayout:
    """Contiguous split of one request's positions over ``world`` ranks."""

    shard_tokens: int   # S: positions per non-tail shard
    world: int

    def __post_init__(self):
        if self.world < 1:
            raise ValueError("world must be >= 1")
        if self.shard_tokens < 1:
            raise ValueError("shard_tokens must be >= 1")

    def offset(self, rank: int) -> int:
        """Positions held by earlier shards (the shard's ``kv_offset``)."""
        self._check(rank)
        return rank * self.shard_tokens

    def limit(self, rank: int) -> int:
        """Positions this shard holds (``kv_limit``); 0 = unbounded (the tail shard)."""
        self._check(rank)
        return 0 if rank == self.world - 1 else self.shard_tokens

    def owner(self, pos: int) -> int:
        """Rank holding 1-based position ``pos``."""
        if pos < 1:
            raise ValueError("positions are 1-based")
        return min((pos - 1) // self.shard_tokens, self.world - 1)

    def local_range(self, rank: int, m: int) -> tuple[int, int]:
        """Positions of ``[1, m]`` held by ``rank`` (inclusive; empty when lo > hi)."""
        lo = self.offset(rank) + 1
        lim = self.limit(rank)
        hi = m if lim == 0 else min(m, self.offset(rank) + lim)
        return lo, hi

    @staticmethod
    def for_context(total_tokens: int, world: int, min_tail: int = 0) -> "ShardLayout":
        """Even split of ``total_tokens``; the tail shard keeps at least ``min_tail`` of them
        (W + r, so that hit spans never leave it)."""
        s = -(-total_tokens // world)
        if world > 1 and total_tokens - (world - 1) * s < min_tail:
            s = max(1, (total_tokens - min_tail) // (world - 1))
        return ShardLayout(shard_tokens=s, world=world)

    def _check(self, rank: int):
        if not 0 <= rank < self.world:
            raise ValueError(f"rank {rank} outside world {self.world}")


def exchange(send: torch.Tensor, parts: torch.Tensor, group=None) -> None:
    """All-gather every rank's ``send`` into ``parts[rank]`` (one collective)."""
    import torch.distributed as dist

    if not dist.is_available() or not dist.is_initialized():
        if parts.shape[0] != 1:
            raise RuntimeError("a multi-shard exchange needs an initialised process group")
        parts[0].copy_(send)
        return
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(parts.view(-1), send.reshape(-1), group=group)
    else:  # gloo (CPU tests): list form
        dist.all_gather(list(parts.unbind(0)), send, group=group)


class ShardedDecodeEngine:
    """This rank's part of a KV-sharded batched decode (B requests, each sharded the same way)."""

    def __init__(self, cfg, batch: int, layout: ShardLayout, rank: int, max_seq_len: int, *, device="cuda",
                 group=None, max_chunks: int | None = None, min_chunk: int = 128):
        self.layout = layout
        self.rank = rank
        self.group = group
        lo = layout.offset(rank)
        lim = layout.limit(rank)
        local_cap = (max_seq_len - lo) if lim == 0 else lim
        if local_cap < 1:
            raise ValueError("this shard holds no positions: max_seq_len too small for the layout")
        self.engine = BatchDecodeEngine(cfg, batch, local_cap, device=device, max_chunks=max_chunks,
                                        min_chunk=min_chunk, kv_offset=lo, kv_limit=lim,
                                        n_shards=layout.world)
        self.cfg = cfg

    # -- state --------------------------------------------------------------------------
    def inject(self, layer: int, k_rot: torch.Tensor, v: torch.Tensor, ring_q, ring_acc, ring_lse, n: int):
        """Load positions 1..n of every request (``k_rot``/``v`` [B, Hkv, n, d]) — this rank keeps its
        own slice — and the full (replicated) ring."""
        lo, hi = self.layout.local_range(self.rank, n)
        eng = self.engine
        hi = max(hi, lo - 1)
        eng.inject(layer, k_rot[:, :, lo - 1:hi], v[:, :, lo - 1:hi], ring_q, ring_acc, ring_lse, hi - lo + 1,
                   seq_len=n)

    # -- step ---------------------------------------------------------------------------
    def partial(self, layer: int, q_pre, k_pre, v):
        """Half 1 (no communication): this shard's (piece, band) summaries into ``shard_send``."""
        eng = self.engine
        eng._layer(layer)
        dt = eng._check_inputs(q_pre, k_pre, v)
        eng._ensure_room(layer)
        _lib.call("mac_shard_partial", eng._params(layer, q_pre, k_pre, v, dt), eng._stream())
        return eng.shard_send

    def complete(self, layer: int, q_pre, k_pre, v) -> BatchStepResult:
        """Half 2, after ``shard_parts`` holds every shard's summaries."""
        eng = self.engine
        dt = eng._check_inputs(q_pre, k_pre, v)
        _lib.call("mac_shard_complete", eng._params(layer, q_pre, k_pre, v, dt), eng._stream())
        eng._len[layer] += 1
        return eng.result()

    def decode_step(self, layer: int, q_pre, k_pre, v) -> BatchStepResult:
        """One sharded MAC step: partial -> all-gather -> complete (identical result on every rank)."""
        send = self.partial(layer, q_pre, k_pre, v)
        exchange(send, self.engine.shard_parts, self.group)
        return self.complete(layer, q_pre, k_pre, v)
