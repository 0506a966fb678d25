"""Decode engines: the batched device engine and the reference-shaped shim.

`BatchDecodeEngine` is the B200 serving form of the path: all state (paged
KV cache, per-(request, head) query ring and summary ring, sequence lengths)
lives in HBM as batched tensors, and one `decode_step(layer, ...)` is four
stream-ordered kernel launches through the C-ABI library (append+RoPE,
match, amend, complete) with no host synchronisation.

`DecodeEngine` keeps the reference's single-request API (engine.py:334-539):
`decode_step(layer, q_pre, k_pre, v, m, oracle_rows=None) -> StepResult`
with host numpy in and out, the same exceptions, metrics and ring views.
It runs the very same device kernels (B = 1) and copies results back.

Data layout in HBM (per layer):
  k_cache, v_cache  [num_pages, Hkv, page_size, d]   post-RoPE keys / values (storage dtype)
  ring_q            [B, Hq, W, d]                    pre-RoPE queries, slot (pos-1) % W
  ring_acc          [B, Hq, W, d_v]  f32 (f64)       prefix summary acc over [1, max(0, pos-r)]
  ring_lse          [B, Hq, W]       f32 (f64)       prefix summary lse, -inf = empty
  seq_lens          [B] int32                        tokens stored
and per engine: page_table [B, pages_per_seq] int32 shared by all layers.
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .store import KvPage, TrafficCounter
from .config import (
    DOWNDATE_REMOVE,
    MATCH_POST_ROPE,
    AttentionSummary,
    DecodeMetrics,
    EngineConfig,
    MatchResult,
    StepResult,
    threshold,
)

_TORCH_STORAGE = {"f32": torch.float32, "bf16": torch.bfloat16, "f64": torch.float64}
_MODE = {"f32": _lib.MODE_F32, "bf16": _lib.MODE_BF16, "f64": _lib.MODE_F64}
_IN_DT = {torch.float32: _lib.DT_F32, torch.bfloat16: _lib.DT_BF16, torch.float64: _lib.DT_F64}

SM_COUNT_B200 = 148


def C_void(ptr: int):
    import ctypes

    return ctypes.c_void_p(ptr)


def mass_bound_check(q_m, q_p, keys, values, band: int, *, device="cuda") -> tuple[float, float]:
    """Reference signature of mass_bound_check (engine.py:246-281): post-RoPE queries q_m, q_p (d,),
    keys [p, d] and values [p, d_v] covering [1, p]; returns (lhs, rhs).  Runs the fp64 CUDA kernel
    (mac_mass_bound) over the arrays laid out as one KV page."""
    keys = np.asarray(keys, dtype=np.float64)
    values = np.asarray(values, dtype=np.float64)
    if keys.ndim != 2 or values.ndim != 2 or values.shape[0] != keys.shape[0]:
        raise ValueError("keys and values must be [p, d] and [p, d_v]")
    n, d = keys.shape
    if n < 1:
        raise ValueError("mass_bound_check needs at least one token")
    dv = values.shape[1]
    lib = _lib.load()
    dev = torch.device(device)
    kc = torch.from_numpy(np.ascontiguousarray(keys)).to(dev)
    vc = torch.from_numpy(np.ascontiguousarray(values)).to(dev)
    qs = torch.from_numpy(np.stack([np.asarray(q_m, dtype=np.float64), np.asarray(q_p, dtype=np.float64)])).to(dev)
    zeros = torch.zeros(4, dtype=torch.int32, device=dev)
    item_pm = torch.tensor([n], dtype=torch.int32, device=dev)
    out = torch.zeros(2, dtype=torch.float64, device=dev)
    P = _lib.MacDecodeParams()
    P.batch = P.n_q_heads = P.n_kv_heads = 1
    P.head_dim, P.head_dim_v = d, dv
    P.page_size, P.pages_per_seq = n, 1
    P.storage = _lib.MODE_F64
    P.page_table = zeros.data_ptr()
    P.k_cache, P.v_cache = kc.data_ptr(), vc.data_ptr()
    mb = _lib.MacMassBoundParams()
    mb.n_items, mb.band, mb.rotate = 1, int(band), 0
    mb.item_req = mb.item_kv_head = zeros.data_ptr()
    mb.item_m = mb.item_p = item_pm.data_ptr()
    mb.q_m, mb.q_p, mb.out = qs[0].data_ptr(), qs[1].data_ptr(), out.data_ptr()
    _lib.check(lib.mac_mass_bound(P, mb, torch.cuda.current_stream(dev).cuda_stream), "mac_mass_bound")
    lhs, rhs = out.cpu().tolist()
    return float(lhs), float(rhs)


def rope_freqs(d: int, base: float) -> np.ndarray:
    """omega_j = base**(-2j/d) evaluated exactly as attention.py:208-209 (numpy f64)."""
    j = np.arange(d // 2, dtype=np.float64)
    return base ** (-2.0 * j / d)


def default_max_chunks(batch: int, n_kv_heads: int, max_seq_len: int = 0) -> int:
    """Split-KV slots per (request, kv head), i.e. the items a full-length (miss) span is cut
    into: at least two per resident amend warp (6 per SM) so the dynamic scheduler balances
    the tail, and items of at most ~8K tokens.  Measured on B200 (profiles/r01): C4 (one
    512K request, 8 groups) 470 us at 222-256 slots vs 523 us at 592 and 783 us at 64; C3
    full attention (256 groups, 128K) 2.50 ms at 16-19 slots vs 2.83 ms at 8."""
    groups = batch * n_kv_heads
    return int(min(2048, max(8, math.ceil(SM_COUNT_B200 * 6 * 2 / groups), math.ceil(max_seq_len / 8192))))


def default_slot_cap(max_chunks: int, max_seq_len: int) -> int:
    """Partial slots per (request, kv head) in the workspace (MacDecodeParams.max_chunks), with
    max_chunks the split of a full span (MacDecodeParams.span_chunks): room for a hit step's
    missing groups to cut their context into items of ~512 tokens, up to 64 (C3 geometry, 2 %
    misses: 16K 113 -> 96 us, 128K 476 -> 301 us; full attention keeps its best split — 16K
    339 us at 8 vs 385 at 64; profiles/r02/mc.jsonl)."""
    return int(max(max_chunks, min(64, math.ceil(max_seq_len / 512))))


class _Ptr:
    """A raw device address where _params expects a tensor."""

    def __init__(self, ptr: int):
        self._p = int(ptr)

    def data_ptr(self) -> int:
        return self._p


@dataclass
class BatchStepResult:
    """Device tensors of one batched step (views of engine-owned buffers; valid until the next step)."""

    out: torch.Tensor          # [B, Hq, d_v]
    match_hit: torch.Tensor    # [B, Hq] int32, raw decision
    use_hit: torch.Tensor      # [B, Hq] int32, after gates
    match_pos: torch.Tensor    # [B, Hq] int32, -1 on raw miss
    match_dist: torch.Tensor   # [B, Hq] f64
    match_scanned: torch.Tensor
    full_lse: torch.Tensor
    band_mass: torch.Tensor
    cached_acc: torch.Tensor | None
    cached_lse: torch.Tensor | None
    fallbacks: torch.Tensor


class BatchDecodeEngine:
    """Batched MAC decode state on one GPU; B independent requests, n_layers layers."""

    def __init__(self, cfg: EngineConfig, batch: int, max_seq_len: int, *, device="cuda",
                 max_chunks: int | None = None, min_chunk: int = 128, page_perm_seed: int | None = None,
                 record_cached: bool = False, kv_offset: int = 0, kv_limit: int = 0, n_shards: int = 0,
                 track_stats: bool = False, allocate_kv: bool = True, slot_cap: int | None = None):
        if batch < 1:
            raise ValueError("batch must be >= 1")
        if max_seq_len < 1:
            raise ValueError("max_seq_len must be >= 1")
        _lib.load()
        self.cfg = cfg
        self.batch = batch
        self.device = torch.device(device)
        if self.device.type == "cuda" and self.device.index is None and torch.cuda.is_available():
            self.device = torch.device("cuda", torch.cuda.current_device())
        self.sdt = _TORCH_STORAGE[cfg.storage]
        self.sumdt = torch.float64 if cfg.storage == "f64" else torch.float32
        self.group = cfg.n_q_heads // cfg.n_kv_heads
        self.page_size = cfg.page_size
        # max_chunks: splits of a full span; slot_cap: partial slots per group (>= max_chunks; an
        # explicit max_chunks without slot_cap pins both, as before)
        self.max_chunks = max_chunks or default_max_chunks(batch, cfg.n_kv_heads, max_seq_len)
        if slot_cap is None:
            slot_cap = self.max_chunks if max_chunks else default_slot_cap(self.max_chunks, max_seq_len)
        if slot_cap < self.max_chunks:
            raise ValueError("slot_cap must be >= max_chunks")
        self.slot_cap = int(slot_cap)
        self.min_chunk = min_chunk
        if kv_offset < 0 or kv_limit < 0 or n_shards < 0:
            raise ValueError("kv_offset, kv_limit and n_shards must be >= 0")
        self.kv_offset = kv_offset
        self.kv_limit = kv_limit
        self.n_shards = n_shards
        self.record_cached = record_cached
        self._page_perm_seed = page_perm_seed
        dev = self.device
        self.freqs = torch.from_numpy(rope_freqs(cfg.d, cfg.rope_base)).to(dev)
        self.capacity = 0
        # host mirror of the tokens stored per layer (max over requests): the engine grows the
        # paged pool before a step would need a page it does not have (the reference KvStore
        # grows on demand, kvstore.py:105-119); the appends also refuse such tokens on the device
        # and raise a sticky flag (check_overflow)
        self._len = [0] * cfg.n_layers
        self.k_cache: list[torch.Tensor] = []
        self.v_cache: list[torch.Tensor] = []
        self.page_table = None
        # allocate_kv=False: the KV pool and block table are the caller's (attach_kv); the engine
        # then owns only the rings, the per-layer positions and the workspace
        self.external_kv = not allocate_kv
        if allocate_kv:
            self._alloc_kv(max_seq_len)
        else:  # placeholders until attach_kv (never read: capacity 0 refuses every step)
            self.page_table = torch.zeros(batch, 1, dtype=torch.int32, device=self.device)
            self.k_cache = [torch.zeros(1, cfg.n_kv_heads, self.page_size, cfg.d, dtype=self.sdt, device=self.device)
                            for _ in range(cfg.n_layers)]
            self.v_cache = [torch.zeros(1, cfg.n_kv_heads, self.page_size, cfg.d_v, dtype=self.sdt,
                                        device=self.device) for _ in range(cfg.n_layers)]
        B, Hq, W, d, dv = batch, cfg.n_q_heads, cfg.window, cfg.d, cfg.d_v
        L = cfg.n_layers
        self.ring_q = [torch.zeros(B, Hq, W, d, dtype=self.sdt, device=dev) for _ in range(L)]
        self.ring_acc = [torch.zeros(B, Hq, W, dv, dtype=self.sumdt, device=dev) for _ in range(L)]
        self.ring_lse = [torch.full((B, Hq, W), -math.inf, dtype=self.sumdt, device=dev) for _ in range(L)]
        # bf16 d = 128: dims 0..PLANAR_DIMS-1 of every ring row, contiguous per head, for pass 1
        # of the two-pass scan (kept in step by the ring write-back; call sync_ring_qp after
        # writing ring_q directly)
        self.ring_qp = ([torch.zeros(B, Hq, W, _lib.PLANAR_DIMS, dtype=self.sdt, device=dev) for _ in range(L)]
                         if cfg.storage == "bf16" and cfg.d == 128 else None)
        self.seq_lens = [torch.zeros(B, dtype=torch.int32, device=dev) for _ in range(L)]
        i32 = dict(dtype=torch.int32, device=dev)
        self.o_out = torch.empty(B, Hq, dv, dtype=self.sumdt, device=dev)
        self.o_hit = torch.zeros(B, Hq, **i32)
        self.o_use = torch.zeros(B, Hq, **i32)
        self.o_pos = torch.full((B, Hq), -1, **i32)
        self.o_dist = torch.zeros(B, Hq, dtype=torch.float64, device=dev)
        self.o_scanned = torch.zeros(B, Hq, **i32)
        self.o_full_lse = torch.zeros(B, Hq, dtype=self.sumdt, device=dev)
        self.o_band_mass = torch.zeros(B, Hq, dtype=self.sumdt, device=dev)
        self.o_fallbacks = torch.zeros(B, Hq, **i32)
        # Match-scan choice: every 8th step the kernels store {heads that missed, heads} since
        # the last publication into this pinned buffer through its device alias; the engine
        # reads it WITHOUT a synchronisation (so it may be ~8-16 steps old) and takes the
        # one-pass scan unless misses are rare (< 1% of heads) — the two-pass match is built for
        # the hit path.  Both scans take the argmin of an fp32 sum of squares but
        # associate it differently (one-pass: 8-dim lane chunks + xor tree; two-pass: 16 planar
        # dims + the other 112), so a near-tie below fp32 resolution (|Δd| ~ 1e-6 relative) may
        # resolve differently between them — inside SURVEY §8c's documented near-tie band, never
        # elsewhere.  match_mode="two_pass" / "dense" / "one_pass" pin the scan for bitwise reproducible
        # decisions; "adaptive" (the default) trades that for speed on miss-heavy steps.
        self.match_mode = "adaptive"
        self._fb_host = self._fb_alias = None
        if dev.type == "cuda":
            self._fb_host = torch.zeros(2, dtype=torch.int32).pin_memory()
            self._fb_alias = C.c_void_p()
            _lib.check(_lib.load().mac_host_alias(C.c_void_p(self._fb_host.data_ptr()), C.byref(self._fb_alias)),
                       "mac_host_alias")
        self._step_mode = 0
        self.o_cached_acc = torch.zeros(B, Hq, dv, dtype=self.sumdt, device=dev) if record_cached else None
        self.o_cached_lse = torch.zeros(B, Hq, dtype=self.sumdt, device=dev) if record_cached else None
        # KV-sharded path (n_shards >= 1, sharded.py): this shard's (piece, band) summaries and
        # every shard's, gathered in rank order
        self.shard_send = torch.zeros(B, Hq, 2, dv + 1, dtype=self.sumdt, device=dev) if n_shards else None
        self.shard_parts = (torch.zeros(n_shards, B, Hq, 2, dv + 1, dtype=self.sumdt, device=dev)
                            if n_shards else None)
        # device-side decision statistics per (layer, head) (mac_step_stats)
        self.track_stats = track_stats
        self.head_stats = torch.zeros(L, Hq, len(_lib.STAT_FIELDS), dtype=torch.float64, device=dev)
        self.group_stats = torch.zeros(L, cfg.n_kv_heads, len(_lib.GSTAT_FIELDS), dtype=torch.float64, device=dev)
        probe = self._params(0, self.o_out, self.o_out, self.o_out, _lib.DT_F32)
        # zeroed once: the match kernel keeps its cross-CTA keys/counters zero between steps
        self.workspace = torch.zeros(int(_lib.load().mac_workspace_bytes(probe)), dtype=torch.uint8, device=dev)

    # ------------------------------------------------------------------ memory
    def _alloc_kv(self, tokens: int):
        cfg, B, ps = self.cfg, self.batch, self.page_size
        pps = -(-tokens // ps)
        n_pages = B * pps
        dev = self.device
        if self._page_perm_seed is not None:
            g = torch.Generator().manual_seed(self._page_perm_seed)
            ids = torch.randperm(n_pages, generator=g).to(torch.int32)
        else:
            ids = torch.arange(n_pages, dtype=torch.int32)
        table = ids.view(B, pps).to(dev)
        new_k, new_v = [], []
        for layer in range(cfg.n_layers):
            k = torch.zeros(n_pages, cfg.n_kv_heads, ps, cfg.d, dtype=self.sdt, device=dev)
            v = torch.zeros(n_pages, cfg.n_kv_heads, ps, cfg.d_v, dtype=self.sdt, device=dev)
            if self.page_table is not None:
                old_pps = self.page_table.shape[1]
                src = self.page_table.long()
                dst = table[:, :old_pps].long()
                k[dst.reshape(-1)] = self.k_cache[layer][src.reshape(-1)]
                v[dst.reshape(-1)] = self.v_cache[layer][src.reshape(-1)]
            new_k.append(k)
            new_v.append(v)
        self.k_cache, self.v_cache, self.page_table = new_k, new_v, table
        self.__dict__.pop("_pcache", None)  # cached launch params hold the old pointers
        self.capacity = pps * ps

    def attach_kv(self, k_cache, v_cache, block_table: torch.Tensor, seq_lens: torch.Tensor | None = None):
        """Serve from a caller-owned paged KV pool — the serving-engine contract (vLLM / SGLang
        block tables; the reference reads pages at kvstore.py:121-165).

        k_cache / v_cache: one tensor per layer (a list, or a [n_layers, ...] tensor), each
        [num_blocks, Hkv, page_size, d] (HND) in the storage dtype, post-RoPE keys as the append
        writes them.  block_table: [B, max_blocks] int32 on the device; row b lists batch slot
        b's blocks in token order (token t in block (t-1) // page_size).  Rows may share blocks
        (a common prompt prefix) and may be permuted or edited in place between steps — the
        kernels read the table every step; a decode step appends into the block holding its
        position, so that block must belong to the request alone.  seq_lens: [B] tokens already
        in the pool (default 0), applied to every layer.

        The engine keeps its rings and per-layer positions; it never allocates or grows KV again
        (reserve() raises once a request would pass max_blocks * page_size)."""
        cfg, L = self.cfg, self.cfg.n_layers
        ks = list(k_cache.unbind(0)) if isinstance(k_cache, torch.Tensor) else list(k_cache)
        vs = list(v_cache.unbind(0)) if isinstance(v_cache, torch.Tensor) else list(v_cache)
        if len(ks) != L or len(vs) != L:
            raise ValueError(f"expected {L} per-layer K and V caches, got {len(ks)} and {len(vs)}")
        nb = ks[0].shape[0]
        for t, dv in [(k, cfg.d) for k in ks] + [(v, cfg.d_v) for v in vs]:
            if (t.dim() != 4 or tuple(t.shape[1:]) != (cfg.n_kv_heads, self.page_size, dv) or t.shape[0] != nb
                    or t.dtype != self.sdt or t.device != self.device or not t.is_contiguous()):
                raise ValueError(f"KV cache must be contiguous [num_blocks, {cfg.n_kv_heads}, {self.page_size}, "
                                 f"d] {self.sdt} on {self.device}; got {tuple(t.shape)} {t.dtype} {t.device}")
        bt = block_table
        if (bt.dim() != 2 or bt.shape[0] != self.batch or bt.dtype != torch.int32 or bt.device != self.device
                or not bt.is_contiguous()):
            raise ValueError(f"block_table must be a contiguous [{self.batch}, max_blocks] int32 tensor on "
                             f"{self.device}")
        self.k_cache, self.v_cache, self.page_table = ks, vs, bt
        self.external_kv = True
        self.capacity = bt.shape[1] * self.page_size
        self.__dict__.pop("_pcache", None)
        if seq_lens is not None:
            for layer in range(L):
                self.seq_lens[layer].copy_(seq_lens.to(self.device, torch.int32))
                self._len[layer] = int(seq_lens.max().item())

    def reserve(self, tokens: int):
        """Grow the paged KV pool so every request can hold `tokens` tokens (doubling)."""
        if tokens > self.capacity and self.external_kv:
            raise ValueError(f"position {tokens} exceeds the caller-owned block table ({self.capacity} tokens per "
                             f"request): extend block_table and attach_kv again")
        if tokens > self.capacity:
            self._alloc_kv(max(tokens, 2 * self.capacity))

    def _local_tokens(self, layer: int, n_new: int) -> int:
        """Shard-local tokens this layer holds after n_new more appends."""
        need = self._len[layer] + n_new - self.kv_offset
        return min(need, self.kv_limit) if self.kv_limit > 0 else need

    def _ensure_room(self, layer: int, n_new: int = 1, *, grow: bool = True):
        need = self._local_tokens(layer, n_new)
        if need > self.capacity:
            if not grow:
                raise ValueError(f"layer {layer}: position {self._len[layer] + n_new} exceeds the KV capacity "
                                 f"{self.capacity}; reserve() before capturing a StepGraph")
            self.reserve(need)

    def check_overflow(self) -> bool:
        """True when any append since construction found no page for its token (synchronises)."""
        off = int(_lib.load().mac_overflow_flag_offset(self._params(0, self.o_out, self.o_out, self.o_out,
                                                                    _lib.DT_F32)))
        return int(self.workspace[off:off + 4].view(torch.int32).item()) != 0

    # ------------------------------------------------------------------ launch
    def _params(self, layer: int, q, k, v, in_dt: int, force_miss: bool = False) -> _lib.MacDecodeParams:
        key = (layer, q.data_ptr(), k.data_ptr(), v.data_ptr(), in_dt, force_miss)
        cache = self.__dict__.setdefault("_pcache", {})
        P = cache.get(key)
        if P is None:
            P = self._build_params(layer, q, k, v, in_dt, force_miss)
            if hasattr(self, "workspace"):
                if len(cache) > 256:
                    cache.clear()
                cache[key] = P
        # per-call fields: the step's scan choice, no output narrowing and device-resident inputs
        # unless the caller sets them
        P.match_mode = self._step_mode
        P.out_bf16 = None
        P.inputs_host = 0
        return P

    def _build_params(self, layer: int, q, k, v, in_dt: int, force_miss: bool) -> _lib.MacDecodeParams:
        cfg = self.cfg
        P = _lib.MacDecodeParams()
        P.batch = self.batch
        P.n_q_heads, P.n_kv_heads = cfg.n_q_heads, cfg.n_kv_heads
        P.head_dim, P.head_dim_v = cfg.d, cfg.d_v
        P.window, P.band = cfg.window, cfg.band
        P.page_size = self.page_size
        P.pages_per_seq = self.page_table.shape[1]
        P.storage = _MODE[cfg.storage]
        P.in_dtype = in_dt
        P.max_chunks, P.span_chunks, P.min_chunk = self.slot_cap, self.max_chunks, self.min_chunk
        P.kv_offset = self.kv_offset
        P.kv_limit = self.kv_limit
        P.n_shards = self.n_shards
        if self.shard_send is not None:
            P.shard_out = self.shard_send.data_ptr()
            P.shard_parts = self.shard_parts.data_ptr()
        P.thr_sq = threshold(cfg.d, cfg.tau_for(layer)) ** 2
        P.delta_max = cfg.delta_max or 0
        P.match_space = _lib.MATCH_POST_ROPE if cfg.match_space == MATCH_POST_ROPE else _lib.MATCH_PRE_ROPE
        P.refresh_every = cfg.refresh_every
        costs = cfg.byte_costs()
        P.roi_gate = int(cfg.roi_gate)
        P.roi_b_kv, P.roi_b_q = float(costs.b_kv), float(costs.b_q)
        P.downdate = _lib.DOWNDATE_REMOVE if cfg.downdate_mode == DOWNDATE_REMOVE else _lib.DOWNDATE_SPLIT
        P.force_miss = int(force_miss)
        P.eps_cancel = 1e-6
        P.seq_lens = self.seq_lens[layer].data_ptr()
        P.page_table = self.page_table.data_ptr()
        P.k_cache, P.v_cache = self.k_cache[layer].data_ptr(), self.v_cache[layer].data_ptr()
        P.ring_q = self.ring_q[layer].data_ptr()
        P.ring_acc = self.ring_acc[layer].data_ptr()
        P.ring_lse = self.ring_lse[layer].data_ptr()
        P.ring_qp = self.ring_qp[layer].data_ptr() if self.ring_qp is not None else None
        P.rope_freqs = self.freqs.data_ptr()
        P.q_pre, P.k_pre, P.v_in = q.data_ptr(), k.data_ptr(), v.data_ptr()
        P.out = self.o_out.data_ptr()
        P.match_hit, P.use_hit = self.o_hit.data_ptr(), self.o_use.data_ptr()
        P.match_pos, P.match_dist = self.o_pos.data_ptr(), self.o_dist.data_ptr()
        P.match_scanned = self.o_scanned.data_ptr()
        P.full_lse, P.band_mass = self.o_full_lse.data_ptr(), self.o_band_mass.data_ptr()
        P.cached_acc = self.o_cached_acc.data_ptr() if self.o_cached_acc is not None else None
        P.cached_lse = self.o_cached_lse.data_ptr() if self.o_cached_lse is not None else None
        P.fallbacks = self.o_fallbacks.data_ptr()
        P.match_mode = self._step_mode
        P.feedback = self._fb_alias.value if self._fb_alias is not None else None
        if hasattr(self, "workspace"):
            P.workspace = self.workspace.data_ptr()
            P.workspace_bytes = self.workspace.numel()
        else:
            P.workspace = 1
            P.workspace_bytes = 0
        return P

    def _check_inputs(self, q, k, v):
        cfg, B = self.cfg, self.batch
        if tuple(q.shape) != (B, cfg.n_q_heads, cfg.d):
            raise ValueError(f"expected queries {(B, cfg.n_q_heads, cfg.d)}, got {tuple(q.shape)}")
        if tuple(k.shape) != (B, cfg.n_kv_heads, cfg.d) or tuple(v.shape) != (B, cfg.n_kv_heads, cfg.d_v):
            raise ValueError("key/value shapes do not match the configured kv heads")
        if not (q.dtype == k.dtype == v.dtype) or q.dtype not in _IN_DT:
            raise ValueError("q_pre, k_pre and v must share one dtype among float32/bfloat16/float64")
        for t in (q, k, v):
            if t.device != self.device and not (t.is_cuda and self.device.type == "cuda"):
                raise ValueError("inputs must live on the engine's device")
            if not t.is_contiguous():
                raise ValueError("inputs must be contiguous")
        return _IN_DT[q.dtype]

    def _layer(self, layer: int):
        if not 0 <= layer < self.cfg.n_layers:
            raise ValueError(f"layer {layer} out of range")

    def _stream(self) -> int:
        return torch.cuda.current_stream(self.device).cuda_stream

    def decode_step(self, layer: int, q_pre: torch.Tensor, k_pre: torch.Tensor, v: torch.Tensor, *,
                    force_miss: bool = False) -> BatchStepResult:
        """One MAC step for every request: append -> match -> amend -> complete (engine.py:410-539).
        force_miss: every head takes the miss path (exact attention), as the reference's
        refresh gate does (engine.py:456-459)."""
        self._layer(layer)
        dt = self._check_inputs(q_pre, k_pre, v)
        self._ensure_room(layer)
        self._choose_match_mode()
        P = self._params(layer, q_pre, k_pre, v, dt, force_miss)
        self.last_params = P  # what the library was given (tests: mac_match_path(last_params))
        _lib.call("mac_decode_step", P, self._stream())
        self._len[layer] += 1
        if self.track_stats and not getattr(self, "_in_prefill", False):
            self._accumulate_stats(layer, P)
        return self.result()

    def _decode_step_ptrs(self, layer: int, q_ptr: int, k_ptr: int, v_ptr: int, in_dt: int, out_bf16: int = 0,
                          inputs_host: bool = False):
        """decode_step on raw device pointers, optionally also writing the output narrowed to
        bf16 at `out_bf16` (a pinned host buffer's device alias: StepGraph's zero-copy output);
        inputs_host: q/k/v are device aliases of pinned host memory (MacDecodeParams.inputs_host)."""
        P = self._params(layer, _Ptr(q_ptr), _Ptr(k_ptr), _Ptr(v_ptr), in_dt, False)
        P.out_bf16 = out_bf16 or None
        P.inputs_host = 1 if inputs_host else 0
        self.last_params = P
        _lib.call("mac_decode_step", P, self._stream())
        if self.track_stats and not getattr(self, "_in_prefill", False):
            self._accumulate_stats(layer, P)

    # ------------------------------------------------------------------ diagnostics
    def _accumulate_stats(self, layer: int, P):
        code = _lib.load().mac_step_stats(P, C_void(self.head_stats[layer].data_ptr()),
                                          C_void(self.group_stats[layer].data_ptr()), self._stream())
        _lib.check(code, "mac_step_stats")

    def reset_stats(self):
        self.head_stats.zero_()
        self.group_stats.zero_()

    def stats(self, layer: int | None = None, *, per_head: bool = False) -> dict:
        """Decision statistics accumulated on the device since the last reset (track_stats=True),
        in the reference's report schema (compute_metrics, engine.py:226-243) plus the raw
        DecodeMetrics counters; `layer=None` sums every layer.  per_head adds per-head arrays of
        acceptance, skip ratio, kv fraction and mean band mass (one host copy, on request)."""
        hs = (self.head_stats.sum(0) if layer is None else self.head_stats[layer]).cpu().numpy()
        gs = (self.group_stats.sum(0) if layer is None else self.group_stats[layer]).cpu().numpy()
        f = {name: hs[:, i] for i, name in enumerate(_lib.STAT_FIELDS)}
        tot = {name: float(v.sum()) for name, v in f.items()}
        steps = tot["steps"]
        rep = {
            "schema_version": 1,
            "steps": int(steps),
            "hits": int(tot["hits"]),
            "acceptance_rate": tot["hits"] / steps if steps else None,
            "skip_ratio": tot["skip_sum"] / steps if steps else None,
            "kv_fraction": tot["kv_tokens_read"] / tot["kv_tokens_full"] if tot["kv_tokens_full"] else None,
            "err_mean": None, "err_p50": None, "err_p99": None,
            "mean_gap": tot["gap_sum"] / tot["hits"] if tot["hits"] else None,
            "mean_band_mass": tot["band_mass_sum"] / steps if steps else None,
            "forced_misses": int(tot["forced_misses"]),
            "fallbacks": int(tot["fallbacks"]),
            "kv_tokens_read": int(tot["kv_tokens_read"]),
            "kv_tokens_full": int(tot["kv_tokens_full"]),
            "match_candidates": int(tot["match_candidates"]),
            "group_kv_tokens": int(gs[:, 0].sum()),
            "group_kv_total": int(gs[:, 1].sum()),
        }
        if per_head:
            with np.errstate(invalid="ignore", divide="ignore"):
                rep["per_head"] = {
                    "steps": f["steps"].astype(np.int64),
                    "acceptance_rate": f["hits"] / f["steps"],
                    "skip_ratio": f["skip_sum"] / f["steps"],
                    "kv_fraction": f["kv_tokens_read"] / f["kv_tokens_full"],
                    "mean_band_mass": f["band_mass_sum"] / f["steps"],
                    "mean_gap": f["gap_sum"] / f["hits"],
                }
                rep["per_group_kv_fraction"] = gs[:, 0] / gs[:, 1]
        return rep

    def mass_bound(self, layer: int, req, kv_head, m, p, q_m: torch.Tensor, q_p: torch.Tensor) -> torch.Tensor:
        """mass_bound_check (engine.py:246-281) for n hits over this layer's paged cache: keys and
        values [1, p] of (req, kv_head), pre-RoPE queries q_m (rotated at m) and q_p (the ring query
        stored at p, rotated at p), [n, d] float64.  Returns [n, 2] float64 (lhs, rhs) on the device."""
        self._layer(layer)
        cfg, dev = self.cfg, self.device
        i32 = lambda x: torch.as_tensor(x, dtype=torch.int32).reshape(-1).to(dev)
        req, kvh, mm, pp = i32(req), i32(kv_head), i32(m), i32(p)
        n = req.numel()
        if not (kvh.numel() == mm.numel() == pp.numel() == n):
            raise ValueError("req, kv_head, m and p must have the same length")
        if n and int(pp.min().item()) < 1:
            raise ValueError("mass_bound_check needs at least one token")
        qm = q_m.to(device=dev, dtype=torch.float64).reshape(n, cfg.d).contiguous()
        qp = q_p.to(device=dev, dtype=torch.float64).reshape(n, cfg.d).contiguous()
        out = torch.zeros(n, 2, dtype=torch.float64, device=dev)
        P = self._params(layer, self.o_out, self.o_out, self.o_out, _lib.DT_F32)
        mb = _lib.MacMassBoundParams()
        mb.n_items, mb.band, mb.rotate = n, cfg.band, 1
        mb.item_req, mb.item_kv_head, mb.item_m, mb.item_p = (req.data_ptr(), kvh.data_ptr(), mm.data_ptr(),
                                                              pp.data_ptr())
        mb.q_m, mb.q_p, mb.out = qm.data_ptr(), qp.data_ptr(), out.data_ptr()
        _lib.check(_lib.load().mac_mass_bound(P, mb, self._stream()), "mac_mass_bound")
        return out

    def prefill(self, layer: int, q_pre: torch.Tensor, k_pre: torch.Tensor, v: torch.Tensor,
                *, ring_build: str = "auto") -> BatchStepResult | None:
        """Append a prompt of n tokens to every request ([B, n, H, d] tensors, token-major) and
        leave exactly the state of n forced-miss decode steps: KV of
        positions 1..n and ring slots holding (q_t, AS[1, t-r] under q_t) for the last min(n, W)
        positions.  Returns the last token's step result (its output is exact attention over
        [1, n]).

        GEMM form (ring_build="auto" on the bf16 d = 128 path, or "gemm"): tokens 1..n-1 in one
        bulk append (mac_prefill_kv), the ring entries of positions n-c..n-1 (c = min(W, n) - 1)
        in one tensor-core pass over the cache (mac_build_ring: every key tile read once per
        block of query rows), then token n as one forced-miss decode step.  ring_build="steps"
        (and every other storage / shape) runs the last min(n, W) tokens as forced-miss decode
        steps instead."""
        self._layer(layer)
        cfg, B = self.cfg, self.batch
        if q_pre.dim() != 4 or q_pre.shape[0] != B or q_pre.shape[2:] != (cfg.n_q_heads, cfg.d):
            raise ValueError(f"expected queries [B={B}, n, {cfg.n_q_heads}, {cfg.d}], got {tuple(q_pre.shape)}")
        n = q_pre.shape[1]
        if tuple(k_pre.shape) != (B, n, cfg.n_kv_heads, cfg.d) or tuple(v.shape) != (B, n, cfg.n_kv_heads, cfg.d_v):
            raise ValueError("key/value shapes do not match [B, n, Hkv, d]")
        if ring_build not in ("auto", "gemm", "steps"):
            raise ValueError(f"ring_build must be 'auto', 'gemm' or 'steps', got {ring_build!r}")
        if n == 0:
            return None
        stored = int(self.seq_lens[layer].max().item()) if self.capacity else 0
        self._len[layer] = max(self._len[layer], stored)
        self._ensure_room(layer, n + 1)
        gemm = ring_build != "steps" and self.ring_build_supported()
        if ring_build == "gemm" and not gemm:
            raise ValueError("the GEMM-form ring build needs bf16 storage, d = d_v = 128, 8 % (Hq/Hkv) == 0, "
                             "page_size % 16 == 0 and an unsharded cache")
        n_steps = 1 if gemm else min(n, cfg.window)
        n_bulk = n - n_steps
        if n_bulk:
            kb, vb = k_pre[:, :n_bulk].contiguous(), v[:, :n_bulk].contiguous()
            dt = _IN_DT[kb.dtype]
            q0 = q_pre[:, 0].contiguous()
            P = self._build_params(layer, q0, kb, vb, dt, False)
            code = _lib.load().mac_prefill_kv(P, n_bulk, self._stream())
            _lib.check(code, "mac_prefill_kv")
            self._len[layer] += n_bulk
        if gemm:
            rows = min(cfg.window, n) - 1
            if rows > 0:
                self.build_ring(layer, q_pre[:, n_bulk - rows:n_bulk])
        res = None
        self._in_prefill = True  # prompt tokens are not decode decisions: no statistics
        try:
            for t in range(n_bulk, n):
                res = self.decode_step(layer, q_pre[:, t].contiguous(), k_pre[:, t].contiguous(),
                                       v[:, t].contiguous(), force_miss=True)
        finally:
            self._in_prefill = False
        return res

    def ring_build_supported(self) -> bool:
        cfg = self.cfg
        g = cfg.n_q_heads // cfg.n_kv_heads
        return (cfg.storage == "bf16" and cfg.d == 128 and cfg.d_v == 128 and 8 % g == 0
                and self.page_size % 16 == 0 and self.kv_offset == 0 and self.kv_limit == 0)

    def build_ring(self, layer: int, q_rows: torch.Tensor, n_chunks: int | None = None, variant: str = "auto"):
        """Ring entries of the last q_rows.shape[1] stored positions of every request from the KV
        already in the cache (mac_build_ring): slot (t-1) % W <- (q_t, AS[1, t-r] under R_t q_t).
        q_rows: [B, n_rows, Hq, d] pre-RoPE queries of positions seq_len-n_rows+1 .. seq_len (a
        caller-owned pool filled by the serving system's own prefill works the same way).
        n_chunks splits each row block's keys for parallelism (default: enough CTAs for ~4
        waves on 148 SMs).  variant: "auto" (the tcgen05 kernel where it applies), "mma"
        (mma.sync, 8-row warps) or "tcgen05" (UMMA, 128-row CTAs)."""
        cfg, B = self.cfg, self.batch
        if not self.ring_build_supported():
            raise ValueError("mac_build_ring needs the bf16 d = 128 path (see prefill)")
        if q_rows.dim() != 4 or q_rows.shape[0] != B or q_rows.shape[2:] != (cfg.n_q_heads, cfg.d):
            raise ValueError(f"expected queries [B={B}, n_rows, {cfg.n_q_heads}, {cfg.d}]")
        n_rows = q_rows.shape[1]
        if n_rows > cfg.window:
            raise ValueError(f"{n_rows} rows exceed the ring window {cfg.window}")
        if n_rows == 0:
            return
        q_rows = q_rows.contiguous()
        g = cfg.n_q_heads // cfg.n_kv_heads
        vid = {"auto": 0, "mma": 1, "tcgen05": 2}[variant]
        rows_per_cta = 8 * (8 // g) if vid == 1 else 256 // g
        blocks = B * cfg.n_kv_heads * -(-n_rows // rows_per_cta)
        if n_chunks is None:
            longest = int(self.seq_lens[layer].max().item())
            n_chunks = max(1, min(-(-4 * SM_COUNT_B200 // blocks), -(-longest // 2048)))
        part = None
        if n_chunks > 1:
            part = torch.empty(B * n_rows * cfg.n_q_heads * n_chunks * (cfg.d_v + 1), dtype=torch.float32,
                               device=self.device)
        P = self._build_params(layer, q_rows, q_rows, q_rows, _IN_DT[q_rows.dtype], False)
        rb = _lib.MacRingBuildParams(n_rows=n_rows, n_chunks=n_chunks, part=part.data_ptr() if part is not None else None,
                                     variant=vid)
        # (part is freed back to the caching allocator on this stream: stream order keeps it live
        # until the merge kernel has read it)
        _lib.check(_lib.load().mac_build_ring(C.byref(P), C.byref(rb), C.c_void_p(self._stream())), "mac_build_ring")

    def match_path(self, P=None) -> int:
        """mac_match_path of a parameter set (default: the last step's): which scan, verify layout
        and amend the library launches for it (MAC_PATH_* bits, split-band items << 8)."""
        P = P if P is not None else self.last_params
        return int(_lib.load().mac_match_path(P))

    # miss fraction above which the adaptive engine takes the one-pass scan even where the dense
    # kernel is available (C3 geometry at 16K, final build: 10 % misses 180 us dense vs 201
    # one-pass, 20 % 263 vs 269, 30 % 330 vs 317, 40 % 349 vs 331; profiles/r02/SUMMARY.md)
    DENSE_MAX_MISS = 0.2

    def _choose_match_mode(self):
        """The step's match scan (MacDecodeParams.match_mode), fixed for all of its stages:
        0 two-pass (the hit path), 2 two-pass with the dense walks of heads without a near-repeat
        spread over the GPU (dense_kernel), 1 one-pass scan."""
        if self.match_mode == "one_pass":
            self._step_mode = 1
        elif self.match_mode == "two_pass" or self._fb_host is None:
            self._step_mode = 0
        elif self.match_mode == "dense":
            self._step_mode = 2
        else:
            # Plain two-pass only while (almost) nothing misses: a head without a near-repeat makes
            # its verify warp walk the whole ring and the verify ends with its last head — C3
            # geometry at 16K (profiles/r02/miss_sweep_final): 0 % 48.9 us two-pass vs 63.5 dense;
            # 1 % already 344 vs 82 (one-pass 131); 10 % 440 / 194 / 215.  So any recurring miss
            # (two or more heads in the feedback window of 8 steps) leaves mode 0: the per-group
            # verify geometry hands the walks to dense_kernel (mode 2); other geometries, and
            # miss-dominated steps, take the one-pass scan.
            missed, heads = (int(x) for x in self._fb_host.tolist())
            f = missed / heads if heads > 0 else 0.0
            if missed < 2:
                self._step_mode = 0
            elif f <= self.DENSE_MAX_MISS and self._dense_capable():
                self._step_mode = 2
            else:
                self._step_mode = 1

    def _dense_capable(self) -> bool:
        cap = self.__dict__.get("_dense_cap")
        if cap is None:
            P = self._params(0, self.o_out, self.o_out, self.o_out, _lib.DT_BF16)
            saved = P.match_mode
            P.match_mode = 2
            path = int(_lib.load().mac_match_path(P))
            P.match_mode = saved
            cap = self._dense_cap = path > 0 and bool(path & _lib.PATH_DENSE_KERNEL)
        return cap

    def stage(self, name: str, layer: int, q_pre, k_pre, v, force_miss: bool = False):
        """Launch one stage (mac_append_kv | mac_match | mac_amend | mac_complete) — for profiling/tests."""
        self._layer(layer)
        if name == "mac_append_kv":  # a step's first stage: its match scan is chosen here
            self._ensure_room(layer)
            self._choose_match_mode()
        dt = self._check_inputs(q_pre, k_pre, v)
        _lib.call(name, self._params(layer, q_pre, k_pre, v, dt, force_miss), self._stream())
        if name == "mac_complete":  # the step's last stage advances seq_lens
            self._len[layer] += 1

    def full_decode(self, layer: int, q_pre, k_pre, v) -> torch.Tensor:
        """Full-attention decode (append + exact attention over [1, m]): the baseline; no ring work."""
        self._layer(layer)
        dt = self._check_inputs(q_pre, k_pre, v)
        self._ensure_room(layer)
        _lib.call("mac_full_decode", self._params(layer, q_pre, k_pre, v, dt, True), self._stream())
        self._len[layer] += 1
        return self.o_out

    def attend_full(self, layer: int, q_pre) -> torch.Tensor:
        """Exact attention of R_m q over the stored [1, m] (m = seq_lens), without appending."""
        self._layer(layer)
        cfg = self.cfg
        dt = _IN_DT[q_pre.dtype]
        kv_dummy_k = torch.empty(self.batch, cfg.n_kv_heads, cfg.d, dtype=q_pre.dtype, device=self.device)
        kv_dummy_v = torch.empty(self.batch, cfg.n_kv_heads, cfg.d_v, dtype=q_pre.dtype, device=self.device)
        _lib.call("mac_attend_full", self._params(layer, q_pre, kv_dummy_k, kv_dummy_v, dt, True), self._stream())
        return self.o_out

    def result(self) -> BatchStepResult:
        return BatchStepResult(self.o_out, self.o_hit, self.o_use, self.o_pos, self.o_dist, self.o_scanned,
                               self.o_full_lse, self.o_band_mass, self.o_cached_acc, self.o_cached_lse,
                               self.o_fallbacks)

    # ------------------------------------------------------------------ state injection
    def inject(self, layer: int, k_rot: torch.Tensor, v: torch.Tensor, ring_q: torch.Tensor, ring_acc: torch.Tensor,
               ring_lse: torch.Tensor, n: int, *, seq_len: int | None = None):
        """Load a prefix state for every request: local K/V rows 1..n (post-RoPE, [B, Hkv, n, d]) and
        the ring entries of positions L-cnt+1..L ([B, Hq, cnt, ...], cnt <= W, oldest first), where
        L = seq_len (default n; a KV shard passes the request's global length)."""
        cfg, B, ps = self.cfg, self.batch, self.page_size
        L = n if seq_len is None else seq_len
        self.reserve(n + 1)
        pages = -(-n // ps)
        for b in range(B):
            ids = self.page_table[b, :pages].long()
            kk = torch.zeros(pages * ps, cfg.n_kv_heads, cfg.d, dtype=self.sdt, device=self.device)
            vv = torch.zeros(pages * ps, cfg.n_kv_heads, cfg.d_v, dtype=self.sdt, device=self.device)
            kk[:n] = k_rot[b].transpose(0, 1).to(self.device, self.sdt)
            vv[:n] = v[b].transpose(0, 1).to(self.device, self.sdt)
            self.k_cache[layer][ids] = kk.view(pages, ps, cfg.n_kv_heads, cfg.d).transpose(1, 2)
            self.v_cache[layer][ids] = vv.view(pages, ps, cfg.n_kv_heads, cfg.d_v).transpose(1, 2)
        cnt = ring_q.shape[2]
        W = cfg.window
        pos = torch.arange(L - cnt + 1, L + 1, device=self.device)
        slots = (pos - 1) % W
        self.ring_q[layer][:, :, slots] = ring_q.to(self.device, self.sdt)
        self.ring_acc[layer][:, :, slots] = ring_acc.to(self.device, self.sumdt)
        self.ring_lse[layer][:, :, slots] = ring_lse.to(self.device, self.sumdt)
        self.seq_lens[layer].fill_(L)
        self._len[layer] = L
        self.sync_ring_qp(layer)

    def sync_ring_qp(self, layer: int):
        """Refresh the planar copy of the query ring's first PLANAR_DIMS dims after ring_q was
        written from outside the kernels (state injection)."""
        if self.ring_qp is not None:
            self.ring_qp[layer].copy_(self.ring_q[layer][..., :_lib.PLANAR_DIMS])


class StepGraph:
    """One decode step of a BatchDecodeEngine as a replayable CUDA graph, with the step's host
    I/O inside it: pinned host inputs -> device, the step's kernels, output -> pinned host.
    The serving loop writes a step's q/k/v into `q_host`/`k_host`/`v_host`, calls `replay()`,
    and reads `out_host` after the stream syncs.  Replays are stream-ordered and advance the
    engine like `decode_step` (every kernel reads its position from `seq_lens`, every
    workspace counter returns to zero by the end of the step), so one graph serves every step.

    `layer` is one layer index, or a sequence of layers captured back to back in one graph
    (one token of a trace replay across the model: one H2D copy of every
    layer's q/k/v, one launch of the graph, one D2H copy of every layer's output); the host
    buffers then carry a leading layer dimension in the order given.

    The host legs never use the copy engines: the inputs are pulled over the host link by a
    zero-copy kernel on the pinned buffer's device alias (`mac_io_copy`, csrc/io.cu; 18 vs
    30 us for the two legs at C3 in tools/zerocopy_probe.cu), and on the bf16 d = 128 path
    with a bf16 output (the serving configuration) the complete kernel writes the narrowed
    output straight into the pinned output buffer (`out_bf16`); otherwise a second zero-copy
    kernel pushes it.  (Letting the front kernel read q/k/v from the host alias directly,
    with no pull launch, measured slower: every scan CTA then waits on a host-link read.)"""

    def __init__(self, eng: "BatchDecodeEngine", layer, dtype=torch.bfloat16, out_dtype=None,
                 host_inputs: bool = True):
        """dtype: the q/k/v input dtype; out_dtype: the host output dtype (default the engine's
        summary dtype, f32 for bf16 storage; bf16 halves the device-to-host bytes);
        host_inputs: on the bf16 two-pass path let the step read q/k/v from the pinned buffer
        (inputs_host) instead of pulling them first."""
        cfg, B = eng.cfg, eng.batch
        self.multi = not isinstance(layer, int)
        self.layers = [int(x) for x in layer] if self.multi else [int(layer)]
        if not self.layers or len(set(self.layers)) != len(self.layers):
            raise ValueError("layers must be a non-empty sequence of distinct layer indices")
        for lay in self.layers:
            eng._layer(lay)
        self.eng, self.layer = eng, (self.layers if self.multi else self.layers[0])
        self.host_inputs = host_inputs
        n_l = len(self.layers)
        dev = eng.device
        # q, k and v of every layer share one pinned staging buffer and one device buffer:
        # one H2D copy per step
        nq, nk, nv = B * cfg.n_q_heads * cfg.d, B * cfg.n_kv_heads * cfg.d, B * cfg.n_kv_heads * cfg.d_v
        per = nq + nk + nv
        self.in_host = torch.zeros(n_l * per, dtype=dtype).pin_memory()
        self.in_dev = torch.zeros(n_l * per, dtype=dtype, device=dev)

        def split(t):
            v = t.view(n_l, per)
            q = v[:, :nq].view(n_l, B, cfg.n_q_heads, cfg.d)
            k = v[:, nq:nq + nk].view(n_l, B, cfg.n_kv_heads, cfg.d)
            vv = v[:, nq + nk:].view(n_l, B, cfg.n_kv_heads, cfg.d_v)
            return (q, k, vv) if self.multi else (q[0], k[0], vv[0])

        self.q_host, self.k_host, self.v_host = split(self.in_host)
        self._qkv_dev = [(self.in_dev[i * per:i * per + nq].view(B, cfg.n_q_heads, cfg.d),
                          self.in_dev[i * per + nq:i * per + nq + nk].view(B, cfg.n_kv_heads, cfg.d),
                          self.in_dev[i * per + nq + nk:(i + 1) * per].view(B, cfg.n_kv_heads, cfg.d_v))
                         for i in range(n_l)]
        self.q_dev, self.k_dev, self.v_dev = self._qkv_dev[0]
        self.out_dtype = out_dtype or eng.sumdt
        if self.out_dtype != eng.sumdt and not (eng.sumdt == torch.float32 and self.out_dtype == torch.bfloat16):
            raise ValueError(f"StepGraph output {self.out_dtype} from {eng.sumdt} summaries: same dtype or f32 -> bf16")
        oshape = (n_l, B, cfg.n_q_heads, cfg.d_v) if self.multi else (B, cfg.n_q_heads, cfg.d_v)
        self.out_host = torch.zeros(oshape, dtype=self.out_dtype).pin_memory()
        # device aliases of the pinned buffers (UVA): the I/O kernels load / store them directly
        lib = _lib.load()
        self._in_alias, self._out_alias = C.c_void_p(), C.c_void_p()
        _lib.check(lib.mac_host_alias(C.c_void_p(self.in_host.data_ptr()), C.byref(self._in_alias)), "mac_host_alias")
        _lib.check(lib.mac_host_alias(C.c_void_p(self.out_host.data_ptr()), C.byref(self._out_alias)),
                   "mac_host_alias")
        # bf16 d = 128 engine with a bf16 output: no I/O kernels at all (see _body)
        self.direct = (cfg.storage == "bf16" and cfg.d == 128 and cfg.d_v == 128 and
                       self.out_dtype == torch.bfloat16)
        self.h2d_bytes = self.in_host.numel() * self.in_host.element_size()
        self.d2h_bytes = self.out_host.numel() * self.out_host.element_size()
        # A graph pins the kernels it captured, so the match scan (MacDecodeParams.match_mode) is
        # fixed per graph: an adaptive engine whose geometry runs the two-pass scan gets one graph
        # per scan and replay() picks one from the engine's misses feedback, like decode_step.
        modes = [eng._step_mode]
        if eng.match_mode == "adaptive":
            P = eng._params(self.layers[0], eng.o_out, eng.o_out, eng.o_out, _lib.DT_BF16)
            P.match_mode = 0
            two = _lib.load().mac_match_path(P)
            modes = [0, 1] if two > 0 and two & _lib.PATH_TWO_PASS else [0]
            if 1 in modes and eng._dense_capable():
                modes.append(2)
        elif eng.match_mode == "one_pass":
            modes = [1]
        elif eng.match_mode == "dense":
            modes = [2]
        else:
            modes = [0]
        self.graphs = {}
        saved = eng._step_mode
        s = torch.cuda.Stream(device=dev)
        s.wait_stream(torch.cuda.current_stream(dev))
        try:
            for mode in modes:
                eng._step_mode = mode
                g = torch.cuda.CUDAGraph()
                # thread-local capture: the launchers' one-time setup (function attributes, occupancy
                # queries) is not a stream operation and may run during the first capture
                with torch.cuda.graph(g, stream=s, capture_error_mode="thread_local"):
                    self._body()
                self.graphs[mode] = g
        finally:
            eng._step_mode = saved
        self.graph = self.graphs[modes[0]]

    def _io(self, src: int, src_dt: int, dst: int, dst_dt: int, n: int):
        lib = _lib.load()
        _lib.check(lib.mac_io_copy(C.c_void_p(src), src_dt, C.c_void_p(dst), dst_dt, n,
                                   C.c_void_p(torch.cuda.current_stream(self.eng.device).cuda_stream)), "mac_io_copy")

    def _body(self):
        eng = self.eng
        dt = {torch.float32: _lib.DT_F32, torch.bfloat16: _lib.DT_BF16, torch.float64: _lib.DT_F64}
        per_out = eng.o_out.numel()
        osz = self.out_host.element_size()
        if self.direct and self.host_inputs and eng._step_mode in (0, 2):
            # the two-pass step reads its inputs from the pinned buffer itself (inputs_host): the
            # scan its MAC_PLANAR_DIMS query dims, the append warps the rest, staged for the later kernels; the
            # complete kernel writes the bf16 output into the pinned output buffer — no I/O launch
            for i, lay in enumerate(self.layers):
                q, k, v = self._qkv_dev[i]
                base = self.in_dev.data_ptr()
                al = self._in_alias.value
                eng._decode_step_ptrs(lay, al + q.data_ptr() - base, al + k.data_ptr() - base,
                                      al + v.data_ptr() - base, dt[q.dtype], self._out_alias.value + i * per_out * osz,
                                      inputs_host=True)
            return
        if self.direct:
            # inputs pulled by one zero-copy kernel; the complete kernel writes the bf16 output
            # straight into the pinned output buffer (no output launch)
            self._io(self._in_alias.value, dt[self.in_host.dtype], self.in_dev.data_ptr(), dt[self.in_dev.dtype],
                     self.in_host.numel())
            for i, lay in enumerate(self.layers):
                q, k, v = self._qkv_dev[i]
                eng._decode_step_ptrs(lay, q.data_ptr(), k.data_ptr(), v.data_ptr(), dt[q.dtype],
                                      self._out_alias.value + i * per_out * osz)
            return
        self._io(self._in_alias.value, dt[self.in_host.dtype], self.in_dev.data_ptr(), dt[self.in_dev.dtype],
                 self.in_host.numel())
        for i, lay in enumerate(self.layers):
            q, k, v = self._qkv_dev[i]
            eng._decode_step_ptrs(lay, q.data_ptr(), k.data_ptr(), v.data_ptr(), dt[q.dtype])
            if self.multi:  # each layer's output leaves before the next layer reuses o_out
                self._io(eng.o_out.data_ptr(), dt[eng.o_out.dtype], self._out_alias.value + i * per_out * osz,
                         dt[self.out_dtype], per_out)
        if not self.multi:
            self._io(eng.o_out.data_ptr(), dt[eng.o_out.dtype], self._out_alias.value, dt[self.out_dtype], per_out)

    def replay(self):
        """One step of every captured layer.  Raises ValueError (before launching) when a layer's
        next position has no KV page: a graph cannot grow the pool (reserve() before capture)."""
        eng = self.eng
        for lay in self.layers:
            eng._ensure_room(lay, grow=False)
        if len(self.graphs) > 1:
            eng._choose_match_mode()
            self.graph = self.graphs.get(eng._step_mode, self.graph)
        self.graph.replay()
        for lay in self.layers:
            eng._len[lay] += 1


# ----------------------------------------------------------------------------
# reference-shaped single-request shim
# ----------------------------------------------------------------------------

class QueryRingView:
    """Read-only view of one (layer, head) query ring (matching.py:67-126)."""

    def __init__(self, eng: "DecodeEngine", layer: int, head: int):
        self._e, self._l, self._h = eng, layer, head
        self.capacity = eng.cfg.window
        self.d = eng.cfg.d

    def _count(self) -> int:
        return int(self._e._ring_last[self._l, self._h])

    def __len__(self):
        return min(self._count(), self.capacity)

    @property
    def last_position(self) -> int:
        return self._count()

    def _positions(self) -> np.ndarray:
        n, W = self._count(), self.capacity
        slots = np.arange(len(self))
        # latest position p <= n with (p - 1) % W == slot
        return n - ((n - 1 - slots) % W)

    def view(self):
        n = len(self)
        q = self._e.batch.ring_q[self._l][0, self._h, :n].double().cpu().numpy()
        return q, np.einsum("ij,ij->i", q, q), self._positions()

    def slot_of(self, pos: int) -> int:
        slot = (pos - 1) % self.capacity
        n = len(self)
        if n == 0 or slot >= n or int(self._positions()[slot]) != pos:
            raise KeyError(f"position {pos} is not in the ring")
        return slot

    def query_at(self, pos: int) -> np.ndarray:
        return self._e.batch.ring_q[self._l][0, self._h, self.slot_of(pos)].double().cpu().numpy()


class SummaryRingView:
    """Read-only view of one (layer, head) summary ring (engine.py:284-320)."""

    def __init__(self, eng: "DecodeEngine", layer: int, head: int):
        self._q = QueryRingView(eng, layer, head)
        self._e, self._l, self._h = eng, layer, head
        self.capacity = eng.cfg.window

    def __len__(self):
        return len(self._q)

    @property
    def last_position(self) -> int:
        return self._q.last_position

    def summary_at(self, pos: int) -> AttentionSummary:
        slot = self._q.slot_of(pos)
        b = self._e.batch
        acc = b.ring_acc[self._l][0, self._h, slot].double().cpu().numpy()
        lse = float(b.ring_lse[self._l][0, self._h, slot].item())
        return AttentionSummary(acc=acc, lse=lse, count=max(0, pos - self._e.cfg.band))


class KvStoreView:
    """Host view of the paged device KV cache with the KvStore read API (kvstore.py:62-165)."""

    def __init__(self, eng: "DecodeEngine", page_rounded_bytes: bool = False):
        self._e = eng
        self.d, self.d_v, self.page_size = eng.cfg.d, eng.cfg.d_v, eng.cfg.page_size
        self.page_rounded_bytes = page_rounded_bytes

    @property
    def token_bytes(self) -> int:
        return (self.d + self.d_v) * self._e.cfg.storage_itemsize

    def length(self, layer: int, kv_head: int) -> int:
        return int(self._e._n[layer])

    def read_range(self, layer: int, kv_head: int, span, counter=None):
        lo, hi = span
        n = self.length(layer, kv_head)
        if lo < 1 or hi < lo:
            raise ValueError(f"invalid token range [{lo}, {hi}]")
        if hi > n:
            raise ValueError(f"token range [{lo}, {hi}] exceeds stored length {n}")
        b = self._e.batch
        idx = torch.arange(lo - 1, hi, device=b.device)
        pages = b.page_table[0, idx // b.page_size].long()
        slots = idx % b.page_size
        keys = b.k_cache[layer][pages, kv_head, slots].double().cpu().numpy()
        vals = b.v_cache[layer][pages, kv_head, slots].double().cpu().numpy()
        if counter is not None:
            tokens = hi - lo + 1
            if self.page_rounded_bytes:  # kvstore.py:137-140
                n_pages = (hi - 1) // self.page_size - (lo - 1) // self.page_size + 1
                counter.record(tokens, n_pages * self.page_size * self.token_bytes)
            else:
                counter.record(tokens, tokens * self.token_bytes)
        return keys, vals

    def n_pages(self, layer: int, kv_head: int) -> int:
        return -(-self.length(layer, kv_head) // self.page_size)

    def page(self, layer: int, kv_head: int, index: int) -> KvPage:
        """Page `index` of (layer, kv head) from the paged device cache (kvstore.py:150-165):
        page_size rows, zero beyond the stored tokens."""
        n_pages = self.n_pages(layer, kv_head)
        if not 0 <= index < n_pages:
            raise IndexError(f"page {index} out of range ({n_pages} pages)")
        b = self._e.batch
        phys = int(b.page_table[0, index].item())
        fill = min(self.length(layer, kv_head) - index * self.page_size, self.page_size)
        keys = b.k_cache[layer][phys, kv_head].double().cpu().numpy()
        vals = b.v_cache[layer][phys, kv_head].double().cpu().numpy()
        keys[fill:] = 0.0
        vals[fill:] = 0.0
        return KvPage(keys=keys, values=vals, fill=fill)


class DecodeEngine:
    """Single-request decoder with the reference API (engine.py:334-539) on the CUDA path."""

    def __init__(self, cfg: EngineConfig, *, device="cuda", capacity: int = 1024):
        self.cfg = cfg
        self.batch = BatchDecodeEngine(cfg, 1, max(capacity, 16), device=device, record_cached=True)
        self.device = self.batch.device
        self.costs = cfg.byte_costs()
        self.metrics = DecodeMetrics()
        self.traffic = TrafficCounter()
        self.oracle_traffic = TrafficCounter()
        self.store = KvStoreView(self)
        self._n = [0] * cfg.n_layers
        # last ring position per (layer, head): the engine's step writes every head's slot, a
        # caller's rectify_append one head's
        self._ring_last = np.zeros((cfg.n_layers, cfg.n_q_heads), dtype=np.int64)
        self._group = cfg.n_q_heads // cfg.n_kv_heads

    def rectify_append(self, layer: int, head: int, m: int, q_pre, full: AttentionSummary, band: AttentionSummary,
                       prefix: AttentionSummary):
        """Push (q_pre, prefix) as the (layer, head) ring entry of position m (engine.py:374-402):
        the same count checks and storage rounding, written into ring slot (m - 1) % W of the
        device rings (and the planar copy the two-pass scan reads).  The device rings are
        slot-aligned, so m must follow the ring's last position by exactly one."""
        cfg = self.cfg
        if full.count != m:
            raise ValueError(f"full summary covers {full.count} tokens, expected {m}")
        if prefix.count != max(0, m - cfg.band):
            raise ValueError(f"prefix summary covers {prefix.count} tokens, expected {max(0, m - cfg.band)}")
        if not 0 <= layer < cfg.n_layers or not 0 <= head < cfg.n_q_heads:
            raise ValueError(f"(layer, head) = ({layer}, {head}) out of range")
        last = int(self._ring_last[layer, head])
        if m <= last:
            raise ValueError(f"ring positions must increase: got {m} after {last}")
        if m != last + 1:
            raise ValueError(f"device rings are slot-aligned: position {m} must follow {last} directly")
        q = np.asarray(q_pre, dtype=np.float64)
        if q.shape != (cfg.d,):
            raise ValueError(f"expected query of dim {cfg.d}, got shape {q.shape}")
        b = self.batch
        slot = (m - 1) % cfg.window
        b.ring_q[layer][0, head, slot] = torch.from_numpy(q).to(self.device, b.ring_q[layer].dtype)
        b.ring_acc[layer][0, head, slot] = torch.from_numpy(np.asarray(prefix.acc, dtype=np.float64)).to(
            self.device, b.ring_acc[layer].dtype)
        b.ring_lse[layer][0, head, slot] = float(prefix.lse)
        if b.ring_qp is not None:
            b.ring_qp[layer][0, head, slot] = b.ring_q[layer][0, head, slot, :_lib.PLANAR_DIMS].to(
                b.ring_qp[layer].dtype)
        self._ring_last[layer, head] = m

    def rings(self, layer: int, head: int):
        return QueryRingView(self, layer, head), SummaryRingView(self, layer, head)

    def decode_step(self, layer: int, q_pre, k_pre, v, m: int, oracle_rows=None) -> StepResult:
        cfg = self.cfg
        r = cfg.band
        q_pre = np.asarray(q_pre, dtype=np.float64)
        k_pre = np.asarray(k_pre, dtype=np.float64)
        v = np.asarray(v, dtype=np.float64)
        if q_pre.shape != (cfg.n_q_heads, cfg.d):
            raise ValueError(f"expected queries ({cfg.n_q_heads}, {cfg.d}), got {q_pre.shape}")
        if k_pre.shape != (cfg.n_kv_heads, cfg.d) or v.shape != (cfg.n_kv_heads, cfg.d_v):
            raise ValueError("key/value shapes do not match the configured kv heads")
        if not 0 <= layer < cfg.n_layers:
            raise ValueError(f"layer {layer} out of range")
        if m != self._n[layer] + 1:
            raise ValueError(f"steps must be consecutive: store is at {self._n[layer] + 1}, step is {m}")
        if int(self._ring_last[layer].max()) >= m:
            raise ValueError(f"ring positions must increase: got {m} after {int(self._ring_last[layer].max())}")
        self.batch.reserve(m)
        dev = self.device
        q = torch.from_numpy(q_pre).to(dev)[None].contiguous()
        k = torch.from_numpy(k_pre).to(dev)[None].contiguous()
        vv = torch.from_numpy(v).to(dev)[None].contiguous()
        mass_check = cfg.mass_check and cfg.oracle_mode
        if mass_check:  # the step overwrites ring slot (m-1) % W, which may hold q at p = m - W
            ring_prev = self.batch.ring_q[layer][0, :, (m - 1) % cfg.window].clone()
        res = self.batch.decode_step(layer, q, k, vv)
        host = {name: t[0].cpu().numpy() for name, t in (
            ("out", res.out), ("hit", res.match_hit), ("use", res.use_hit), ("pos", res.match_pos),
            ("dist", res.match_dist), ("scan", res.match_scanned), ("flse", res.full_lse),
            ("rho", res.band_mass), ("cacc", res.cached_acc), ("clse", res.cached_lse), ("fb", res.fallbacks))}
        self._n[layer] = m
        self._ring_last[layer] = m
        ref_rows = None
        if cfg.oracle_mode:
            if oracle_rows is not None:
                ref_rows = np.asarray(oracle_rows, dtype=np.float64)
            elif host["use"].any():
                ref_rows = self.batch.attend_full(layer, q)[0].double().cpu().numpy()
                for h in range(cfg.n_q_heads):
                    if host["use"][h]:
                        self.oracle_traffic.record(m, m * self.store.token_bytes)

        delta = DecodeMetrics()
        if mass_check and host["use"].any():
            # engine.py:480-483: per hit, q_m at m and the ring query at p, keys [1, p]
            hs = [h for h in range(cfg.n_q_heads) if host["use"][h]]
            ps = [int(host["pos"][h]) for h in hs]
            ring = self.batch.ring_q[layer][0]
            q_p = torch.stack([ring_prev[h] if p == m - cfg.window else ring[h, (p - 1) % cfg.window]
                               for h, p in zip(hs, ps)]).double()
            mb = self.batch.mass_bound(layer, [0] * len(hs), [h // self._group for h in hs], [m] * len(hs), ps,
                                       q[0, hs], q_p).cpu().numpy()
            delta.mass_bound_samples.extend((float(a), float(b)) for a, b in mb)
            for p in ps:
                self.oracle_traffic.record(p, p * self.store.token_bytes)
        outputs = host["out"].astype(np.float64)
        matches, fulls, cacheds, masses = [], [], [], []
        errs = [] if cfg.oracle_mode else None
        for h in range(cfg.n_q_heads):
            hit = bool(host["hit"][h])
            mres = MatchResult(hit, int(host["pos"][h]), float(host["dist"][h]), int(host["scan"][h]))
            delta.match_candidates += mres.candidates_scanned
            delta.match_bytes += mres.candidates_scanned * self.costs.b_q
            use = bool(host["use"][h])
            if hit and not use:
                delta.forced_misses += 1
            delta.fallbacks += int(host["fb"][h])
            if use:
                tokens = delta.record_hit(m, mres.p, r, self.costs.b_kv)
                cached = AttentionSummary(host["cacc"][h].astype(np.float64), float(host["clse"][h]),
                                          max(0, mres.p - r))
            else:
                delta.record_miss(m, self.costs.b_kv)
                tokens = m
                cached = None
            self.traffic.record(tokens, tokens * self.store.token_bytes)
            if errs is not None:
                ref = outputs[h] if (ref_rows is None or (oracle_rows is None and not use)) else ref_rows[h]
                num = float(np.linalg.norm(outputs[h] - ref))
                den = float(np.linalg.norm(ref))
                err = 0.0 if num == 0.0 else (math.inf if den == 0.0 else num / den)
                errs.append(err)
                delta.err_samples.append(err)
            rho = float(host["rho"][h])
            matches.append(mres)
            fulls.append(AttentionSummary(outputs[h], float(host["flse"][h]), m))
            cacheds.append(cached)
            masses.append(rho)
            delta.band_mass_samples.append(rho)
        for g in range(cfg.n_kv_heads):
            grp = matches[g * self._group:(g + 1) * self._group]
            delta.group_kv_tokens += m - min((max(mr.p - r, 0) if mr.hit else 0) for mr in grp)
            delta.group_kv_total += m
        self.metrics.merge(delta)
        return StepResult(outputs=outputs, matches=tuple(matches), full_summaries=tuple(fulls),
                          cached_summaries=tuple(cacheds), band_masses=tuple(masses),
                          errs=tuple(errs) if errs is not None else None, delta=delta)


def oracle_outputs(trace, cfg: EngineConfig, *, chunk: int = 256, device="cuda") -> np.ndarray:
    """Exact causal attention outputs for every (layer, step, q head) of a trace
    (engine.py:542-572), batched on the device: keys rotated at their positions and rounded
    through the storage dtype exactly as the engine stores them, query t rotated at t and
    attended over keys [1, t] in f64 (mac_rope_rotate + mac_summarize, one summarize launch
    per layer).  Returns (n_layers, L, n_q_heads, d_v) f64; `chunk` bounds the query rows of
    one launch."""
    from .summary import rope_rotate_rows, summarize_rows

    dev = torch.device(device)
    L, Hq, Hkv, d, dv = int(trace.seq_len), cfg.n_q_heads, cfg.n_kv_heads, cfg.d, cfg.d_v
    g = Hq // Hkv
    freqs = torch.from_numpy(rope_freqs(d, cfg.rope_base)).to(dev)
    pos = torch.arange(1, L + 1, dtype=torch.float64, device=dev)
    out = np.empty((cfg.n_layers, L, Hq, dv), dtype=np.float64)
    store = {"f32": torch.float32, "bf16": torch.bfloat16, "f64": torch.float64}[cfg.storage]
    for layer in range(cfg.n_layers):
        k = torch.from_numpy(np.ascontiguousarray(trace.k_pre[:, layer], dtype=np.float64)).to(dev)  # [L, Hkv, d]
        v = torch.from_numpy(np.ascontiguousarray(trace.v[:, layer], dtype=np.float64)).to(dev)
        k_rot = rope_rotate_rows(k.permute(1, 0, 2).reshape(Hkv * L, d), pos.repeat(Hkv), freqs).view(Hkv, L, d)
        vv = v.permute(1, 0, 2).contiguous()
        k_rot, vv = k_rot.to(store).double(), vv.to(store).double()  # storage rounding
        q = torch.from_numpy(np.ascontiguousarray(trace.q_pre[:, layer], dtype=np.float64)).to(dev)
        q = q.permute(1, 0, 2).contiguous()  # [Hq, L, d]
        step = max(1, int(chunk))
        for lo in range(0, L, step):
            hi = min(L, lo + step)
            t = torch.arange(lo + 1, hi + 1, dtype=torch.int32, device=dev).expand(Hq, hi - lo).contiguous()
            acc, _ = summarize_rows(q[:, lo:hi], k_rot[:, :hi], vv[:, :hi], hi=t, rope_t=t, rope_freqs=freqs,
                                    sets_per_kv=g)
            out[layer, lo:hi] = acc.permute(1, 0, 2).cpu().numpy()
    return out


def run_decode(trace, cfg: EngineConfig, *, per_step_oracle: bool = False, on_step=None,
               device="cuda") -> DecodeEngine:
    """Drive a whole trace through a fresh engine (engine.py:575-607).  With oracle_mode the
    reference rows come from one batched device pass (oracle_outputs) unless per_step_oracle
    is set, in which case every step computes its own (mac_attend_full on the stored cache)."""
    if (trace.d, trace.d_v, trace.n_layers, trace.n_q_heads, trace.n_kv_heads) != (
            cfg.d, cfg.d_v, cfg.n_layers, cfg.n_q_heads, cfg.n_kv_heads):
        raise ValueError("trace dimensions do not match the engine config")
    eng = DecodeEngine(cfg, device=device, capacity=int(trace.seq_len))
    oracle = oracle_outputs(trace, cfg, device=eng.device) if cfg.oracle_mode and not per_step_oracle else None
    for m in range(1, int(trace.seq_len) + 1):
        for layer in range(cfg.n_layers):
            rows = oracle[layer, m - 1] if oracle is not None else None
            res = eng.decode_step(layer, trace.q_pre[m - 1, layer], trace.k_pre[m - 1, layer],
                                  trace.v[m - 1, layer], m, oracle_rows=rows)
            if on_step is not None:
                on_step(m, layer, res)
    return eng
