"""Configuration and result types of the decode path, mirroring `attnreuse`.

Names, fields, defaults and validation follow the reference so a caller can
switch imports: EngineConfig (engine.py:108-164), MatchConfig / MatchResult /
threshold (matching.py:29-64), AttentionSummary / empty_summary / finalize
(attention.py:35-58,175-179), DecodeMetrics / compute_metrics
(engine.py:167-243), StepResult (engine.py:323-331), ByteCostModel /
break_even_gate / group_kv_span and the sizing helpers (engine.py:45-105).
These are host-side bookkeeping only; every attention number is produced by
the CUDA library.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

MATCH_PRE_ROPE = "pre_rope"
MATCH_POST_ROPE = "post_rope"
DOWNDATE_SPLIT = "split"
DOWNDATE_REMOVE = "remove"
STORAGES = ("f32", "f64", "bf16")


class CancellationError(ArithmeticError):
    """Removing the band would cancel catastrophically (attention.py:23-24)."""


class MassExceededError(ValueError):
    """Band mass exceeds the summary it is removed from (attention.py:27-28)."""


class EmptySummaryError(ValueError):
    """finalize() on a summary over zero tokens (attention.py:31-32)."""


@dataclass(frozen=True)
class AttentionSummary:
    """acc = S/Z, lse = ln Z, count tokens; empty is (0, -inf, 0) (attention.py:35-54)."""

    acc: np.ndarray
    lse: float
    count: int

    def astype(self, dtype) -> "AttentionSummary":
        """The summary as stored in `dtype` (acc and a finite lse rounded through it)."""
        dt = np.dtype(dtype)
        lse = self.lse if math.isinf(self.lse) else float(dt.type(self.lse))
        return AttentionSummary(acc=self.acc.astype(dt), lse=lse, count=self.count)


def empty_summary(d_v: int, dtype=np.float64) -> AttentionSummary:
    return AttentionSummary(acc=np.zeros(d_v, dtype=dtype), lse=-math.inf, count=0)


def finalize(s: AttentionSummary) -> np.ndarray:
    if s.count == 0:
        raise EmptySummaryError("cannot finalize a summary over zero tokens")
    return s.acc


def threshold(d: int, tau: float) -> float:
    """Acceptance radius sqrt(2d)(1 - tau) (matching.py:58-64)."""
    if d < 1:
        raise ValueError("head dim must be positive")
    if not 0.0 <= tau < 1.0:
        raise ValueError(f"tau must lie in [0, 1), got {tau}")
    return math.sqrt(2.0 * d) * (1.0 - tau)


@dataclass
class MatchConfig:
    d: int
    tau: float = 0.45
    delta_max: int | None = None
    space: str = MATCH_PRE_ROPE
    rope_base: float = 10000.0

    def __post_init__(self):
        if self.d < 1:
            raise ValueError("head dim must be positive")
        if not 0.0 <= self.tau < 1.0:
            raise ValueError(f"tau must lie in [0, 1), got {self.tau}")
        if self.delta_max is not None and self.delta_max < 1:
            raise ValueError("delta_max must be >= 1 when set")
        if self.space not in (MATCH_PRE_ROPE, MATCH_POST_ROPE):
            raise ValueError(f"unknown match space {self.space!r}")


@dataclass(frozen=True)
class MatchResult:
    hit: bool
    p: int
    sq_dist: float
    candidates_scanned: int

    MISS_POS = -1


@dataclass(frozen=True)
class ByteCostModel:
    """Bytes per cached token read (b_kv) and per ring candidate scanned (b_q)."""

    b_kv: float
    b_q: float

    def __post_init__(self):
        if self.b_kv < 0 or self.b_q < 0:
            raise ValueError("byte costs must be non-negative")


def break_even_gate(p: int, band: int, window: int, costs: ByteCostModel) -> bool:
    """p*b_kv >= window*b_q + band*b_kv (engine.py:57-63)."""
    return p * costs.b_kv >= window * costs.b_q + band * costs.b_kv


def group_kv_span(matches, m: int, band: int) -> int:
    """KV rows a GQA group streams at step m (engine.py:66-77)."""
    matches = list(matches)
    if not matches:
        raise ValueError("group_kv_span needs at least one head")
    return m - min((max(mr.p - band, 0) if mr.hit else 0) for mr in matches)


def aux_overhead_ratio(cfg: "EngineConfig", seq_len: int) -> float:
    """Ring state over KV cache size at seq_len (engine.py:80-91)."""
    if seq_len < 1:
        raise ValueError("seq_len must be >= 1")
    return (cfg.window * cfg.n_q_heads * (cfg.d + cfg.d_v + 2)) / (seq_len * cfg.n_kv_heads * 2 * cfg.d)


def aux_overhead_rule_of_thumb(window: int, seq_len: int) -> float:
    """5% of the KV cache at window 1024 and 120k context (engine.py:94-98)."""
    if window < 0 or seq_len < 1:
        raise ValueError("window must be >= 0 and seq_len >= 1")
    return 0.05 * (window / 1024.0) * (120_000.0 / seq_len)


def fidelity_efficiency(err_mean: float, kv_fraction: float) -> float:
    if kv_fraction <= 0:
        raise ValueError("kv_fraction must be positive")
    return (1.0 - min(max(err_mean, 0.0), 1.0)) / kv_fraction


@dataclass
class EngineConfig:
    """Decode-path parameters (engine.py:108-164).  storage adds 'bf16' (B200 serving)."""

    d: int
    d_v: int
    n_layers: int = 1
    n_q_heads: int = 1
    n_kv_heads: int = 1
    window: int = 1024
    band: int = 256
    tau: float = 0.45
    tau_per_layer: tuple | None = None
    delta_max: int | None = None
    match_space: str = MATCH_PRE_ROPE
    rope_base: float = 10000.0
    storage: str = "f32"
    oracle_mode: bool = False
    roi_gate: bool = False
    economics: ByteCostModel | None = None
    downdate_mode: str = DOWNDATE_SPLIT
    refresh_every: int = 0
    mass_check: bool = False
    page_size: int = 16

    def __post_init__(self):
        if self.d < 2 or self.d % 2:
            raise ValueError(f"head dim must be even and >= 2 (rotary pairs), got {self.d}")
        if self.d_v < 1:
            raise ValueError("value dim must be >= 1")
        if self.n_layers < 1 or self.n_q_heads < 1 or self.n_kv_heads < 1:
            raise ValueError("layer and head counts must be >= 1")
        if self.n_q_heads % self.n_kv_heads:
            raise ValueError("n_q_heads must be a multiple of n_kv_heads")
        if self.window < 1:
            raise ValueError("ring window must be >= 1")
        if self.band < 0:
            raise ValueError("band must be >= 0")
        if not 0.0 <= self.tau < 1.0:
            raise ValueError(f"tau must lie in [0, 1), got {self.tau}")
        if self.tau_per_layer is not None:
            self.tau_per_layer = tuple(self.tau_per_layer)
            if len(self.tau_per_layer) != self.n_layers:
                raise ValueError("tau_per_layer must list one tau per layer")
            if any(not 0.0 <= t < 1.0 for t in self.tau_per_layer):
                raise ValueError("per-layer taus must lie in [0, 1)")
        if self.storage not in STORAGES:
            raise ValueError(f"storage must be one of {STORAGES}, got {self.storage!r}")
        if self.downdate_mode not in (DOWNDATE_SPLIT, DOWNDATE_REMOVE):
            raise ValueError(f"unknown downdate mode {self.downdate_mode!r}")
        if self.refresh_every < 0:
            raise ValueError("refresh_every must be >= 0 (0 disables)")
        if self.match_space not in (MATCH_PRE_ROPE, MATCH_POST_ROPE):
            raise ValueError(f"unknown match space {self.match_space!r}")
        if self.delta_max is not None and self.delta_max < 1:
            raise ValueError("delta_max must be >= 1 when set")
        if self.rope_base <= 1.0:
            raise ValueError("rope base must exceed 1")
        if self.page_size < 1:
            raise ValueError("page_size must be >= 1")

    @property
    def storage_itemsize(self) -> int:
        return {"f32": 4, "f64": 8, "bf16": 2}[self.storage]

    def tau_for(self, layer: int) -> float:
        return self.tau_per_layer[layer] if self.tau_per_layer is not None else self.tau

    def byte_costs(self) -> ByteCostModel:
        """Default economics (engine.py:340-343): b_kv = (d + d_v)*s, b_q = d*s (s = 4 for f32, 8 for f64)."""
        if self.economics is not None:
            return self.economics
        isize = 8 if self.storage == "f64" else 4
        return ByteCostModel(b_kv=(self.d + self.d_v) * isize, b_q=self.d * isize)


@dataclass
class DecodeMetrics:
    """Accumulator over per-(step, layer, q head) decisions (engine.py:167-223)."""

    steps: int = 0
    hits: int = 0
    fallbacks: int = 0
    forced_misses: int = 0
    skip_sum: float = 0.0
    kv_tokens_read: int = 0
    kv_tokens_full: int = 0
    kv_bytes: float = 0.0
    match_candidates: int = 0
    match_bytes: float = 0.0
    group_kv_tokens: int = 0
    group_kv_total: int = 0
    err_samples: list = field(default_factory=list)
    band_mass_samples: list = field(default_factory=list)
    delta_gaps: list = field(default_factory=list)
    mass_bound_samples: list = field(default_factory=list)

    def record_hit(self, m: int, p: int, band: int, kv_cost: float = 0.0) -> int:
        skipped = max(p - band, 0)
        tokens = m - skipped
        self.steps += 1
        self.hits += 1
        self.skip_sum += skipped / m
        self.kv_tokens_read += tokens
        self.kv_tokens_full += m
        self.kv_bytes += tokens * kv_cost
        self.delta_gaps.append(m - p)
        return tokens

    def record_miss(self, m: int, kv_cost: float = 0.0):
        self.steps += 1
        self.kv_tokens_read += m
        self.kv_tokens_full += m
        self.kv_bytes += m * kv_cost

    def merge(self, other: "DecodeMetrics"):
        for name in ("steps", "hits", "fallbacks", "forced_misses", "skip_sum", "kv_tokens_read", "kv_tokens_full",
                     "kv_bytes", "match_candidates", "match_bytes", "group_kv_tokens", "group_kv_total"):
            setattr(self, name, getattr(self, name) + getattr(other, name))
        for name in ("err_samples", "band_mass_samples", "delta_gaps", "mass_bound_samples"):
            getattr(self, name).extend(getattr(other, name))


def compute_metrics(metrics: DecodeMetrics) -> dict:
    """Report schema v1 (engine.py:226-243)."""
    if metrics.steps < 1:
        raise ValueError("metrics cover zero decisions")
    errs = np.asarray(metrics.err_samples, dtype=np.float64) if metrics.err_samples else None
    return {
        "schema_version": 1,
        "steps": metrics.steps,
        "hits": metrics.hits,
        "acceptance_rate": metrics.hits / metrics.steps,
        "skip_ratio": metrics.skip_sum / metrics.steps,
        "kv_fraction": metrics.kv_tokens_read / metrics.kv_tokens_full,
        "err_mean": float(errs.mean()) if errs is not None else None,
        "err_p50": float(np.percentile(errs, 50)) if errs is not None else None,
        "err_p99": float(np.percentile(errs, 99)) if errs is not None else None,
        "mean_gap": float(np.mean(metrics.delta_gaps)) if metrics.delta_gaps else None,
        "mean_band_mass": float(np.mean(metrics.band_mass_samples)) if metrics.band_mass_samples else None,
    }


@dataclass
class StepResult:
    """One decode_step's host-side result (engine.py:323-331)."""

    outputs: np.ndarray
    matches: tuple
    full_summaries: tuple
    cached_summaries: tuple
    band_masses: tuple
    errs: tuple | None
    delta: DecodeMetrics
