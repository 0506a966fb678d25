"""CPU oracle for the MAC-Attention decode path — TEST INFRASTRUCTURE ONLY.

This module is the parity checker, never the product.  Only `tests/`,
`__graft_entry__.smoke()` and `bench.py` (its `cpu_baseline` leg and the
`--impl reference` arm) may import it.  The product path
(`paper_2604_00235_b200`) never imports it and fails loudly when its CUDA
library is missing.

It is a numpy restatement of the reference package `attnreuse`
(/root/reference/pkg/src/attnreuse, pure Python + numpy), step for step:

* summary algebra        attention.py:35-135  (AttentionSummary, summarize, merge)
* interleaved RoPE       attention.py:195-232 (RopeTable, rope_rotate)
* query-ring match       matching.py:58-175   (threshold, QueryRing, match_query)
* paged KV store         kvstore.py:105-144   (append rounding, read_range)
* decode step            engine.py:410-539    (DecodeEngine.decode_step)
* ring write-back        engine.py:374-402    (rectify_append)
* metrics                engine.py:167-243    (DecodeMetrics, compute_metrics)
* batched oracle         engine.py:542-572    (oracle_outputs)
* prefix mass bound      engine.py:246-281    (mass_bound_check)

One extension beyond the reference: storage "bf16" (keys, values and ring
queries rounded through bfloat16, summaries through float32), the storage
the GPU bf16 path uses.  With bf16-representable inputs this equals the
reference fed the storage-matched keys R_m^-1(bf16(R_m k)).

Parity pinning: `tests/golden/make_golden.py` runs the real reference (this
container only) and commits its outputs under `tests/golden/`;
`tests/test_oracle_golden.py` checks this module against them.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

__all__ = [
    "round_bf16",
    "round_storage",
    "rope_freqs",
    "rope_rotate",
    "Summary",
    "EMPTY_LSE",
    "summarize",
    "merge",
    "remove",
    "threshold",
    "OracleConfig",
    "OracleEngine",
    "OracleStep",
    "oracle_outputs",
    "metrics_report",
    "mass_bound_check",
]

EMPTY_LSE = -math.inf


# ----------------------------------------------------------------------------
# storage rounding (kvstore.py:113-115, engine.py:396-399, attention.py:49-54)
# ----------------------------------------------------------------------------

def round_bf16(x) -> np.ndarray:
    """Round-to-nearest-even through bfloat16, returned as float64."""
    f = np.ascontiguousarray(np.asarray(x, dtype=np.float32))
    u = f.view(np.uint32).astype(np.uint64)
    lsb = (u >> 16) & 1
    u = (u + 0x7FFF + lsb) & 0xFFFF0000
    out = u.astype(np.uint32).view(np.float32)
    # NaN/inf pass through unchanged (not produced by this workload)
    bad = ~np.isfinite(f)
    if bad.any():
        out = np.where(bad, f, out)
    return out.astype(np.float64)


def round_storage(x, storage: str) -> np.ndarray:
    x = np.asarray(x, dtype=np.float64)
    if storage == "f64":
        return x.copy()
    if storage == "f32":
        return x.astype(np.float32).astype(np.float64)
    if storage == "bf16":
        return round_bf16(x)
    raise ValueError(f"unknown storage {storage!r}")


def round_summary_scalar(v: float, storage: str) -> float:
    # attention.py:53 — lse rounded unless infinite; summaries stay f32 under bf16
    if math.isinf(v) or storage == "f64":
        return v
    return float(np.float32(v))


# ----------------------------------------------------------------------------
# RoPE (attention.py:195-232)
# ----------------------------------------------------------------------------

def rope_freqs(d: int, base: float = 10000.0) -> np.ndarray:
    """omega_j = base**(-2j/d), j = 0..d/2-1 (attention.py:208-209)."""
    if d < 2 or d % 2:
        raise ValueError("rotary embedding needs an even head dim >= 2")
    if base <= 1.0:
        raise ValueError("rope base must exceed 1")
    j = np.arange(d // 2, dtype=np.float64)
    return base ** (-2.0 * j / d)


def rope_rotate(x, t, freqs: np.ndarray) -> np.ndarray:
    """Rotate adjacent pairs (x[2j], x[2j+1]) by t*omega_j (attention.py:212-232)."""
    x = np.asarray(x, dtype=np.float64)
    t = np.asarray(t, dtype=np.float64)
    angles = t[..., None] * freqs if t.ndim else t * freqs
    c = np.cos(angles)
    s = np.sin(angles)
    pairs = x.reshape(*x.shape[:-1], freqs.shape[0], 2)
    out = np.empty_like(pairs)
    out[..., 0] = pairs[..., 0] * c - pairs[..., 1] * s
    out[..., 1] = pairs[..., 0] * s + pairs[..., 1] * c
    return out.reshape(x.shape)


# ----------------------------------------------------------------------------
# summary algebra (attention.py:35-172)
# ----------------------------------------------------------------------------

@dataclass(frozen=True)
class Summary:
    """(acc = S/Z, lse = ln Z, count); empty = (0, -inf, 0) (attention.py:35-58)."""

    acc: np.ndarray
    lse: float
    count: int

    @staticmethod
    def empty(d_v: int) -> "Summary":
        return Summary(np.zeros(d_v, dtype=np.float64), EMPTY_LSE, 0)

    def stored(self, storage: str) -> "Summary":
        """Storage model of attention.py:49-54 (bf16 mode keeps summaries in f32)."""
        if storage == "f64":
            return self
        acc = np.asarray(self.acc, dtype=np.float32).astype(np.float64)
        return Summary(acc, round_summary_scalar(self.lse, storage), self.count)


def summarize(q, keys, values, block: int = 4096) -> Summary:
    """Online-softmax summary of q over keys/values (attention.py:75-116)."""
    n = keys.shape[0]
    if n == 0:
        return Summary.empty(values.shape[1])
    q64 = np.asarray(q, dtype=np.float64)
    scale = 1.0 / math.sqrt(q64.shape[0])
    if n <= block:
        logits = (keys @ q64) * scale
        mx = float(logits.max())
        w = np.exp(logits - mx)
        z = float(w.sum())
        return Summary((w @ values) / z, mx + math.log(z), n)
    run_m, run_z = -math.inf, 0.0
    run_s = np.zeros(values.shape[1], dtype=np.float64)
    for lo in range(0, n, block):
        hi = min(lo + block, n)
        logits = (keys[lo:hi] @ q64) * scale
        new_m = max(run_m, float(logits.max()))
        w = np.exp(logits - new_m)
        run_s = run_s * math.exp(run_m - new_m) + w @ values[lo:hi]
        run_z = run_z * math.exp(run_m - new_m) + float(w.sum())
        run_m = new_m
    return Summary(run_s / run_z, run_m + math.log(run_z), n)


def merge(a: Summary, b: Summary) -> Summary:
    """Log-domain merge, empty is the identity (attention.py:119-135)."""
    if a.count == 0:
        return b
    if b.count == 0:
        return a
    lse = float(np.logaddexp(a.lse, b.lse))
    acc = a.acc * math.exp(a.lse - lse) + b.acc * math.exp(b.lse - lse)
    return Summary(acc, lse, a.count + b.count)


class CancellationError(ArithmeticError):
    pass


def remove(a: Summary, band: Summary, eps_cancel: float = 1e-6) -> Summary:
    """Down-date a band out of a summary (attention.py:138-172)."""
    if band.count == 0:
        return a
    if band.count > a.count:
        raise ValueError("band covers more tokens than the summary")
    if band.count == a.count:
        if band.lse == a.lse:
            return Summary.empty(a.acc.shape[0])
        raise CancellationError("count would reach zero")
    diff = a.lse - band.lse
    if diff < -eps_cancel:
        raise ValueError("band mass exceeds the summary")
    if diff < eps_cancel:
        raise CancellationError("residual below guard")
    lse = band.lse + math.log(math.expm1(diff))
    acc = a.acc * math.exp(a.lse - lse) - band.acc * math.exp(band.lse - lse)
    return Summary(acc, lse, a.count - band.count)


# ----------------------------------------------------------------------------
# matching (matching.py:58-175)
# ----------------------------------------------------------------------------

def threshold(d: int, tau: float) -> float:
    """sqrt(2d)(1 - tau) (matching.py:58-64)."""
    return math.sqrt(2.0 * d) * (1.0 - tau)


def _match(q, m, ring_q, ring_sq, ring_pos, n_live, cfg, tau, freqs):
    """match_query restated (matching.py:141-175). Returns (hit, p, best, scanned)."""
    if n_live == 0:
        return False, -1, math.inf, 0
    cand, sqn, pos = ring_q[:n_live], ring_sq[:n_live], ring_pos[:n_live]
    if cfg.delta_max is not None:
        keep = (m - pos) <= cfg.delta_max
        if not keep.any():
            return False, -1, math.inf, 0
        cand, sqn, pos = cand[keep], sqn[keep], pos[keep]
    if cfg.match_space == "post_rope":
        ang = (pos - m).astype(np.float64)[:, None] * freqs
        c, s = np.cos(ang), np.sin(ang)
        pairs = cand.reshape(cand.shape[0], -1, 2)
        rot = np.empty_like(pairs)
        rot[..., 0] = pairs[..., 0] * c - pairs[..., 1] * s
        rot[..., 1] = pairs[..., 0] * s + pairs[..., 1] * c
        cand = rot.reshape(cand.shape)
    sq = float(q @ q) + sqn - 2.0 * (cand @ q)
    np.maximum(sq, 0.0, out=sq)
    best = sq.min()
    p = int(pos[np.flatnonzero(sq == best)].max())
    hit = bool(best < threshold(cfg.d, tau) ** 2)
    return hit, (p if hit else -1), float(best), int(pos.shape[0])


# ----------------------------------------------------------------------------
# engine (engine.py:108-243, 334-572)
# ----------------------------------------------------------------------------

@dataclass
class OracleConfig:
    """Field names and defaults of EngineConfig (engine.py:108-129); storage adds 'bf16'."""

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
    match_space: str = "pre_rope"
    rope_base: float = 10000.0
    storage: str = "f32"
    roi_gate: bool = False
    b_kv: float | None = None
    b_q: float | None = None
    downdate_mode: str = "split"
    refresh_every: int = 0

    def tau_for(self, layer: int) -> float:
        return self.tau_per_layer[layer] if self.tau_per_layer is not None else self.tau

    @property
    def itemsize(self) -> int:
        return {"f64": 8, "f32": 4, "bf16": 2}[self.storage]


@dataclass
class OracleMetrics:
    """DecodeMetrics counters (engine.py:167-223)."""

    steps: int = 0
    hits: int = 0
    fallbacks: int = 0
    forced_misses: int = 0
    skip_sum: float = 0.0
    kv_tokens_read: int = 0
    kv_tokens_full: int = 0
    match_candidates: int = 0
    group_kv_tokens: int = 0
    group_kv_total: int = 0
    band_mass_samples: list = field(default_factory=list)
    delta_gaps: list = field(default_factory=list)


def metrics_report(mt: OracleMetrics) -> dict:
    """compute_metrics (engine.py:226-243) without the oracle-mode error fields."""
    return {
        "steps": mt.steps,
        "hits": mt.hits,
        "acceptance_rate": mt.hits / mt.steps,
        "skip_ratio": mt.skip_sum / mt.steps,
        "kv_fraction": mt.kv_tokens_read / mt.kv_tokens_full,
        "mean_gap": float(np.mean(mt.delta_gaps)) if mt.delta_gaps else None,
        "mean_band_mass": float(np.mean(mt.band_mass_samples)) if mt.band_mass_samples else None,
        "group_kv_tokens": mt.group_kv_tokens,
        "group_kv_total": mt.group_kv_total,
        "forced_misses": mt.forced_misses,
        "fallbacks": mt.fallbacks,
    }


@dataclass
class OracleStep:
    outputs: np.ndarray          # (Hq, d_v) f64
    hit: np.ndarray              # (Hq,) raw match decision (matching.py:174)
    use_hit: np.ndarray          # (Hq,) after roi/refresh gates (engine.py:452-459)
    p: np.ndarray                # (Hq,) int, -1 on a raw miss
    sq_dist: np.ndarray          # (Hq,) f64, inf when nothing scanned
    scanned: np.ndarray          # (Hq,) int
    full_lse: np.ndarray         # (Hq,)
    prefix_acc: np.ndarray       # (Hq, d_v) stored ring summary (rounded)
    prefix_lse: np.ndarray       # (Hq,)
    band_mass: np.ndarray        # (Hq,)


class OracleEngine:
    """One request's decode state; restates DecodeEngine (engine.py:334-539).

    KV is held per (layer, kv head) in preallocated float64 buffers holding
    storage-rounded values (kvstore.py:42-59, 105-119).
    """

    def __init__(self, cfg: OracleConfig, capacity: int = 1024):
        self.cfg = cfg
        self.freqs = rope_freqs(cfg.d, cfg.rope_base)
        self.group = cfg.n_q_heads // cfg.n_kv_heads
        isz = 4 if cfg.storage in ("f32", "bf16") else 8
        self.b_kv = cfg.b_kv if cfg.b_kv is not None else (cfg.d + cfg.d_v) * isz
        self.b_q = cfg.b_q if cfg.b_q is not None else cfg.d * isz
        L, Hq, Hkv, W = cfg.n_layers, cfg.n_q_heads, cfg.n_kv_heads, cfg.window
        self.cap = max(int(capacity), 16)
        self.K = np.zeros((L, Hkv, self.cap, cfg.d))
        self.V = np.zeros((L, Hkv, self.cap, cfg.d_v))
        self.n = np.zeros(L, dtype=np.int64)
        # query ring (matching.py:67-126): slot = (pos-1) % W
        self.rq = np.zeros((L, Hq, W, cfg.d))
        self.rsq = np.zeros((L, Hq, W))
        self.rpos = np.zeros((L, Hq, W), dtype=np.int64)
        # summary ring (engine.py:284-320), slot-aligned with the query ring
        self.racc = np.zeros((L, Hq, W, cfg.d_v))
        self.rlse = np.full((L, Hq, W), EMPTY_LSE)
        self.count = np.zeros(L, dtype=np.int64)  # ring pushes per layer (== n)
        self.metrics = OracleMetrics()

    # --- state -------------------------------------------------------------
    def _grow(self, need: int):
        if need <= self.cap:
            return
        cap = max(need, 2 * self.cap)
        for name in ("K", "V"):
            old = getattr(self, name)
            buf = np.zeros(old.shape[:2] + (cap,) + old.shape[3:])
            buf[:, :, : self.cap] = old[:, :, : self.cap]
            setattr(self, name, buf)
        self.cap = cap

    def inject(self, layer, k_store, v_store, ring_q, ring_acc, ring_lse):
        """Load a prefix state: K/V rows 1..n (already rotated+rounded) and the last
        min(n, W) ring entries (positions n-len+1..n, oldest first)."""
        cfg = self.cfg
        n = k_store.shape[1]
        self._grow(n + 64)
        self.K[layer, :, :n] = k_store
        self.V[layer, :, :n] = v_store
        self.n[layer] = n
        cnt = ring_q.shape[1]
        W = cfg.window
        for i in range(cnt):
            pos = n - cnt + 1 + i
            slot = (pos - 1) % W
            self.rq[layer, :, slot] = ring_q[:, i]
            self.rsq[layer, :, slot] = np.einsum("hd,hd->h", ring_q[:, i], ring_q[:, i])
            self.rpos[layer, :, slot] = pos
            self.racc[layer, :, slot] = ring_acc[:, i]
            self.rlse[layer, :, slot] = ring_lse[:, i]
        self.count[layer] = n

    def inject_tail(self, layer, n, k_rows, v_rows, row0, ring_q, ring_acc, ring_lse):
        """Like inject(), but only K/V rows row0+1..row0+T are given; older rows stay
        zero (np.zeros pages are mapped lazily, so a 128K-token state costs only its tail)."""
        self._grow(n + 64)
        T = k_rows.shape[1]
        self.K[layer, :, row0 : row0 + T] = k_rows
        self.V[layer, :, row0 : row0 + T] = v_rows
        self.n[layer] = n
        W = self.cfg.window
        cnt = ring_q.shape[1]
        pos = np.arange(n - cnt + 1, n + 1)
        slots = (pos - 1) % W
        self.rq[layer][:, slots] = ring_q
        self.rsq[layer][:, slots] = np.einsum("hwd,hwd->hw", ring_q, ring_q)
        self.rpos[layer][:, slots] = pos
        self.racc[layer][:, slots] = ring_acc
        self.rlse[layer][:, slots] = ring_lse
        self.count[layer] = n

    def _live(self, layer, h):
        """Ring view in push order semantics: entries live if pos >= 1 (matching.py:114-117)."""
        n_live = int(min(self.count[layer], self.cfg.window))
        if n_live < self.cfg.window:
            return self.rq[layer, h, :n_live], self.rsq[layer, h, :n_live], self.rpos[layer, h, :n_live], n_live
        return self.rq[layer, h], self.rsq[layer, h], self.rpos[layer, h], n_live

    # --- one step ------------------------------------------------------------
    def decode_step(self, layer: int, q_pre, k_pre, v, m: int) -> OracleStep:
        cfg = self.cfg
        r, W, st = cfg.band, cfg.window, cfg.storage
        q_pre = np.asarray(q_pre, dtype=np.float64)
        k_pre = np.asarray(k_pre, dtype=np.float64)
        v = np.asarray(v, dtype=np.float64)
        if m != self.n[layer] + 1:
            raise ValueError(f"steps must be consecutive: store is at {self.n[layer] + 1}, step is {m}")
        self._grow(m)
        # engine.py:434-437 — rotate keys at position m, round through storage, append
        k_rot = rope_rotate(k_pre, float(m), self.freqs)
        self.K[layer, :, m - 1] = round_storage(k_rot, st)
        self.V[layer, :, m - 1] = round_storage(v, st)
        self.n[layer] = m

        Hq, dv = cfg.n_q_heads, cfg.d_v
        out = np.empty((Hq, dv))
        hit = np.zeros(Hq, dtype=bool)
        use = np.zeros(Hq, dtype=bool)
        ps = np.full(Hq, -1, dtype=np.int64)
        dist = np.full(Hq, math.inf)
        scanned = np.zeros(Hq, dtype=np.int64)
        flse = np.empty(Hq)
        pacc = np.empty((Hq, dv))
        plse = np.empty(Hq)
        rho_all = np.zeros(Hq)
        empty = Summary.empty(dv)
        tau = cfg.tau_for(layer)
        mt = self.metrics
        for h in range(Hq):
            rq, rsq, rpos, n_live = self._live(layer, h)
            # matching.py:141-175 (ring holds exactly positions < m)
            hh, p, best, nscan = _match(q_pre[h], m, rq, rsq, rpos, n_live, cfg, tau, self.freqs)
            mt.match_candidates += nscan
            u = hh
            # engine.py:453-459 — break-even and refresh gates force misses
            if u and cfg.roi_gate and not (p * self.b_kv >= W * self.b_q + r * self.b_kv):
                u = False
                mt.forced_misses += 1
            if cfg.refresh_every and m % cfg.refresh_every == 0:
                if u:
                    mt.forced_misses += 1
                u = False
            q_rot = rope_rotate(q_pre[h], float(m), self.freqs)
            j = h // self.group
            if u:
                # engine.py:464-479 — hit: reuse cached(p), recompute [lo, m] split at m-r
                lo = max(1, p - r + 1)
                keys = self.K[layer, j, lo - 1 : m]
                vals = self.V[layer, j, lo - 1 : m]
                slot = (p - 1) % W
                cached = Summary(self.racc[layer, h, slot].copy(), float(self.rlse[layer, h, slot]), max(0, p - r))
                n1 = max(0, (m - r) - lo + 1)
                piece = summarize(q_rot, keys[:n1], vals[:n1]) if n1 > 0 else empty
                band = summarize(q_rot, keys[n1:], vals[n1:]) if n1 < keys.shape[0] else empty
                prefix = merge(cached, piece)
                full = merge(prefix, band)
                o = full.acc
                if cfg.downdate_mode == "remove" and band.count:
                    try:
                        prefix = remove(full, band)
                    except CancellationError:
                        mt.fallbacks += 1
                skipped = max(p - r, 0)
                mt.steps += 1
                mt.hits += 1
                mt.skip_sum += skipped / m
                mt.kv_tokens_read += m - skipped
                mt.kv_tokens_full += m
                mt.delta_gaps.append(m - p)
            else:
                # engine.py:484-499 — miss: exact attention over [1, m] plus split summaries
                keys = self.K[layer, j, :m]
                vals = self.V[layer, j, :m]
                full = summarize(q_rot, keys, vals)
                o = full.acc
                mid = max(0, m - r)
                if r == 0:
                    prefix, band = full, empty
                elif mid == 0:
                    prefix, band = empty, full
                else:
                    prefix = summarize(q_rot, keys[:mid], vals[:mid])
                    band = summarize(q_rot, keys[mid:], vals[mid:])
                if cfg.downdate_mode == "remove" and band.count and prefix.count:
                    try:
                        prefix = remove(full, band)
                    except CancellationError:
                        mt.fallbacks += 1
                mt.steps += 1
                mt.kv_tokens_read += m
                mt.kv_tokens_full += m
            # engine.py:501 — band mass
            rho = math.exp(band.lse - full.lse) if band.count else 0.0
            # engine.py:374-402 — ring write at slot (m-1) % W
            slot = (m - 1) % W
            qs = round_storage(q_pre[h], st)
            ps_ = prefix.stored(st)
            self.rq[layer, h, slot] = qs
            self.rsq[layer, h, slot] = float(qs @ qs)
            self.rpos[layer, h, slot] = m
            self.racc[layer, h, slot] = ps_.acc
            self.rlse[layer, h, slot] = ps_.lse
            out[h] = o
            hit[h], use[h], ps[h], dist[h], scanned[h] = hh, u, p, best, nscan
            flse[h] = full.lse
            pacc[h], plse[h] = ps_.acc, ps_.lse
            rho_all[h] = rho
            mt.band_mass_samples.append(rho)
        self.count[layer] = m
        # engine.py:525-528 — GQA group span uses the raw match decisions
        for g in range(cfg.n_kv_heads):
            hs = range(g * self.group, (g + 1) * self.group)
            floor = min((max(int(ps[h]) - r, 0) if hit[h] else 0) for h in hs)
            mt.group_kv_tokens += m - floor
            mt.group_kv_total += m
        return OracleStep(out, hit, use, ps, dist, scanned, flse, pacc, plse, rho_all)


def mass_bound_check(q_m, q_p, keys, values, band: int) -> tuple[float, float]:
    """Drift of the reused non-band prefix vs its first-order bound (engine.py:246-281).

    Softmaxes of both post-RoPE queries over keys [1, p]; cut = (p - band)+;
    lhs = ||sum_{t<=cut} (a_p - a_m)_t v_t||, rhs = expm1(max_{t<=cut}|l_m - l_p|)
    * (1 - rho) * E_{a_p}[||v||] over the prefix, rho = a_p's band share."""
    keys = np.asarray(keys, dtype=np.float64)
    values = np.asarray(values, dtype=np.float64)
    n = keys.shape[0]
    if n < 1:
        raise ValueError("mass_bound_check needs at least one token")
    sc = 1.0 / math.sqrt(keys.shape[1])
    lp = keys @ np.asarray(q_p, dtype=np.float64) * sc
    lm = keys @ np.asarray(q_m, dtype=np.float64) * sc
    wp = np.exp(lp - lp.max())
    wm = np.exp(lm - lm.max())
    zp, zm = wp.sum(), wm.sum()
    cut = max(0, n - band)
    if cut == 0:
        return 0.0, 0.0
    rho = float(wp[cut:].sum() / zp)
    drift = (wp[:cut] / zp - wm[:cut] / zm) @ values[:cut]
    lhs = float(np.sqrt(drift @ drift))
    dl = float(np.max(np.abs(lm[:cut] - lp[:cut])))
    pre = float(wp[:cut].sum())
    ev = float(wp[:cut] @ np.sqrt((values[:cut] ** 2).sum(axis=1))) / pre if pre > 0 else 0.0
    return lhs, math.expm1(dl) * (1.0 - rho) * ev


def oracle_outputs(q_pre, k_pre, v, cfg: OracleConfig, chunk: int = 256) -> np.ndarray:
    """Exact causal attention for every (layer, step, q head) (engine.py:542-572).

    q_pre (L, n_layers, Hq, d), k_pre (L, n_layers, Hkv, d), v (L, n_layers, Hkv, d_v).
    """
    freqs = rope_freqs(cfg.d, cfg.rope_base)
    L = q_pre.shape[0]
    pos = np.arange(1, L + 1, dtype=np.float64)
    scale = 1.0 / math.sqrt(cfg.d)
    out = np.empty((cfg.n_layers, L, cfg.n_q_heads, cfg.d_v))
    g = cfg.n_q_heads // cfg.n_kv_heads
    for layer in range(cfg.n_layers):
        for j in range(cfg.n_kv_heads):
            k_rot = round_storage(rope_rotate(k_pre[:, layer, j], pos, freqs), cfg.storage)
            v_all = round_storage(v[:, layer, j], cfg.storage)
            for h in range(j * g, (j + 1) * g):
                q_rot = rope_rotate(q_pre[:, layer, h], pos, freqs)
                for lo in range(0, L, chunk):
                    hi = min(lo + chunk, L)
                    lg = (q_rot[lo:hi] @ k_rot[:hi].T) * scale
                    cols = np.arange(hi)
                    lg[cols[None, :] > (lo + np.arange(hi - lo))[:, None]] = -np.inf
                    lg -= lg.max(axis=1, keepdims=True)
                    w = np.exp(lg)
                    out[layer, lo:hi, h] = (w @ v_all[:hi]) / w.sum(axis=1, keepdims=True)
    return out
