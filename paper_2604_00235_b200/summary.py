"""Summary algebra and rotary embedding of the reference, on the device.

The reference's public building blocks (attention.py): `summarize`, `merge`,
`remove`, `finalize`, `attend_full`, `RopeTable`, `rope_rotate`, `avg_cos` —
same names, signatures, return types and exceptions, so a caller can switch
imports.  The attention math runs in the CUDA library (csrc/summary.cu,
csrc/merge.cu) in f64 like the reference; inputs are host arrays (as in the
reference) and results come back as host arrays.  Batched forms that keep
device tensors (`summarize_rows`) serve the device oracle (`oracle_outputs`).
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .config import (AttentionSummary, CancellationError, EmptySummaryError, MassExceededError, empty_summary,
                     finalize)

__all__ = [
    "AttentionSummary", "CancellationError", "EmptySummaryError", "MassExceededError", "RopeTable",
    "attend_full", "avg_cos", "empty_summary", "finalize", "merge", "remove", "rope_rotate", "rope_rotate_rows",
    "summarize", "summarize_rows",
]


def _device(device=None) -> torch.device:
    if device is not None:
        return torch.device(device)
    if not torch.cuda.is_available():
        raise RuntimeError("the summary algebra runs on the CUDA library: no CUDA device is visible")
    return torch.device("cuda", torch.cuda.current_device())


def _stream(dev: torch.device) -> int:
    return torch.cuda.current_stream(dev).cuda_stream


def _f64(x, dev) -> torch.Tensor:
    return torch.from_numpy(np.array(x, dtype=np.float64, order="C")).to(dev)  # a writable host copy


def _ptr(t) -> int | None:
    return None if t is None else t.data_ptr()


def summarize_rows(q: torch.Tensor, keys: torch.Tensor, values: torch.Tensor, *, lo=None, hi=None, rope_t=None,
                   rope_freqs=None, sets_per_kv: int = 1) -> tuple[torch.Tensor, torch.Tensor]:
    """Batched summarize on device tensors (mac_summarize): q [S, n_q, d], keys [S/g, n, d],
    values [S/g, n, d_v] (f32 or f64, same dtype), optional per-row key ranges lo / hi
    (int32 [S, n_q], 1-based inclusive) and per-row RoPE positions rope_t for q.  Returns
    (acc [S, n_q, d_v], lse [S, n_q]) in f64; an empty range gives (0, -inf)."""
    S, nq, d = q.shape
    dv = values.shape[-1]
    dt = {torch.float64: _lib.DT_F64, torch.float32: _lib.DT_F32}[q.dtype]
    if keys.dtype != q.dtype or values.dtype != q.dtype:
        raise ValueError("q, keys and values must share one dtype")
    dev = q.device
    acc = torch.empty((S, nq, dv), dtype=torch.float64, device=dev)
    lse = torch.empty((S, nq), dtype=torch.float64, device=dev)
    q, keys, values = q.contiguous(), keys.contiguous(), values.contiguous()
    cvt = lambda t: None if t is None else t.to(dev, torch.int32).contiguous()
    lo, hi, rope_t = cvt(lo), cvt(hi), cvt(rope_t)
    P = _lib.MacSummarizeParams(n_sets=S, q_per_set=nq, n_keys=keys.shape[1], sets_per_kv=sets_per_kv, head_dim=d,
                                head_dim_v=dv, dtype=dt, q=q.data_ptr(), keys=keys.data_ptr(),
                                values=values.data_ptr(), lo=_ptr(lo), hi=_ptr(hi), rope_t=_ptr(rope_t),
                                rope_freqs=_ptr(rope_freqs), out_acc=acc.data_ptr(), out_lse=lse.data_ptr())
    _lib.check(_lib.load().mac_summarize(C.byref(P), C.c_void_p(_stream(dev))), "mac_summarize")
    return acc, lse


def summarize(q, keys, values, *, dtype=np.float64, block: int = 4096, device=None) -> AttentionSummary:
    """Summary of `keys`/`values` under query `q` (attention.py:75-116): acc = softmax-weighted
    value mean, lse = ln Z of the 1/sqrt(d)-scaled logits, count = rows.  f64 accumulation on
    the device; `dtype` is the storage dtype of the result.  `block` is accepted for signature
    compatibility (the kernel streams keys with an online softmax at any length)."""
    keys = np.asarray(keys)
    values = np.asarray(values)
    if keys.ndim != 2 or values.ndim != 2 or keys.shape[0] != values.shape[0]:
        raise ValueError("keys and values must be 2-D with matching row counts")
    n = keys.shape[0]
    if n == 0:
        return empty_summary(values.shape[1], dtype=dtype)
    dev = _device(device)
    q64 = np.asarray(q, dtype=np.float64)
    acc, lse = summarize_rows(_f64(q64, dev)[None, None], _f64(keys, dev)[None], _f64(values, dev)[None])
    s = AttentionSummary(acc=acc[0, 0].cpu().numpy(), lse=float(lse[0, 0].item()), count=n)
    return s if np.dtype(dtype) == np.float64 else s.astype(dtype)


def merge(a: AttentionSummary, b: AttentionSummary, *, device=None) -> AttentionSummary:
    """Summary of the union of two disjoint token sets (attention.py:119-135), through the
    library's log-domain merge (mac_merge_partials).  The empty summary is the identity."""
    if a.count == 0:
        return b
    if b.count == 0:
        return a
    out_dtype = np.result_type(a.acc, b.acc)
    dev = _device(device)
    acc = _f64(np.stack([a.acc, b.acc]), dev)
    lse = torch.tensor([a.lse, b.lse], dtype=torch.float64, device=dev)
    oacc = torch.empty(acc.shape[1], dtype=torch.float64, device=dev)
    olse = torch.empty(1, dtype=torch.float64, device=dev)
    P = _lib.MacMergeParams(n_parts=2, n_rows=1, head_dim_v=acc.shape[1], dtype=_lib.DT_F64,
                            part_acc=acc.data_ptr(), part_lse=lse.data_ptr(), out_acc=oacc.data_ptr(),
                            out_lse=olse.data_ptr())
    _lib.check(_lib.load().mac_merge_partials(C.byref(P), C.c_void_p(_stream(dev))), "mac_merge_partials")
    s = AttentionSummary(acc=oacc.cpu().numpy(), lse=float(olse.item()), count=a.count + b.count)
    return s if out_dtype == np.float64 else s.astype(out_dtype)


def remove(a: AttentionSummary, band: AttentionSummary, *, eps_cancel: float = 1e-6,
           device=None) -> AttentionSummary:
    """Down-date: the summary of a's tokens without `band`'s (attention.py:138-172).  Raises
    ValueError when the band covers more tokens than `a`, CancellationError when the residual
    log-mass is inside the guard, MassExceededError when the band outweighs `a`."""
    if band.count == 0:
        return a
    if band.count > a.count:
        raise ValueError("band covers more tokens than the summary it is removed from")
    if band.count == a.count:
        if band.lse == a.lse:
            return empty_summary(a.acc.shape[0], dtype=a.acc.dtype)
        raise CancellationError("count would reach zero but band mass differs from the whole")
    out_dtype = np.result_type(a.acc, band.acc)
    dev = _device(device)
    aa, ba = _f64(a.acc, dev), _f64(band.acc, dev)
    al = torch.tensor([a.lse], dtype=torch.float64, device=dev)
    bl = torch.tensor([band.lse], dtype=torch.float64, device=dev)
    oacc, olse = torch.empty_like(aa), torch.empty(1, dtype=torch.float64, device=dev)
    st = torch.empty(1, dtype=torch.int32, device=dev)
    code = _lib.load().mac_remove_summaries(1, aa.numel(), aa.data_ptr(), al.data_ptr(), ba.data_ptr(), bl.data_ptr(),
                                            eps_cancel, oacc.data_ptr(), olse.data_ptr(), st.data_ptr(),
                                            C.c_void_p(_stream(dev)))
    _lib.check(code, "mac_remove_summaries")
    status = int(st.item())
    diff = a.lse - band.lse
    if status == 2:
        raise MassExceededError("band mass exceeds the summary it is removed from")
    if status == 1:
        raise CancellationError(f"residual log-mass {diff:.3e} below cancellation guard {eps_cancel:.1e}")
    s = AttentionSummary(acc=oacc.cpu().numpy(), lse=float(olse.item()), count=a.count - band.count)
    return s if out_dtype == np.float64 else s.astype(out_dtype)


def attend_full(q, keys, values, *, device=None) -> tuple[np.ndarray, AttentionSummary]:
    """Exact attention of `q` over every row (attention.py:182-189): (output, summary)."""
    s = summarize(q, keys, values, device=device)
    return finalize(s), s


@dataclass(frozen=True)
class RopeTable:
    """Rotation frequencies freqs[j] = base**(-2j/d), j < d/2 (attention.py:195-209)."""

    d: int
    base: float = 10000.0
    freqs: np.ndarray = field(init=False, repr=False)

    def __post_init__(self):
        if self.d < 2 or self.d % 2 != 0:
            raise ValueError(f"rotary embedding needs an even head dim >= 2, got d={self.d}")
        if self.base <= 1.0:
            raise ValueError("rope base must exceed 1")
        j = np.arange(self.d // 2, dtype=np.float64)
        object.__setattr__(self, "freqs", self.base ** (-2.0 * j / self.d))


def rope_rotate(x, t, table: RopeTable, *, device=None) -> np.ndarray:
    """Rotate interleaved pairs (x[2j], x[2j+1]) by t * freqs[j] (attention.py:212-232) on the
    device with f64 angles.  x is (d,) or (..., d); t a scalar or per-row positions."""
    x = np.asarray(x, dtype=np.float64)
    if x.shape[-1] != table.d:
        raise ValueError(f"vector dim {x.shape[-1]} does not match table dim {table.d}")
    rows = x.reshape(-1, table.d)
    t = np.broadcast_to(np.asarray(t, dtype=np.float64), x.shape[:-1]).reshape(-1)
    if rows.shape[0] == 0:
        return x.copy()
    dev = _device(device)
    out = rope_rotate_rows(_f64(rows, dev), _f64(t, dev), _f64(table.freqs, dev))
    return out.cpu().numpy().reshape(x.shape)


def rope_rotate_rows(x: torch.Tensor, t: torch.Tensor, freqs: torch.Tensor) -> torch.Tensor:
    """Device form of rope_rotate: x [n, d] f64, t [n] f64 positions, freqs [d/2] f64."""
    x, t = x.contiguous(), t.to(torch.float64).contiguous()
    out = torch.empty_like(x)
    if x.shape[0]:
        code = _lib.load().mac_rope_rotate(x.shape[0], x.shape[1], x.data_ptr(), t.data_ptr(), freqs.data_ptr(),
                                           out.data_ptr(), C.c_void_p(_stream(x.device)))
        _lib.check(code, "mac_rope_rotate")
    return out


def avg_cos(x, delta, table: RopeTable) -> float:
    """Energy-weighted mean of cos(freqs[j] * delta) over the pair planes of x
    (attention.py:235-249): ||x - R(delta) x||^2 = 2 ||x||^2 (1 - avg_cos).  A host-side
    diagnostic of one vector, like `threshold`."""
    x = np.asarray(x, dtype=np.float64)
    if x.shape != (table.d,):
        raise ValueError(f"expected a single vector of dim {table.d}")
    w = (x.reshape(-1, 2) ** 2).sum(axis=1)
    total = float(w.sum())
    if total == 0.0:
        raise ValueError("avg_cos is undefined for the zero vector")
    return float(np.cos(table.freqs * float(delta)) @ w / total)
