"""Helpers shared by the oracle and GPU parity tests: load golden fixtures and
rebuild the exact inputs the reference saw (with this repo's trace generator)."""

from __future__ import annotations

import json
import os

import numpy as np

from conftest import GOLDEN
from paper_2604_00235_b200.workload import SyntheticSpec, gen_synthetic

SCENARIOS = ["gqa_f32", "gqa_f64", "bf16_matched", "independent", "post_rope", "gates", "roi", "remove",
             "small_window"]


def load(name: str) -> dict:
    z = np.load(os.path.join(GOLDEN, f"{name}.npz"), allow_pickle=False)
    return {k: z[k] for k in z.files}


def bf16_round(x) -> np.ndarray:
    f = np.ascontiguousarray(np.asarray(x, dtype=np.float32))
    u = f.view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32).astype(np.float64)


def scenario_inputs(rec: dict):
    """(spec_kw, cfg_kw, q, k, v) as float64 arrays (token, layer, head, dim)."""
    spec_kw = json.loads(str(rec["spec"]))
    cfg_kw = json.loads(str(rec["cfg"]))
    tr = gen_synthetic(SyntheticSpec(**spec_kw))
    q, k, v = (a.astype(np.float64) for a in (tr.q_pre, tr.k_pre, tr.v))
    if int(rec["storage_matched_bf16"]):
        q, k, v = bf16_round(q), bf16_round(k), bf16_round(v)
        cfg_kw = dict(cfg_kw, storage="bf16")
    if "tau_per_layer" in cfg_kw and cfg_kw["tau_per_layer"] is not None:
        cfg_kw["tau_per_layer"] = tuple(cfg_kw["tau_per_layer"])
    return spec_kw, cfg_kw, q, k, v, tr


def rel_err(a, b) -> float:
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    den = float(np.linalg.norm(b))
    num = float(np.linalg.norm(a - b))
    return 0.0 if num == 0.0 else num / den
