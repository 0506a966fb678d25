"""B200-native MAC-Attention decode path (match -> amend -> complete, full-attention fallback).

Drop-in for the decode path of the reference package `attnreuse`: the same
public names for the engine, its configuration and result types, the metrics
and the trace format, backed by hand-written sm_100a CUDA kernels behind the
C-ABI library `lib/libmacattn.so` (include/macattn.h).  There is no CPU path:
decode calls fail loudly when the library or a CUDA device is missing.
"""

from .config import (
    DOWNDATE_REMOVE,
    DOWNDATE_SPLIT,
    MATCH_POST_ROPE,
    MATCH_PRE_ROPE,
    AttentionSummary,
    ByteCostModel,
    CancellationError,
    DecodeMetrics,
    EmptySummaryError,
    EngineConfig,
    MassExceededError,
    MatchConfig,
    MatchResult,
    StepResult,
    aux_overhead_ratio,
    aux_overhead_rule_of_thumb,
    break_even_gate,
    compute_metrics,
    empty_summary,
    fidelity_efficiency,
    finalize,
    group_kv_span,
    threshold,
)
from .workload import PRESETS, SyntheticSpec, Trace, TraceError, gen_synthetic, read_trace, write_trace

__version__ = "0.1.0"


_LAZY = {
    # the device modules import torch; load them on first use
    "engine": ("BatchDecodeEngine", "BatchStepResult", "DecodeEngine", "StepGraph", "run_decode", "oracle_outputs",
               "KvStoreView", "QueryRingView", "SummaryRingView", "rope_freqs", "mass_bound_check"),
    "summary": ("RopeTable", "attend_full", "avg_cos", "merge", "remove", "rope_rotate", "summarize",
                "summarize_rows", "rope_rotate_rows"),
    "rings": ("QueryRing", "SummaryRing", "match_query", "match_queries"),
    "store": ("KvPage", "KvStore", "TrafficCounter"),
}


def __getattr__(name):
    import importlib

    for mod, names in _LAZY.items():
        if name in names:
            return getattr(importlib.import_module(f".{mod}", __name__), name)
    raise AttributeError(name)


# the reference's public names on the decode path (attnreuse/__init__.py:3-65) minus the
# out-of-scope offline scheduler (sched.py) and tau calibration (calibrate_tau, chi2_cdf),
# plus this package's batched device API
__all__ = [
    "KvPage", "KvStore", "QueryRing", "RopeTable", "SummaryRing", "attend_full", "avg_cos", "match_queries",
    "match_query", "merge", "oracle_outputs", "remove", "rope_rotate", "summarize",
    "AttentionSummary", "BatchDecodeEngine", "BatchStepResult", "ByteCostModel", "CancellationError",
    "DOWNDATE_REMOVE", "DOWNDATE_SPLIT", "DecodeEngine", "DecodeMetrics", "EmptySummaryError", "EngineConfig",
    "MATCH_POST_ROPE", "MATCH_PRE_ROPE", "MassExceededError", "MatchConfig", "MatchResult", "PRESETS",
    "StepGraph", "StepResult", "SyntheticSpec", "Trace", "TraceError", "TrafficCounter", "aux_overhead_ratio",
    "aux_overhead_rule_of_thumb", "break_even_gate", "compute_metrics", "empty_summary", "fidelity_efficiency",
    "finalize", "gen_synthetic", "group_kv_span", "mass_bound_check", "read_trace", "run_decode", "threshold", "write_trace",
]
