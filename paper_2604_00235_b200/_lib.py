"""ctypes binding of the C-ABI library lib/libmacattn.so (include/macattn.h).

This is the ONLY way the product reaches compute: there is no CPU or
PyTorch fallback.  A missing or stale library raises immediately.
"""

from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# MACATTN_LIB points at an alternative build of the same library (e.g. a tracing build)
LIB_PATH = os.environ.get("MACATTN_LIB") or os.path.join(_HERE, "lib", "libmacattn.so")

ABI_VERSION = 14
PLANAR_DIMS = 8  # MAC_PLANAR_DIMS: dims of the planar query-ring copy (ring_qp)

MODE_F32, MODE_BF16, MODE_F64 = 0, 1, 2
DT_F32, DT_BF16, DT_F64 = 0, 1, 2
MATCH_PRE_ROPE, MATCH_POST_ROPE = 0, 1
DOWNDATE_SPLIT, DOWNDATE_REMOVE = 0, 1
PATH_TWO_PASS, PATH_VERIFY_GROUP, PATH_VERIFY_HEAD, PATH_AMEND_MMA, PATH_DENSE_KERNEL, PATH_AMEND_TMA = 1, 2, 4, 8, 16, 32

EXPORTS = (
    "mac_abi_version",
    "mac_params_size",
    "mac_error_string",
    "mac_workspace_bytes",
    "mac_overflow_flag_offset",
    "mac_amend_variant",
    "mac_match_path",
    "mac_append_kv",
    "mac_match",
    "mac_match_scan",
    "mac_match_verify",
    "mac_amend",
    "mac_complete",
    "mac_decode_step",
    "mac_full_decode",
    "mac_attend_full",
    "mac_merge_partials",
    "mac_shard_partial",
    "mac_shard_complete",
    "mac_prefill_kv",
    "mac_step_stats",
    "mac_mass_bound",
    "mac_host_alias",
    "mac_io_copy",
    "mac_summarize",
    "mac_remove_summaries",
    "mac_rope_rotate",
    "mac_match_rows",
    "mac_build_ring",
)

# per-head / per-group statistics fields of mac_step_stats (include/macattn.h)
STAT_FIELDS = ("steps", "hits", "forced_misses", "fallbacks", "skip_sum", "kv_tokens_read",
               "kv_tokens_full", "gap_sum", "band_mass_sum", "match_candidates")
GSTAT_FIELDS = ("group_kv_tokens", "group_kv_total")


class MacDecodeParams(C.Structure):
    _fields_ = [
        ("batch", C.c_int32),
        ("n_q_heads", C.c_int32),
        ("n_kv_heads", C.c_int32),
        ("head_dim", C.c_int32),
        ("head_dim_v", C.c_int32),
        ("window", C.c_int32),
        ("band", C.c_int32),
        ("page_size", C.c_int32),
        ("pages_per_seq", C.c_int32),
        ("storage", C.c_int32),
        ("in_dtype", C.c_int32),
        ("max_chunks", C.c_int32),
        ("min_chunk", C.c_int32),
        ("kv_offset", C.c_int32),
        ("kv_limit", C.c_int32),
        ("n_shards", C.c_int32),
        ("span_chunks", C.c_int32),
        ("thr_sq", C.c_double),
        ("delta_max", C.c_int32),
        ("match_space", C.c_int32),
        ("refresh_every", C.c_int32),
        ("roi_gate", C.c_int32),
        ("roi_b_kv", C.c_double),
        ("roi_b_q", C.c_double),
        ("downdate", C.c_int32),
        ("force_miss", C.c_int32),
        ("eps_cancel", C.c_double),
        ("seq_lens", C.c_void_p),
        ("page_table", C.c_void_p),
        ("k_cache", C.c_void_p),
        ("v_cache", C.c_void_p),
        ("ring_q", C.c_void_p),
        ("ring_acc", C.c_void_p),
        ("ring_lse", C.c_void_p),
        ("ring_qp", C.c_void_p),
        ("rope_freqs", C.c_void_p),
        ("q_pre", C.c_void_p),
        ("k_pre", C.c_void_p),
        ("v_in", C.c_void_p),
        ("out", C.c_void_p),
        ("match_hit", C.c_void_p),
        ("use_hit", C.c_void_p),
        ("match_pos", C.c_void_p),
        ("match_dist", C.c_void_p),
        ("match_scanned", C.c_void_p),
        ("full_lse", C.c_void_p),
        ("band_mass", C.c_void_p),
        ("cached_acc", C.c_void_p),
        ("cached_lse", C.c_void_p),
        ("fallbacks", C.c_void_p),
        ("out_bf16", C.c_void_p),
        ("shard_out", C.c_void_p),
        ("shard_parts", C.c_void_p),
        ("workspace", C.c_void_p),
        ("workspace_bytes", C.c_size_t),
        ("match_mode", C.c_int32),
        ("feedback", C.c_void_p),
        ("inputs_host", C.c_int32),
    ]


class MacMergeParams(C.Structure):
    _fields_ = [
        ("n_parts", C.c_int32),
        ("n_rows", C.c_int32),
        ("head_dim_v", C.c_int32),
        ("dtype", C.c_int32),
        ("part_acc", C.c_void_p),
        ("part_lse", C.c_void_p),
        ("out_acc", C.c_void_p),
        ("out_lse", C.c_void_p),
    ]


class MacMassBoundParams(C.Structure):
    _fields_ = [
        ("n_items", C.c_int32),
        ("band", C.c_int32),
        ("rotate", C.c_int32),
        ("item_req", C.c_void_p),
        ("item_kv_head", C.c_void_p),
        ("item_m", C.c_void_p),
        ("item_p", C.c_void_p),
        ("q_m", C.c_void_p),
        ("q_p", C.c_void_p),
        ("out", C.c_void_p),
    ]


class MacSummarizeParams(C.Structure):
    _fields_ = [
        ("n_sets", C.c_int32),
        ("q_per_set", C.c_int32),
        ("n_keys", C.c_int32),
        ("sets_per_kv", C.c_int32),
        ("head_dim", C.c_int32),
        ("head_dim_v", C.c_int32),
        ("dtype", C.c_int32),
        ("q", C.c_void_p),
        ("keys", C.c_void_p),
        ("values", C.c_void_p),
        ("lo", C.c_void_p),
        ("hi", C.c_void_p),
        ("rope_t", C.c_void_p),
        ("rope_freqs", C.c_void_p),
        ("out_acc", C.c_void_p),
        ("out_lse", C.c_void_p),
    ]


class MacMatchRowsParams(C.Structure):
    _fields_ = [
        ("n_rings", C.c_int32),
        ("capacity", C.c_int32),
        ("head_dim", C.c_int32),
        ("delta_max", C.c_int32),
        ("post_rope", C.c_int32),
        ("thr_sq", C.c_double),
        ("rope_freqs", C.c_void_p),
        ("q", C.c_void_p),
        ("ring_q", C.c_void_p),
        ("ring_sqnorm", C.c_void_p),
        ("ring_pos", C.c_void_p),
        ("n_live", C.c_void_p),
        ("m", C.c_void_p),
        ("out_hit", C.c_void_p),
        ("out_pos", C.c_void_p),
        ("out_dist", C.c_void_p),
        ("out_scanned", C.c_void_p),
    ]


class MacRingBuildParams(C.Structure):
    _fields_ = [("n_rows", C.c_int32), ("n_chunks", C.c_int32), ("part", C.c_void_p), ("variant", C.c_int32)]


_lib = None


def load() -> C.CDLL:
    """Load and check the library once; raise loudly if it is absent or mismatched."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(
            f"macattn CUDA library not found at {LIB_PATH}; build it with "
            "`python -m paper_2604_00235_b200.build` (there is no CPU fallback)"
        )
    lib = C.CDLL(LIB_PATH)
    for name in EXPORTS:
        if not hasattr(lib, name):
            raise RuntimeError(f"{LIB_PATH} does not export {name}")
    lib.mac_abi_version.restype = C.c_int
    lib.mac_params_size.restype = C.c_size_t
    lib.mac_error_string.restype = C.c_char_p
    lib.mac_error_string.argtypes = [C.c_int]
    lib.mac_workspace_bytes.restype = C.c_size_t
    lib.mac_workspace_bytes.argtypes = [C.POINTER(MacDecodeParams)]
    lib.mac_overflow_flag_offset.restype = C.c_size_t
    lib.mac_overflow_flag_offset.argtypes = [C.POINTER(MacDecodeParams)]
    lib.mac_amend_variant.restype = C.c_int
    lib.mac_amend_variant.argtypes = [C.POINTER(MacDecodeParams)]
    lib.mac_match_path.restype = C.c_int
    lib.mac_match_path.argtypes = [C.POINTER(MacDecodeParams)]
    for name in ("mac_append_kv", "mac_match", "mac_match_scan", "mac_match_verify", "mac_amend", "mac_complete", "mac_decode_step", "mac_full_decode",
                 "mac_attend_full", "mac_shard_partial", "mac_shard_complete"):
        fn = getattr(lib, name)
        fn.restype = C.c_int
        fn.argtypes = [C.POINTER(MacDecodeParams), C.c_void_p]
    lib.mac_prefill_kv.restype = C.c_int
    lib.mac_prefill_kv.argtypes = [C.POINTER(MacDecodeParams), C.c_int32, C.c_void_p]
    lib.mac_step_stats.restype = C.c_int
    lib.mac_step_stats.argtypes = [C.POINTER(MacDecodeParams), C.c_void_p, C.c_void_p, C.c_void_p]
    lib.mac_mass_bound.restype = C.c_int
    lib.mac_mass_bound.argtypes = [C.POINTER(MacDecodeParams), C.POINTER(MacMassBoundParams), C.c_void_p]
    lib.mac_host_alias.restype = C.c_int
    lib.mac_host_alias.argtypes = [C.c_void_p, C.POINTER(C.c_void_p)]
    lib.mac_io_copy.restype = C.c_int
    lib.mac_io_copy.argtypes = [C.c_void_p, C.c_int32, C.c_void_p, C.c_int32, C.c_size_t, C.c_void_p]
    lib.mac_merge_partials.restype = C.c_int
    lib.mac_merge_partials.argtypes = [C.POINTER(MacMergeParams), C.c_void_p]
    lib.mac_summarize.restype = C.c_int
    lib.mac_summarize.argtypes = [C.POINTER(MacSummarizeParams), C.c_void_p]
    lib.mac_match_rows.restype = C.c_int
    lib.mac_match_rows.argtypes = [C.POINTER(MacMatchRowsParams), C.c_void_p]
    lib.mac_remove_summaries.restype = C.c_int
    lib.mac_remove_summaries.argtypes = [C.c_int32, C.c_int32] + [C.c_void_p] * 4 + [C.c_double] + [C.c_void_p] * 4
    lib.mac_rope_rotate.restype = C.c_int
    lib.mac_rope_rotate.argtypes = [C.c_int32, C.c_int32] + [C.c_void_p] * 5
    lib.mac_build_ring.restype = C.c_int
    lib.mac_build_ring.argtypes = [C.POINTER(MacDecodeParams), C.POINTER(MacRingBuildParams), C.c_void_p]
    if lib.mac_abi_version() != ABI_VERSION:
        raise RuntimeError(f"libmacattn ABI {lib.mac_abi_version()} != expected {ABI_VERSION}; rebuild")
    if lib.mac_params_size() != C.sizeof(MacDecodeParams):
        raise RuntimeError("libmacattn MacDecodeParams layout differs from the ctypes mirror; rebuild")
    _lib = lib
    return lib


def check(code: int, what: str):
    if code != 0:
        msg = load().mac_error_string(code).decode()
        raise RuntimeError(f"{what} failed ({code}): {msg}")


def call(name: str, params, stream_handle: int):
    lib = load()
    code = getattr(lib, name)(C.byref(params), C.c_void_p(stream_handle))
    check(code, name)
