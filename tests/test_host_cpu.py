"""CPU-only checks: configuration/metrics parity with the reference, trace I/O,
and the C-ABI library surface (it loads and exports every declared symbol)."""

import math
import os
import sys
import re

import numpy as np
import pytest

from conftest import ROOT
from paper_2604_00235_b200 import (
    ByteCostModel,
    DecodeMetrics,
    EngineConfig,
    MatchConfig,
    MatchResult,
    SyntheticSpec,
    TraceError,
    aux_overhead_ratio,
    aux_overhead_rule_of_thumb,
    break_even_gate,
    compute_metrics,
    gen_synthetic,
    group_kv_span,
    read_trace,
    threshold,
    write_trace,
)


def hit_at(p):
    return MatchResult(hit=True, p=p, sq_dist=0.0, candidates_scanned=1)


MISS = MatchResult(hit=False, p=-1, sq_dist=math.inf, candidates_scanned=0)


def test_threshold_formula():
    assert threshold(128, 0.45) ** 2 == pytest.approx(2 * 128 * 0.55 ** 2)
    assert threshold(2, 0.5) == pytest.approx(1.0)
    with pytest.raises(ValueError):
        threshold(4, 1.0)


def test_break_even_and_group_span():
    unit = ByteCostModel(b_kv=1.0, b_q=1.0)
    assert break_even_gate(1280, 256, 1024, unit) and not break_even_gate(1279, 256, 1024, unit)
    assert group_kv_span([hit_at(1000), hit_at(1500)], 2000, 256) == 1256
    assert group_kv_span([hit_at(1000), MISS], 2000, 256) == 2000
    assert group_kv_span([hit_at(100)], 2000, 256) == 2000
    with pytest.raises(ValueError):
        group_kv_span([], 10, 2)


def test_aux_overhead():
    cfg = EngineConfig(d=64, d_v=64, n_q_heads=8, n_kv_heads=8, window=1024)
    want = 1024 * 8 * (64 + 64 + 2) / (120_000 * 8 * 2 * 64)
    assert aux_overhead_ratio(cfg, 120_000) == pytest.approx(want, rel=1e-15)
    assert aux_overhead_rule_of_thumb(1024, 120_000) == pytest.approx(0.05)


def test_engine_config_validation():
    EngineConfig(d=2, d_v=1)
    EngineConfig(d=128, d_v=128, storage="bf16")
    for bad in (dict(d=3, d_v=1), dict(d=4, d_v=0), dict(d=4, d_v=4, n_q_heads=3, n_kv_heads=2),
                dict(d=4, d_v=4, window=0), dict(d=4, d_v=4, band=-1), dict(d=4, d_v=4, tau=1.0),
                dict(d=4, d_v=4, n_layers=2, tau_per_layer=(0.4,)), dict(d=4, d_v=4, storage="f16"),
                dict(d=4, d_v=4, downdate_mode="subtract"), dict(d=4, d_v=4, refresh_every=-1)):
        with pytest.raises(ValueError):
            EngineConfig(**bad)
    cfg = EngineConfig(d=4, d_v=4, n_layers=2, tau_per_layer=(0.3, 0.6))
    assert cfg.tau_for(0) == 0.3 and cfg.tau_for(1) == 0.6
    with pytest.raises(ValueError):
        MatchConfig(d=4, tau=1.0)


def test_metrics_algebra():
    m = DecodeMetrics()
    assert m.record_hit(2000, 1000, 256) == 1256
    for _ in range(3):
        m.record_miss(2000)
    got = compute_metrics(m)
    assert got["acceptance_rate"] == 0.25
    assert got["kv_fraction"] == pytest.approx((1256 + 6000) / 8000)
    assert got["mean_gap"] == 1000.0
    with pytest.raises(ValueError):
        compute_metrics(DecodeMetrics())


def test_trace_roundtrip_and_errors(tmp_path):
    tr = gen_synthetic(SyntheticSpec(seq_len=20, d=8, d_v=4, n_layers=2, n_q_heads=4, n_kv_heads=2))
    write_trace(tr, str(tmp_path / "t"))
    back = read_trace(str(tmp_path / "t"))
    for a, b in ((tr.q_pre, back.q_pre), (tr.k_pre, back.k_pre), (tr.v, back.v)):
        np.testing.assert_array_equal(a, b)
    with pytest.raises(TraceError):
        read_trace(str(tmp_path / "missing"))
    with open(tmp_path / "t" / "v.bin", "wb") as fh:
        fh.write(b"\0" * 12)
    with pytest.raises(TraceError):
        read_trace(str(tmp_path / "t"))


def test_synthetic_spec_validation():
    with pytest.raises(ValueError):
        SyntheticSpec(seq_len=0)
    with pytest.raises(ValueError):
        SyntheticSpec(seq_len=4, d=3)
    tr = gen_synthetic(SyntheticSpec(seq_len=50, d=16, d_v=8))
    np.testing.assert_allclose(np.linalg.norm(tr.q_pre.astype(np.float64), axis=-1), 4.0, rtol=1e-6)


def _declared_functions():
    with open(os.path.join(ROOT, "include", "macattn.h")) as fh:
        src = fh.read()
    return re.findall(r"^\w[\w\s\*]*?\b(mac_\w+)\s*\(", src, flags=re.M)


def test_library_exports_every_declared_symbol():
    from paper_2604_00235_b200 import _lib

    lib = _lib.load()  # raises if missing or ABI/layout mismatched
    declared = _declared_functions()
    assert set(declared) == set(_lib.EXPORTS)
    for name in declared:
        assert hasattr(lib, name), name
    import ctypes

    assert lib.mac_params_size() == ctypes.sizeof(_lib.MacDecodeParams)
    assert lib.mac_error_string(1002).decode().startswith("macattn")


def test_library_rejects_bad_params_without_gpu():
    """Validation happens before any launch, so it is testable on a CPU box."""
    from paper_2604_00235_b200 import _lib

    lib = _lib.load()
    p = _lib.MacDecodeParams()
    assert lib.mac_decode_step(p, None) == 1002  # zero batch -> shape error
    p.batch, p.n_q_heads, p.n_kv_heads, p.head_dim, p.head_dim_v = 1, 4, 2, 8, 8
    p.window, p.band, p.max_chunks, p.min_chunk, p.page_size, p.pages_per_seq = 4, 1, 1, 16, 16, 1
    assert lib.mac_decode_step(p, None) == 1001  # null pointers
    p.storage = 7
    assert lib.mac_decode_step(p, None) == 1003


def test_stat_fields_follow_the_header():
    from paper_2604_00235_b200 import _lib

    with open(os.path.join(ROOT, "include", "macattn.h")) as fh:
        src = fh.read()
    stat = dict((k, int(v)) for k, v in re.findall(r"MAC_STAT_(\w+)\s*=\s*(\d+)", src))
    gstat = dict((k, int(v)) for k, v in re.findall(r"MAC_GSTAT_(\w+)\s*=\s*(\d+)", src))
    assert stat.pop("COUNT") == len(_lib.STAT_FIELDS) and sorted(stat.values()) == list(range(len(stat)))
    assert gstat.pop("COUNT") == len(_lib.GSTAT_FIELDS)
    names = {"STEPS": "steps", "HITS": "hits", "FORCED": "forced_misses", "FALLBACKS": "fallbacks",
             "SKIP_SUM": "skip_sum", "KV_READ": "kv_tokens_read", "KV_FULL": "kv_tokens_full",
             "GAP_SUM": "gap_sum", "RHO_SUM": "band_mass_sum", "CANDIDATES": "match_candidates"}
    for k, i in stat.items():
        assert _lib.STAT_FIELDS[i] == names[k]


def test_diagnostic_entry_points_validate_without_gpu():
    import ctypes

    from paper_2604_00235_b200 import _lib

    lib = _lib.load()
    p = _lib.MacDecodeParams()
    assert lib.mac_step_stats(p, None, None, None) == 1001
    buf = (ctypes.c_double * 64)()
    assert lib.mac_step_stats(p, buf, buf, None) == 1002  # zero batch
    p.batch, p.n_q_heads, p.n_kv_heads = 1, 4, 2
    assert lib.mac_step_stats(p, buf, buf, None) == 1001  # decision buffers missing
    mb = _lib.MacMassBoundParams()
    p.head_dim, p.head_dim_v, p.page_size, p.pages_per_seq = 8, 8, 16, 1
    assert lib.mac_mass_bound(p, mb, None) == 1001  # no cache
    p.head_dim = 512
    assert lib.mac_mass_bound(p, mb, None) == 1002  # d > 256


def test_io_entry_points_validate_without_gpu():
    """mac_io_copy / mac_host_alias (StepGraph's zero-copy I/O) reject bad arguments before any
    launch; the planar ring width of the Python mirror follows the header."""
    import ctypes

    from paper_2604_00235_b200 import _lib

    lib = _lib.load()
    out = ctypes.c_void_p()
    assert lib.mac_host_alias(None, ctypes.byref(out)) == 1001
    buf = (ctypes.c_uint8 * 64)()
    base = ctypes.addressof(buf)
    aligned = base + (-base) % 16
    assert lib.mac_io_copy(None, _lib.DT_F32, aligned, _lib.DT_F32, 4, None) == 1001
    assert lib.mac_io_copy(aligned + 4, _lib.DT_F32, aligned, _lib.DT_F32, 4, None) == 1002  # misaligned
    assert lib.mac_io_copy(aligned, _lib.DT_F32, aligned, _lib.DT_F32, 3, None) == 1002  # 12 bytes
    assert lib.mac_io_copy(aligned, _lib.DT_F64, aligned, _lib.DT_BF16, 8, None) == 1003  # no f64 -> bf16
    with open(os.path.join(ROOT, "include", "macattn.h")) as fh:
        src = fh.read()
    assert int(re.search(r"#define MAC_PLANAR_DIMS (\d+)", src).group(1)) == _lib.PLANAR_DIMS
    assert int(re.search(r"#define MACATTN_ABI_VERSION (\d+)", src).group(1)) == _lib.ABI_VERSION


def test_ncu_traffic_summary_matches_committed_capture():
    """profiles/r02/ncu_traffic.json (the bench's roofline.traffic) is what tools/ncu_traffic.py
    derives from the committed ncu capture of the decode step."""
    import json
    import subprocess
    import sys

    res = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_traffic.py"),
                          os.path.join(ROOT, "profiles", "r02", "ncu_kernels_c3.csv")],
                         capture_output=True, text=True, check=True)
    got = json.loads(res.stdout)
    with open(os.path.join(ROOT, "profiles", "r02", "ncu_traffic.json")) as fh:
        want = json.load(fh)
    for stage in ("mac_match_scan", "mac_match_verify", "mac_amend", "mac_complete"):
        assert got[stage]["traffic_bytes"] == want[stage]["traffic_bytes"], stage
        assert got[stage]["kernel"] == want[stage]["kernel"], stage
    # the dominant kernel moves at least its algorithmic bytes and no more than 10 % on top
    assert 87.1e6 <= want["mac_amend"]["traffic_bytes"] <= 1.1 * 87.1e6


def test_algorithmic_step_bytes_by_hand():
    """bench.step_bytes (the roofline's algorithmic bytes) on a case worked by hand:
    one request, 2 q heads sharing one kv head, d = 128, W = 64, r = 16, m = 100, both heads hit
    (p = 90 and 80) -> the group reads [min(75, 65), 100] = 36 tokens of K and V."""
    import numpy as np

    sys.path.insert(0, ROOT)
    import bench
    from paper_2604_00235_b200._lib import PLANAR_DIMS as P

    use = np.array([[1, 1]])
    pos = np.array([[90, 80]])
    b = bench.step_bytes(use, pos, np.array([100]), hq=2, hkv=1, d=128, window=64, band=16)
    assert b["amend"] == 36 * 2 * 128 * 2
    assert b["match"] == 2 * (64 * P * 2 + 64 * 4 + 1 * 16 + 128 * 2)
    assert b["verify"] == 2 * (1 * 16 + 2 * (128 - P) * 2 + 128 * 2)
    assert b["complete"] == 2 * (128 * 4 + 4) + 2 * (128 * 2 + P * 2 + 128 * 4 + 4) + 2 * 128 * 4
    assert b["append"] == 1 * 2 * 128 * 2
    assert b["total"] == sum(b[k] for k in ("match", "verify", "amend", "complete", "append"))
    # a miss reads the group's whole context
    b2 = bench.step_bytes(np.array([[0, 1]]), pos, np.array([100]), hq=2, hkv=1, d=128, window=64, band=16)
    assert b2["amend"] == 100 * 2 * 128 * 2


def test_public_names_cover_reference(golden_dir):
    """Every public name of the reference package (attnreuse/__init__.py:3-65, recorded by
    tests/golden/make_api_list.py) except the out-of-scope scheduler / calibration is exported,
    and each resolves (the device modules import lazily; nothing here launches)."""
    import json

    import paper_2604_00235_b200 as pkg

    with open(os.path.join(golden_dir, "reference_api.json")) as fh:
        ref = json.load(fh)
    want = set(ref["reference_all"]) - set(ref["out_of_scope"])
    assert not want - set(pkg.__all__), sorted(want - set(pkg.__all__))
    for name in pkg.__all__:
        assert getattr(pkg, name) is not None, name


def test_new_entry_points_validate_without_gpu():
    """mac_summarize / mac_match_rows / mac_remove_summaries / mac_rope_rotate reject bad
    parameter sets before any launch."""
    import ctypes

    from paper_2604_00235_b200 import _lib

    lib = _lib.load()
    s = _lib.MacSummarizeParams()
    assert lib.mac_summarize(s, None) == 1001
    buf = (ctypes.c_double * 16)()
    a = ctypes.addressof(buf)
    s.q = s.keys = s.values = s.out_acc = s.out_lse = a
    assert lib.mac_summarize(s, None) == 1002  # sets_per_kv 0, head_dim 0
    s.sets_per_kv, s.head_dim, s.head_dim_v, s.dtype = 1, 4, 4, 5
    assert lib.mac_summarize(s, None) == 0  # zero rows: nothing to launch
    s.n_sets = s.q_per_set = 1
    assert lib.mac_summarize(s, None) == 1003  # unknown dtype
    s.rope_t = a
    assert lib.mac_summarize(s, None) == 1001  # rotation without frequencies
    m = _lib.MacMatchRowsParams()
    assert lib.mac_match_rows(m, None) == 1001
    assert lib.mac_remove_summaries(1, 4, None, a, a, a, 1e-6, a, a, a, None) == 1001
    assert lib.mac_rope_rotate(1, 3, a, a, a, a, None) == 1002


def test_split_defaults_and_span_chunks_field():
    """The engine's split-KV defaults (engine.py default_max_chunks / default_slot_cap) and the ABI
    13 span_chunks field: the slot capacity never falls below the full-span split, grows with the
    context up to 64, and the ctypes mirror carries the field where the header declares it."""
    from paper_2604_00235_b200 import _lib
    from paper_2604_00235_b200.engine import default_max_chunks, default_slot_cap

    mc = default_max_chunks(32, 8, 16384 + 64)  # C3 geometry at 16K: 8 splits of a full span
    assert mc == 8
    assert default_slot_cap(mc, 16384 + 64) == 33  # ~512-token items for a missing group
    assert default_slot_cap(17, 131072) == 64  # capped
    assert default_slot_cap(222, 524288) == 222  # never below the span split (C4)
    for n in (64, 1024, 8192, 65536):
        assert default_slot_cap(default_max_chunks(4, 8, n), n) >= default_max_chunks(4, 8, n)
    names = [f[0] for f in _lib.MacDecodeParams._fields_]
    assert names.index("span_chunks") == names.index("n_shards") + 1
    with open(os.path.join(ROOT, "include", "macattn.h")) as fh:
        hdr = fh.read()
    assert re.search(r"int32_t n_shards;.*\n\s*int32_t span_chunks;", hdr)


def test_adaptive_scan_policy():
    """BatchDecodeEngine._choose_match_mode on the published {missed, heads} feedback: the plain
    two-pass scan while at most one head missed in the window, dense mode up to DENSE_MAX_MISS
    where the geometry has it (else the one-pass scan), the one-pass scan above; pinned modes win."""
    import torch

    from paper_2604_00235_b200 import BatchDecodeEngine

    def mode(missed, heads, dense=True, pin="adaptive"):
        e = object.__new__(BatchDecodeEngine)
        e.match_mode = pin
        e._fb_host = torch.tensor([missed, heads], dtype=torch.int32)
        e._dense_cap = dense
        e._choose_match_mode()
        return e._step_mode

    H = 8 * 1024
    assert mode(0, H) == 0 and mode(1, H) == 0
    assert mode(2, H) == 2 and mode(int(0.2 * H), H) == 2
    assert mode(2, H, dense=False) == 1
    assert mode(int(0.3 * H), H) == 1
    assert mode(0, H, pin="one_pass") == 1 and mode(H, H, pin="two_pass") == 0 and mode(0, H, pin="dense") == 2
