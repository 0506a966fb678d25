"""GPU: diagnostics beside the decode step.

* mac_mass_bound (mass_bound_check, engine.py:246-281) against the reference's
  own outputs (tests/golden/mass_bound.npz): direct cases, and every sample a
  reference decode run with oracle_mode + mass_check produced (engine.py:480-483);
* mac_step_stats (DecodeMetrics record_hit/record_miss, engine.py:188-205, and
  group_kv_span, engine.py:66-77) accumulated on the device, against the
  reference's metrics for the same scenario and against the shim's host fold.
"""

import json

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from golden_util import load, scenario_inputs  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_cuda():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")


def test_mass_bound_direct_cases():
    from paper_2604_00235_b200 import mass_bound_check

    z = load("mass_bound")
    for i in range(int(z["n_cases"])):
        got = mass_bound_check(z[f"c{i}__q_m"], z[f"c{i}__q_p"], z[f"c{i}__keys"], z[f"c{i}__values"],
                               int(z[f"c{i}__band"]))
        want = z[f"c{i}__out"]
        np.testing.assert_allclose(got, want, rtol=1e-10, atol=1e-15, err_msg=f"case {i}")
    # test_engine.py:369-382 edge behaviour
    rng = np.random.default_rng(11)
    keys, vals, q = rng.standard_normal((50, 8)), rng.standard_normal((50, 8)), rng.standard_normal(8)
    assert mass_bound_check(q, q, keys, vals, 8) == (0.0, 0.0)
    assert mass_bound_check(q, rng.standard_normal(8), keys, vals, 50) == (0.0, 0.0)
    for _ in range(20):
        lhs, rhs = mass_bound_check(q + 1e-3 * rng.standard_normal(8), q, keys, vals, 8)
        assert lhs <= rhs
    with pytest.raises(ValueError):
        mass_bound_check(q, q, np.zeros((0, 8)), np.zeros((0, 8)), 8)


def test_mass_check_samples_match_reference_run():
    from paper_2604_00235_b200 import DecodeEngine, EngineConfig, SyntheticSpec, gen_synthetic

    z = load("mass_bound")
    spec_kw = json.loads(str(z["run_spec"]))
    cfg_kw = json.loads(str(z["run_cfg"]))
    tr = gen_synthetic(SyntheticSpec(**spec_kw))
    cfg = EngineConfig(d=spec_kw["d"], d_v=spec_kw["d_v"], n_q_heads=spec_kw["n_q_heads"],
                       n_kv_heads=spec_kw["n_kv_heads"], **cfg_kw)
    eng = DecodeEngine(cfg, capacity=spec_kw["seq_len"])
    q, k, v = (a.astype(np.float64) for a in (tr.q_pre, tr.k_pre, tr.v))
    for m in range(1, spec_kw["seq_len"] + 1):
        eng.decode_step(0, q[m - 1, 0], k[m - 1, 0], v[m - 1, 0], m)
    got = np.array(eng.metrics.mass_bound_samples).reshape(-1, 2)
    want = z["run_samples"]
    assert got.shape == want.shape  # same hits, same order
    np.testing.assert_allclose(got, want, rtol=1e-7, atol=1e-12)
    # the fraction the reference reports (cli.py:355) is identical
    assert np.mean(got[:, 0] <= got[:, 1]) == np.mean(want[:, 0] <= want[:, 1])


@pytest.mark.parametrize("name", ["gqa_f32", "gates", "roi", "remove"])
def test_device_stats_equal_reference_metrics(name):
    from paper_2604_00235_b200 import DecodeEngine, EngineConfig, compute_metrics

    rec = load(name)
    spec_kw, cfg_kw, q, k, v, _ = scenario_inputs(rec)
    cfg = EngineConfig(d=spec_kw["d"], d_v=spec_kw["d_v"], n_layers=spec_kw.get("n_layers", 1),
                       n_q_heads=spec_kw.get("n_q_heads", 1), n_kv_heads=spec_kw.get("n_kv_heads", 1), **cfg_kw)
    eng = DecodeEngine(cfg, capacity=q.shape[0])
    eng.batch.track_stats = True
    for m in range(1, q.shape[0] + 1):
        for layer in range(cfg.n_layers):
            eng.decode_step(layer, q[m - 1, layer], k[m - 1, layer], v[m - 1, layer], m)
    dev = eng.batch.stats(per_head=True)
    host = compute_metrics(eng.metrics)
    for key in ("steps", "hits", "acceptance_rate", "skip_ratio", "kv_fraction", "mean_gap", "mean_band_mass"):
        assert dev[key] == pytest.approx(host[key], rel=1e-9), key
    mt = eng.metrics
    assert dev["group_kv_tokens"] == mt.group_kv_tokens and dev["group_kv_total"] == mt.group_kv_total
    assert dev["forced_misses"] == mt.forced_misses and dev["fallbacks"] == mt.fallbacks
    assert dev["match_candidates"] == mt.match_candidates and dev["kv_tokens_read"] == mt.kv_tokens_read
    want = json.loads(str(rec["metrics"]))  # the reference's own run of this scenario
    assert dev["steps"] == want["steps"] and dev["group_kv_total"] == want["group_kv_total"]
    assert abs(dev["hits"] - want["hits"]) <= 2  # decisions may differ only at documented near-ties
    # per-layer split sums back to the total; per-head steps are L per head per layer
    per_layer = [eng.batch.stats(layer) for layer in range(cfg.n_layers)]
    assert sum(r["steps"] for r in per_layer) == dev["steps"]
    assert (dev["per_head"]["steps"] == q.shape[0] * cfg.n_layers).all()
    eng.batch.reset_stats()
    assert eng.batch.stats()["steps"] == 0


def test_batch_stats_skip_prefill_and_count_batch():
    from paper_2604_00235_b200 import BatchDecodeEngine, EngineConfig

    cfg = EngineConfig(d=32, d_v=32, n_q_heads=4, n_kv_heads=2, window=16, band=4, storage="bf16")
    B, n = 3, 40
    eng = BatchDecodeEngine(cfg, B, 128, track_stats=True)
    g = torch.Generator().manual_seed(0)
    qs = torch.randn(B, n + 5, 4, 32, generator=g).cuda()
    ks = torch.randn(B, n + 5, 2, 32, generator=g).cuda()
    vs = torch.randn(B, n + 5, 2, 32, generator=g).cuda()
    eng.prefill(0, qs[:, :n], ks[:, :n], vs[:, :n])
    assert eng.stats()["steps"] == 0  # prompt tokens are not decisions
    hits, reads, span = 0, 0, 0
    for t in range(n, n + 5):
        qs[:, t] = qs[:, t - 3]  # repeats: hits at p = m - 3
        res = eng.decode_step(0, qs[:, t].contiguous(), ks[:, t].contiguous(), vs[:, t].contiguous())
        m = t + 1
        use, pos, hit = res.use_hit.cpu().numpy(), res.match_pos.cpu().numpy(), res.match_hit.cpu().numpy()
        hits += int(use.sum())
        reads += int(sum((m - max(p - cfg.band, 0)) if u else m for u, p in zip(use.ravel(), pos.ravel())))
        for b in range(B):
            for grp in range(2):
                hh = range(grp * 2, grp * 2 + 2)
                span += m - min(max(pos[b, h] - cfg.band, 0) if hit[b, h] else 0 for h in hh)
    st = eng.stats()
    assert st["steps"] == 5 * B * 4
    assert st["hits"] == hits and hits > 0
    assert st["kv_tokens_read"] == reads
    assert st["group_kv_tokens"] == span
