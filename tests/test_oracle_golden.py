"""Pin the CPU oracle (oracle/mac_oracle.py) against the reference's own outputs.

The fixtures under tests/golden/ were produced by tests/golden/make_golden.py
running the unmodified reference package (attnreuse) in the build container.
Traces are regenerated here with this repo's generator, pinned by SHA-256.
"""

import hashlib
import json
import os

import numpy as np
import pytest

import mac_oracle as orc
from golden_util import GOLDEN, SCENARIOS, load, rel_err, scenario_inputs
from paper_2604_00235_b200.workload import SyntheticSpec, gen_synthetic


def _sha(tr):
    h = hashlib.sha256()
    for a in (tr.q_pre, tr.k_pre, tr.v):
        h.update(np.ascontiguousarray(a, dtype="<f4").tobytes())
    return h.hexdigest()


def test_trace_generator_matches_reference_bytes():
    with open(os.path.join(GOLDEN, "trace_sha.json")) as fh:
        want = json.load(fh)
    for kw, sha in want.items():
        assert _sha(gen_synthetic(SyntheticSpec(**json.loads(kw)))) == sha, kw


def run_oracle(cfg_kw, spec_kw, q, k, v):
    cfg = orc.OracleConfig(d=spec_kw["d"], d_v=spec_kw["d_v"], n_layers=spec_kw.get("n_layers", 1),
                           n_q_heads=spec_kw.get("n_q_heads", 1), n_kv_heads=spec_kw.get("n_kv_heads", 1),
                           **cfg_kw)
    eng = orc.OracleEngine(cfg, capacity=q.shape[0])
    steps = []
    for m in range(1, q.shape[0] + 1):
        steps.append([eng.decode_step(layer, q[m - 1, layer], k[m - 1, layer], v[m - 1, layer], m)
                      for layer in range(cfg.n_layers)])
    return eng, steps


@pytest.mark.parametrize("name", SCENARIOS)
def test_oracle_matches_reference(name):
    rec = load(name)
    spec_kw, cfg_kw, q, k, v, tr = scenario_inputs(rec)
    assert _sha(tr) == str(rec["trace_sha"])
    eng, steps = run_oracle(cfg_kw, spec_kw, q, k, v)
    hit = np.array([[s.hit for s in row] for row in steps])
    p = np.array([[s.p for s in row] for row in steps])
    dist = np.array([[s.sq_dist for s in row] for row in steps])
    np.testing.assert_array_equal(hit, rec["hit"].astype(bool))
    np.testing.assert_array_equal(p, rec["p"])
    fin = np.isfinite(rec["dist"])
    np.testing.assert_array_equal(np.isfinite(dist), fin)
    np.testing.assert_allclose(dist[fin], rec["dist"][fin], rtol=1e-9, atol=1e-9)
    rho = np.array([[s.band_mass for s in row] for row in steps])
    np.testing.assert_allclose(rho, rec["rho"], rtol=1e-9, atol=1e-12)
    for i, m in enumerate(rec["out_steps"]):
        for layer in range(q.shape[1]):
            assert rel_err(steps[m - 1][layer].outputs, rec["outputs"][i, layer]) <= 1e-9
    met = orc.metrics_report(eng.metrics)
    want = json.loads(str(rec["metrics"]))
    for key in ("steps", "hits", "group_kv_tokens", "group_kv_total", "forced_misses", "fallbacks"):
        assert met[key] == want[key], key
    for key in ("acceptance_rate", "skip_ratio", "kv_fraction"):
        assert met[key] == pytest.approx(want[key], rel=1e-12), key


def test_oracle_kats():
    z = np.load(os.path.join(GOLDEN, "kat.npz"))
    for name in ("kat_d2", "kat_d8_f32", "kat_pband"):
        cfg_kw = json.loads(str(z[f"{name}__cfg"]))
        q, k, v = z[f"{name}__q"], z[f"{name}__k"], z[f"{name}__v"]
        cfg = orc.OracleConfig(**cfg_kw)
        eng = orc.OracleEngine(cfg)
        for m in range(1, q.shape[0] + 1):
            st = eng.decode_step(0, q[m - 1][None], k[m - 1][None], v[m - 1][None], m)
            assert st.hit[0] == z[f"{name}__hit"][m - 1]
            assert st.p[0] == z[f"{name}__p"][m - 1]
            assert rel_err(st.outputs[0], z[f"{name}__outputs"][m - 1]) <= 1e-12


def test_oracle_outputs_batched():
    z = np.load(os.path.join(GOLDEN, "oracle_outputs.npz"))
    kw = json.loads(str(z["spec"]))
    tr = gen_synthetic(SyntheticSpec(**kw))
    cfg = orc.OracleConfig(d=kw["d"], d_v=kw["d_v"], n_layers=kw["n_layers"], n_q_heads=kw["n_q_heads"],
                           n_kv_heads=kw["n_kv_heads"])
    got = orc.oracle_outputs(tr.q_pre.astype(np.float64), tr.k_pre.astype(np.float64), tr.v.astype(np.float64),
                             cfg, chunk=16)
    np.testing.assert_allclose(got, z["out"], rtol=1e-12, atol=1e-14)


def test_bf16_rounding_is_rne():
    x = np.array([1.0, 1.0 + 2 ** -8, 1.0 + 3 * 2 ** -9, -2.5, 3.140625, 1e-30], dtype=np.float32)
    got = orc.round_bf16(x)
    import torch

    want = torch.from_numpy(x).bfloat16().double().numpy()
    np.testing.assert_array_equal(got, want)


def test_oracle_mass_bound_matches_reference():
    """mass_bound_check (engine.py:246-281) restated; pinned on the reference's outputs."""
    from mac_oracle import mass_bound_check

    z = load("mass_bound")
    for i in range(int(z["n_cases"])):
        got = mass_bound_check(z[f"c{i}__q_m"], z[f"c{i}__q_p"], z[f"c{i}__keys"], z[f"c{i}__values"],
                               int(z[f"c{i}__band"]))
        np.testing.assert_allclose(got, z[f"c{i}__out"], rtol=1e-12, atol=1e-16, err_msg=f"case {i}")
    samples = z["run_samples"]
    assert samples.shape[1] == 2 and (samples >= 0).all()
