"""GPU tests of the reference's public building blocks on the CUDA library.

Summary algebra and RoPE (attention.py, its tests pkg/tests/test_attention.py),
QueryRing / match_query (matching.py, pkg/tests/test_matching.py), KvStore
(kvstore.py, pkg/tests/test_kvstore.py), SummaryRing, rectify_append,
oracle_outputs and run_decode (engine.py, pkg/tests/test_engine.py) — each
against naive f64 formulas or the CPU oracle (oracle/mac_oracle.py).
"""

import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import mac_oracle as orc  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_cuda():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")


def naive(q, keys, values):
    """softmax(keys q / sqrt(d)) values and ln Z, written out (test_attention.py:44-56)."""
    lg = keys @ q / math.sqrt(q.shape[0])
    mx = lg.max()
    w = np.exp(lg - mx)
    return (w @ values) / w.sum(), mx + math.log(w.sum())


# ---------------------------------------------------------------- summary algebra
def test_summarize_matches_naive_and_oracle():
    from paper_2604_00235_b200 import summarize

    rng = np.random.default_rng(0)
    for n, d, dv in ((1, 2, 3), (37, 16, 8), (5000, 64, 32), (300, 128, 128)):
        q, k, v = rng.standard_normal(d) * 2, rng.standard_normal((n, d)), rng.standard_normal((n, dv))
        s = summarize(q, k, v)
        acc, lse = naive(q, k, v)
        assert s.count == n
        np.testing.assert_allclose(s.acc, acc, rtol=1e-12, atol=1e-13)
        assert abs(s.lse - lse) < 1e-11
        o = orc.summarize(q, k, v)  # streaming-block oracle (n > 4096 takes the online path)
        np.testing.assert_allclose(s.acc, o.acc, rtol=1e-12, atol=1e-13)


def test_summarize_empty_validation_and_storage_dtype():
    from paper_2604_00235_b200 import summarize

    e = summarize(np.ones(4), np.zeros((0, 4)), np.zeros((0, 3)))
    assert e.count == 0 and e.lse == -math.inf and e.acc.shape == (3,)
    with pytest.raises(ValueError):
        summarize(np.ones(4), np.ones((3, 4)), np.ones((2, 3)))
    with pytest.raises(ValueError):
        summarize(np.ones(4), np.ones(4), np.ones((1, 3)))
    rng = np.random.default_rng(1)
    s = summarize(rng.standard_normal(8), rng.standard_normal((9, 8)), rng.standard_normal((9, 8)), dtype=np.float32)
    assert s.acc.dtype == np.float32 and float(np.float32(s.lse)) == s.lse


def test_merge_reproduces_monolith_at_every_cut():
    from paper_2604_00235_b200 import merge, summarize

    rng = np.random.default_rng(2)
    q, k, v = rng.standard_normal(16), rng.standard_normal((24, 16)), rng.standard_normal((24, 5))
    whole = summarize(q, k, v)
    for cut in range(0, 25, 3):
        m = merge(summarize(q, k[:cut], v[:cut]), summarize(q, k[cut:], v[cut:]))
        assert m.count == 24
        np.testing.assert_allclose(m.acc, whole.acc, rtol=1e-12, atol=1e-13)
        assert abs(m.lse - whole.lse) < 1e-12


def test_merge_identity_commutativity_association():
    from paper_2604_00235_b200 import empty_summary, merge, summarize

    rng = np.random.default_rng(3)
    q = rng.standard_normal(8)
    a, b, c = (summarize(q, rng.standard_normal((n, 8)), rng.standard_normal((n, 4))) for n in (3, 5, 7))
    e = empty_summary(4)
    assert merge(a, e) is a and merge(e, b) is b
    ab, ba = merge(a, b), merge(b, a)
    np.testing.assert_allclose(ab.acc, ba.acc, rtol=1e-14)
    x, y = merge(merge(a, b), c), merge(a, merge(b, c))
    np.testing.assert_allclose(x.acc, y.acc, rtol=1e-13)
    assert x.count == 15 and abs(x.lse - y.lse) < 1e-13
    f = merge(a.astype(np.float32), b.astype(np.float32))
    assert f.acc.dtype == np.float32  # result_type of the stored operands


def test_remove_inverts_merge_and_guards():
    from paper_2604_00235_b200 import (CancellationError, MassExceededError, empty_summary, merge, remove,
                                       summarize)

    rng = np.random.default_rng(4)
    q, k, v = rng.standard_normal(16), rng.standard_normal((40, 16)), rng.standard_normal((40, 6))
    head, band = summarize(q, k[:30], v[:30]), summarize(q, k[30:], v[30:])
    back = remove(merge(head, band), band)
    assert back.count == 30
    np.testing.assert_allclose(back.acc, head.acc, rtol=1e-9, atol=1e-10)
    assert abs(back.lse - head.lse) < 1e-9
    assert remove(head, empty_summary(6)) is head
    same = remove(head, head)
    assert same.count == 0 and same.lse == -math.inf
    with pytest.raises(ValueError):
        remove(band, head)  # more tokens than the whole
    bogus = type(head)(acc=head.acc, lse=head.lse + 1.0, count=head.count)
    with pytest.raises(CancellationError):
        remove(head, bogus)  # all tokens, different mass
    heavy = type(band)(acc=band.acc, lse=head.lse + 1.0, count=5)
    with pytest.raises(MassExceededError):
        remove(head, heavy)
    near = type(band)(acc=band.acc, lse=head.lse - 1e-8, count=5)
    with pytest.raises(CancellationError):
        remove(head, near)


def test_attend_full_and_finalize():
    from paper_2604_00235_b200 import EmptySummaryError, attend_full, empty_summary, finalize

    rng = np.random.default_rng(5)
    q, k, v = rng.standard_normal(32), rng.standard_normal((50, 32)), rng.standard_normal((50, 32))
    out, s = attend_full(q, k, v)
    np.testing.assert_array_equal(out, s.acc)
    np.testing.assert_allclose(out, naive(q, k, v)[0], rtol=1e-12, atol=1e-13)
    with pytest.raises(EmptySummaryError):
        finalize(empty_summary(3))


def test_rope_table_rotate_and_avg_cos():
    from paper_2604_00235_b200 import RopeTable, avg_cos, rope_rotate

    with pytest.raises(ValueError):
        RopeTable(3)
    with pytest.raises(ValueError):
        RopeTable(4, base=1.0)
    tab = RopeTable(128)
    np.testing.assert_array_equal(tab.freqs, orc.rope_freqs(128))
    rng = np.random.default_rng(6)
    x = rng.standard_normal((9, 128))
    t = np.array([1, 2, 7, 100, 4097, 32768, 131072, 524288, 3])
    y = rope_rotate(x, t, tab)
    ref = np.stack([orc.rope_rotate(x[i], t[i], tab.freqs) for i in range(9)])
    np.testing.assert_allclose(y, ref, rtol=0, atol=1e-12)
    np.testing.assert_allclose(np.linalg.norm(y, axis=1), np.linalg.norm(x, axis=1), rtol=1e-13)
    np.testing.assert_allclose(rope_rotate(x[0], 0, tab), x[0], rtol=0, atol=0)
    np.testing.assert_allclose(rope_rotate(x[:2], 5, tab), rope_rotate(x[:2], [5, 5], tab), rtol=0, atol=0)
    # ||x - R(delta) x||^2 == 2 ||x||^2 (1 - avg_cos)   (attention.py:235-249)
    r = rope_rotate(x[1], 37, tab)
    lhs = float(np.sum((x[1] - r) ** 2))
    assert abs(lhs - 2 * float(x[1] @ x[1]) * (1 - avg_cos(x[1], 37, tab))) < 1e-9
    with pytest.raises(ValueError):
        rope_rotate(np.ones(6), 1, RopeTable(4))


# ---------------------------------------------------------------- rings + matching
def test_query_ring_basics_and_eviction():
    from paper_2604_00235_b200 import QueryRing

    ring = QueryRing(3, 4)
    assert len(ring) == 0 and ring.last_position == 0
    for pos in (1, 2, 3):
        assert ring.push(pos, np.full(4, float(pos))) is None
    ev = ring.push(4, np.full(4, 4.0))
    assert ev[0] == 1 and ev[2] == 4.0 and len(ring) == 3 and ring.last_position == 4
    assert ring.slot_of(4) == 0 and ring.query_at(3)[0] == 3.0
    with pytest.raises(KeyError):
        ring.slot_of(1)
    with pytest.raises(ValueError):
        ring.push(4, np.zeros(4))
    with pytest.raises(ValueError):
        ring.push(9, np.zeros(5))
    with pytest.raises(ValueError):
        QueryRing(0, 4)
    q, sq, pos = ring.view()
    assert sorted(pos.tolist()) == [2, 3, 4]
    np.testing.assert_array_equal(sq, (q * q).sum(axis=1))


def test_match_query_kats():
    """Empty ring, exact duplicate, tie -> most recent, strict radius, Δmax, stale stream
    (pkg/tests/test_matching.py:65-121)."""
    from paper_2604_00235_b200 import MatchConfig, QueryRing, match_query, threshold

    d = 16
    cfg = MatchConfig(d=d, tau=0.45)
    ring = QueryRing(8, d)
    r = match_query(np.ones(d), 1, ring, cfg)
    assert not r.hit and r.p == -1 and r.candidates_scanned == 0 and r.sq_dist == math.inf
    rng = np.random.default_rng(7)
    qs = rng.standard_normal((5, d))
    for i in range(5):
        ring.push(i + 1, qs[i])
    r = match_query(qs[2], 6, ring, cfg)
    assert r.hit and r.p == 3 and r.sq_dist == 0.0 and r.candidates_scanned == 5
    ring.push(6, qs[2])  # duplicate of position 3: tie, the most recent wins
    r = match_query(qs[2], 7, ring, cfg)
    assert r.hit and r.p == 6
    thr = threshold(d, 0.45)
    ring2 = QueryRing(4, d)
    base = np.zeros(d)
    ring2.push(1, base)
    at = base.copy()
    at[0] = thr  # distance exactly thr: a miss (strict)
    assert not match_query(at, 2, ring2, cfg).hit
    inside = base.copy()
    inside[0] = np.nextafter(thr, 0.0)
    assert match_query(inside, 2, ring2, cfg).hit
    ring3 = QueryRing(8, d)
    for i in range(5):
        ring3.push(i + 1, qs[i])
    far = MatchConfig(d=d, tau=0.45, delta_max=2)
    r = match_query(qs[0], 6, ring3, far)  # position 1 is 5 back: filtered
    assert r.candidates_scanned == 2 and r.p != 1
    r = match_query(qs[0], 20, ring3, far)
    assert not r.hit and r.candidates_scanned == 0
    with pytest.raises(ValueError):
        match_query(qs[0], 5, ring3, cfg)  # ring already holds position 5


def test_match_queries_batched_equals_oracle_incl_post_rope():
    from paper_2604_00235_b200 import MATCH_POST_ROPE, MatchConfig, QueryRing, match_queries

    rng = np.random.default_rng(8)
    d, W, n_rings = 32, 16, 24
    freqs = orc.rope_freqs(d)
    for space in ("pre_rope", MATCH_POST_ROPE):
        cfg = MatchConfig(d=d, tau=0.3, space=space)
        rings, qs, ms = [], [], []
        for i in range(n_rings):
            ring = QueryRing(W, d)
            n = int(rng.integers(1, 3 * W))
            hist = rng.standard_normal((n, d))
            for p in range(n):
                ring.push(p + 1, hist[p])
            rings.append(ring)
            q = hist[int(rng.integers(max(0, n - W), n))] + 0.05 * rng.standard_normal(d)
            qs.append(q if i % 3 else rng.standard_normal(d))
            ms.append(n + 1)
        got = match_queries(np.array(qs), ms, rings, cfg)
        ocfg = orc.OracleConfig(d=d, d_v=d, window=W, tau=0.3, match_space=space)
        for ring, q, m, g in zip(rings, qs, ms, got):
            cand, sq, pos = ring.view()
            hit, p, dist, n_scan = orc._match(q, m, cand, sq, pos, len(ring), ocfg, 0.3, freqs)
            assert (g.hit, g.p, g.candidates_scanned) == (bool(hit), int(p), int(n_scan))
            assert abs(g.sq_dist - dist) <= 1e-9 * max(1.0, dist)


def test_summary_ring():
    from paper_2604_00235_b200 import AttentionSummary, SummaryRing

    ring = SummaryRing(2)
    s = [AttentionSummary(acc=np.full(3, float(i), dtype=np.float32), lse=float(i), count=i) for i in range(4)]
    assert ring.push(1, s[1]) is None and ring.push(2, s[2]) is None
    ev = ring.push(3, s[3])
    assert ev[0] == 1 and ev[1].count == 1
    got = ring.summary_at(3)
    assert got.count == 3 and got.lse == 3.0 and got.acc.dtype == np.float32 and got.acc[0] == 3.0
    with pytest.raises(KeyError):
        ring.summary_at(1)
    with pytest.raises(ValueError):
        ring.push(3, s[0])
    assert len(ring) == 2 and ring.last_position == 3


# ---------------------------------------------------------------- KvStore
def test_kvstore_semantics():
    from paper_2604_00235_b200 import KvStore, TrafficCounter

    st = KvStore(4, 2)
    assert st.append(0, 0, np.ones(4), np.ones(2)) == 1 and st.append(0, 0, np.ones(4), np.ones(2)) == 2
    assert st.length(0, 0) == 2 and st.length(0, 1) == 0
    rng = np.random.default_rng(9)
    k, v = rng.standard_normal(8), rng.standard_normal(8)
    f32 = KvStore(8, 8)
    f32.append(0, 0, k, v)
    kk, vv = f32.read_range(0, 0, (1, 1))
    assert kk.dtype == np.float64
    np.testing.assert_array_equal(kk[0], k.astype(np.float32).astype(np.float64))
    np.testing.assert_array_equal(vv[0], v.astype(np.float32).astype(np.float64))
    f64 = KvStore(8, 8, storage_dtype=np.float64)
    f64.append(0, 0, k, v)
    np.testing.assert_array_equal(f64.read_range(0, 0, (1, 1))[0][0], k)
    with pytest.raises(ValueError):
        KvStore(4, 4, storage_dtype=np.float16)
    with pytest.raises(ValueError):
        KvStore(4, 4, page_size=0)
    with pytest.raises(ValueError):
        st.append(0, 0, np.ones(3), np.ones(2))
    rows = rng.standard_normal((300, 2)).astype(np.float32).astype(np.float64)
    big = KvStore(2, 2)
    for i in range(300):  # grows the page pool several times
        big.append(0, 0, rows[i], rows[i])
    np.testing.assert_array_equal(big.read_range(0, 0, (3, 7))[0], rows[2:7])
    np.testing.assert_array_equal(big.read_range(0, 0, (1, 300))[1], rows)
    for bad in ((0, 5), (5, 301), (6, 5), (1, 0)):
        with pytest.raises(ValueError):
            big.read_range(0, 0, bad)
    with pytest.raises(ValueError):
        big.read_range(1, 0, (1, 1))
    t = TrafficCounter()
    tb = KvStore(4, 4)
    for _ in range(20):
        tb.append(0, 0, np.ones(4), np.ones(4))
    tb.read_range(0, 0, (1, 20), t)
    tb.read_range(0, 0, (5, 8), t)
    assert t.tokens_read == 24 and tb.token_bytes == 32 and t.bytes_read == 24 * 32
    assert t.read_histogram[(20).bit_length()] == 1 and t.read_histogram[(4).bit_length()] == 1
    pr = KvStore(4, 4, page_size=16, page_rounded_bytes=True)
    for _ in range(20):
        pr.append(0, 0, np.ones(4), np.ones(4))
    t1, t2 = TrafficCounter(), TrafficCounter()
    pr.read_range(0, 0, (1, 1), t1)
    pr.read_range(0, 0, (16, 17), t2)
    assert t1.tokens_read == 1 and t1.bytes_read == 16 * pr.token_bytes and t2.bytes_read == 32 * pr.token_bytes
    pg = KvStore(2, 2, page_size=4)
    for i in range(1, 7):
        pg.append(0, 0, np.full(2, float(i)), np.full(2, float(i)))
    assert pg.n_pages(0, 0) == 2
    p0, p1 = pg.page(0, 0, 0), pg.page(0, 0, 1)
    assert p0.fill == 4 and p1.fill == 2
    np.testing.assert_array_equal(p0.keys[:, 0], [1.0, 2.0, 3.0, 4.0])
    np.testing.assert_array_equal(p1.keys[:, 0], [5.0, 6.0, 0.0, 0.0])
    np.testing.assert_array_equal(p1.values[2:], np.zeros((2, 2)))
    with pytest.raises(IndexError):
        pg.page(0, 0, 2)
    kd, _ = pg.read_range_device(0, 0, (2, 5))
    assert kd.is_cuda and kd.shape == (4, 2) and float(kd[0, 0]) == 2.0


# ---------------------------------------------------------------- engine surface
def _small_trace(seed=11, L=96, layers=1, hq=4, hkv=2, d=16):
    from paper_2604_00235_b200 import SyntheticSpec, gen_synthetic

    return gen_synthetic(SyntheticSpec(seq_len=L, d=d, d_v=d, n_layers=layers, n_q_heads=hq, n_kv_heads=hkv,
                                       seed=seed))


def test_oracle_outputs_matches_cpu_oracle():
    from paper_2604_00235_b200 import EngineConfig, oracle_outputs

    tr = _small_trace(layers=2)
    for storage in ("f32", "f64"):
        cfg = EngineConfig(d=16, d_v=16, n_layers=2, n_q_heads=4, n_kv_heads=2, window=16, band=4, storage=storage)
        got = oracle_outputs(tr, cfg, chunk=40)
        ocfg = orc.OracleConfig(d=16, d_v=16, n_layers=2, n_q_heads=4, n_kv_heads=2, window=16, band=4,
                                storage=storage)
        ref = orc.oracle_outputs(tr.q_pre, tr.k_pre, tr.v, ocfg)
        assert got.shape == (2, 96, 4, 16)
        np.testing.assert_allclose(got, ref, rtol=1e-11, atol=1e-12)


def test_run_decode_oracle_modes_and_traffic_identity():
    """Batched vs per-step oracle give the same errors on miss steps (0) and agree on hits
    (test_engine.py:317-328); traffic.tokens_read == metrics.kv_tokens_read
    (test_engine.py:255,328)."""
    from paper_2604_00235_b200 import EngineConfig, compute_metrics, run_decode

    tr = _small_trace(L=120)
    cfg = EngineConfig(d=16, d_v=16, n_q_heads=4, n_kv_heads=2, window=32, band=8, oracle_mode=True)
    a = run_decode(tr, cfg)
    b = run_decode(tr, cfg, per_step_oracle=True)
    ea, eb = np.array(a.metrics.err_samples), np.array(b.metrics.err_samples)
    assert ea.shape == eb.shape and ea.size == 120 * 4
    # (the reference's own test uses atol 1e-6 with f64 math; the f32-storage kernels differ from the
    # f64 batched oracle by f32 roundoff on miss steps)
    np.testing.assert_allclose(ea, eb, atol=5e-6)
    assert b.oracle_traffic.tokens_read > 0 and a.oracle_traffic.tokens_read == 0
    for eng in (a, b):
        assert eng.traffic.tokens_read == eng.metrics.kv_tokens_read
        assert eng.metrics.hits > 0
    assert compute_metrics(a.metrics)["acceptance_rate"] == compute_metrics(b.metrics)["acceptance_rate"]


def test_rectify_append_validation_and_ring_write():
    from paper_2604_00235_b200 import AttentionSummary, DecodeEngine, EngineConfig

    cfg = EngineConfig(d=8, d_v=8, n_q_heads=2, n_kv_heads=1, window=4, band=2)
    eng = DecodeEngine(cfg, capacity=32)
    full = AttentionSummary(acc=np.zeros(8), lse=0.0, count=3)
    band = AttentionSummary(acc=np.zeros(8), lse=0.0, count=2)
    good = AttentionSummary(acc=np.arange(8.0), lse=1.5, count=1)
    with pytest.raises(ValueError):
        eng.rectify_append(0, 0, 3, np.ones(8), AttentionSummary(np.zeros(8), 0.0, 2), band, good)
    with pytest.raises(ValueError):
        eng.rectify_append(0, 0, 3, np.ones(8), full, band, AttentionSummary(np.zeros(8), 0.0, 2))
    with pytest.raises(ValueError):
        eng.rectify_append(0, 0, 3, np.ones(8), full, band, good)  # not slot-aligned after 0
    rng = np.random.default_rng(12)
    for m in (1, 2):
        eng.decode_step(0, rng.standard_normal((2, 8)), rng.standard_normal((1, 8)), rng.standard_normal((1, 8)), m)
    q3 = rng.standard_normal(8)
    eng.rectify_append(0, 1, 3, q3, full, band, good)
    qr, sr = eng.rings(0, 1)
    np.testing.assert_array_equal(qr.query_at(3), q3.astype(np.float32).astype(np.float64))
    got = sr.summary_at(3)
    np.testing.assert_array_equal(got.acc, good.acc)
    assert got.lse == 1.5 and got.count == 1
    with pytest.raises(ValueError):
        eng.rectify_append(0, 1, 3, q3, full, band, good)  # position does not increase
    with pytest.raises(ValueError):
        eng.decode_step(0, rng.standard_normal((2, 8)), rng.standard_normal((1, 8)), rng.standard_normal((1, 8)), 3)
