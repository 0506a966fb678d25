"""GPU parity of the KV-sharded decode path (sharded.py, mac_shard_partial / mac_shard_complete).

The box has one GPU, so G shard engines share it and the all-gather is a
stack of their `shard_send` buffers — everything else (per-shard plans,
appends, partial summaries, rank-order merge, ring write-back) is exactly
the multi-GPU code path.  Checked against the unsharded CPU oracle and
against each other (every shard must produce the identical result).
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import mac_oracle as orc  # noqa: E402
from golden_util import bf16_round, rel_err  # noqa: E402

TOL = 1e-4


def _setup(world, hq=8, hkv=2, W=64, r=16, n0=3000, S=6, rep_prob=0.6, seed=7):
    from paper_2604_00235_b200 import EngineConfig
    from paper_2604_00235_b200.sharded import ShardedDecodeEngine, ShardLayout
    from paper_2604_00235_b200.synth import request_state

    cfg = EngineConfig(d=128, d_v=128, n_q_heads=hq, n_kv_heads=hkv, window=W, band=r, storage="bf16")
    st = request_state(seed, n0=n0, steps=S, hq=hq, hkv=hkv, d=128, dv=128, window=W, band=r, rep_prob=rep_prob)
    rng = np.random.default_rng(seed + 1)
    kf = bf16_round(rng.standard_normal((hkv, n0, 128))).astype(np.float32)
    vf = bf16_round(rng.standard_normal((hkv, n0, 128))).astype(np.float32)
    T = st.tail_k.shape[1]
    kf[:, n0 - T:] = st.tail_k
    vf[:, n0 - T:] = st.tail_v
    layout = ShardLayout.for_context(n0 + S, world, min_tail=W + r)
    engs = [ShardedDecodeEngine(cfg, 1, layout, rk, n0 + S + 8, min_chunk=64) for rk in range(world)]
    kt, vt = torch.from_numpy(kf[None]).cuda(), torch.from_numpy(vf[None]).cuda()
    rq, ra, rl = (torch.from_numpy(a[None]).cuda() for a in (st.ring_q, st.ring_acc, st.ring_lse))
    for e in engs:
        e.inject(0, kt, vt, rq, ra, rl, n0)
    ocfg = orc.OracleConfig(d=128, d_v=128, n_q_heads=hq, n_kv_heads=hkv, window=W, band=r, storage="bf16")
    oe = orc.OracleEngine(ocfg, capacity=n0 + S + 8)
    oe.inject(0, kf.astype(np.float64), vf.astype(np.float64), st.ring_q.astype(np.float64),
              st.ring_acc.astype(np.float64), st.ring_lse.astype(np.float64))
    return engs, oe, st, n0, S, layout


@pytest.mark.parametrize("world", [1, 2, 3, 4])
def test_sharded_step_matches_oracle(world):
    engs, oe, st, n0, S, layout = _setup(world)
    hits = misses = 0
    worst = 0.0
    for s in range(S):
        q, k, v = (torch.from_numpy(a[s][None]).to("cuda", torch.bfloat16).contiguous()
                   for a in (st.step_q, st.step_k, st.step_v))
        sends = [e.partial(0, q, k, v).clone() for e in engs]
        gathered = torch.stack(sends)
        outs, rings = [], []
        for e in engs:
            e.engine.shard_parts.copy_(gathered)
            res = e.complete(0, q, k, v)
            outs.append(res.out.clone())
            rings.append((e.engine.ring_acc[0].clone(), e.engine.ring_lse[0].clone(), e.engine.ring_q[0].clone()))
            assert (res.match_hit.cpu().numpy()[0] == engs[0].engine.o_hit.cpu().numpy()[0]).all()
        ref = oe.decode_step(0, st.step_q[s], st.step_k[s], st.step_v[s], n0 + s + 1)
        for i in range(1, world):  # identical on every shard, rings included
            assert torch.equal(outs[i], outs[0])
            for a, b in zip(rings[i], rings[0]):
                assert torch.equal(a, b)
        e0 = engs[0].engine
        np.testing.assert_array_equal(e0.o_hit.cpu().numpy()[0].astype(bool), ref.hit)
        np.testing.assert_array_equal(e0.o_pos.cpu().numpy()[0], ref.p)
        got = outs[0].double().cpu().numpy()[0]
        for h in range(got.shape[0]):
            worst = max(worst, rel_err(got[h], ref.outputs[h]))
        ring_acc = e0.ring_acc[0][0, :, (n0 + s) % e0.cfg.window].double().cpu().numpy()
        for h in range(got.shape[0]):
            if np.linalg.norm(ref.prefix_acc[h]) > 0:
                assert rel_err(ring_acc[h], ref.prefix_acc[h]) <= TOL
        hits += int(ref.use_hit.sum())
        misses += int((~ref.use_hit).sum())
        assert all(int(e.engine.seq_lens[0][0]) == n0 + s + 1 for e in engs)
    assert hits > 0 and misses > 0
    assert worst <= TOL, worst


def test_sharded_append_lands_on_the_tail_shard():
    engs, oe, st, n0, S, layout = _setup(3, S=2)
    q, k, v = (torch.from_numpy(a[0][None]).to("cuda", torch.bfloat16).contiguous()
               for a in (st.step_q, st.step_k, st.step_v))
    before = [e.engine.k_cache[0].clone() for e in engs]
    for e in engs:
        e.partial(0, q, k, v)
    torch.cuda.synchronize()
    for rk, e in enumerate(engs):
        changed = not torch.equal(before[rk], e.engine.k_cache[0])
        assert changed == (rk == layout.owner(n0 + 1)), rk


def _nccl_worker(rank, world, port, result_path):
    """One rank per GPU over NCCL: the KV-sharded step through ShardedDecodeEngine.decode_step
    (partial -> all_gather_into_tensor -> complete), checked against the unsharded oracle."""
    import os

    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    from paper_2604_00235_b200 import EngineConfig
    from paper_2604_00235_b200.sharded import ShardedDecodeEngine, ShardLayout
    from paper_2604_00235_b200.synth import request_state

    hq, hkv, W, r, n0, S = 8, 2, 64, 16, 3000, 6
    cfg = EngineConfig(d=128, d_v=128, n_q_heads=hq, n_kv_heads=hkv, window=W, band=r, storage="bf16")
    st = request_state(7, n0=n0, steps=S, hq=hq, hkv=hkv, d=128, dv=128, window=W, band=r, rep_prob=0.6)
    rng = np.random.default_rng(8)
    kf = bf16_round(rng.standard_normal((hkv, n0, 128))).astype(np.float32)
    vf = bf16_round(rng.standard_normal((hkv, n0, 128))).astype(np.float32)
    T = st.tail_k.shape[1]
    kf[:, n0 - T:] = st.tail_k
    vf[:, n0 - T:] = st.tail_v
    dev = torch.device("cuda", rank)
    layout = ShardLayout.for_context(n0 + S, world, min_tail=W + r)
    eng = ShardedDecodeEngine(cfg, 1, layout, rank, n0 + S + 8, device=dev, min_chunk=64)
    eng.inject(0, torch.from_numpy(kf[None]).to(dev), torch.from_numpy(vf[None]).to(dev),
               *(torch.from_numpy(a[None]).to(dev) for a in (st.ring_q, st.ring_acc, st.ring_lse)), n0)
    ocfg = orc.OracleConfig(d=128, d_v=128, n_q_heads=hq, n_kv_heads=hkv, window=W, band=r, storage="bf16")
    oe = orc.OracleEngine(ocfg, capacity=n0 + S + 8)
    oe.inject(0, kf.astype(np.float64), vf.astype(np.float64), st.ring_q.astype(np.float64),
              st.ring_acc.astype(np.float64), st.ring_lse.astype(np.float64))
    worst, flips = 0.0, 0
    for s in range(S):
        q, k, v = (torch.from_numpy(a[s][None]).to(dev, torch.bfloat16).contiguous()
                   for a in (st.step_q, st.step_k, st.step_v))
        res = eng.decode_step(0, q, k, v)
        ref = oe.decode_step(0, st.step_q[s], st.step_k[s], st.step_v[s], n0 + s + 1)
        flips += int((res.match_hit.cpu().numpy()[0].astype(bool) != ref.hit).sum())
        got = res.out.double().cpu().numpy()[0]
        worst = max(worst, max(rel_err(got[h], ref.outputs[h]) for h in range(hq)))
        out0 = res.out.clone()
        dist.broadcast(out0, 0)  # every rank holds the identical result
        if not torch.equal(out0, res.out):
            flips += 1000
    if rank == 0:
        with open(result_path, "w") as fh:
            fh.write(f"{worst!r} {flips} {dist.get_backend()} {world}")
    dist.destroy_process_group()


def test_nccl_kv_sharded_step_across_visible_gpus(tmp_path):
    """NCCL exercised for real: one rank per visible GPU (a 1-GPU box runs a one-rank NCCL
    group, so the all_gather_into_tensor path still executes)."""
    import socket

    import torch.multiprocessing as tmp

    world = torch.cuda.device_count()
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    out = tmp_path / "nccl.txt"
    tmp.spawn(_nccl_worker, args=(world, port, str(out)), nprocs=world, join=True)
    worst, flips, backend, n = out.read_text().split()
    assert backend == "nccl" and int(n) == world
    assert int(flips) == 0
    assert float(worst) <= TOL, worst
