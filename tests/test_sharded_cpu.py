"""Host logic of the KV-sharded miss path on CPU: the shard layout, and the
exchange (the product's `exchange`, over a world-size-2 gloo group) followed
by the rank-order log-domain merge, checked against unsharded attention
computed by the oracle.  No GPU: each rank's (piece, band) partials are the
oracle's summaries over that rank's KV slice, in the exact `shard_send`
layout [B, Hq, 2, d_v+1] the CUDA path exports."""

import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as tmp

import mac_oracle as orc
from paper_2604_00235_b200.sharded import ShardLayout, exchange


def test_layout_offsets_limits_owner():
    lay = ShardLayout(shard_tokens=100, world=3)
    assert [lay.offset(r) for r in range(3)] == [0, 100, 200]
    assert [lay.limit(r) for r in range(3)] == [100, 100, 0]
    assert lay.owner(1) == 0 and lay.owner(100) == 0 and lay.owner(101) == 1 and lay.owner(10_000) == 2
    assert lay.local_range(0, 50) == (1, 50)
    assert lay.local_range(1, 50) == (101, 50)  # empty
    assert lay.local_range(2, 260) == (201, 260)
    with pytest.raises(ValueError):
        lay.offset(3)
    with pytest.raises(ValueError):
        ShardLayout(shard_tokens=0, world=2)


def test_layout_for_context_keeps_tail():
    lay = ShardLayout.for_context(1000, 4, min_tail=400)
    lo, hi = lay.local_range(3, 1000)
    assert hi - lo + 1 >= 400
    covered = sum(max(0, b - a + 1) for a, b in (lay.local_range(r, 1000) for r in range(4)))
    assert covered == 1000
    assert ShardLayout.for_context(1000, 1).local_range(0, 1000) == (1, 1000)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _pack(s: orc.Summary, dv: int) -> np.ndarray:
    out = np.zeros(dv + 1, dtype=np.float32)
    out[:dv] = s.acc
    out[dv] = s.lse
    return out


def _unpack(row: np.ndarray, count: int) -> orc.Summary:
    lse = float(row[-1])
    return orc.Summary(row[:-1].astype(np.float64), lse, 0 if lse == -math.inf else count)


def _worker(rank, world, port, result_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(0)  # same data on every rank
    Hq, Hkv, d, m, r = 4, 2, 16, 50, 8
    g = Hq // Hkv
    K = rng.standard_normal((Hkv, m, d))
    V = rng.standard_normal((Hkv, m, d))
    q = rng.standard_normal((Hq, d))
    lay = ShardLayout.for_context(m, world, min_tail=r)
    lo, hi = lay.local_range(rank, m)
    send = torch.zeros(1, Hq, 2, d + 1)
    for h in range(Hq):
        j = h // g
        p_lo, p_hi = lo, min(hi, m - r)            # piece: t <= m - r
        b_lo, b_hi = max(lo, m - r + 1), hi         # band:  t >  m - r
        piece = orc.summarize(q[h], K[j, p_lo - 1:p_hi], V[j, p_lo - 1:p_hi]) if p_hi >= p_lo else orc.Summary.empty(d)
        band = orc.summarize(q[h], K[j, b_lo - 1:b_hi], V[j, b_lo - 1:b_hi]) if b_hi >= b_lo else orc.Summary.empty(d)
        send[0, h, 0] = torch.from_numpy(_pack(piece, d))
        send[0, h, 1] = torch.from_numpy(_pack(band, d))
    parts = torch.zeros(world, 1, Hq, 2, d + 1)
    exchange(send, parts)
    worst = 0.0
    for h in range(Hq):
        j = h // g
        prefix, band = orc.Summary.empty(d), orc.Summary.empty(d)
        for rk in range(world):  # rank order
            prefix = orc.merge(prefix, _unpack(parts[rk, 0, h, 0].numpy(), 1))
            band = orc.merge(band, _unpack(parts[rk, 0, h, 1].numpy(), 1))
        full = orc.merge(prefix, band)
        ref = orc.summarize(q[h], K[j], V[j])
        worst = max(worst, float(np.linalg.norm(full.acc - ref.acc) / np.linalg.norm(ref.acc)),
                    abs(full.lse - ref.lse))
        ref_prefix = orc.summarize(q[h], K[j, : m - r], V[j, : m - r])
        worst = max(worst, float(np.linalg.norm(prefix.acc - ref_prefix.acc) / np.linalg.norm(ref_prefix.acc)))
    if rank == 0:
        with open(result_path, "w") as fh:
            fh.write(repr(worst))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_gloo_exchange_and_rank_order_merge(tmp_path, world):
    out = tmp_path / "worst.txt"
    tmp.spawn(_worker, args=(world, _free_port(), str(out)), nprocs=world, join=True)
    worst = float(out.read_text())
    assert worst < 1e-5, worst  # f32 exchange of f64 summaries


def test_exchange_single_process_copies():
    send = torch.arange(6.0).view(1, 1, 2, 3)
    parts = torch.zeros(1, 1, 1, 2, 3)
    exchange(send, parts)
    assert torch.equal(parts[0], send)
