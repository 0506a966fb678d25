"""GPU parity of the serving contract: a caller-owned paged KV pool and block table
(BatchDecodeEngine(allocate_kv=False).attach_kv).

Three requests over one pool whose block table is permuted; requests 0 and 1 share
the blocks of a common 160-token prompt (10 full pages) and then decode different
tokens into blocks of their own.  Every request must match the CPU oracle run on its
own token stream, and the shared prefix blocks must be left untouched by the decode.
"""

import dataclasses

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import mac_oracle as orc  # noqa: E402
from golden_util import bf16_round, rel_err  # noqa: E402


def test_external_block_table_shared_prefix_matches_oracle():
    from paper_2604_00235_b200 import BatchDecodeEngine, EngineConfig, SyntheticSpec, gen_synthetic

    B, hq, hkv, W, r, ps = 3, 8, 2, 64, 16, 16
    n0, S = 160, 48
    L = n0 + S
    trs = [gen_synthetic(SyntheticSpec(seq_len=L, d=128, d_v=128, n_q_heads=hq, n_kv_heads=hkv, seed=70 + s))
           for s in range(B)]
    q = np.stack([bf16_round(t.q_pre[:, 0]) for t in trs])
    k = np.stack([bf16_round(t.k_pre[:, 0]) for t in trs])
    v = np.stack([bf16_round(t.v[:, 0]) for t in trs])
    q[1, :n0], k[1, :n0], v[1, :n0] = q[0, :n0], k[0, :n0], v[0, :n0]  # common prompt
    cfg = EngineConfig(d=128, d_v=128, n_q_heads=hq, n_kv_heads=hkv, window=W, band=r, storage="bf16")

    # the caller's pool and table: permuted blocks, rows 0 and 1 share the prompt blocks
    max_blocks = -(-(L + 1) // ps)
    n_blocks = 3 * max_blocks + 7
    perm = np.random.default_rng(3).permutation(n_blocks).astype(np.int32)
    table = np.zeros((B, max_blocks), dtype=np.int32)
    shared = n0 // ps
    table[0] = perm[:max_blocks]
    table[1, :shared] = table[0, :shared]
    table[1, shared:] = perm[max_blocks:2 * max_blocks - shared]
    table[2] = perm[2 * max_blocks:3 * max_blocks]
    kc = torch.zeros(n_blocks, hkv, ps, 128, dtype=torch.bfloat16, device="cuda")
    vc = torch.zeros_like(kc)
    bt = torch.from_numpy(table).cuda()

    eng = BatchDecodeEngine(cfg, B, L + 8, allocate_kv=False, min_chunk=32)
    with pytest.raises(ValueError):  # nothing attached yet: no room
        eng.reserve(1)
    with pytest.raises(ValueError):
        eng.attach_kv([kc], [vc], bt[:2].contiguous())
    eng.attach_kv([kc], [vc], bt)
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to("cuda", torch.bfloat16)  # noqa: E731
    eng.prefill(0, dev(q[:, :n0]), dev(k[:, :n0]), dev(v[:, :n0]))
    assert eng.seq_lens[0].tolist() == [n0] * B
    shared_ids = torch.from_numpy(table[0, :shared]).long().cuda()
    prefix_k = kc[shared_ids].clone()

    ocfg = orc.OracleConfig(d=128, d_v=128, n_q_heads=hq, n_kv_heads=hkv, window=W, band=r, storage="bf16")
    oes = [orc.OracleEngine(ocfg, capacity=L + 8) for _ in range(B)]
    forced = dataclasses.replace(ocfg, refresh_every=1)
    for b, oe in enumerate(oes):
        oe.cfg = forced
        for m in range(1, n0 + 1):
            oe.decode_step(0, q[b, m - 1], k[b, m - 1], v[b, m - 1], m)
        oe.cfg = ocfg
    worst, hits = 0.0, 0
    for m in range(n0 + 1, L + 1):
        res = eng.decode_step(0, dev(q[:, m - 1]), dev(k[:, m - 1]), dev(v[:, m - 1]))
        gh = res.match_hit.cpu().numpy().astype(bool)
        gp = res.match_pos.cpu().numpy()
        go = res.out.double().cpu().numpy()
        for b, oe in enumerate(oes):
            st = oe.decode_step(0, q[b, m - 1], k[b, m - 1], v[b, m - 1], m)
            np.testing.assert_array_equal(gh[b], st.hit)
            np.testing.assert_array_equal(gp[b], st.p)
            hits += int(st.use_hit.sum())
            for h in range(hq):
                worst = max(worst, rel_err(go[b, h], st.outputs[h]))
    assert hits > 0
    assert worst <= 1e-4, worst
    assert torch.equal(kc[shared_ids], prefix_k)  # decode appends never touched the shared prompt
    # request 0's own tail blocks hold its keys, request 1's blocks its own
    last = (L - 1) // ps
    assert not torch.equal(kc[int(table[0, last])], kc[int(table[1, last])])
    assert not eng.check_overflow()
    with pytest.raises(ValueError):  # a position past the caller's table cannot be stepped
        eng.reserve(max_blocks * ps + 1)
