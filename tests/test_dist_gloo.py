"""Multi-process host logic of the head-parallel split (gloo, world size 2, CPU).

The CUDA kernels cannot run here; these tests cover what the multi-GPU path
adds on top of them: the head partition (whole GQA groups per rank), the
output reassembly collective, and the max/sum-over-ranks timing reductions
bench.py uses.
"""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2605_19726_b200.dist import (gather_heads, gather_units, head_range, max_over_ranks, sum_over_ranks,
                                        unit_heads, unit_range)


def test_head_range_partitions():
    for hq, hkv in ((32, 8), (32, 32), (28, 28), (24, 24), (12, 3)):
        for world in (1, 2, 3, 4, 8):
            if world > hkv:
                continue
            got_q, got_kv = [], []
            for r in range(world):
                q0, q1, k0, k1 = head_range(hq, hkv, world, r)
                got_q += list(range(q0, q1))
                got_kv += list(range(k0, k1))
                # every q-head of the slice reads a kv-head of the slice (whole GQA groups)
                grp = hq // hkv
                assert all(k0 <= h // grp < k1 for h in range(q0, q1))
            assert got_q == list(range(hq)) and got_kv == list(range(hkv))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, hq, hkv, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        b, L, d = 2, 5, 4
        full = torch.arange(b * hq * L * d, dtype=torch.float32).reshape(b, hq, L, d)
        q0, q1, _, _ = head_range(hq, hkv, world, rank)
        got = gather_heads(full[:, q0:q1].contiguous(), hq)
        ok = torch.equal(got, full)
        mx = max_over_ranks(float(rank + 1), "cpu")
        sm = sum_over_ranks(float(rank + 1), "cpu")
        q.put((rank, ok, mx, sm))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("hq,hkv", [(32, 8), (6, 3)])
def test_gather_heads_world2(hq, hkv):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, hq, hkv, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(ok for _, ok, _, _ in res), res
    assert all(mx == 2.0 and sm == 3.0 for _, _, mx, sm in res), res


def test_peer_slice_ptrs():
    """out_peers of the fused head-parallel epilogue: every rank's buffer base
    advanced by q0 heads of the full buffer (element strides x element size)."""
    from paper_2605_19726_b200.dist import peer_slice_ptrs
    b, hq, L, d = 2, 32, 1000, 128
    full = torch.empty(b, hq, L, d, dtype=torch.bfloat16)
    for world in (1, 2, 4, 8):
        bases = [0x10000000 * (r + 1) for r in range(world)]
        for rank in range(world):
            q0, q1, _, _ = head_range(hq, 8, world, rank)
            ptrs = peer_slice_ptrs(bases, q0, full.stride(1), full.element_size())
            assert ptrs == [bb + q0 * L * d * 2 for bb in bases]
            # the local head h of this rank lands on global head q0 + h of every copy
            h = q1 - q0 - 1
            assert ptrs[0] + h * full.stride(1) * 2 == bases[0] + (q0 + h) * L * d * 2


def test_unit_range_partitions():
    """SURVEY §8(e) uneven split: flattened (head, q-block) units, contiguous,
    balanced to one unit, every unit owned once; the head span a rank selects
    over covers its units with whole GQA groups."""
    for hq, hkv, nq in ((28, 28, 1024), (32, 8, 1024), (24, 24, 591), (6, 3, 7), (1, 1, 16)):
        for world in (1, 2, 3, 4, 5, 8):
            owned, sizes = [], []
            for r in range(world):
                u0, u1 = unit_range(hq, nq, world, r)
                owned += list(range(u0, u1))
                sizes.append(u1 - u0)
                assert u0 % nq % 2 == 0  # starts on a q-block pair (2p, 2p+1)
                q0, q1, k0, k1 = unit_heads(u0, u1, nq, hq, hkv)
                grp = hq // hkv
                if u1 > u0:
                    assert q0 <= u0 // nq and (u1 - 1) // nq < q1
                    assert q0 == k0 * grp and q1 == k1 * grp
            assert owned == list(range(hq * nq))
            # one pair, plus the one-block tail pairs of odd N_q (at most one per head a rank touches)
            assert max(sizes) - min(sizes) <= 2 + (nq % 2) * (hq // world + 2)
    # M on 8 GPUs: 3.5 heads of work per rank instead of 4/4/4/4/3/3/3/3 (speedup cap 7.0x -> 8x)
    sizes = [unit_range(28, 1024, 8, r)[1] - unit_range(28, 1024, 8, r)[0] for r in range(8)]
    assert sizes == [3584] * 8


def _unit_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        hq, L, d, B = 5, 37, 4, 8  # ragged last block, 5 heads over 3 ranks
        nq = (L + B - 1) // B
        g = torch.Generator().manual_seed(7)
        full = torch.randn(1, hq, L, d, generator=g)
        perm = torch.stack([torch.randperm(L, generator=g) for _ in range(hq)])  # sorted position -> token
        u0, u1 = unit_range(hq, nq, world, rank)
        mine = torch.zeros_like(full)
        for u in range(u0, u1):  # what ba_sparse_attn_units stores: the unit's rows at pi_q positions
            h, gq = divmod(u, nq)
            rows = perm[h, gq * B:min(L, (gq + 1) * B)]
            mine[0, h, rows] = full[0, h, rows]
        keep = mine.clone()
        got = gather_units(mine)
        ok = torch.equal(got, full) and torch.equal(mine, keep)  # out-of-place: the local rows stay as stored
        # a second step on the same (unchanged) local buffer reassembles the same O (no stale rows summed in)
        got2 = gather_units(mine, torch.empty_like(full))
        q.put((rank, ok and torch.equal(got2, full)))
    finally:
        dist.destroy_process_group()


def test_gather_units_world3():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_unit_worker, args=(r, 3, port, q)) for r in range(3)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(ok for _, ok in res), res
