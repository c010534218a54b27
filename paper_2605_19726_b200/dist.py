"""Multi-GPU plumbing for the BA-Att hot path (one process per GPU).

Every (batch, head) problem is independent (Alg. 1 is per head, PAPER.md
P:527-569), so the path shards with no data-path collective:

  * weak scaling (default, bench.py): rank r processes its own batch element;
    nothing crosses NVLink.
  * head-parallel (north star's 1/2/4/8-GPU split): rank r owns a contiguous
    range of KV heads — whole GQA groups, so K/V never need replicating — and
    the q-heads that read them; the only collective is one all-gather of O
    along the head dimension to reassemble the output (NCCL over NVLink /
    NVSwitch; gloo in the CPU tests).
"""
from __future__ import annotations

from typing import Tuple

import torch
import torch.distributed as dist


def head_range(heads_q: int, heads_kv: int, world: int, rank: int) -> Tuple[int, int, int, int]:
    """(q0, q1, kv0, kv1): the q-head and kv-head ranges owned by `rank`.
    KV heads are split as evenly as possible; q-heads follow their group."""
    if heads_q % heads_kv:
        raise ValueError("heads_q must be a multiple of heads_kv")
    grp = heads_q // heads_kv
    base, extra = divmod(heads_kv, world)
    kv0 = rank * base + min(rank, extra)
    kv1 = kv0 + base + (1 if rank < extra else 0)
    return kv0 * grp, kv1 * grp, kv0, kv1


def even_split(heads_q: int, heads_kv: int, world: int) -> bool:
    return heads_kv % world == 0


def unit_range(heads: int, n_q: int, world: int, rank: int, pair: int = 2) -> Tuple[int, int]:
    """[u0, u1): rank's share of the flattened work units u = (b*Hq + h)*Nq + g_q
    (SURVEY §8(e) fallback when the heads do not divide by the world size, e.g.
    M's 28 heads on 8 GPUs).  Contiguous; boundaries fall on pairs of query
    blocks (2p, 2p+1) of a head — the tiles the attention kernels pair — so the
    reassembled output is bit-identical to one GPU's; shares differ by at most
    one pair.  `heads` = b*Hq for batched problems."""
    n_p = (n_q + pair - 1) // pair
    base, extra = divmod(heads * n_p, world)
    p0 = rank * base + min(rank, extra)
    p1 = p0 + base + (1 if rank < extra else 0)

    def unit(p):
        return (p // n_p) * n_q + min(pair * (p % n_p), n_q)
    return unit(p0), unit(p1)


def unit_heads(u0: int, u1: int, n_q: int, heads_q: int, heads_kv: int) -> Tuple[int, int, int, int]:
    """(q0, q1, kv0, kv1): the head span (batch 1) a rank must select over to
    run units [u0, u1) — the q-heads they touch, widened to whole GQA groups so
    that the K'/V' copies of every KV head it reads are its own."""
    grp = heads_q // heads_kv
    if u1 <= u0:
        return 0, 0, 0, 0
    h0, h1 = u0 // n_q, (u1 - 1) // n_q + 1
    kv0, kv1 = h0 // grp, (h1 + grp - 1) // grp
    return kv0 * grp, kv1 * grp, kv0, kv1


def gather_units(out_local: torch.Tensor, out_full: torch.Tensor = None, group=None) -> torch.Tensor:
    """Reassemble O after a unit split.  out_local: this rank's zero-filled full-size
    O into which only its own units' rows were ever stored; it is NOT modified, so
    it can be reused step after step (its other rows stay zero).  Every row has
    exactly one writer across the ranks, so a SUM reduction reproduces the 1-GPU
    output bit for bit (x + 0 is exact).  out_full: the reassembled O (allocated
    if None).  NCCL: an out-of-place all-reduce as reduce-scatter + all-gather of
    the flat buffer; gloo: copy + in-place all-reduce."""
    if out_full is None:
        out_full = torch.empty_like(out_local)
    world = dist.get_world_size(group)
    flat, full = out_local.reshape(-1), out_full.view(-1)
    if dist.get_backend(group) == "nccl" and flat.numel() % world == 0:
        chunk = torch.empty(flat.numel() // world, dtype=flat.dtype, device=flat.device)
        dist.reduce_scatter_tensor(chunk, flat, op=dist.ReduceOp.SUM, group=group)
        dist.all_gather_into_tensor(full, chunk, group=group)
    else:
        out_full.copy_(out_local)
        dist.all_reduce(out_full, op=dist.ReduceOp.SUM, group=group)
    return out_full


def gather_heads(out_local: torch.Tensor, heads_q: int, group=None) -> torch.Tensor:
    """Reassemble O [b, Hq, L, d] from per-rank head slices [b, Hq_r, L, d].
    Uses one all_gather_into_tensor when every rank holds the same number of
    heads (the only collective of the path), else all_gather of padded slices."""
    world = dist.get_world_size(group)
    b, hr, L, d = out_local.shape
    if hr * world == heads_q and dist.get_backend(group) == "nccl":
        # gather along a leading dim, then move heads into place
        flat = out_local.transpose(0, 1).contiguous()  # [hr, b, L, d]
        full = torch.empty((world * hr, b, L, d), dtype=out_local.dtype, device=out_local.device)
        dist.all_gather_into_tensor(full, flat, group=group)
        return full.transpose(0, 1).contiguous()
    counts_t = [torch.zeros(1, dtype=torch.int64, device=out_local.device) for _ in range(world)]
    dist.all_gather(counts_t, torch.tensor([hr], dtype=torch.int64, device=out_local.device), group=group)
    counts = [int(c.item()) for c in counts_t]
    hmax = max(counts)
    pad = torch.zeros((hmax, b, L, d), dtype=out_local.dtype, device=out_local.device)
    pad[:hr] = out_local.transpose(0, 1)
    bufs = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(bufs, pad, group=group)
    parts = [bufs[r][:counts[r]] for r in range(world)]
    return torch.cat(parts, dim=0).transpose(0, 1).contiguous()


def max_over_ranks(x: float, device) -> float:
    t = torch.tensor([x], dtype=torch.float64, device=device)
    if dist.is_available() and dist.is_initialized():
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(x: float, device) -> float:
    t = torch.tensor([x], dtype=torch.float64, device=device)
    if dist.is_available() and dist.is_initialized():
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def peer_slice_ptrs(buffer_ptrs, q0: int, head_stride_elems: int, elem_size: int):
    """Device pointers of every rank's full-O buffer advanced to this rank's first
    head q0 — the out_peers of ba_sparse_attn_peers (its kernel adds the local
    head / token offsets with the full buffer's strides)."""
    off = q0 * head_stride_elems * elem_size
    return [int(p) + off for p in buffer_ptrs]


class FusedHeadGather:
    """Head-parallel output reassembly fused into the attention epilogue: the
    full O [b, Hq, L, d] lives in symmetric memory on every rank, and each
    rank's kernel stores its heads' rows into all ranks' copies over NVLink /
    NVSwitch — once per row through the NVLS multicast address when the system
    supports it (ba_sparse_attn_multicast, mc_ptr), else one unicast store per
    peer (ba_sparse_attn_peers); a symmetric-memory barrier then orders the
    reads.  Replaces the NCCL all-gather of gather_heads."""

    def __init__(self, shape_full, dtype, device, q0: int, group=None):
        import torch.distributed._symmetric_memory as symm_mem
        if not dist.is_initialized():
            raise RuntimeError("FusedHeadGather needs an initialised process group (launch under torchrun)")
        group = group or dist.group.WORLD
        self.full = symm_mem.empty(*shape_full, dtype=dtype, device=device)
        self.handle = symm_mem.rendezvous(self.full, group)
        self.peer_ptrs = peer_slice_ptrs(self.handle.buffer_ptrs, q0, self.full.stride(1), self.full.element_size())
        # NVLS multicast address of the same buffer (0 when the NVSwitch / driver has no
        # multicast support): one multimem.st reaches every rank's copy
        mc = int(getattr(self.handle, "multicast_ptr", 0) or 0)
        self.mc_ptr = peer_slice_ptrs([mc], q0, self.full.stride(1), self.full.element_size())[0] if mc else 0

    def barrier(self):
        self.handle.barrier()
