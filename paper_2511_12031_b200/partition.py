"""Batch x KV-head partitioner for multi-GPU BMC decode (north_star item 5).

Every (batch row b, kv head g) unit of the cache, with its G query heads, is
independent at every decode step (the attention of one unit never reads
another unit), so shards need no collective on the hot path.  A shard is a
rectangle of batch rows x kv heads, so each rank holds ordinary handles of
shape [B_local][H_kv_local].

Rule: split the batch dimension into contiguous, near-equal ranges when
B >= P; otherwise split kv heads (keeping each head's G query heads with it)
when H_kv % (P / B) == 0 with P % B == 0.  Anything else is rejected.
"""
from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class Shard:
    rank: int
    b0: int      # first batch row
    nb: int      # batch rows
    g0: int      # first kv head
    ng: int      # kv heads
    G: int       # query heads per kv head

    @property
    def h_q0(self) -> int:
        return self.g0 * self.G

    @property
    def nh_q(self) -> int:
        return self.ng * self.G

    @property
    def units(self) -> int:
        return self.nb * self.ng


def partition(B: int, H_kv: int, H_q: int, world: int) -> list[Shard]:
    if B < 1 or H_kv < 1 or world < 1 or H_q % H_kv:
        raise ValueError("bad dims")
    G = H_q // H_kv
    if B >= world:
        base, extra = divmod(B, world)
        out, b0 = [], 0
        for r in range(world):
            nb = base + (1 if r < extra else 0)
            out.append(Shard(r, b0, nb, 0, H_kv, G))
            b0 += nb
        return out
    if world % B == 0 and H_kv % (world // B) == 0:
        per_b = world // B
        ng = H_kv // per_b
        return [Shard(r, r // per_b, 1, (r % per_b) * ng, ng, G) for r in range(world)]
    raise ValueError(f"cannot shard B={B}, H_kv={H_kv} over {world} ranks")


def shard_of(B: int, H_kv: int, H_q: int, world: int, rank: int) -> Shard:
    return partition(B, H_kv, H_q, world)[rank]


# ---------------------------------------------------------------- check path
# Collectives used OUTSIDE the hot path only (north_star item 5: "NCCL over
# NVLink is used only to gather outputs for checking").  They move bytes and
# integers; no arithmetic of the method happens here.

LEDGER_KEYS = ("alloc_events", "copy_events", "copied_bytes", "init_written_bytes",
               "append_written_bytes", "kv_bytes_read", "macs", "sdpa_calls", "capacity")


def gather_global(o_local, shard: Shard, B: int, H_q: int, group=None):
    """All ranks' outputs [nb][nh_q][t][D] -> the global [B][H_q][t_max][D] on
    every rank.  One all_gather_into_tensor of equal-size (zero-padded)
    blocks: NCCL for device tensors, gloo for host tensors.  Under
    speculation each rank admits its own draft count (admission uses the
    shard's longest row, reading R10/R11), so t may differ per rank: an
    all_reduce(MAX) of t first, rows tau >= a rank's t stay zero.  Returns
    (global tensor, bytes each rank contributed)."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    shards = partition(B, H_q // shard.G, H_q, world)
    t, D = o_local.shape[2], o_local.shape[3]
    tt = torch.tensor([t], dtype=torch.int64, device=o_local.device)
    dist.all_reduce(tt, op=dist.ReduceOp.MAX, group=group)
    t_max = int(tt.item())
    if t_max != t:
        pad = torch.zeros(o_local.shape[0], o_local.shape[1], t_max, D, dtype=o_local.dtype,
                          device=o_local.device)
        pad[:, :, :t] = o_local
        o_local, t = pad, t_max
    blk = max(s.nb * s.nh_q for s in shards) * t * D
    send = torch.zeros(blk, dtype=o_local.dtype, device=o_local.device)
    send[:o_local.numel()] = o_local.reshape(-1)
    recv = torch.empty(world * blk, dtype=o_local.dtype, device=o_local.device)
    dist.all_gather_into_tensor(recv, send, group=group)
    out = torch.empty(B, H_q, t, D, dtype=o_local.dtype, device=o_local.device)
    for s in shards:
        n = s.nb * s.nh_q * t * D
        out[s.b0:s.b0 + s.nb, s.h_q0:s.h_q0 + s.nh_q] = \
            recv[s.rank * blk:s.rank * blk + n].reshape(s.nb, s.nh_q, t, D)
    return out, blk * o_local.element_size()


def reduce_ledger(stats: list, device, group=None) -> dict:
    """Ledgers (bmc_stats dicts of this rank's layers) reduced over ranks:
    per key the min and max over ranks and layers (allocation / copy counts
    and capacities must agree: every shard sees the same step sequence) and
    the sum (bytes and MACs add up over the disjoint units)."""
    import torch
    import torch.distributed as dist
    vals = torch.tensor([[s[k] for k in LEDGER_KEYS] for s in stats], dtype=torch.int64,
                        device=device)
    lo, hi, tot = vals.min(0).values.clone(), vals.max(0).values.clone(), vals.sum(0).clone()
    dist.all_reduce(lo, op=dist.ReduceOp.MIN, group=group)
    dist.all_reduce(hi, op=dist.ReduceOp.MAX, group=group)
    dist.all_reduce(tot, op=dist.ReduceOp.SUM, group=group)
    return {k: {"min": int(lo[i]), "max": int(hi[i]), "sum": int(tot[i])}
            for i, k in enumerate(LEDGER_KEYS)}
