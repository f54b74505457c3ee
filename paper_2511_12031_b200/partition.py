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
