"""Batch x KV-head partitioner (north_star item 5) and the multi-process
check path, on CPU with the gloo backend (world_size 2 and 4).

Each rank runs its shard of a small decode through the oracle (the compute
stand-in on CPU), all-gathers its outputs, and rank 0 checks that the
gathered result equals a single-process run over the whole batch: shards are
independent units, no collective is needed inside the step.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2511_12031_b200.partition import Shard, partition, shard_of


def test_partition_covers_every_unit_once():
    for B, H_kv, H_q, P in [(16, 32, 32, 1), (16, 32, 32, 8), (64, 8, 32, 8), (8, 8, 64, 8),
                            (10, 4, 8, 4), (2, 8, 16, 8), (1, 8, 64, 8), (3, 2, 2, 2)]:
        shards = partition(B, H_kv, H_q, P)
        assert len(shards) == P
        seen = np.zeros((B, H_kv), dtype=int)
        for s in shards:
            seen[s.b0:s.b0 + s.nb, s.g0:s.g0 + s.ng] += 1
            assert s.G == H_q // H_kv and s.nh_q == s.ng * s.G
        assert (seen == 1).all(), (B, H_kv, P)
        sizes = [s.units for s in shards]
        assert max(sizes) - min(sizes) <= H_kv      # balanced to within one batch row


def test_partition_rejects_unshardable():
    with pytest.raises(ValueError):
        partition(2, 3, 3, 4)        # 4 ranks cannot split 2 rows x 3 heads evenly
    with pytest.raises(ValueError):
        partition(1, 3, 4, 1)        # H_q % H_kv


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, B, H_kv, H_q, D, N, r, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle as O
    from paper_2511_12031_b200 import synth
    sh = shard_of(B, H_kv, H_q, world, rank)
    orc = O.Oracle(sh.nb, sh.ng, sh.nh_q, D, r, N, dtype=O.BF16, policy=O.POLICY_BMC)
    outs = []
    for n in range(1, N + 1):
        x = synth.step_inputs(5, 0, n, B=B, H_kv=H_kv, H_q=H_q, D=D, dtype="bf16")
        k = x["k"][sh.b0:sh.b0 + sh.nb, sh.g0:sh.g0 + sh.ng].contiguous()
        v = x["v"][sh.b0:sh.b0 + sh.nb, sh.g0:sh.g0 + sh.ng].contiguous()
        qq = x["q"][sh.b0:sh.b0 + sh.nb, sh.h_q0:sh.h_q0 + sh.nh_q].contiguous()
        orc.append(k, v)
        outs.append(torch.from_numpy(orc.sdpa(qq, n)))
    mine = torch.stack(outs)                                     # [N][nb][nh_q][1][D]
    flat = mine.reshape(-1).contiguous()
    sizes = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(sizes, torch.tensor([flat.numel()]))
    bufs = [torch.zeros(int(s.item()), dtype=torch.float64) for s in sizes]
    dist.all_gather(bufs, flat)                                  # check path only
    if rank == 0:
        full = torch.zeros(N, B, H_q, 1, D, dtype=torch.float64)
        for rr, buf in enumerate(bufs):
            s = shard_of(B, H_kv, H_q, world, rr)
            full[:, s.b0:s.b0 + s.nb, s.h_q0:s.h_q0 + s.nh_q] = buf.reshape(
                N, s.nb, s.nh_q, 1, D)
        ref = O.Oracle(B, H_kv, H_q, D, r, N, dtype=O.BF16, policy=O.POLICY_BMC)
        ok = True
        for n in range(1, N + 1):
            x = synth.step_inputs(5, 0, n, B=B, H_kv=H_kv, H_q=H_q, D=D, dtype="bf16")
            ref.append(x["k"], x["v"])
            o = ref.sdpa(x["q"], n)
            ok &= bool(np.array_equal(full[n - 1].numpy(), o))
        q.put(ok)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,B,H_kv,H_q", [(2, 4, 2, 4), (4, 2, 4, 8)])
def test_gloo_sharded_decode_equals_single_process(world, B, H_kv, H_q):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, B, H_kv, H_q, 16, 24, 5, q))
             for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
        assert p.exitcode == 0
    assert q.get(timeout=5) is True
