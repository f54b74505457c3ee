"""Multi-rank plumbing of the batch x kv-head partitioner:
the check path's gather (all_gather_into_tensor) and ledger reduction on
gloo (CPU), and two libbmc ranks sharing the one GPU (gloo) whose gathered
outputs are compared element by element with the oracle of the global batch.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2511_12031_b200.partition import LEDGER_KEYS, gather_global, reduce_ledger, shard_of


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _spawn(fn, world, *args):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=fn, args=(r, world, port, q, *args)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=600)
        assert p.exitcode == 0, p.exitcode
    return q.get(timeout=5)


def _gather_worker(rank, world, port, q, B, H_kv, H_q, t, D):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sh = shard_of(B, H_kv, H_q, world, rank)
    # every element encodes its global (b, h_q, tau, d) coordinates
    b = torch.arange(sh.b0, sh.b0 + sh.nb).view(-1, 1, 1, 1)
    h = torch.arange(sh.h_q0, sh.h_q0 + sh.nh_q).view(1, -1, 1, 1)
    tau = torch.arange(t).view(1, 1, -1, 1)
    d = torch.arange(D).view(1, 1, 1, -1)
    mine = (((b * H_q + h) * t + tau) * D + d).to(torch.float32)
    out, nbytes = gather_global(mine.contiguous(), sh, B, H_q)
    stats = [{k: (rank + 1) * (i + 1) * (10 if k != "alloc_events" else 1) for k in LEDGER_KEYS}
             for i in range(2)]
    led = reduce_ledger(stats, "cpu")
    if rank == 0:
        ref = torch.arange(B * H_q * t * D, dtype=torch.float32).view(B, H_q, t, D)
        ok = torch.equal(out, ref) and nbytes > 0
        ok &= led["alloc_events"]["min"] == 1 and led["alloc_events"]["max"] == 2 * world
        ok &= led["copied_bytes"]["sum"] == sum(10 * (r + 1) * 3 for r in range(world))
        q.put(bool(ok))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,B,H_kv,H_q", [(2, 4, 2, 8), (3, 5, 2, 4), (4, 2, 4, 8)])
def test_gather_global_and_ledger_gloo(world, B, H_kv, H_q):
    """Uneven batch shards (B=5 over 3 ranks) and kv-head shards (B < P):
    the padded all_gather_into_tensor reassembles the global [B][H_q][t][D]
    exactly; the ledger reduction gives min / max / sum over ranks and layers."""
    assert _spawn(_gather_worker, world, B, H_kv, H_q, 3, 4) is True


def _libbmc_worker(rank, world, port, q, B, H_kv, H_q, D, r, N, L):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)                 # both ranks share the box's one GPU
    import oracle as O
    from paper_2511_12031_b200 import bmc, synth
    from paper_2511_12031_b200.partition import partition
    sh = shard_of(B, H_kv, H_q, world, rank)
    caches = [bmc.KVCache(sh.nb, sh.ng, sh.nh_q, D, r, N, dtype="bf16") for _ in range(L)]
    plan = bmc.StepPlan(caches)
    # rank 0 checks: one oracle per (shard, layer).  Each rank is an
    # independent BMC instance over its units: under per-row acceptance the
    # draft admission (cap - longest row of the shard, reading R10/R11) and
    # the growth schedule are the shard's own, so the reference of a shard is
    # the oracle of that shard's rows and heads.
    shards = partition(B, H_kv, H_q, world)
    orcs = {(s.rank, l): O.Oracle(s.nb, s.ng, s.nh_q, D, r, N, dtype=O.BF16,
                                  policy=O.POLICY_BMC)
            for s in shards for l in range(L)} if rank == 0 else None
    cut = lambda x, s, h0, nh: x[s.b0:s.b0 + s.nb, h0:h0 + nh].contiguous()
    kvcut = lambda x, s: cut(x, s, s.g0, s.ng)
    qcut = lambda x, s: cut(x, s, s.h_q0, s.nh_q)
    worst, ok, step, n = 0.0, True, 0, 0
    for it in range(28):                       # 24 decode steps, then 4 speculative iterations
        spec = it >= 24
        k = 4 if spec else 0
        k_adm = bmc.bmc_admissible(caches[0].h, k) if spec else 0
        t = 1 + k_adm
        xs = [synth.step_inputs(77, l, step, B=B, H_kv=H_kv, H_q=H_q, D=D, t=1 + k,
                                k_draft=max(k, 1)) for l in range(L)]
        step += 1
        dv = [{"k": kvcut(x["k"], sh).cuda(), "v": kvcut(x["v"], sh).cuda(),
               "kd": kvcut(x["kd"], sh).cuda(), "vd": kvcut(x["vd"], sh).cuda(),
               "q": qcut(x["q"], sh)[:, :, :t].contiguous().cuda()} for x in xs]
        outs = [torch.empty(sh.nb, sh.nh_q, t, D, device="cuda") for _ in range(L)]
        P = plan.ptrs
        if spec:
            got = bmc.bmc_spec_step(plan, P([d["k"] for d in dv]), P([d["v"] for d in dv]),
                                    P([d["kd"] for d in dv]), P([d["vd"] for d in dv]), k,
                                    P([d["q"] for d in dv]), P(outs))
            ok &= got == k_adm
        else:
            n += 1
            bmc.bmc_decode_step(plan, P([d["k"] for d in dv]), P([d["v"] for d in dv]),
                                P([d["q"] for d in dv]), P(outs), n)
        torch.cuda.synchronize()
        m = synth.acceptance(5, it, B, k) if spec else None
        for l in range(L):
            full, _ = gather_global(outs[l].cpu(), sh, B, H_q)      # [B][H_q][t_max][D]
            if rank == 0:
                for s in shards:
                    o = orcs[(s.rank, l)]
                    x = xs[l]
                    o.append(kvcut(x["k"], s), kvcut(x["v"], s))
                    ka = o.spec_write(kvcut(x["kd"], s), kvcut(x["vd"], s), k) if spec else 0
                    st = o.stats()
                    nv = st["valid_max"] if st["valid_min"] == st["valid_max"] else -1
                    ref = o.sdpa(qcut(x["q"], s)[:, :, :1 + ka].contiguous(), nv)
                    got_s = full[s.b0:s.b0 + s.nb, s.h_q0:s.h_q0 + s.nh_q, :1 + ka].numpy()
                    worst = max(worst, float(np.abs(got_s - ref).max()))
                    if spec:
                        o.commit_rows([min(mb, ka) for mb in m[s.b0:s.b0 + s.nb]])
        if spec:
            bmc.bmc_commit_step(plan, [min(mb, k_adm) for mb in m[sh.b0:sh.b0 + sh.nb]])
    torch.cuda.synchronize()
    led = reduce_ledger([c.stats() for c in caches], "cpu")
    if rank == 0:
        so = [o.stats() for o in orcs.values()]
        for key in ("alloc_events", "copy_events", "capacity", "sdpa_calls"):
            ok &= led[key]["min"] == min(s[key] for s in so)
            ok &= led[key]["max"] == max(s[key] for s in so)
        for key in ("copied_bytes", "init_written_bytes", "append_written_bytes",
                    "kv_bytes_read", "macs"):
            ok &= led[key]["sum"] == sum(s[key] for s in so)
        q.put((bool(ok), worst))
    for c in caches:
        c.close()
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("B,H_kv,H_q", [(4, 2, 8), (1, 4, 16)])
def test_two_libbmc_ranks_vs_oracle(B, H_kv, H_q):
    """Two ranks (one process each, sharing the GPU, gloo) decode their shard
    (batch rows, or kv heads when B < P) of 2 layers through bmc_decode_step
    and speculative bmc_spec_step / bmc_commit_step iterations; at every
    step the outputs are gathered with all_gather_into_tensor and rank 0
    compares them element by element with the oracles of the shards
    (max-abs <= 2e-3; plain decode: identical to the global batch's oracle,
    speculation: each shard admits its own drafts); the all-reduced ledgers
    equal the oracles' (count min / max over ranks, bytes and MACs summed)."""
    import __graft_entry__
    __graft_entry__.build()
    ok, worst = _spawn(_libbmc_worker, 2, B, H_kv, H_q, 128, 8, 64, 2)
    assert ok and worst <= 2e-3, (ok, worst)
