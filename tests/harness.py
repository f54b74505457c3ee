"""Lock-step driver: the same call sequence on libbmc (GPU, through the C ABI)
and on the CPU oracle, with the same seeded inputs, comparing every output.

Tolerances (BASELINE.json north_star): bf16 inputs max-abs <= 2e-3;
fp32 inputs max|diff| <= 1e-5 * max(1, max|O_oracle|) (normwise reading of
"1e-5 relative", R18).  Cache contents, capacities, counters and
committed lengths must be bit-exact / equal.
"""
from __future__ import annotations

import numpy as np
import torch

import oracle as O
from paper_2511_12031_b200 import bmc, synth

TOL_BF16 = 2e-3
TOL_F32 = 1e-5
STAT_KEYS = ("valid_min", "valid_max", "capacity", "staged", "alloc_events", "copy_events",
             "copied_bytes", "init_written_bytes", "append_written_bytes", "kv_bytes_read",
             "macs", "sdpa_calls")


def err_of(o: np.ndarray, ref: np.ndarray, dtype: str) -> float:
    """Error in the units of the tolerance (<= 1 passes)."""
    d = float(np.abs(o.astype(np.float64) - ref).max()) if o.size else 0.0
    if dtype == "bf16":
        return d / TOL_BF16
    return d / (TOL_F32 * max(1.0, float(np.abs(ref).max())))


class Pair:
    def __init__(self, B, H_kv, H_q, D, r, N, dtype="bf16", policy="bmc", seed=1,
                 layer=0, ctas=0, host_io=False, variant="normal"):
        self.B, self.H_kv, self.H_q, self.D, self.r, self.N = B, H_kv, H_q, D, r, N
        self.dtype, self.seed, self.layer, self.variant = dtype, seed, layer, variant
        self.host_io = host_io
        self.gpu = bmc.KVCache(B, H_kv, H_q, D, r, N, dtype=dtype, policy=policy)
        if ctas:
            self.gpu.set_option(bmc.BMC_OPT_ATTN_CTAS, ctas)
        pol = {"bmc": O.POLICY_BMC, "iterative": O.POLICY_ITERATIVE,
               "upfront": O.POLICY_UPFRONT}[policy]
        self.orc = O.Oracle(B, H_kv, H_q, D, r, N, dtype=O.F32 if dtype == "f32" else O.BF16,
                            policy=pol)
        self.step = 0
        self.worst = 0.0
        self.pending = []

    def _dev(self, x: torch.Tensor):
        if self.host_io == "pinned":        # copied on the handle's upload stream
            return x.contiguous().pin_memory()
        return x.contiguous() if self.host_io else x.cuda()

    def append(self):
        x = synth.step_inputs(self.seed, self.layer, self.step, B=self.B, H_kv=self.H_kv,
                              H_q=self.H_q, D=self.D, dtype=self.dtype, want=("k", "v"),
                              variant=self.variant)
        self.step += 1
        self.gpu.append(self._dev(x["k"]), self._dev(x["v"]))
        self.orc.append(x["k"], x["v"])

    def append_n(self, n):
        """Bulk (prompt) append of n rows (the draft stream's [B][H_kv][n][D] layout)."""
        x = synth.step_inputs(self.seed, self.layer, self.step, B=self.B, H_kv=self.H_kv,
                              H_q=self.H_q, D=self.D, dtype=self.dtype, k_draft=max(n, 1),
                              want=("kd", "vd"), variant=self.variant)
        self.step += 1
        kd, vd = x["kd"][:, :, :n].contiguous(), x["vd"][:, :, :n].contiguous()
        self.gpu.append_n(self._dev(kd), self._dev(vd), n)
        self.orc.append_n(kd, vd, n)

    def spec_write(self, k):
        x = synth.step_inputs(self.seed, self.layer, self.step, B=self.B, H_kv=self.H_kv,
                              H_q=self.H_q, D=self.D, dtype=self.dtype, k_draft=k,
                              want=("kd", "vd"))
        self.step += 1
        a = self.gpu.spec_write(self._dev(x["kd"]), self._dev(x["vd"]), k)
        b = self.orc.spec_write(x["kd"], x["vd"], k)
        assert a == b, (a, b)
        return a

    def spec_write_tree(self, k, parent):
        x = synth.step_inputs(self.seed, self.layer, self.step, B=self.B, H_kv=self.H_kv,
                              H_q=self.H_q, D=self.D, dtype=self.dtype, k_draft=k,
                              want=("kd", "vd"))
        self.step += 1
        a = self.gpu.spec_write_tree(self._dev(x["kd"]), self._dev(x["vd"]), k, parent)
        b = self.orc.spec_write_tree(x["kd"], x["vd"], k, parent)
        assert a == b, (a, b)
        return a

    def commit_path(self, paths):
        self.gpu.commit_path(paths)
        self.orc.commit_path(paths)

    def sdpa(self, n_valid=None):
        st = self.orc.stats()
        t = 1 + st["staged"]
        if n_valid is None:
            n_valid = st["valid_max"] if st["valid_min"] == st["valid_max"] else -1
        x = synth.step_inputs(self.seed, self.layer, self.step, B=self.B, H_kv=self.H_kv,
                              H_q=self.H_q, D=self.D, t=t, dtype=self.dtype, want=("q",),
                              variant=self.variant)
        self.step += 1
        if self.host_io == "pinned":
            # asynchronous end to end: checked after the next sync (check_state)
            o = torch.empty(self.B, self.H_q, t, self.D, dtype=torch.float32).pin_memory()
            self.gpu.sdpa(self._dev(x["q"]), n_valid, o)
            ref = self.orc.sdpa(x["q"], n_valid)
            self.pending.append((o, ref, self.step))
            return None, ref
        if self.host_io:
            o = torch.empty(self.B, self.H_q, t, self.D, dtype=torch.float32).pin_memory()
            self.gpu.sdpa(x["q"], n_valid, o)
            self.gpu.sync()              # pinned host output is written asynchronously
            og = o.numpy()
        else:
            og = self.gpu.sdpa(x["q"].cuda(), n_valid).cpu().numpy()
        ref = self.orc.sdpa(x["q"], n_valid)
        e = err_of(og, ref, self.dtype)
        self.worst = max(self.worst, e)
        assert e <= 1.0, f"sdpa mismatch at step {self.step}: {e:.3f} x tolerance"
        return og, ref

    def commit(self, m):
        self.gpu.commit(m)
        self.orc.commit(m)

    def commit_rows(self, m):
        self.gpu.commit_rows(m)
        self.orc.commit_rows(m)

    def drain(self):
        """Compare the outputs of asynchronous (pinned) SDPA calls."""
        if self.pending:
            self.gpu.sync()
            for o, ref, step in self.pending:
                e = err_of(o.numpy(), ref, self.dtype)
                self.worst = max(self.worst, e)
                assert e <= 1.0, f"sdpa mismatch at step {step}: {e:.3f} x tolerance"
            self.pending = []

    def check_state(self):
        self.drain()
        sg, so = self.gpu.stats(), self.orc.stats()
        for key in STAT_KEYS:
            assert sg[key] == so[key], (key, sg[key], so[key])
        assert self.gpu.valid() == list(self.orc.valid())
        Kg, Vg = self.gpu.kv()
        Ko, Vo = self.orc.read_cache()
        if self.dtype == "bf16":
            kg = Kg.cpu().view(torch.int16).numpy().view(np.uint16)
            vg = Vg.cpu().view(torch.int16).numpy().view(np.uint16)
        else:
            kg, vg = Kg.cpu().numpy().view(np.uint32), Vg.cpu().numpy().view(np.uint32)
            Ko, Vo = Ko.view(np.uint32), Vo.view(np.uint32)
        assert kg.shape == Ko.shape, (kg.shape, Ko.shape)
        assert np.array_equal(kg, Ko), "K cache differs"
        assert np.array_equal(vg, Vo), "V cache differs"

    def close(self):
        self.drain()
        self.gpu.close()
        self.orc.close()


class Model:
    """L layers stepped together through the fused C-ABI calls
    (bmc_decode_step / bmc_spec_step / bmc_commit_step, the calls bench.py
    times), each layer in lock-step with its own oracle on the same seeded
    inputs.  check: compare every layer's outputs (else only `check_layers`)."""

    def __init__(self, L, B, H_kv, H_q, D, r, N, dtype="bf16", policy="bmc", seed=5,
                 check_layers=None, options=()):
        self.L, self.B, self.H_kv, self.H_q, self.D = L, B, H_kv, H_q, D
        self.dtype, self.seed = dtype, seed
        self.gpu = [bmc.KVCache(B, H_kv, H_q, D, r, N, dtype=dtype, policy=policy)
                    for _ in range(L)]
        for c in self.gpu:
            for key, val in options:
                c.set_option(key, val)
        pol = {"bmc": O.POLICY_BMC, "iterative": O.POLICY_ITERATIVE,
               "upfront": O.POLICY_UPFRONT}[policy]
        self.orc = [O.Oracle(B, H_kv, H_q, D, r, N, dtype=O.F32 if dtype == "f32" else O.BF16,
                             policy=pol) for _ in range(L)]
        self.plan = bmc.StepPlan(self.gpu)
        self.check_layers = range(L) if check_layers is None else check_layers
        self.step = 0
        self.worst = 0.0
        self.keep = []
        # SDPA ledger of every call (the oracle runs SDPA only on checked steps):
        # per layer K+V bytes of all cap rows, MACs 2*B*H_q*t*cap*D, calls
        self.sdpa_ledger = [dict(kv_bytes_read=0, macs=0, sdpa_calls=0) for _ in range(L)]
        self.eb = 4 if dtype == "f32" else 2

    def _inputs(self, t, k):
        xs = [synth.step_inputs(self.seed, l, self.step, B=self.B, H_kv=self.H_kv,
                                H_q=self.H_q, D=self.D, t=t, k_draft=k, dtype=self.dtype)
              for l in range(self.L)]
        self.step += 1
        return xs

    def _account(self, l, t):
        st = self.orc[l].stats()
        led = self.sdpa_ledger[l]
        led["kv_bytes_read"] += 2 * self.B * self.H_kv * st["capacity"] * self.D * self.eb
        led["macs"] += 2 * self.B * self.H_q * t * st["capacity"] * self.D
        led["sdpa_calls"] += 1

    def _compare(self, outs, refs):
        for l in self.check_layers:
            e = err_of(outs[l].cpu().numpy(), refs[l], self.dtype)
            self.worst = max(self.worst, e)
            assert e <= 1.0, f"layer {l} step {self.step}: {e:.3f} x tolerance"

    def decode_step(self, check=True):
        xs = self._inputs(1, 0)
        st = self.orc[0].stats()
        n = st["valid_max"] + 1 if st["valid_min"] == st["valid_max"] else -1   # BMC_PER_ROW
        dev = [{k: v.cuda() for k, v in x.items()} for x in xs]
        outs = [torch.empty(self.B, self.H_q, 1, self.D, device="cuda") for _ in range(self.L)]
        p = self.plan
        bmc.bmc_decode_step(p, p.ptrs([d["k"] for d in dev]), p.ptrs([d["v"] for d in dev]),
                            p.ptrs([d["q"] for d in dev]), p.ptrs(outs), n)
        self.keep = dev
        refs = []
        for l in range(self.L):
            self.orc[l].append(xs[l]["k"], xs[l]["v"])
            self._account(l, 1)
            refs.append(self.orc[l].sdpa(xs[l]["q"], n) if check else None)
        if check:
            torch.cuda.synchronize()
            self._compare(outs, refs)
        return outs

    def spec_step(self, k, check=True):
        """One speculative iteration (append + k chain drafts + verify) of
        every layer; returns k_adm."""
        k_adm = bmc.bmc_admissible(self.gpu[0].h, k)
        t = 1 + k_adm
        xs = self._inputs(t, max(k, 1))
        dev = [{key: v.cuda() for key, v in x.items()} for x in xs]
        outs = [torch.empty(self.B, self.H_q, t, self.D, device="cuda") for _ in range(self.L)]
        p = self.plan
        got = bmc.bmc_spec_step(p, p.ptrs([d["k"] for d in dev]), p.ptrs([d["v"] for d in dev]),
                                p.ptrs([d["kd"] for d in dev]), p.ptrs([d["vd"] for d in dev]),
                                k, p.ptrs([d["q"] for d in dev]), p.ptrs(outs))
        assert got == k_adm, (got, k_adm)
        self.keep = dev
        refs = []
        for l in range(self.L):
            o = self.orc[l]
            o.append(xs[l]["k"], xs[l]["v"])
            if k > 0:
                assert o.spec_write(xs[l]["kd"], xs[l]["vd"], k) == k_adm
            st = o.stats()
            self._account(l, t)
            nv = st["valid_max"] if st["valid_min"] == st["valid_max"] else -1
            refs.append(o.sdpa(xs[l]["q"], nv) if check else None)
        if check:
            torch.cuda.synchronize()
            self._compare(outs, refs)
        return k_adm

    def spec_step_tree(self, k, parent, check=True):
        """One token-tree iteration (append + a k-node tree + verify) of every
        layer through bmc_spec_step_tree; returns k_adm."""
        k_adm = bmc.bmc_admissible(self.gpu[0].h, k)
        t = 1 + k_adm
        xs = self._inputs(t, max(k, 1))
        dev = [{key: v.cuda() for key, v in x.items()} for x in xs]
        outs = [torch.empty(self.B, self.H_q, t, self.D, device="cuda") for _ in range(self.L)]
        p = self.plan
        got = bmc.bmc_spec_step_tree(p, p.ptrs([d["k"] for d in dev]),
                                     p.ptrs([d["v"] for d in dev]), p.ptrs([d["kd"] for d in dev]),
                                     p.ptrs([d["vd"] for d in dev]), k, parent,
                                     p.ptrs([d["q"] for d in dev]), p.ptrs(outs))
        assert got == k_adm, (got, k_adm)
        self.keep = dev
        refs = []
        for l in range(self.L):
            o = self.orc[l]
            o.append(xs[l]["k"], xs[l]["v"])
            if k > 0:
                assert o.spec_write_tree(xs[l]["kd"], xs[l]["vd"], k, parent) == k_adm
            self._account(l, t)
            refs.append(o.sdpa(xs[l]["q"], -1) if check else None)
        if check:
            torch.cuda.synchronize()
            self._compare(outs, refs)
        return k_adm

    def commit_path_step(self, paths):
        bmc.bmc_commit_path_step(self.plan, paths)
        for o in self.orc:
            o.commit_path(paths)

    def commit_step(self, m):
        bmc.bmc_commit_step(self.plan, m)
        for o in self.orc:
            o.commit_rows(m)

    def check_state(self, layers=None):
        torch.cuda.synchronize()
        for l in (range(self.L) if layers is None else layers):
            sg, so = self.gpu[l].stats(), self.orc[l].stats()
            so.update(self.sdpa_ledger[l])
            for key in STAT_KEYS:
                assert sg[key] == so[key], (l, key, sg[key], so[key])
            assert self.gpu[l].valid() == list(self.orc[l].valid())
            Kg, Vg = self.gpu[l].kv()
            Ko, Vo = self.orc[l].read_cache()
            if self.dtype == "bf16":
                kg = Kg.cpu().view(torch.int16).numpy().view(np.uint16)
                vg = Vg.cpu().view(torch.int16).numpy().view(np.uint16)
            else:
                kg, vg = Kg.cpu().numpy().view(np.uint32), Vg.cpu().numpy().view(np.uint32)
                Ko, Vo = Ko.view(np.uint32), Vo.view(np.uint32)
            assert np.array_equal(kg, Ko) and np.array_equal(vg, Vo), f"layer {l} cache differs"

    def close(self):
        for c in self.gpu:
            c.close()
        for o in self.orc:
            o.close()
