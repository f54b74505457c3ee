"""Seeded synthetic inputs for the BMC decode path (no method arithmetic here).

This module is the ONLY code shared by the CUDA path's callers (bench.py,
tests) and the oracle's callers: it draws random numbers and nothing else.
It holds no allocation, masking, softmax or attention logic.

Recipe:
  * Q, K_new, V_new, K_draft, V_draft: iid N(0, 1) drawn in fp32 by a seeded
    torch CPU generator, then rounded to the cache dtype by round-to-nearest-
    even (torch's ``.to(torch.bfloat16)``); both sides receive the rounded
    bits.  Seed of one (layer, step) stream = hash of (seed, layer, step).
  * variants: "normal"; "peaky" (Q scaled by 8 -> near one-hot softmax);
    "outlier" (K of ~3% of steps scaled by 16 -> scores of O(100), exercises
    max subtraction).
  * acceptance for speculative iterations: m_b = number of leading successes
    of iid Bernoulli(p_accept) over the k_adm drafts of batch row b.
"""
from __future__ import annotations

import torch

_DT = {"bf16": torch.bfloat16, "f32": torch.float32}


def _gen(seed: int, *idx: int) -> torch.Generator:
    h = (int(seed) * 0x9E3779B1) & 0xFFFFFFFFFFFF
    for i in idx:
        h = (h * 1000003 + int(i) + 0x51ED27) & 0xFFFFFFFFFFFF
    g = torch.Generator(device="cpu")
    g.manual_seed(h)
    return g


def torch_dtype(dtype: str) -> torch.dtype:
    return _DT[dtype]


def step_inputs(seed: int, layer: int, step: int, *, B: int, H_kv: int, H_q: int, D: int,
                t: int = 1, k_draft: int = 0, dtype: str = "bf16",
                variant: str = "normal", want=("q", "k", "v", "kd", "vd")) -> dict:
    """Inputs of one decode (or speculative) iteration of one layer.

    Every tensor has its own stream (seed, layer, step, tensor), so any subset
    can be drawn alone.  Returns CPU tensors: q [B][H_q][t][D],
    k/v [B][H_kv][D], kd/vd [B][H_kv][k_draft][D] (when k_draft > 0)."""
    shapes = {"q": (B, H_q, t, D), "k": (B, H_kv, D), "v": (B, H_kv, D),
              "kd": (B, H_kv, k_draft, D), "vd": (B, H_kv, k_draft, D)}
    out = {}
    for tag, name in enumerate(("q", "k", "v", "kd", "vd")):
        if name not in want or (name in ("kd", "vd") and k_draft == 0):
            continue
        x = torch.randn(*shapes[name], generator=_gen(seed, layer, step, tag),
                        dtype=torch.float32)
        if variant == "peaky" and name == "q":
            x = x * 8.0
        elif variant == "outlier" and name == "k":
            if torch.rand(1, generator=_gen(seed, layer, step, 99)).item() < 0.03:
                x = x * 16.0
        elif variant not in ("normal", "peaky", "outlier"):
            raise ValueError(variant)
        out[name] = x.to(_DT[dtype])
    return out


def acceptance(seed: int, it: int, B: int, k_adm: int, p_accept: float = 0.7) -> list:
    """Per-row accepted-draft counts m_b (leading successes of Bernoulli(p))."""
    if k_adm == 0:
        return [0] * B
    g = _gen(seed ^ 0xACCE97, it)
    u = torch.rand(B, k_adm, generator=g)
    m = []
    for b in range(B):
        n = 0
        while n < k_adm and u[b, n].item() < p_accept:
            n += 1
        m.append(n)
    return m


def device_ring(seed: int, n_steps: int, n_layers: int, *, B: int, H_kv: int, H_q: int,
                D: int, t: int = 1, k_draft: int = 0, dtype: str = "bf16",
                device: str = "cuda") -> dict:
    """A ring of n_steps x n_layers iterations' inputs generated on the device
    (benchmark only: keeps the RNG outside the timed region)."""
    g = torch.Generator(device=device)
    g.manual_seed(int(seed))
    dt = _DT[dtype]
    ring = {
        "q": torch.randn(n_steps, n_layers, B, H_q, t, D, generator=g, device=device).to(dt),
        "k": torch.randn(n_steps, n_layers, B, H_kv, D, generator=g, device=device).to(dt),
        "v": torch.randn(n_steps, n_layers, B, H_kv, D, generator=g, device=device).to(dt),
    }
    if k_draft > 0:
        ring["kd"] = torch.randn(n_steps, n_layers, B, H_kv, k_draft, D, generator=g,
                                 device=device).to(dt)
        ring["vd"] = torch.randn(n_steps, n_layers, B, H_kv, k_draft, D, generator=g,
                                 device=device).to(dt)
    return ring
