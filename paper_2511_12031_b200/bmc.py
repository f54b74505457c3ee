"""Thin Python binding of libbmc.so (include/bmc.h): argument marshalling only.

Every step of the hot path runs in the library's sm_100a kernels; this module
only passes pointers, sizes and the stream.  It never falls back to a CPU or
PyTorch implementation: if libbmc.so is missing or no CUDA device is present,
the first call raises.

Function names mirror the C ABI (bmc_create, bmc_append, bmc_spec_write,
bmc_sdpa, bmc_commit, bmc_destroy, ...).  ``KVCache`` is a small convenience
wrapper holding one handle (= one layer).
"""
from __future__ import annotations

import ctypes
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
SO_PATH = os.path.join(_HERE, "libbmc.so")

BMC_OK, BMC_ERR_ARG, BMC_ERR_STATE, BMC_ERR_CAPACITY = 0, -1, -2, -3
BMC_ERR_OOM, BMC_ERR_CUDA, BMC_ERR_UNSUPPORTED = -4, -5, -6
BMC_F32, BMC_BF16 = 0, 1
BMC_POLICY_BMC, BMC_POLICY_ITERATIVE, BMC_POLICY_UPFRONT = 0, 1, 2
BMC_PER_ROW = -1
BMC_MAX_B = 256
BMC_OPT_ATTN_CTAS, BMC_OPT_ATTN_PATH, BMC_OPT_ARENA, BMC_OPT_SKIP_PADDING = 1, 2, 3, 4
BMC_OPT_COPY_ON_READ = 5
BMC_OPT_TCK_GROUPS = 6
BMC_OPT_FAULT_OOM = 7
ARENA_VMM, ARENA_POOL, ARENA_REGION = 0, 1, 2
BMC_OPT_TCK_PREFETCH = 8
POLICIES = {"bmc": BMC_POLICY_BMC, "iterative": BMC_POLICY_ITERATIVE,
            "upfront": BMC_POLICY_UPFRONT}
DTYPES = {"f32": BMC_F32, "bf16": BMC_BF16}
_TORCH_DT = {BMC_F32: torch.float32, BMC_BF16: torch.bfloat16}
_NAMES = {0: "OK", -1: "ARG", -2: "STATE", -3: "CAPACITY", -4: "OOM", -5: "CUDA",
          -6: "UNSUPPORTED"}

EXPORTS = ["bmc_create", "bmc_create_ex", "bmc_append", "bmc_append_n", "bmc_spec_write",
           "bmc_sdpa", "bmc_admissible", "bmc_spec_step",
           "bmc_commit", "bmc_commit_rows", "bmc_commit_step", "bmc_commit_path", "bmc_pool_reserve", "bmc_pool_trim", "bmc_spec_write_tree",
           "bmc_spec_step_tree", "bmc_commit_path_step", "bmc_region_reserve",
           "bmc_decode_step", "bmc_destroy", "bmc_stats", "bmc_kv_view",
           "bmc_valid", "bmc_read_cache", "bmc_sync", "bmc_set_option", "bmc_launch_count", "bmc_host_profile", "bmc_last_error"]


class BMCError(RuntimeError):
    def __init__(self, code: int, where: str, msg: str):
        super().__init__(f"{where}: {_NAMES.get(code, code)} ({code}): {msg}")
        self.code = code


class Stats(ctypes.Structure):
    _fields_ = [(n, ctypes.c_longlong) for n in (
        "valid_min", "valid_max", "capacity", "staged", "alloc_events", "copy_events",
        "copied_bytes", "init_written_bytes", "append_written_bytes", "kv_bytes_read",
        "macs", "sdpa_calls")]

    def as_dict(self) -> dict:
        return {n: int(getattr(self, n)) for n, _ in self._fields_}


_lib = None


class _missing:
    """Stand-in for a symbol an experiment build of the library lacks."""

    def __init__(self, name):
        self.name = name
        self.argtypes = self.restype = None

    def __call__(self, *a):
        raise RuntimeError(f"{self.name} is not in this build of libbmc")


def load(path: str = SO_PATH):
    """Load libbmc.so (raises if it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    path = os.environ.get("BMC_LIB", path)   # experiment builds only
    if not os.path.exists(path):
        raise RuntimeError(f"libbmc.so not built at {path}: run __graft_entry__.build()")
    L = ctypes.CDLL(path)
    if path != SO_PATH:   # experiment builds may predate newer diagnostics
        for name in ("bmc_pool_trim", "bmc_host_profile", "bmc_spec_step_tree",
                     "bmc_commit_path_step", "bmc_region_reserve"):
            if not hasattr(L, name):
                setattr(L, name, _missing(name))
    vp, i, ll = ctypes.c_void_p, ctypes.c_int, ctypes.c_longlong
    L.bmc_create.argtypes = [i, i, i, i, i, i, ctypes.POINTER(vp)]
    L.bmc_create_ex.argtypes = [i, i, i, i, i, i, i, i, i, vp, ctypes.POINTER(vp)]
    L.bmc_append.argtypes = [vp, vp, vp]
    L.bmc_append_n.argtypes = [vp, vp, vp, ctypes.c_int]
    L.bmc_admissible.argtypes = [vp, ctypes.c_int]
    L.bmc_spec_step.argtypes = [vp, ctypes.c_int, vp, vp, vp, vp, ctypes.c_int, vp, vp]
    L.bmc_spec_write.argtypes = [vp, vp, vp, i]
    L.bmc_sdpa.argtypes = [vp, vp, i, vp]
    L.bmc_commit.argtypes = [vp, i]
    L.bmc_commit_rows.argtypes = [vp, ctypes.POINTER(ctypes.c_int)]
    L.bmc_commit_step.argtypes = [vp, ctypes.c_int, ctypes.POINTER(ctypes.c_int)]
    L.bmc_pool_reserve.argtypes = [ctypes.c_int, ctypes.c_longlong]
    L.bmc_pool_trim.argtypes = [ctypes.c_int]
    L.bmc_region_reserve.argtypes = [ctypes.c_int, ctypes.c_longlong]
    L.bmc_destroy.argtypes = [vp]
    L.bmc_spec_write_tree.argtypes = [vp, vp, vp, i, ctypes.POINTER(ctypes.c_int)]
    L.bmc_commit_path.argtypes = [vp, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int), i]
    L.bmc_spec_step_tree.argtypes = [vp, i, vp, vp, vp, vp, i, ctypes.POINTER(ctypes.c_int), vp, vp]
    L.bmc_commit_path_step.argtypes = [vp, i, ctypes.POINTER(ctypes.c_int),
                                       ctypes.POINTER(ctypes.c_int), i]
    L.bmc_decode_step.argtypes = [vp, i, vp, vp, vp, vp, i]
    L.bmc_stats.argtypes = [vp, ctypes.POINTER(Stats)]
    L.bmc_kv_view.argtypes = [vp, ctypes.POINTER(vp), ctypes.POINTER(vp), ctypes.POINTER(i)]
    L.bmc_valid.argtypes = [vp, ctypes.POINTER(ctypes.c_int)]
    L.bmc_read_cache.argtypes = [vp, vp, vp]
    L.bmc_sync.argtypes = [vp]
    L.bmc_set_option.argtypes = [vp, i, ll]
    L.bmc_launch_count.argtypes = []
    L.bmc_host_profile.argtypes = [ctypes.POINTER(ll), ctypes.POINTER(ll), i]
    L.bmc_launch_count.restype = ctypes.c_ulonglong
    L.bmc_last_error.argtypes = []
    L.bmc_last_error.restype = ctypes.c_char_p
    for f in EXPORTS:
        if f not in ("bmc_launch_count", "bmc_last_error"):
            getattr(L, f).restype = ctypes.c_int
    _lib = L
    return L


def _check(rc: int, where: str) -> int:
    if rc < 0:
        raise BMCError(rc, where, load().bmc_last_error().decode())
    return rc


def _ptr(x) -> ctypes.c_void_p:
    if x is None:
        return ctypes.c_void_p(0)
    if isinstance(x, torch.Tensor):
        assert x.is_contiguous(), "tensors passed to libbmc must be contiguous"
        return ctypes.c_void_p(x.data_ptr())
    return ctypes.c_void_p(int(x))


# ------------------------------------------------------------- C-ABI mirror

def bmc_create(B, H_kv, H_q, D, r, N_max) -> ctypes.c_void_p:
    h = ctypes.c_void_p()
    _check(load().bmc_create(B, H_kv, H_q, D, r, N_max, ctypes.byref(h)), "bmc_create")
    return h


def bmc_create_ex(B, H_kv, H_q, D, r, N_max, dtype=BMC_BF16, policy=BMC_POLICY_BMC,
                  device=-1, stream=None) -> ctypes.c_void_p:
    h = ctypes.c_void_p()
    s = ctypes.c_void_p(0 if stream is None else int(stream))
    _check(load().bmc_create_ex(B, H_kv, H_q, D, r, N_max, dtype, policy, device, s,
                                ctypes.byref(h)), "bmc_create_ex")
    return h


def bmc_append(h, K, V) -> int:
    return _check(load().bmc_append(h, _ptr(K), _ptr(V)), "bmc_append")


def bmc_append_n(h, K, V, n: int) -> int:
    return _check(load().bmc_append_n(h, _ptr(K), _ptr(V), n), "bmc_append_n")


def bmc_spec_write(h, K_draft, V_draft, k: int) -> int:
    return _check(load().bmc_spec_write(h, _ptr(K_draft), _ptr(V_draft), k), "bmc_spec_write")


def bmc_sdpa(h, Q, n_valid: int, O) -> int:
    return _check(load().bmc_sdpa(h, _ptr(Q), n_valid, _ptr(O)), "bmc_sdpa")


def bmc_pool_reserve(device: int, nbytes: int) -> int:
    """Map nbytes of device memory into the library's growth pool now."""
    return _check(load().bmc_pool_reserve(device, nbytes), "bmc_pool_reserve")


def bmc_pool_trim(device: int = -1) -> int:
    return _check(load().bmc_pool_trim(device), "bmc_pool_trim")


def bmc_region_reserve(device: int, nbytes: int) -> int:
    """(Re)create the two-ended growth region (BMC_OPT_ARENA = 2); 0 frees it."""
    return _check(load().bmc_region_reserve(device, nbytes), "bmc_region_reserve")


def bmc_commit(h, n_accepted: int) -> int:
    return _check(load().bmc_commit(h, n_accepted), "bmc_commit")


def bmc_commit_rows(h, n_accepted) -> int:
    arr = (ctypes.c_int * len(n_accepted))(*[int(x) for x in n_accepted])
    return _check(load().bmc_commit_rows(h, arr), "bmc_commit_rows")


class StepPlan:
    """Pointer arrays for bmc_decode_step over L handles (build once, reuse)."""

    def __init__(self, caches):
        self.L = len(caches)
        self.hs = (ctypes.c_void_p * self.L)(*[c.h.value for c in caches])

    def ptrs(self, tensors):
        return (ctypes.c_void_p * self.L)(*[t.data_ptr() for t in tensors])


def bmc_decode_step(plan: StepPlan, K, V, Q, O, n_valid: int) -> int:
    """K, V, Q, O: ctypes pointer arrays from plan.ptrs(...)."""
    return _check(load().bmc_decode_step(plan.hs, plan.L, K, V, Q, O, n_valid),
                  "bmc_decode_step")


def bmc_admissible(h, k: int) -> int:
    return _check(load().bmc_admissible(h, k), "bmc_admissible")


def bmc_spec_step(plan: StepPlan, K, V, Kd, Vd, k: int, Q, O) -> int:
    """One speculative iteration over the plan's layers; returns k_adm.
    K, V, Kd, Vd, Q, O: ctypes pointer arrays from plan.ptrs(...)."""
    return _check(load().bmc_spec_step(plan.hs, plan.L, K, V, Kd, Vd, k, Q, O), "bmc_spec_step")


def bmc_commit_step(plan: StepPlan, n_accepted) -> int:
    """Per-row commit of every layer of the plan (one zero-fill launch)."""
    arr = (ctypes.c_int * len(n_accepted))(*[int(x) for x in n_accepted])
    return _check(load().bmc_commit_step(plan.hs, plan.L, arr), "bmc_commit_step")


def bmc_spec_write_tree(h, K_draft, V_draft, k: int, parent) -> int:
    par = (ctypes.c_int * max(1, k))(*[int(x) for x in parent])
    return _check(load().bmc_spec_write_tree(h, _ptr(K_draft), _ptr(V_draft), k, par),
                  "bmc_spec_write_tree")


def _paths(paths):
    depth = max([len(p) for p in paths] + [1])
    flat = (ctypes.c_int * (len(paths) * depth))()
    m = (ctypes.c_int * len(paths))()
    for b, pth in enumerate(paths):
        m[b] = len(pth)
        for i, x in enumerate(pth):
            flat[b * depth + i] = int(x)
    return flat, m, depth


def bmc_commit_path(h, paths) -> int:
    """paths: one list of node indices (root first) per batch row."""
    flat, m, depth = _paths(paths)
    return _check(load().bmc_commit_path(h, flat, m, depth), "bmc_commit_path")


def bmc_spec_step_tree(plan: StepPlan, K, V, Kd, Vd, k: int, parent, Q, O) -> int:
    """One token-tree iteration over the plan's layers (parent: k ints,
    breadth-first, -1 = child of the last committed token); returns k_adm."""
    par = (ctypes.c_int * max(1, k))(*[int(x) for x in parent])
    return _check(load().bmc_spec_step_tree(plan.hs, plan.L, K, V, Kd, Vd, k, par, Q, O),
                  "bmc_spec_step_tree")


def bmc_commit_path_step(plan: StepPlan, paths) -> int:
    """Commit one accepted path per batch row in every layer of the plan."""
    flat, m, depth = _paths(paths)
    return _check(load().bmc_commit_path_step(plan.hs, plan.L, flat, m, depth),
                  "bmc_commit_path_step")


def bmc_destroy(h) -> int:
    return _check(load().bmc_destroy(h), "bmc_destroy")


def bmc_stats(h) -> dict:
    s = Stats()
    _check(load().bmc_stats(h, ctypes.byref(s)), "bmc_stats")
    return s.as_dict()


def bmc_kv_view(h):
    k, v, cap = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_int()
    _check(load().bmc_kv_view(h, ctypes.byref(k), ctypes.byref(v), ctypes.byref(cap)),
           "bmc_kv_view")
    return k.value, v.value, cap.value


def bmc_read_cache(h, K_dst, V_dst) -> int:
    return _check(load().bmc_read_cache(h, _ptr(K_dst), _ptr(V_dst)), "bmc_read_cache")


def bmc_valid(h, B: int) -> list:
    arr = (ctypes.c_int * B)()
    _check(load().bmc_valid(h, arr), "bmc_valid")
    return list(arr)


def bmc_sync(h) -> int:
    return _check(load().bmc_sync(h), "bmc_sync")


def bmc_set_option(h, key: int, value: int) -> int:
    return _check(load().bmc_set_option(h, key, value), "bmc_set_option")


HOST_CATS = ("alloc", "release", "launch", "premap", "sync_map")


def bmc_host_profile(reset: bool = True) -> dict:
    """Host time (ms) and calls per growth-path category (include/bmc.h)."""
    ns = (ctypes.c_longlong * 5)()
    calls = (ctypes.c_longlong * 5)()
    _check(load().bmc_host_profile(ns, calls, int(reset)), "bmc_host_profile")
    return {k: (ns[i] / 1e6, int(calls[i])) for i, k in enumerate(HOST_CATS)}


def bmc_launch_count() -> int:
    return int(load().bmc_launch_count())


def bmc_last_error() -> str:
    return load().bmc_last_error().decode()


# ------------------------------------------------------------- convenience

class KVCache:
    """One layer's BMC cache (one handle) on the current CUDA device/stream."""

    def __init__(self, B, H_kv, H_q, D, r, N_max, dtype="bf16", policy="bmc",
                 device=None, stream=None):
        if not torch.cuda.is_available():
            raise RuntimeError("libbmc needs a CUDA device (no CPU fallback exists)")
        self.B, self.H_kv, self.H_q, self.D, self.r, self.N_max = B, H_kv, H_q, D, r, N_max
        self.dtype = DTYPES[dtype] if isinstance(dtype, str) else dtype
        self.policy = POLICIES[policy] if isinstance(policy, str) else policy
        self.device = torch.cuda.current_device() if device is None else device
        self.stream = torch.cuda.current_stream(self.device) if stream is None else stream
        self.h = bmc_create_ex(B, H_kv, H_q, D, r, N_max, self.dtype, self.policy,
                               self.device, self.stream.cuda_stream)
        self.torch_dtype = _TORCH_DT[self.dtype]

    # Rows passed to append / spec_write are read by the next call that
    # touches the cache (include/bmc.h): keep them referenced until then so the
    # torch caching allocator cannot hand their memory to another tensor first.
    # Host tensors are copied on the handle's own copy streams (pinned) and
    # may still be read after the call returns: they are held until sync().
    _keep = ()
    _hold = None

    def _hold_host(self, *xs):
        hs = [x for x in xs if isinstance(x, torch.Tensor) and x.device.type == "cpu"]
        if hs:
            if self._hold is None:
                self._hold = []
            self._hold.extend(hs)

    def append(self, K, V):
        rc = bmc_append(self.h, K, V)
        self._keep = (K, V)
        self._hold_host(K, V)
        return rc

    def append_n(self, K, V, n):
        """Bulk (prompt) append, K/V [B][H_kv][n][D]."""
        rc = bmc_append_n(self.h, K, V, n)
        self._keep = (K, V)
        self._hold_host(K, V)
        return rc

    def spec_write(self, Kd, Vd, k):
        rc = bmc_spec_write(self.h, Kd, Vd, k)
        self._keep = self._keep + (Kd, Vd)
        self._hold_host(Kd, Vd)
        return rc

    def spec_write_tree(self, Kd, Vd, k, parent):
        rc = bmc_spec_write_tree(self.h, Kd, Vd, k, parent)
        self._keep = self._keep + (Kd, Vd)
        self._hold_host(Kd, Vd)
        return rc

    def commit_path(self, paths):
        rc = bmc_commit_path(self.h, paths)
        self._keep = ()
        return rc

    def sdpa(self, Q, n_valid, O=None):
        if O is None:
            t = 1 + self.stats()["staged"]
            O = torch.empty(self.B, self.H_q, t, self.D, dtype=torch.float32,
                            device=Q.device if isinstance(Q, torch.Tensor) else "cuda")
        bmc_sdpa(self.h, Q, n_valid, O)
        self._keep = ()
        self._hold_host(Q, O)
        return O

    def commit(self, n):
        rc = bmc_commit(self.h, n)
        self._keep = ()
        return rc

    def commit_rows(self, n):
        rc = bmc_commit_rows(self.h, n)
        self._keep = ()
        return rc

    def stats(self):
        return bmc_stats(self.h)

    def valid(self):
        return bmc_valid(self.h, self.B)

    def set_option(self, key, value):
        return bmc_set_option(self.h, key, value)

    def kv(self):
        """(K, V) cache contents as torch tensors [B*H_kv][cap][D] (device copies)."""
        cap = self.stats()["capacity"]
        K = torch.empty(self.B * self.H_kv, cap, self.D, dtype=self.torch_dtype,
                        device=f"cuda:{self.device}")
        V = torch.empty_like(K)
        bmc_read_cache(self.h, K, V)
        self._keep = ()
        return K, V

    def sync(self):
        rc = bmc_sync(self.h)
        self._keep = ()
        self._hold = None
        return rc

    def close(self):
        if getattr(self, "h", None) is not None:
            bmc_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


