"""CPU oracle for the BMC decode hot path (ctypes wrapper over liboracle.so).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  The product package ``paper_2511_12031_b200`` never imports it and
shares no code with it (see oracle/oracle.h for what it computes and the
PAPER.md passages each function follows).

Parity status: every function is pinned by ``tests/test_oracle_pins.py``
(incl. the ITERATIVE+SD exact-size ledger and kv_bytes_read closed forms;
``tools/mutate_oracle.sh`` checks that 11 plausible mutations each fail a pin)
(closed forms P:L392/L410/L437, the SD worked example P:L863-866, brute-force
SDPA, fp64 torch SDPA, GQA replication, policy degeneracy).  No function is
"parity unpinned".
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SRC = os.path.join(_HERE, "oracle.c")

F32, BF16 = 0, 1
POLICY_BMC, POLICY_ITERATIVE, POLICY_UPFRONT = 0, 1, 2
STATUS = {0: "OK", -1: "ARG", -2: "STATE", -3: "CAPACITY", -4: "OOM", -6: "UNSUPPORTED"}


class OracleError(RuntimeError):
    def __init__(self, code: int, where: str):
        super().__init__(f"{where}: oracle status {code} ({STATUS.get(code, '?')})")
        self.code = code


class Stats(ctypes.Structure):
    _fields_ = [(n, ctypes.c_longlong) for n in (
        "valid_min", "valid_max", "capacity", "staged", "alloc_events", "copy_events",
        "copied_bytes", "init_written_bytes", "append_written_bytes", "kv_bytes_read",
        "macs", "sdpa_calls")]

    def as_dict(self) -> dict:
        return {n: int(getattr(self, n)) for n, _ in self._fields_}


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (plain C, OpenMP over (b, h) rows)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < max(
            os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "oracle.h"))):
        cmd = ["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-fPIC",
               "-shared", "-std=c11", "-o", _SO, _SRC, "-lm"]
        subprocess.run(cmd, check=True)
    return _SO


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_SO)
        vp, ip, i = ctypes.c_void_p, ctypes.POINTER(ctypes.c_int), ctypes.c_int
        L.oracle_create.argtypes = [i, i, i, i, i, i, i, i, ctypes.POINTER(vp)]
        L.oracle_append.argtypes = [vp, vp, vp]
        L.oracle_append_n.argtypes = [vp, vp, vp, i]
        L.oracle_spec_write.argtypes = [vp, vp, vp, i]
        L.oracle_sdpa.argtypes = [vp, vp, i, vp]
        L.oracle_commit.argtypes = [vp, i]
        L.oracle_commit_rows.argtypes = [vp, ip]
        L.oracle_stats.argtypes = [vp, ctypes.POINTER(Stats)]
        L.oracle_valid.argtypes = [vp, ip]
        L.oracle_read_cache.argtypes = [vp, vp, vp]
        L.oracle_destroy.argtypes = [vp]
        L.oracle_exact_sdpa.argtypes = [vp, vp, vp, i, i, vp]
        L.oracle_spec_write_tree.argtypes = [vp, vp, vp, i, ip]
        L.oracle_commit_path.argtypes = [vp, ip, ip, i]
        for f in ("oracle_create", "oracle_append", "oracle_append_n", "oracle_spec_write", "oracle_sdpa",
                  "oracle_commit", "oracle_commit_rows", "oracle_stats", "oracle_valid",
                  "oracle_read_cache", "oracle_destroy", "oracle_exact_sdpa",
                  "oracle_spec_write_tree", "oracle_commit_path"):
            getattr(L, f).restype = ctypes.c_int
        _lib = L
    return _lib


def set_threads(n: int) -> None:
    """OpenMP threads of the oracle's SDPA loop (the libgomp the oracle
    library loaded; used for bench.py's all-cores and single-core timings)."""
    lib()
    import ctypes.util
    name = ctypes.util.find_library("gomp") or "libgomp.so.1"
    ctypes.CDLL(name).omp_set_num_threads(int(max(1, n)))


def _raw(x, dtype: int) -> np.ndarray:
    """Contiguous raw element bits: fp32 -> float32, bf16 -> uint16 bit patterns.

    Accepts numpy arrays or CPU torch tensors (bf16 tensors are reinterpreted
    as int16 bits, never converted)."""
    try:
        import torch
        if isinstance(x, torch.Tensor):
            x = x.detach().cpu().contiguous()
            if dtype == BF16:
                assert x.dtype == torch.bfloat16, x.dtype
                return x.view(torch.int16).numpy().view(np.uint16)
            assert x.dtype == torch.float32, x.dtype
            return x.numpy()
    except ImportError:  # pragma: no cover
        pass
    x = np.ascontiguousarray(x)
    if dtype == BF16:
        assert x.dtype == np.uint16, x.dtype
    else:
        assert x.dtype == np.float32, x.dtype
    return x


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


class Oracle:
    """One layer's K/V cache under one policy, mirroring the bmc_* call sequence."""

    def __init__(self, B, H_kv, H_q, D, r, N_max, dtype=BF16, policy=POLICY_BMC):
        self.B, self.H_kv, self.H_q, self.D = B, H_kv, H_q, D
        self.r, self.N_max, self.dtype, self.policy = r, N_max, dtype, policy
        h = ctypes.c_void_p()
        rc = lib().oracle_create(B, H_kv, H_q, D, r, N_max, dtype, policy, ctypes.byref(h))
        if rc != 0:
            raise OracleError(rc, "oracle_create")
        self._h = h

    def _check(self, rc, where):
        if rc < 0:
            raise OracleError(rc, where)
        return rc

    def append(self, K, V):
        k, v = _raw(K, self.dtype), _raw(V, self.dtype)
        assert k.size == self.B * self.H_kv * self.D and v.size == k.size
        return self._check(lib().oracle_append(self._h, _ptr(k), _ptr(v)), "oracle_append")

    def append_n(self, K, V, n: int):
        """Bulk (prompt) append of n rows per unit, K/V [B][H_kv][n][D]."""
        if n == 0:
            return self._check(lib().oracle_append_n(self._h, None, None, 0), "append_n")
        k, v = _raw(K, self.dtype), _raw(V, self.dtype)
        assert k.size == self.B * self.H_kv * n * self.D and v.size == k.size
        return self._check(lib().oracle_append_n(self._h, _ptr(k), _ptr(v), n), "oracle_append_n")

    def spec_write(self, Kd, Vd, k: int) -> int:
        if k == 0:
            return self._check(lib().oracle_spec_write(self._h, None, None, 0), "spec_write")
        kd, vd = _raw(Kd, self.dtype), _raw(Vd, self.dtype)
        assert kd.size == self.B * self.H_kv * k * self.D and vd.size == kd.size
        return self._check(lib().oracle_spec_write(self._h, _ptr(kd), _ptr(vd), k),
                           "oracle_spec_write")

    def sdpa(self, Q, n_valid: int) -> np.ndarray:
        q = _raw(Q, self.dtype)
        t = 1 + self.stats()["staged"]
        assert q.size == self.B * self.H_q * t * self.D, (q.size, t)
        out = np.zeros((self.B, self.H_q, t, self.D), dtype=np.float64)
        self._check(lib().oracle_sdpa(self._h, _ptr(q), n_valid, _ptr(out)), "oracle_sdpa")
        return out

    def spec_write_tree(self, Kd, Vd, k: int, parent) -> int:
        par = np.ascontiguousarray(np.asarray(parent, dtype=np.int32))
        assert par.size == k
        if k == 0:
            return self._check(lib().oracle_spec_write_tree(
                self._h, None, None, 0, par.ctypes.data_as(ctypes.POINTER(ctypes.c_int))),
                "spec_write_tree")
        kd, vd = _raw(Kd, self.dtype), _raw(Vd, self.dtype)
        assert kd.size == self.B * self.H_kv * k * self.D and vd.size == kd.size
        return self._check(lib().oracle_spec_write_tree(
            self._h, _ptr(kd), _ptr(vd), k, par.ctypes.data_as(ctypes.POINTER(ctypes.c_int))),
            "oracle_spec_write_tree")

    def commit_path(self, paths):
        """paths: list (one per batch row) of node-index lists (root first)."""
        assert len(paths) == self.B
        depth = max([len(p) for p in paths] + [1])
        arr = np.zeros((self.B, depth), dtype=np.int32)
        m = np.zeros(self.B, dtype=np.int32)
        for b, pth in enumerate(paths):
            arr[b, :len(pth)] = pth
            m[b] = len(pth)
        ip = ctypes.POINTER(ctypes.c_int)
        return self._check(lib().oracle_commit_path(
            self._h, arr.ctypes.data_as(ip), m.ctypes.data_as(ip), depth), "oracle_commit_path")

    def commit(self, n_accepted: int):
        return self._check(lib().oracle_commit(self._h, n_accepted), "oracle_commit")

    def commit_rows(self, n_accepted):
        arr = np.ascontiguousarray(np.asarray(n_accepted, dtype=np.int32))
        assert arr.size == self.B
        return self._check(lib().oracle_commit_rows(
            self._h, arr.ctypes.data_as(ctypes.POINTER(ctypes.c_int))), "oracle_commit_rows")

    def stats(self) -> dict:
        s = Stats()
        self._check(lib().oracle_stats(self._h, ctypes.byref(s)), "oracle_stats")
        return s.as_dict()

    def valid(self) -> np.ndarray:
        arr = np.zeros(self.B, dtype=np.int32)
        self._check(lib().oracle_valid(self._h, arr.ctypes.data_as(
            ctypes.POINTER(ctypes.c_int))), "oracle_valid")
        return arr

    def read_cache(self):
        """Raw cache contents [B*H_kv][cap][D] (float32 or uint16 bf16 bits)."""
        cap = self.stats()["capacity"]
        npdt = np.float32 if self.dtype == F32 else np.uint16
        K = np.zeros((self.B * self.H_kv, cap, self.D), dtype=npdt)
        V = np.zeros_like(K)
        self._check(lib().oracle_read_cache(self._h, _ptr(K), _ptr(V)), "oracle_read_cache")
        return K, V

    def close(self):
        if getattr(self, "_h", None):
            lib().oracle_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def exact_sdpa(q, K, V) -> np.ndarray:
    """Textbook SDPA over exactly the given rows, fp64."""
    q = np.ascontiguousarray(q, dtype=np.float64)
    K = np.ascontiguousarray(K, dtype=np.float64)
    V = np.ascontiguousarray(V, dtype=np.float64)
    n, D = K.shape
    o = np.zeros(D, dtype=np.float64)
    rc = lib().oracle_exact_sdpa(_ptr(q), _ptr(K), _ptr(V), n, D, _ptr(o))
    if rc != 0:
        raise OracleError(rc, "oracle_exact_sdpa")
    return o
