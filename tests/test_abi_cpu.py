"""CPU-side checks of the C-ABI boundary: libbmc.so loads without a GPU,
exports every symbol include/bmc.h declares, and rejects bad arguments
before touching CUDA."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_2511_12031_b200 import build, bmc
    build.build()
    return bmc.load()


def _declared():
    with open(os.path.join(ROOT, "include", "bmc.h")) as f:
        src = f.read()
    return sorted(set(re.findall(r"^\s*(?:int|unsigned long long|const char\*)\s+(bmc_\w+)\(",
                                 src, re.M)))


def test_exports_every_declared_symbol(lib):
    names = _declared()
    assert len(names) >= 15, names
    for n in names:
        assert hasattr(lib, n), n
    from paper_2511_12031_b200 import bmc
    assert sorted(bmc.EXPORTS) == names


def test_no_libcuda_link():
    so = os.path.join(ROOT, "paper_2511_12031_b200", "libbmc.so")
    out = os.popen(f"ldd {so}").read()
    assert "libcuda.so" not in out


def test_argument_errors_before_cuda(lib):
    from paper_2511_12031_b200 import bmc
    h = ctypes.c_void_p()
    cases = [((0, 1, 1, 128, 1, 8), bmc.BMC_ERR_ARG),       # B < 1
             ((1, 3, 4, 128, 1, 8), bmc.BMC_ERR_ARG),       # H_q % H_kv
             ((1, 1, 1, 128, 0, 8), bmc.BMC_ERR_ARG),       # r < 1
             ((1, 1, 1, 128, 9, 8), bmc.BMC_ERR_ARG),       # r > N_max
             ((1, 1, 1, 96, 1, 8), bmc.BMC_ERR_UNSUPPORTED),  # D
             ((300, 1, 1, 128, 1, 8), bmc.BMC_ERR_UNSUPPORTED)]  # B > BMC_MAX_B
    for dims, code in cases:
        rc = lib.bmc_create_ex(*dims, bmc.BMC_BF16, bmc.BMC_POLICY_BMC, -1, None,
                               ctypes.byref(h))
        assert rc == code, (dims, rc, bmc.bmc_last_error())
        assert bmc.bmc_last_error()
    assert lib.bmc_append(None, None, None) == bmc.BMC_ERR_ARG
    assert lib.bmc_destroy(None) == bmc.BMC_ERR_ARG
    assert lib.bmc_pool_reserve(0, ctypes.c_longlong(-5)) == bmc.BMC_ERR_ARG
    assert lib.bmc_commit_step(None, 1, None) == bmc.BMC_ERR_ARG
    assert lib.bmc_launch_count() == 0


def test_no_oracle_in_product():
    """The product package never imports or links the oracle."""
    pkg = os.path.join(ROOT, "paper_2511_12031_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cpp", ".h")):
                src = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in src.replace("oracle_", "").lower() or f == "synth.py", f
