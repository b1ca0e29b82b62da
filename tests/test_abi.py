"""C ABI: the in-tree library builds, loads and exports every declared symbol.
No compute here (no GPU in the CPU suite); error paths only."""
import ctypes
import os
import re

import numpy as np
import pytest

import __graft_entry__ as ge
from paper_1510_07244_b200 import _native, kernels, pairquad, quadrature

HEADER = os.path.join(ge.ROOT, "include", "gcabem_b200.h")


@pytest.fixture(scope="module")
def lib():
    ge.build_library()
    return _native.lib()


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(gcabem_[a-z0-9_]+)\s*\(", text)))


def test_header_and_binding_agree(lib):
    syms = declared_symbols()
    assert len(syms) >= 18
    assert sorted(_native.EXPORTED) == syms
    raw = ctypes.CDLL(_native.LIB_PATH)
    for s in syms:
        assert hasattr(raw, s), s


def test_sm100a_code_in_library(lib):
    """The fatbin carries sm_100a SASS (cuobjdump lists the ELF arch)."""
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", _native.LIB_PATH], capture_output=True,
                         text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_version_and_argument_errors(lib):
    assert lib.gcabem_version() >= 100
    n = 1
    a = np.zeros((n, 3))
    g = np.ones(n)
    w = np.ones(1)
    out = np.zeros(2 * n)
    rc = lib.gcabem_pair_values(0, 7, 0, 0.0, n, *[a.ctypes.data] * 3, g.ctypes.data,
                                *[a.ctypes.data] * 3, g.ctypes.data, None, 1,
                                np.zeros(2).ctypes.data, np.zeros(2).ctypes.data,
                                w.ctypes.data, out.ctypes.data)
    assert rc == _native.ERR_ARG
    assert "equation" in lib.gcabem_last_error().decode()
    with pytest.raises(ValueError):
        _native.check(rc)


@pytest.mark.skipif(_native.device_count() > 0 if os.path.exists(_native.LIB_PATH) else False,
                    reason="a device is present")
def test_no_device_fails_loudly(lib):
    """No CPU fallback: without a device the product raises BackendError."""
    spec = kernels.KernelSpec("laplace", "single")
    r = quadrature.build_rule("disjoint", 2)
    e = np.zeros((1, 3))
    with pytest.raises(_native.BackendError):
        pairquad.pair_values(spec, e, e, e, np.ones(1), e + 2, e, e, np.ones(1), None,
                             r.x_points, r.y_points, r.weights)


def test_pinned_pool_views_keep_memory(lib):
    if _native.device_count() == 0:
        pytest.skip("cudaHostAlloc needs a driver with a device")
    a = _native.pinned_empty((4, 2), np.complex128)
    a[:] = 1
    v = a[1:3]
    del a
    assert np.all(v == 1)
