"""The C-ABI library loads and exports exactly what include/okt.h declares
(no GPU needed), and the host-only entry points behave."""
import ctypes
import os
import re

import pytest

from paper_2201_07598_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared():
    hdr = open(os.path.join(ROOT, "include", "okt.h")).read()
    return set(re.findall(r"^(?:int|const char\*)\s+(okt_\w+)\s*\(", hdr, re.M))


def test_library_loads_and_exports_every_declared_symbol():
    L = _lib.lib()
    names = declared()
    assert names == set(_lib.EXPORTS)
    for name in names:
        assert hasattr(L, name), name


def test_library_is_sm100a_cuda_code():
    # The shared object embeds sm_100a SASS (built with -gencode
    # arch=compute_100a,code=sm_100a); no other architecture is present.
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    archs = set(re.findall(r"sm_\d+a?", out.stdout))
    assert archs == {"sm_100a"}, archs


def test_abi_version_and_status_strings():
    L = _lib.lib()
    assert L.okt_abi_version() == 1
    assert L.okt_status_string(0) == b"ok"
    assert L.okt_status_string(2) == b"NumericError"
    assert L.okt_status_string(3) == b"ProtocolError"
    assert L.okt_status_string(4) == b"TransportError"
    assert L.okt_status_string(5) == b"ConfigError"


def test_world_size_must_be_a_power_of_two():
    # ConfigError (transport.cpp:105-107) before any device work.
    L = _lib.lib()
    w = ctypes.c_void_p()
    assert L.okt_world_create_local(ctypes.byref(w), 3, None) == 5
    assert b"power of two" in L.okt_last_error()
    assert L.okt_world_create_local(ctypes.byref(w), 16, None) == 5
    assert L.okt_world_create_local(ctypes.byref(w), 0, None) == 1


def test_null_handles_are_rejected():
    L = _lib.lib()
    assert L.okt_sparse_allreduce(None, None, 0, 1, 1, None, None) == 1
    assert L.okt_get_state(None, None) == 1
    assert L.okt_comm_destroy(None) == 0
