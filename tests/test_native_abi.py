"""The C-ABI library loads and exports every symbol include/clover.h declares (no GPU needed)."""

import ctypes
import os
import re

import pytest

from paper_2304_09781_b200 import _native as N
from paper_2304_09781_b200.core import derive_seed
from paper_2304_09781_b200.errors import DeviceError, InfeasibleGraphError

HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "clover.h")


def declared():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(clv_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    from paper_2304_09781_b200 import build
    build.build()
    lib = N.load()
    names = declared()
    assert len(names) >= 20
    for name in names:
        assert hasattr(lib, name), name
        assert name in N.SIGNATURES, name
    assert lib.clv_abi_version() == 3


def test_host_derive_seed_through_abi():
    lib = N.load()
    import random
    rnd = random.Random(3)
    for _ in range(200):
        parts = [rnd.getrandbits(64) for _ in range(rnd.randint(0, 6))]
        arr = (ctypes.c_uint64 * max(1, len(parts)))(*parts)
        assert lib.clv_derive_seed(arr, len(parts)) == derive_seed(*parts)


def test_status_mapping():
    with pytest.raises(InfeasibleGraphError):
        N.check(5)
    with pytest.raises(DeviceError):
        N.check(100)
    N.check(0)
