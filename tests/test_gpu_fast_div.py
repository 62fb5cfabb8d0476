"""The chain kernel's branch-free division (clv_common.cuh div_rn_fast) against IEEE
division over the operand ranges fast_div_safe() admits: 3 x 10^8 random quotients,
every one bit-identical (for rho^8 / (m (1 - rho)) at the level the epilogue uses it,
1 + quotient).  The parity suite then checks whole chains against the oracle."""

import ctypes

import pytest

pytestmark = pytest.mark.gpu


def test_fast_div_matches_ieee():
    from paper_2304_09781_b200 import _native as N
    lib = N.load()
    lib.clv_debug_fast_div_check.argtypes = [ctypes.c_longlong, ctypes.c_ulonglong, ctypes.POINTER(ctypes.c_longlong)]
    lib.clv_debug_fast_div_check.restype = ctypes.c_int
    bad = ctypes.c_longlong(-1)
    assert lib.clv_debug_fast_div_check(300_000_000, 230409781, ctypes.byref(bad)) == 0
    assert bad.value == 0
