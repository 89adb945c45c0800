"""The C-ABI library loads on a GPU-less host and exports every symbol include/bfpp.h declares."""
import ctypes as C

from paper_2211_05953_b200 import _native as N


def test_exports_every_declared_symbol():
    L = N.lib()
    names = N.declared_symbols()
    assert len(names) > 20
    missing = [n for n in names if not hasattr(L, n)]
    assert not missing, missing


def test_error_codes_and_last_error():
    L = N.lib()
    m = N.ModelSpecC(16, 64, 4, 16, 256, 128, 1000)
    c = N.ParallelConfigC(1, 1, 5, 5, 1, 1, 0, 4)
    assert L.bfpp_validate(C.byref(m), C.byref(c), None) == 2
    assert b"divisibility" in L.bfpp_last_error()
    h = C.c_void_p()
    assert L.bfpp_build_tasks(C.byref(m), C.byref(c), C.byref(h)) == 2
    assert not h.value
