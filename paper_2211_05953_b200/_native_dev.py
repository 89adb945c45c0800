"""Prototypes of the device-side C ABI entry points (kernels + executor)."""
from __future__ import annotations

import ctypes as C

PROTOS: dict = {}


def bind(L):
    for name, (res, args) in PROTOS.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
