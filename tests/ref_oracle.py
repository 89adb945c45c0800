"""TEST INFRASTRUCTURE: ctypes loader for the reference-built oracle.

oracle/_ref/libpipesim_ref.so is the reference's own schedule/simulator
(/root/reference/proj/src, unmodified) behind oracle/ref_shim.cpp. Built by
``make -C oracle`` (called from __graft_entry__.build()). Only tests, smoke()
and bench.py's cpu_baseline leg use it.
"""
from __future__ import annotations

import ctypes as C
import os

from paper_2211_05953_b200 import _native as N

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_LIB = os.path.join(ROOT, "oracle", "_ref", "libpipesim_ref.so")

_ref = None


def available() -> bool:
    return os.path.exists(REF_LIB)


def ref():
    global _ref
    if _ref is None:
        L = C.CDLL(REF_LIB)
        P = C.c_void_p
        M, Cf, T = C.POINTER(N.ModelSpecC), C.POINTER(N.ParallelConfigC), C.POINTER(N.TimingModelC)
        sig = {
            "ref_last_error": (C.c_char_p, []),
            "ref_validate": (C.c_int, [M, Cf]),
            "ref_place_stages": (C.c_int, [M, Cf, C.POINTER(C.c_int64), C.c_int64, C.POINTER(C.c_int64),
                                           C.POINTER(C.c_int64)]),
            "ref_build_tasks": (C.c_int, [M, Cf, C.POINTER(P)]),
            "ref_build_accumulation_tasks": (C.c_int, [M, C.c_int32, C.c_int32, C.c_int64, C.POINTER(P)]),
            "ref_graph_n_tasks": (C.c_int64, [P]),
            "ref_graph_n_devices": (C.c_int64, [P]),
            "ref_graph_n_deps": (C.c_int64, [P]),
            "ref_graph_n_program_steps": (C.c_int64, [P]),
            "ref_graph_dump": (None, [P, C.POINTER(N.TaskC), C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                                      C.POINTER(C.c_int32), C.POINTER(C.c_int32)]),
            "ref_graph_destroy": (None, [P]),
            "ref_simulate": (C.c_int, [P, T] + [C.POINTER(C.c_double)] * 5),
            "ref_peak_inflight": (C.c_int, [M, Cf, T, C.POINTER(C.c_int64)]),
            "ref_compute_per_gpu": (C.c_double, [M, Cf]),
            "ref_total_memory": (C.c_int, [M, Cf, C.c_double, C.POINTER(C.c_double)]),
            "ref_feasible": (C.c_int, [M, Cf, C.c_double, C.c_double, C.c_double, C.POINTER(C.c_int32)]),
            "ref_cluster_preset": (C.c_int, [C.c_char_p, C.POINTER(N.ClusterSpecC)]),
            "ref_rank_configs": (C.c_int, [M, C.POINTER(N.ClusterSpecC), C.POINTER(C.c_int32), C.c_int64,
                                           C.POINTER(C.c_int32), C.c_int64]
                                 + [C.POINTER(C.c_int64), C.c_int64] * 5
                                 + [C.c_int32, C.c_int64, C.POINTER(N.ParallelConfigC), C.POINTER(C.c_double),
                                    C.POINTER(C.c_int64)]),
            "ref_timeline_text": (C.c_int, [P, T, C.c_int32, C.c_char_p, C.c_int64, C.POINTER(C.c_int64)]),
            "ref_time_schedule_path": (C.c_int, [M, Cf, T, C.c_int, C.POINTER(C.c_double),
                                                 C.POINTER(C.c_double), C.POINTER(C.c_int64)]),
        }
        for k, (r, a) in sig.items():
            f = getattr(L, k)
            f.restype, f.argtypes = r, a
        _ref = L
    return _ref


def dump_ref_graph(h):
    """(tasks tuple list, dep CSR, prog CSR) from a reference graph handle."""
    L = ref()
    n, nd = L.ref_graph_n_tasks(h), L.ref_graph_n_devices(h)
    tasks = (N.TaskC * max(n, 1))()
    doff = (C.c_int32 * (n + 1))()
    dids = (C.c_int32 * max(1, L.ref_graph_n_deps(h)))()
    poff = (C.c_int32 * (nd + 1))()
    pids = (C.c_int32 * max(1, L.ref_graph_n_program_steps(h)))()
    L.ref_graph_dump(h, tasks, doff, dids, poff, pids)
    return _canon(n, nd, tasks, doff, dids, poff, pids)


def dump_our_graph(h):
    L = N.lib()
    n, nd = L.bfpp_graph_n_tasks(h), L.bfpp_graph_n_devices(h)
    tasks = (N.TaskC * max(n, 1))()
    assert L.bfpp_graph_tasks(h, tasks, n) == 0
    doff = (C.c_int32 * (n + 1))()
    dids = (C.c_int32 * max(1, L.bfpp_graph_n_deps(h)))()
    assert L.bfpp_graph_deps(h, doff, dids) == 0
    poff = (C.c_int32 * (nd + 1))()
    pids = (C.c_int32 * max(1, L.bfpp_graph_n_program_steps(h)))()
    assert L.bfpp_graph_programs(h, poff, pids) == 0
    return _canon(n, nd, tasks, doff, dids, poff, pids)


def _canon(n, nd, tasks, doff, dids, poff, pids):
    ts = [(t.id, t.lane, t.kind, t.priority, t.device, t.peer_device, t.micro_batch, t.stage,
           tuple(dids[doff[i]:doff[i + 1]])) for i, t in enumerate(tasks[:n])]
    progs = [tuple(pids[poff[d]:poff[d + 1]]) for d in range(nd)]
    return {"n_devices": nd, "tasks": ts, "programs": progs}


def ref_build(m: N.ModelSpecC, c: N.ParallelConfigC):
    """Returns (status, dump or error message)."""
    L = ref()
    h = C.c_void_p()
    st = L.ref_build_tasks(C.byref(m), C.byref(c), C.byref(h))
    if st != 0:
        return st, L.ref_last_error().decode()
    try:
        return 0, (dump_ref_graph(h), h)
    finally:
        pass


def ref_simulate(h, t: N.TimingModelC, n_tasks: int, n_dev: int):
    L = ref()
    st = (C.c_double * max(n_tasks, 1))()
    en = (C.c_double * max(n_tasks, 1))()
    lb = (C.c_double * (3 * n_dev))()
    mk, bub = C.c_double(), C.c_double()
    status = L.ref_simulate(h, C.byref(t), st, en, lb, C.byref(mk), C.byref(bub))
    if status != 0:
        return status, L.ref_last_error().decode()
    return 0, (list(st[:n_tasks]), list(en[:n_tasks]), list(lb), mk.value, bub.value)


def ref_timeline_text(h, t: N.TimingModelC, which: int) -> str:
    """The reference's chrome_trace_json (which=0) / gantt_svg (1) of the simulated timeline."""
    L = ref()
    n = C.c_int64()
    assert L.ref_timeline_text(h, C.byref(t), which, None, 0, C.byref(n)) == 0, L.ref_last_error()
    buf = C.create_string_buffer(n.value + 1)
    assert L.ref_timeline_text(h, C.byref(t), which, buf, n.value + 1, C.byref(n)) == 0, L.ref_last_error()
    return buf.value.decode()
