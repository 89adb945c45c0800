"""Generates tests/golden/schedule_golden.json from the REFERENCE implementation.

Run in the build container (needs oracle/_ref/libpipesim_ref.so, built from
/root/reference/proj/src by `make -C oracle`):
    python tests/golden/make_schedule_golden.py
The fixture pins our schedule layer on hosts where the reference is absent.
Every case stores the reference's full task graph (ids, lanes, kinds,
priorities, devices, peers, micro-batches, stages, ordered deps), the
per-device compute programs, and the simulated timeline (exact doubles as
float.hex) under a fixed timing model.
"""
from __future__ import annotations

import ctypes as C
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
sys.path.insert(0, os.path.dirname(HERE))

from paper_2211_05953_b200 import _native as N  # noqa: E402
import ref_oracle as R  # noqa: E402

DP0, DP_PS, DP_FS = 0, 1, 2
NOP, GP, OFOB, DF, BF = 0, 1, 2, 3, 4

# (name, model (L, h, heads, head, mlp, seq, voc), config (dp, tp, pp, mb, smb, loop, variant, sched))
CASES = [
    ("tiny_bf_fs", (4, 128, 4, 32, 512, 64, 1000), (2, 1, 2, 4, 1, 2, DP_FS, BF)),
    ("tiny_df_dp0", (4, 128, 4, 32, 512, 64, 1000), (2, 1, 2, 4, 1, 2, DP0, DF)),
    ("tiny_gpipe_dp0", (4, 128, 4, 32, 512, 64, 1000), (2, 1, 2, 4, 1, 1, DP0, GP)),
    ("tiny_1f1b_dp0", (4, 128, 4, 32, 512, 64, 1000), (2, 1, 2, 4, 1, 1, DP0, OFOB)),
    ("l16_bf_p4v4_mb8", (16, 64, 4, 16, 256, 128, 1000), (1, 1, 4, 8, 1, 4, DP0, BF)),
    ("l16_df_p4v4_mb8", (16, 64, 4, 16, 256, 128, 1000), (1, 1, 4, 8, 1, 4, DP0, DF)),
    ("l16_gpipe_p4_mb8", (16, 64, 4, 16, 256, 128, 1000), (1, 1, 4, 8, 1, 1, DP0, GP)),
    ("l16_1f1b_p4_mb8", (16, 64, 4, 16, 256, 128, 1000), (1, 1, 4, 8, 1, 1, DP0, OFOB)),
    ("l16_bf_fs_dp2", (16, 64, 4, 16, 256, 128, 1000), (2, 1, 4, 8, 1, 4, DP_FS, BF)),
    ("l16_df_fs_dp2", (16, 64, 4, 16, 256, 128, 1000), (2, 1, 4, 8, 1, 4, DP_FS, DF)),
    ("l4_gpipe_fs_dp2", (4, 64, 4, 16, 256, 128, 1000), (2, 1, 4, 8, 1, 1, DP_FS, GP)),
    ("gpt13b_pp2x4_dp4", (24, 2048, 16, 128, 8192, 2048, 50304), (4, 1, 2, 2, 1, 4, DP_FS, BF)),
    ("gpt67b_bf_pp4x2_dp2_mb8", (32, 4096, 32, 128, 16384, 2048, 50304), (2, 1, 4, 8, 1, 2, DP_FS, BF)),
    ("gpt67b_df_pp4x2_dp2_mb8", (32, 4096, 32, 128, 16384, 2048, 50304), (2, 1, 4, 8, 1, 2, DP_FS, DF)),
    ("gpt67b_1f1b_pp4_dp2_mb8", (32, 4096, 32, 128, 16384, 2048, 50304), (2, 1, 4, 8, 1, 1, DP_FS, OFOB)),
    ("gpt13b_l32_pp8x4_mb8", (32, 5760, 45, 128, 23040, 2048, 50304), (1, 1, 8, 8, 1, 4, DP0, BF)),
    ("f52_bf_pp4x4_dp2_mb4", (64, 8192, 64, 128, 32768, 1024, 50304), (2, 1, 4, 4, 1, 4, DP_FS, BF)),
]
TIMING = (1.0, 3.0, 0.05, 0.01, 0.4, 0.2)
INVALID = [
    ("divisibility", (16, 64, 4, 16, 256, 128, 1000), (1, 1, 5, 5, 1, 1, DP0, BF)),
    ("gpt13b_l40_pp8x4", (40, 5120, 40, 128, 20480, 2048, 50304), (1, 1, 8, 8, 1, 4, DP0, BF)),
    ("df_mb_multiple", (8, 64, 4, 16, 256, 128, 1000), (1, 1, 4, 6, 1, 2, DP0, DF)),
    ("mb_lt_pp", (8, 64, 4, 16, 256, 128, 1000), (1, 1, 4, 2, 1, 2, DP0, BF)),
    ("gpipe_loop", (8, 64, 4, 16, 256, 128, 1000), (1, 1, 4, 4, 1, 2, DP0, GP)),
    ("nopipe_pp", (8, 64, 4, 16, 256, 128, 1000), (1, 1, 2, 4, 1, 1, DP0, NOP)),
    ("zero_field", (8, 64, 4, 16, 256, 128, 1000), (0, 1, 2, 4, 1, 1, DP0, BF)),
    ("heads_mismatch", (8, 64, 4, 15, 256, 128, 1000), (1, 1, 2, 4, 1, 1, DP0, BF)),
]


def main():
    out = {"timing": TIMING, "cases": [], "invalid": []}
    L = R.ref()
    for name, m, c in CASES:
        mc, cc = N.ModelSpecC(*m), N.ParallelConfigC(*c)
        st, res = R.ref_build(mc, cc)
        assert st == 0, (name, res)
        dump, h = res
        t = N.TimingModelC(*TIMING)
        st, sim = R.ref_simulate(h, t, len(dump["tasks"]), dump["n_devices"])
        assert st == 0, (name, sim)
        start, end, lb, mk, bub = sim
        peaks = (C.c_int64 * dump["n_devices"])()
        assert L.ref_peak_inflight(C.byref(mc), C.byref(cc), C.byref(t), peaks) == 0
        ns, lps = C.c_int64(), C.c_int64()
        asg = (C.c_int64 * (c[2] * c[5]))()
        assert L.ref_place_stages(C.byref(mc), C.byref(cc), asg, len(asg), C.byref(ns), C.byref(lps)) == 0
        L.ref_graph_destroy(h)
        out["cases"].append({
            "name": name, "model": m, "config": c,
            "assignment": list(asg), "layers_per_stage": lps.value,
            "tasks": [list(t[:8]) + [list(t[8])] for t in dump["tasks"]],
            "programs": [list(p) for p in dump["programs"]],
            "start": [x.hex() for x in start], "end": [x.hex() for x in end],
            "lane_busy": [x.hex() for x in lb], "makespan": mk.hex(), "bubble": bub.hex(),
            "peak_inflight": list(peaks),
            "compute_per_gpu": L.ref_compute_per_gpu(C.byref(mc), C.byref(cc)).hex(),
        })
    for name, m, c in INVALID:
        st = L.ref_validate(C.byref(N.ModelSpecC(*m)), C.byref(N.ParallelConfigC(*c)))
        out["invalid"].append({"name": name, "model": m, "config": c, "status": st,
                               "message": L.ref_last_error().decode() if st else ""})
    path = os.path.join(HERE, "schedule_golden.json")
    with open(path, "w") as f:
        json.dump(out, f, separators=(",", ":"))
    print("wrote", path, os.path.getsize(path), "bytes")


if __name__ == "__main__":
    main()
