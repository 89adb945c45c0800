"""Generates tests/golden/report_golden.json from the REFERENCE exporters.

Run in the build container (needs oracle/_ref/libpipesim_ref.so, `make -C oracle`):
    python tests/golden/make_report_golden.py
For a few configurations it stores the reference's chrome_trace_json and gantt_svg
(report.cpp:160-212, 248-290) of the simulated timeline under a fixed timing model, so the
exporters stay pinned on hosts where the reference is absent.
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
from make_schedule_golden import CASES, TIMING  # noqa: E402

PICK = ["tiny_bf_fs", "tiny_df_dp0", "tiny_1f1b_dp0", "l4_gpipe_fs_dp2"]


def main():
    out = []
    t = N.TimingModelC(*TIMING)
    for name, m, c in CASES:
        if name not in PICK:
            continue
        h = C.c_void_p()
        assert R.ref().ref_build_tasks(C.byref(N.ModelSpecC(*m)), C.byref(N.ParallelConfigC(*c)), C.byref(h)) == 0
        out.append({"name": name, "model": m, "config": c, "timing": TIMING,
                    "chrome_trace_json": R.ref_timeline_text(h, t, 0), "gantt_svg": R.ref_timeline_text(h, t, 1)})
        R.ref().ref_graph_destroy(h)
    with open(os.path.join(HERE, "report_golden.json"), "w") as f:
        json.dump(out, f, indent=0)
    print("wrote", len(out), "cases")


if __name__ == "__main__":
    main()
