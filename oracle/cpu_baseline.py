"""TEST / BASELINE INFRASTRUCTURE ONLY — times the CPU oracle port on host cores.

The reference has no CPU executor of the model, so the CPU
"reference arm" for tokens/sec is this repository's numpy restatement
(oracle/gpt_oracle.py, kind "port") run in float32 with numpy's BLAS threads.
Bounded sample step (SampleStep): one transformer layer forward+backward on one
full-length sequence plus the LM head + loss forward+backward on a `head_tokens`
slice, counted as the model-flop-weighted number of tokens it represents.
Also times the reference's own schedule path (place_stages + build_tasks +
simulate) from oracle/_ref when it is present.
"""
from __future__ import annotations

import ctypes as C
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
import gpt_oracle as O  # noqa: E402


def blas_threads() -> int:
    try:
        from threadpoolctl import threadpool_info
        info = threadpool_info()
        if info:
            return int(max(i.get("num_threads", 1) for i in info))
    except Exception:
        pass
    return os.cpu_count() or 1


def _layer_params(h, rng):
    m = 4 * h
    f = np.float32
    return {"l.ln1_g": np.ones(h, f), "l.ln1_b": np.zeros(h, f), "l.ln2_g": np.ones(h, f), "l.ln2_b": np.zeros(h, f),
            "l.w_qkv": (rng.standard_normal((3 * h, h)) * 0.02).astype(f),
            "l.w_o": (rng.standard_normal((h, h)) * 0.02).astype(f),
            "l.w_fc1": (rng.standard_normal((m, h)) * 0.02).astype(f),
            "l.w_fc2": (rng.standard_normal((h, m)) * 0.02).astype(f)}


class SampleStep:
    """One bounded CPU step of the workload: one transformer layer forward+backward on a full
    [S x h] sequence plus the LM head + loss forward+backward on `head_tokens` tokens, float32
    numpy on the BLAS threads. Inputs and weights are created once, outside the timed step.
    Its size in tokens is model-flop weighted: the sample's model flops
    S*(72h^2 + 12Sh) + head_tokens*6hV divided by the model's flops per token
    (72Lh^2 + 12Lsh + 6hV), so tokens_equiv / seconds is the model's tokens/s on these cores."""

    def __init__(self, cfg, head_tokens: int = 256, seed: int = 0):
        rng = np.random.default_rng(seed)
        h, S, V = cfg.s_hidden, cfg.s_seq, cfg.s_voc
        head_tokens = min(head_tokens, S)
        self.cfg, self.head_tokens = cfg, head_tokens
        self.P = _layer_params(h, rng)
        self.G = {k: np.zeros_like(v) for k, v in self.P.items()}
        self.x = rng.standard_normal((S, h)).astype(np.float32)
        self.HP = {"lnf_g": np.ones(h, np.float32), "lnf_b": np.zeros(h, np.float32),
                   "w_head": (rng.standard_normal((V, h)) * 0.02).astype(np.float32)}
        self.HG = {k: np.zeros_like(v) for k, v in self.HP.items()}
        self.lab = rng.integers(0, V, head_tokens)
        L = cfg.n_layers
        fpt = 72.0 * L * h * h + 12.0 * L * S * h + 6.0 * h * V
        self.tokens_equiv = (S * (72.0 * h * h + 12.0 * S * h) + head_tokens * 6.0 * h * V) / fpt
        self.desc = (f"1 of {L} layers fwd+bwd at [{S} x {h}] + LM head fwd+bwd on {head_tokens} of {S} tokens per "
                     f"step (float32 numpy); = {self.tokens_equiv:.1f} model-flop-weighted tokens per step")

    def run(self) -> float:
        t0 = time.perf_counter()
        y, cache = O.layer_forward(self.P, "l.", self.x, self.cfg)
        O.layer_backward(self.P, self.G, "l.", np.ones_like(y), cache, self.cfg)
        O.head_forward_backward(self.HP, self.HG, self.x[:self.head_tokens], self.lab, self.head_tokens)
        return time.perf_counter() - t0


def reference_search_path(model_spec_c, n_gpu: int, threads: int):
    """Wall seconds of the reference's configuration search in simulate mode (enumerate_configs +
    rank_configs, search.cpp:136-188) on `threads` host threads."""
    lib = os.path.join(HERE, "_ref", "libpipesim_ref.so")
    if not os.path.exists(lib):
        return None
    L = C.CDLL(lib)
    if not hasattr(L, "ref_time_rank_configs"):
        return None
    L.ref_time_rank_configs.restype = C.c_int
    sec, ne, nr = C.c_double(), C.c_int64(), C.c_int64()
    st = L.ref_time_rank_configs(C.byref(model_spec_c), n_gpu, threads, C.byref(sec), C.byref(ne), C.byref(nr))
    if st != 0:
        return None
    return {"seconds": sec.value, "configs_enumerated": ne.value, "configs_ranked": nr.value, "threads": threads,
            "scoring": "simulate"}


def reference_schedule_path(model_spec_c, config_c, timing_c, reps: int = 100):
    """Seconds per (place_stages + build_tasks) and per simulate() of the compiled reference."""
    lib = os.path.join(HERE, "_ref", "libpipesim_ref.so")
    if not os.path.exists(lib):
        return None
    L = C.CDLL(lib)
    L.ref_time_schedule_path.restype = C.c_int
    b, s, n = C.c_double(), C.c_double(), C.c_int64()
    st = L.ref_time_schedule_path(C.byref(model_spec_c), C.byref(config_c), C.byref(timing_c), reps, C.byref(b),
                                  C.byref(s), C.byref(n))
    if st != 0:
        return None
    return {"build_s": b.value, "simulate_s": s.value, "tasks": n.value, "reps": reps, "threads": 1}
