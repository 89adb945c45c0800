"""TEST / BASELINE INFRASTRUCTURE ONLY — times the CPU oracle port on host cores.

The reference has no CPU executor of the model, so the CPU
"reference arm" for tokens/sec is this repository's numpy restatement
(oracle/gpt_oracle.py, kind "port") run in float32 with numpy's BLAS threads.
Bounded sample: one transformer layer forward+backward on one full-length
sequence plus the LM head + loss forward+backward on a `head_tokens` slice;
extrapolated to the whole model as  t_seq = L * t_layer + t_head * S/head_tokens.
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


def time_sample(cfg, head_tokens: int = 256, reps: int = 1, seed: int = 0):
    """Returns (seconds per sequence for the whole model, t_layer, t_head_slice)."""
    rng = np.random.default_rng(seed)
    h, S, V = cfg.s_hidden, cfg.s_seq, cfg.s_voc
    P = _layer_params(h, rng)
    G = {k: np.zeros_like(v) for k, v in P.items()}
    x = rng.standard_normal((S, h)).astype(np.float32)
    t_layer = 1e30
    for _ in range(reps):
        t0 = time.perf_counter()
        y, cache = O.layer_forward(P, "l.", x, cfg)
        O.layer_backward(P, G, "l.", np.ones_like(y), cache, cfg)
        t_layer = min(t_layer, time.perf_counter() - t0)
    HP = {"lnf_g": np.ones(h, np.float32), "lnf_b": np.zeros(h, np.float32),
          "w_head": (rng.standard_normal((V, h)) * 0.02).astype(np.float32)}
    HG = {k: np.zeros_like(v) for k, v in HP.items()}
    xs = x[:head_tokens]
    lab = rng.integers(0, V, head_tokens)
    t_head = 1e30
    for _ in range(reps):
        t0 = time.perf_counter()
        O.head_forward_backward(HP, HG, xs, lab, head_tokens)
        t_head = min(t_head, time.perf_counter() - t0)
    per_seq = cfg.n_layers * t_layer + t_head * (S / head_tokens)
    return per_seq, t_layer, t_head


def tokens_per_sec(cfg, head_tokens: int = 256):
    per_seq, t_layer, t_head = time_sample(cfg, head_tokens)
    sample = (f"1 layer fwd+bwd at [{cfg.s_seq} x {cfg.s_hidden}] ({t_layer:.2f} s) + LM head fwd+bwd on "
              f"{head_tokens} tokens ({t_head:.2f} s), float32 numpy, extrapolated to {cfg.n_layers} layers x "
              f"{cfg.s_seq} tokens per sequence")
    return cfg.s_seq / per_seq, sample, per_seq


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
