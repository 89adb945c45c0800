"""TEST INFRASTRUCTURE: runs the executor on a config and compares with the CPU oracle.

Used in-process by tests/test_executor_gpu.py (1 GPU) and, per rank, by
tests/dist_worker.py under torchrun (N GPUs)."""
from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.insert(0, ROOT)

import gpt_oracle as O  # noqa: E402

from paper_2211_05953_b200 import pipesim as ps  # noqa: E402
from paper_2211_05953_b200.model import GPTConfig, flatten_stage, unflatten_stage  # noqa: E402,F401

LR = 1e-3
TINY = GPTConfig.preset("tiny")


def make_case(cfg: GPTConfig, config: ps.ParallelConfig, seed=7):
    params = O.init_params(cfg, seed=seed, std=0.05)
    rng = np.random.default_rng(seed + 1)
    tokens = rng.integers(0, cfg.s_voc, (config.n_dp, config.n_mb, config.s_mb, cfg.s_seq + 1)).astype(np.int32)
    return params, tokens


def run_rank(executor_factory, cfg, config, params, tokens, rank):
    """Runs 1 step without optimizer (grads) then 1 step with (weights) on this rank.
    Returns dict with loss, per-stage (grads, lo, hi), per-stage (params, lo, hi)."""
    n_stage = config.n_pp * config.n_loop
    dp = rank // config.n_pp
    ex = executor_factory(skip_optimizer=True)
    for s in ex.local_stages:
        flat = flatten_stage(params, cfg, s, n_stage)
        ex.set_stage_params(s, flat)
        w16, lo, hi = ex.get_stage_weights16(s)
        own = ~np.isnan(w16[lo:hi])  # sharded variants: this rank's slices only
        want = torch_bf16(flat[lo:hi])
        assert own.any() and np.array_equal(w16[lo:hi][own], want[own]), \
            f"stage {s}: bf16 compute weights differ after set_params"
    loss = ex.step(tokens[dp])
    grads = {s: ex.get_stage_grads(s) for s in ex.local_stages}
    ex.close()
    ex = executor_factory(skip_optimizer=False, lr=LR)
    for s in ex.local_stages:
        ex.set_stage_params(s, flatten_stage(params, cfg, s, n_stage))
    loss2 = ex.step(tokens[dp])
    newp = {s: ex.get_stage_params(s) for s in ex.local_stages}
    for s in ex.local_stages:  # the bf16 copy the next step computes with is the rounded master
        w16, lo, hi = ex.get_stage_weights16(s)
        p, plo, phi = newp[s]
        own = ~np.isnan(w16) & ~np.isnan(p)
        assert own.any() and np.array_equal(w16[own], torch_bf16(p[own])), f"stage {s}: bf16 weights != bf16(master)"
    ex.close()
    return {"loss": loss, "loss2": loss2, "grads": grads, "params": newp}


def make_steps_case(cfg: GPTConfig, config: ps.ParallelConfig, n_steps: int, seed=7):
    """Initial parameters + a fresh token batch per step: tokens [n_steps, n_dp, n_mb, s_mb, S+1]."""
    params = O.init_params(cfg, seed=seed, std=0.05)
    rng = np.random.default_rng(seed + 1)
    tokens = rng.integers(0, cfg.s_voc, (n_steps, config.n_dp, config.n_mb, config.s_mb, cfg.s_seq + 1))
    return params, tokens.astype(np.int32)


def run_rank_steps(executor_factory, cfg, config, params, tokens, rank):
    """n_steps optimizer steps on ONE executor (tokens[k] at step k): exercises everything that
    only happens from step 2 on -- gradient buffers overwritten by each unit's first backward,
    Adam moments + bias correction at steps >= 2, re-used receive slots / flags (step-sequence
    waits), the two-step run-ahead ring, per-segment early reduce-scatter across steps.
    Returns {"losses": [...], "params": {stage: (p, lo, hi)}}."""
    n_stage = config.n_pp * config.n_loop
    dp = rank // config.n_pp
    ex = executor_factory(skip_optimizer=False, lr=LR)
    for s in ex.local_stages:
        ex.set_stage_params(s, flatten_stage(params, cfg, s, n_stage))
    losses = [ex.step(tokens[k][dp]) for k in range(tokens.shape[0])]
    newp = {s: ex.get_stage_params(s) for s in ex.local_stages}
    for s in ex.local_stages:
        w16, lo, hi = ex.get_stage_weights16(s)
        p, _, _ = newp[s]
        own = ~np.isnan(w16) & ~np.isnan(p)
        assert own.any() and np.array_equal(w16[own], torch_bf16(p[own])), f"stage {s}: bf16 weights != bf16(master)"
    ex.close()
    return {"losses": losses, "params": newp}


def oracle_steps(cfg, config, params, tokens):
    """The oracle's n_steps of (loss, gradient, Adam) on the same batches: per-step replica
    losses [n_steps][n_dp] and the final float64 parameters."""
    P = {k: np.asarray(a, np.float64) for k, a in params.items()}
    m = {k: np.zeros_like(v) for k, v in P.items()}
    v = {k: np.zeros_like(v) for k, v in P.items()}
    rl = []
    for k in range(tokens.shape[0]):
        rl.append([O.loss_and_grads(P, tokens[k][d].reshape(-1, cfg.s_seq + 1), cfg)[0]
                   for d in range(config.n_dp)])
        _, grads = O.loss_and_grads(P, tokens[k].reshape(-1, cfg.s_seq + 1), cfg)
        P = O.adam_step(P, grads, m, v, k + 1, LR, 0.9, 0.95, 1e-8, 0.0)
    return rl, P


def compare_steps(cfg, config, results, params, tokens):
    """Multi-step parity. Tolerances (bf16 weights/activations, f32 accumulation and optimizer):
      replica loss at every step: |dl| <= 2e-3 * loss
      weights after n steps: |p - p_ref| <= 2 * n * lr everywhere (each Adam step moves an element
      by at most ~lr, so two trajectories can separate by at most 2 lr per step), and within
      0.1 * lr on >= 90 % of the elements of every tensor.
    """
    n_stage = config.n_pp * config.n_loop
    n = tokens.shape[0]
    rloss, newp = oracle_steps(cfg, config, params, tokens)
    report = {"losses": [], "weights_frac_close": {}, "weights_max_dev_lr": {}}
    for r, res in enumerate(results):
        dp, pp = r // config.n_pp, r % config.n_pp
        if pp == (n_stage - 1) % config.n_pp:
            for k in range(n):
                got, ref = res["losses"][k], rloss[k][dp]
                assert abs(got - ref) <= 2e-3 * ref, (k, got, ref)
                report["losses"].append((k, got, ref))
    for s in range(n_stage):
        full_p = np.full(flatten_stage(params, cfg, s, n_stage).size, np.nan, np.float32)
        for res in results:
            if s in res["params"]:
                p, lo, hi = res["params"][s]
                own = ~np.isnan(p[lo:hi])
                full_p[lo:hi][own] = p[lo:hi][own]
        assert not np.isnan(full_p).any(), f"stage {s}: parameter shards do not cover the stage"
        got_p = unflatten_stage(full_p, cfg, s, n_stage)
        for k in got_p:
            dpar = np.abs(got_p[k] - newp[k])
            report["weights_max_dev_lr"][k] = float(dpar.max() / LR)
            assert dpar.max() <= 2 * n * LR + 1e-6, (k, dpar.max() / LR)
            frac = float((dpar <= 0.1 * LR).mean())
            report["weights_frac_close"][k] = frac
            assert frac >= 0.90, (k, frac)
    return report


def torch_bf16(x):
    """Round-to-nearest-even float32 -> bf16 -> float32 (the kernels' __float2bfloat16_rn)."""
    import torch
    return torch.from_numpy(np.ascontiguousarray(x, np.float32)).bfloat16().float().numpy()


def oracle(cfg, config, params, tokens):
    flat_tokens = tokens.reshape(-1, cfg.s_seq + 1)
    loss, grads = O.loss_and_grads(params, flat_tokens, cfg)
    m = {k: np.zeros_like(v) for k, v in params.items()}
    v = {k: np.zeros_like(v) for k, v in params.items()}
    newp = O.adam_step({k: np.asarray(a, np.float64) for k, a in params.items()}, grads, m, v, 1, LR, 0.9, 0.95,
                       1e-8, 0.0)
    replica_loss = [O.loss_and_grads(params, tokens[d].reshape(-1, cfg.s_seq + 1), cfg)[0]
                    for d in range(config.n_dp)]
    return loss, grads, newp, replica_loss


def compare(cfg, config, results, params, tokens):
    """results: list over ranks of run_rank dicts. Returns a report dict; raises AssertionError on mismatch.

    Tolerances (bf16 weights/activations, f32 accumulation):
      replica loss: |dl| <= 2e-3 * loss
      gradients: per tensor ||g - g_ref|| <= 3e-2 * ||g_ref|| (+1e-6 absolute floor)
      weights after one Adam step (first step: update = lr * sign-like): |p - p_ref| <= 2*lr for
      every element and <= 0.05*lr for >= 95% of elements.
    """
    n_stage = config.n_pp * config.n_loop
    loss, grads, newp, rloss = oracle(cfg, config, params, tokens)
    report = {"oracle_loss": loss, "grad_rel": {}, "weights_frac_close": {}}
    for r, res in enumerate(results):
        dp, pp = r // config.n_pp, r % config.n_pp
        if pp == (n_stage - 1) % config.n_pp:
            assert abs(res["loss"] - rloss[dp]) <= 2e-3 * rloss[dp], (res["loss"], rloss[dp])
            report.setdefault("losses", []).append((res["loss"], rloss[dp]))
    for s in range(n_stage):
        full_g = np.full(flatten_stage(params, cfg, s, n_stage).size, np.nan, np.float32)
        full_p = full_g.copy()
        for r, res in enumerate(results):
            if s in res["grads"]:
                g, lo, hi = res["grads"][s]
                own = ~np.isnan(g[lo:hi])  # this rank's elements (slices of every segment when sharded)
                full_g[lo:hi][own] = g[lo:hi][own]
                p, lo, hi = res["params"][s]
                own = ~np.isnan(p[lo:hi])
                full_p[lo:hi][own] = p[lo:hi][own]
        assert not np.isnan(full_g).any(), f"stage {s}: gradient shards do not cover the stage"
        got_g = unflatten_stage(full_g, cfg, s, n_stage)
        got_p = unflatten_stage(full_p, cfg, s, n_stage)
        for k in got_g:
            ref = grads[k]
            err = np.linalg.norm(got_g[k] - ref)
            rel = err / (np.linalg.norm(ref) + 1e-6)
            report["grad_rel"][k] = float(rel)
            assert err <= 3e-2 * np.linalg.norm(ref) + 1e-6, (k, rel)
            dpar = np.abs(got_p[k] - newp[k])
            assert dpar.max() <= 2 * LR + 1e-6, (k, dpar.max())
            frac = float((dpar <= 0.05 * LR).mean())
            report["weights_frac_close"][k] = frac
            assert frac >= 0.95, (k, frac)
    return report
