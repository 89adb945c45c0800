"""Pins the CPU numerics oracle (oracle/gpt_oracle.py) against an independent
implementation: the same GPT written with torch float64 autograd on the CPU.
(The reference has no numerics to pin against.)"""
import math
import os
import sys

import numpy as np
import pytest
import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
import gpt_oracle as O  # noqa: E402

from paper_2211_05953_b200.model import GPTConfig, flatten_stage, stage_layout, unflatten_stage  # noqa: E402


def torch_loss(P, tokens, cfg):
    h, H = cfg.s_hidden, cfg.n_heads
    d = h // H
    N, S = tokens.shape[0], tokens.shape[1] - 1
    inp, lab = tokens[:, :-1], tokens[:, 1:]
    x = P["wte"][inp] + P["wpe"][:S]

    def ln(x, g, b):
        return torch.nn.functional.layer_norm(x, (h,), g, b, O.LN_EPS)

    for l in range(cfg.n_layers):
        p = f"h{l}."
        a = ln(x, P[p + "ln1_g"], P[p + "ln1_b"])
        qkv = a @ P[p + "w_qkv"].T
        q, k, v = qkv.split(h, -1)
        q, k, v = (t.view(N, S, H, d).transpose(1, 2) for t in (q, k, v))
        o = torch.nn.functional.scaled_dot_product_attention(q, k, v, is_causal=True)
        x = x + o.transpose(1, 2).reshape(N, S, h) @ P[p + "w_o"].T
        a = ln(x, P[p + "ln2_g"], P[p + "ln2_b"])
        x = x + torch.nn.functional.gelu(a @ P[p + "w_fc1"].T, approximate="tanh") @ P[p + "w_fc2"].T
    logits = ln(x, P["lnf_g"], P["lnf_b"]) @ P["w_head"].T
    return torch.nn.functional.cross_entropy(logits.reshape(-1, cfg.s_voc), lab.reshape(-1))


@pytest.mark.parametrize("heads", [1, 2])
def test_oracle_matches_torch_autograd(heads):
    cfg = GPTConfig(2, 64, heads, 16, 50)
    params = O.init_params(cfg, seed=3, std=0.2)
    rng = np.random.default_rng(5)
    tokens = rng.integers(0, cfg.s_voc, (3, cfg.s_seq + 1))
    loss, grads = O.loss_and_grads(params, tokens, cfg)
    P = {k: torch.tensor(v, dtype=torch.float64, requires_grad=True) for k, v in params.items()}
    ref = torch_loss(P, torch.tensor(tokens), cfg)
    ref.backward()
    assert loss == pytest.approx(ref.item(), rel=1e-12)
    for k, v in P.items():
        np.testing.assert_allclose(grads[k], v.grad.numpy(), rtol=1e-9, atol=1e-12, err_msg=k)


def test_stage_layout_roundtrip_and_split_independence():
    cfg = GPTConfig.preset("tiny")
    params = O.init_params(cfg, seed=1)
    for n_stage in (1, 2, 4):
        names = []
        for s in range(n_stage):
            lay, numel, padded = stage_layout(cfg, s, n_stage, n_dp=2)
            assert padded % 128 == 0 and padded >= numel
            assert all(off % 64 == 0 for _, off, _ in lay)
            flat = flatten_stage(params, cfg, s, n_stage)
            back = unflatten_stage(flat, cfg, s, n_stage)
            for k, v in back.items():
                np.testing.assert_array_equal(v, params[k].astype(np.float32))
            names += [n for n, _, _ in lay]
        assert sorted(names) == sorted(params)


def test_adam_step_first_update_is_signed_lr():
    p = {"w": np.array([1.0, -2.0, 3.0])}
    g = {"w": np.array([0.5, -1e-3, 0.0])}
    m = {"w": np.zeros(3)}
    v = {"w": np.zeros(3)}
    out = O.adam_step(p, g, m, v, 1, 1e-2, 0.9, 0.95, 1e-8, 0.0)
    np.testing.assert_allclose(out["w"], [1.0 - 1e-2, -2.0 + 1e-2, 3.0], atol=1e-8)
