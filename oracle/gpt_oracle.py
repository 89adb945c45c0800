"""TEST INFRASTRUCTURE ONLY — CPU numerics oracle for the stage executor.

Parity status: UNPINNED by the reference. The reference (pipesim) models a
stage as a scalar duration (proj/src/simulate.cpp:20-29,
proj/include/pipesim/schedule.hpp:24-39) and holds no loss, gradient or
weight computation, so no reference test or fixture constrains these numbers
(SURVEY.md §8c). This file restates the model the paper trains (PAPER.md:604:
identical layers of self-attention + 2-layer MLP, S_mlp = 4h; mixed precision;
Adam; embedding/output folded into the first/last stage) as a
pre-LN GPT in float64 numpy, and is itself checked against an independent
torch float64 autograd implementation in tests/test_oracle.py.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may use it.
"""
from __future__ import annotations

import math
from typing import Dict

import numpy as np

GELU_K0 = math.sqrt(2.0 / math.pi)
GELU_K1 = 0.044715
LN_EPS = 1e-5


def gelu(x):
    return 0.5 * x * (1.0 + np.tanh(GELU_K0 * (x + GELU_K1 * x ** 3)))


def dgelu(x):
    u = GELU_K0 * (x + GELU_K1 * x ** 3)
    t = np.tanh(u)
    return 0.5 * (1.0 + t) + 0.5 * x * (1.0 - t * t) * GELU_K0 * (1.0 + 3.0 * GELU_K1 * x * x)


def layernorm(x, g, b):
    mu = x.mean(-1, keepdims=True)
    var = ((x - mu) ** 2).mean(-1, keepdims=True)
    rstd = 1.0 / np.sqrt(var + LN_EPS)
    xh = (x - mu) * rstd
    return xh * g + b, (xh, rstd)


def layernorm_bwd(dy, cache, g):
    xh, rstd = cache
    gd = dy * g
    w = xh.shape[-1]
    dx = rstd * (gd - gd.sum(-1, keepdims=True) / w - xh * (gd * xh).sum(-1, keepdims=True) / w)
    return dx, (dy * xh).reshape(-1, w).sum(0), dy.reshape(-1, w).sum(0)


def init_params(cfg, seed: int = 0, std: float = 0.02) -> Dict[str, np.ndarray]:
    """N(0, std) weights, output projections std/sqrt(2L), LayerNorm (1, 0)."""
    rng = np.random.default_rng(seed)
    h, m, V, S, L = cfg.s_hidden, cfg.s_mlp, cfg.s_voc, cfg.s_seq, cfg.n_layers
    out_std = std / math.sqrt(2 * L)
    p = {"wte": rng.normal(0, std, (V, h)), "wpe": rng.normal(0, std, (S, h))}
    for l in range(L):
        p[f"h{l}.ln1_g"] = np.ones(h) + rng.normal(0, 0.1, h)
        p[f"h{l}.ln1_b"] = rng.normal(0, 0.1, h)
        p[f"h{l}.w_qkv"] = rng.normal(0, std, (3 * h, h))
        p[f"h{l}.w_o"] = rng.normal(0, out_std, (h, h))
        p[f"h{l}.ln2_g"] = np.ones(h) + rng.normal(0, 0.1, h)
        p[f"h{l}.ln2_b"] = rng.normal(0, 0.1, h)
        p[f"h{l}.w_fc1"] = rng.normal(0, std, (m, h))
        p[f"h{l}.w_fc2"] = rng.normal(0, out_std, (h, m))
    p["lnf_g"] = np.ones(h) + rng.normal(0, 0.1, h)
    p["lnf_b"] = rng.normal(0, 0.1, h)
    p["w_head"] = rng.normal(0, std, (V, h))
    return p


def _attention(q, k, v):
    """Causal softmax attention for one head: q, k, v [S, d]."""
    S, d = q.shape
    s = q @ k.T / math.sqrt(d)
    s = np.where(np.tril(np.ones((S, S), dtype=bool)), s, -np.inf)
    s = s - s.max(-1, keepdims=True)
    p = np.exp(s)
    p /= p.sum(-1, keepdims=True)
    return p @ v, p


def _attention_bwd(do, q, k, v, p):
    d = q.shape[1]
    dv = p.T @ do
    dp = do @ v.T
    ds = p * (dp - (dp * p).sum(-1, keepdims=True))
    dq = ds @ k / math.sqrt(d)
    dk = ds.T @ q / math.sqrt(d)
    return dq, dk, dv


def layer_forward(P, pre, x, cfg):
    """One pre-LN block on one sequence x [S, h]; returns (x_out, cache)."""
    h, H = cfg.s_hidden, cfg.n_heads
    d = h // H
    S = x.shape[0]
    ln1, c1 = layernorm(x, P[pre + "ln1_g"], P[pre + "ln1_b"])
    qkv = ln1 @ P[pre + "w_qkv"].T
    o = np.zeros((S, h), dtype=x.dtype)
    probs = []
    for j in range(H):
        q = qkv[:, j * d:(j + 1) * d]
        k = qkv[:, h + j * d:h + (j + 1) * d]
        v = qkv[:, 2 * h + j * d:2 * h + (j + 1) * d]
        oj, pj = _attention(q, k, v)
        o[:, j * d:(j + 1) * d] = oj
        probs.append(pj)
    x_mid = x + o @ P[pre + "w_o"].T
    ln2, c2 = layernorm(x_mid, P[pre + "ln2_g"], P[pre + "ln2_b"])
    a_pre = ln2 @ P[pre + "w_fc1"].T
    act = gelu(a_pre)
    x_out = x_mid + act @ P[pre + "w_fc2"].T
    return x_out, (ln1, c1, qkv, o, probs, ln2, c2, a_pre, act)


def layer_backward(P, G, pre, dx, cache, cfg):
    """Backward of layer_forward: accumulates parameter grads into G, returns d x_in."""
    h, H = cfg.s_hidden, cfg.n_heads
    d = h // H
    ln1, c1, qkv, o, probs, ln2, c2, a_pre, act = cache
    G[pre + "w_fc2"] += dx.T @ act
    dpre = (dx @ P[pre + "w_fc2"]) * dgelu(a_pre)
    G[pre + "w_fc1"] += dpre.T @ ln2
    dln2 = dpre @ P[pre + "w_fc1"]
    dmid, dg, db = layernorm_bwd(dln2, c2, P[pre + "ln2_g"])
    dmid += dx
    G[pre + "ln2_g"] += dg
    G[pre + "ln2_b"] += db
    G[pre + "w_o"] += dmid.T @ o
    do = dmid @ P[pre + "w_o"]
    dqkv = np.zeros_like(qkv)
    for j in range(H):
        sl = slice(j * d, (j + 1) * d)
        ks = slice(h + j * d, h + (j + 1) * d)
        vs = slice(2 * h + j * d, 2 * h + (j + 1) * d)
        dq, dk, dv = _attention_bwd(do[:, sl], qkv[:, sl], qkv[:, ks], qkv[:, vs], probs[j])
        dqkv[:, sl], dqkv[:, ks], dqkv[:, vs] = dq, dk, dv
    G[pre + "w_qkv"] += dqkv.T @ ln1
    dln1 = dqkv @ P[pre + "w_qkv"]
    dxi, dg, db = layernorm_bwd(dln1, c1, P[pre + "ln1_g"])
    G[pre + "ln1_g"] += dg
    G[pre + "ln1_b"] += db
    return dxi + dmid


def head_forward_backward(P, G, x, lab, n_tok):
    """Final LayerNorm + LM head + cross-entropy (summed over rows) and its backward
    (gradient of the mean over n_tok tokens); returns (loss_sum, d x)."""
    S = x.shape[0]
    lnf, cf = layernorm(x, P["lnf_g"], P["lnf_b"])
    logits = lnf @ P["w_head"].T
    mx = logits.max(-1, keepdims=True)
    lse = mx[:, 0] + np.log(np.exp(logits - mx).sum(-1))
    loss = float((lse - logits[np.arange(S), lab]).sum())
    dlog = np.exp(logits - lse[:, None])
    dlog[np.arange(S), lab] -= 1.0
    dlog /= n_tok
    G["w_head"] += dlog.T @ lnf
    dx, dg, db = layernorm_bwd(dlog @ P["w_head"], cf, P["lnf_g"])
    G["lnf_g"] += dg
    G["lnf_b"] += db
    return loss, dx


def loss_and_grads(params, tokens, cfg):
    """Mean next-token cross-entropy over all sequences of `tokens` [N, S+1] and its
    gradient w.r.t. every parameter (float64)."""
    P = {k: np.asarray(v, dtype=np.float64) for k, v in params.items()}
    G = {k: np.zeros_like(v) for k, v in P.items()}
    tokens = np.asarray(tokens)
    N, S = tokens.shape[0], tokens.shape[1] - 1
    n_tok = N * S
    total = 0.0
    for b in range(N):
        inp, lab = tokens[b, :-1], tokens[b, 1:]
        x = P["wte"][inp] + P["wpe"][:S]
        caches = []
        for l in range(cfg.n_layers):
            x, c = layer_forward(P, f"h{l}.", x, cfg)
            caches.append(c)
        loss, dx = head_forward_backward(P, G, x, lab, n_tok)
        total += loss
        for l in reversed(range(cfg.n_layers)):
            dx = layer_backward(P, G, f"h{l}.", dx, caches[l], cfg)
        np.add.at(G["wte"], inp, dx)
        G["wpe"][:S] += dx
    return total / n_tok, G


def adam_step(params, grads, m, v, step, lr, beta1, beta2, eps, wd):
    """The executor's update (csrc/kernels/elementwise.cu adam_kernel), float64."""
    out = {}
    bc1, bc2 = 1 - beta1 ** step, 1 - beta2 ** step
    for k in params:
        g = grads[k]
        m[k] = beta1 * m[k] + (1 - beta1) * g
        v[k] = beta2 * v[k] + (1 - beta2) * g * g
        out[k] = params[k] - lr * ((m[k] / bc1) / (np.sqrt(v[k] / bc2) + eps) + wd * params[k])
    return out
