"""GPT model description shared by the executor front end and the tests.

Pre-LN decoder-only transformer, the paper's layer structure (self-attention +
2-layer GeLU MLP with S_mlp = 4h) with bias-free linear layers
and untied input/output embeddings. The embedding is folded into stage 0 and
the final LayerNorm + LM head + cross-entropy into the last stage
(SPEC.md:431).

``stage_layout`` mirrors ``make_stage_layout`` in csrc/exec/executor.cu: every
sub-tensor starts at a multiple of 64 elements; stage vectors are padded to a
multiple of 64 * n_dp so DP shards are equal and 128-byte aligned.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Dict, List, Tuple

PRESETS = {
    # name: (n_layers, s_hidden, n_heads, s_seq, s_voc)
    "tiny": (4, 128, 1, 64, 1000),        # BASELINE configs[0]; one head of 128 (kernel head_dim)
    # parity presets at production kernel paths: every GEMM has M, N >= 256 (2-CTA tiles, grouped
    # weight-gradient pairs), several heads and several 128-row attention blocks per sequence
    "small": (2, 256, 2, 512, 2048),
    # + an LM head whose weight-gradient operand (V x tokens) exceeds L2 -> N-fastest tile raster
    "small-v50k": (1, 384, 3, 512, 50304),
    "gpt-1.3b": (24, 2048, 16, 2048, 50304),
    "gpt-2.7b": (32, 2560, 20, 2048, 50304),
    "gpt-6.7b": (32, 4096, 32, 2048, 50304),
    "gpt-13b-l40": (40, 5120, 40, 2048, 50304),
    "gpt-13b-l32": (32, 5760, 45, 2048, 50304),
    "52b": (64, 8192, 64, 1024, 50304),
    # the 52B layer shape at a depth 4 B200s can hold (BASELINE configs[4] needs 8: PP4 x DP2)
    "52b-l16": (16, 8192, 64, 1024, 50304),
}


@dataclass(frozen=True)
class GPTConfig:
    n_layers: int
    s_hidden: int
    n_heads: int
    s_seq: int
    s_voc: int

    @property
    def s_head(self):
        return self.s_hidden // self.n_heads

    @property
    def s_mlp(self):
        return 4 * self.s_hidden

    @staticmethod
    def preset(name: str) -> "GPTConfig":
        return GPTConfig(*PRESETS[name])

    def n_params(self) -> int:
        h, V, S, L = self.s_hidden, self.s_voc, self.s_seq, self.n_layers
        return L * (12 * h * h + 4 * h) + 2 * V * h + S * h + 2 * h

    def model_flops_per_token(self) -> float:
        """72*L*h^2 + 12*L*s*h + 6*h*V (no recompute, full attention)."""
        L, h, s, V = self.n_layers, self.s_hidden, self.s_seq, self.s_voc
        return 72.0 * L * h * h + 12.0 * L * s * h + 6.0 * h * V


def _align(n: int) -> int:
    return (n + 63) // 64 * 64


def stage_layout(cfg: GPTConfig, stage: int, n_stage: int, n_dp: int = 1
                 ) -> Tuple[List[Tuple[str, int, Tuple[int, ...]]], int, int]:
    """[(name, offset, shape)], numel, padded for one stage's flat parameter vector."""
    h, m, V, S = cfg.s_hidden, cfg.s_mlp, cfg.s_voc, cfg.s_seq
    lps = cfg.n_layers // n_stage
    out = []
    off = 0

    def take(name, shape):
        nonlocal off
        n = 1
        for d in shape:
            n *= d
        out.append((name, off, shape))
        off += _align(n)

    if stage == 0:
        take("wte", (V, h))
        take("wpe", (S, h))
    for i in range(lps):
        l = stage * lps + i
        take(f"h{l}.ln1_g", (h,))
        take(f"h{l}.ln1_b", (h,))
        take(f"h{l}.w_qkv", (3 * h, h))
        take(f"h{l}.w_o", (h, h))
        take(f"h{l}.ln2_g", (h,))
        take(f"h{l}.ln2_b", (h,))
        take(f"h{l}.w_fc1", (m, h))
        take(f"h{l}.w_fc2", (h, m))
    if stage == n_stage - 1:
        take("lnf_g", (h,))
        take("lnf_b", (h,))
        take("w_head", (V, h))
    q = 64 * n_dp
    return out, off, (off + q - 1) // q * q


def flatten_stage(params: Dict[str, "object"], cfg: GPTConfig, stage: int, n_stage: int):
    import numpy as np
    layout, numel, _ = stage_layout(cfg, stage, n_stage)
    flat = np.zeros(numel, dtype=np.float32)
    for name, off, shape in layout:
        a = np.asarray(params[name], dtype=np.float32).reshape(-1)
        flat[off:off + a.size] = a
    return flat


def unflatten_stage(flat, cfg: GPTConfig, stage: int, n_stage: int) -> Dict[str, "object"]:
    import numpy as np
    layout, _, _ = stage_layout(cfg, stage, n_stage)
    out = {}
    for name, off, shape in layout:
        n = int(np.prod(shape))
        out[name] = np.asarray(flat[off:off + n]).reshape(shape)
    return out
