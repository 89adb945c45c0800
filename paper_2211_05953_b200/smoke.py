"""One tiny breadth-first training step on cuda:0 checked against the CPU oracle
(called by __graft_entry__.smoke()). Fails loudly if the CUDA path is missing."""
from __future__ import annotations

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run():
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("smoke: no CUDA device")
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import exec_harness as H  # oracle-backed checker (test infrastructure)
    from . import pipesim as ps
    from .executor import Executor
    config = ps.ParallelConfig(n_mb=2, n_loop=2, schedule=ps.Schedule.BreadthFirst)
    cfg = H.TINY
    params, tokens = H.make_case(cfg, config)
    res = H.run_rank(lambda **kw: Executor(cfg, config, device=0, **kw), cfg, config, params, tokens, 0)
    rep = H.compare(cfg, config, [res], params, tokens)
    print(f"smoke ok: loss {res['loss']:.6f} (oracle {rep['oracle_loss']:.6f}), "
          f"max grad rel err {max(rep['grad_rel'].values()):.2e}", flush=True)


if __name__ == "__main__":
    run()
