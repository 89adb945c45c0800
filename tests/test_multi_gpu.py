"""Multi-GPU executor parity vs the CPU oracle: pipeline hand-offs as copy-engine peer copies
into CUDA-IPC-mapped receive slots signalled with cuStreamWriteValue32 / cuStreamWaitValue32,
DP_FS all-gather / reduce-scatter, DP0 all-reduce and DP_PS over NCCL. Each case runs under torchrun, one rank per GPU;
skipped when fewer GPUs are visible than the case needs."""
import os
import pickle
import subprocess
import sys

import pytest

import exec_harness as H
from dist_worker import CASES, config_of, model_of, steps_of

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def _gpus():
    import torch
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


@pytest.mark.parametrize("case", list(CASES))
def test_multi_gpu_parity(case, tmp_path):
    config = config_of(case)
    n = config.n_dp * config.n_pp
    if _gpus() < n:
        pytest.skip(f"needs {n} GPUs")
    port = 29500 + (abs(hash(case)) % 2000)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.join(HERE, "dist_worker.py"),
           "--case", case, "--out", str(tmp_path)]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=240)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    results = []
    for rank in range(n):
        with open(tmp_path / f"rank{rank}.pkl", "rb") as f:
            results.append(pickle.load(f))
    cfg, n_steps = model_of(case), steps_of(case)
    if n_steps:
        params, tokens = H.make_steps_case(cfg, config, n_steps)
        rep = H.compare_steps(cfg, config, results, params, tokens)
        print(case, rep["losses"], min(rep["weights_frac_close"].values()))
    else:
        params, tokens = H.make_case(cfg, config)
        rep = H.compare(cfg, config, results, params, tokens)
        print(case, rep.get("losses"), max(rep["grad_rel"].values()))
