"""bfpp — B200-native executor for Breadth-First Pipeline Parallelism (arXiv 2211.05953).

``pipesim`` mirrors the reference's schedule/stage API (drop-in surface);
``executor`` runs the resulting task graphs on B200s (tcgen05 kernels + NCCL).
"""
import os

# The executor runs 7 streams; with fewer hardware work queues than streams, CUDA maps streams
# onto shared queues and a receive stream blocked in cuStreamWaitValue32 (waiting for its peer's
# copy) can block an unrelated send queued behind it -> cross-GPU deadlock. Must be set before the
# CUDA context exists: import this package before anything initialises CUDA. The executor refuses
# pipeline configs (n_pp >= 2) when a smaller value is already set.
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")  # one hardware queue per executor stream (see executor.py)

from . import pipesim  # noqa: F401
from .pipesim import *  # noqa: F401,F403

__version__ = "0.1.0"
