"""bfpp — B200-native executor for Breadth-First Pipeline Parallelism (arXiv 2211.05953).

``pipesim`` mirrors the reference's schedule/stage API (drop-in surface);
``executor`` runs the resulting task graphs on B200s (tcgen05 kernels + NCCL).
"""
from . import pipesim  # noqa: F401
from .pipesim import *  # noqa: F401,F403

__version__ = "0.1.0"
