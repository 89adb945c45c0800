"""Python front end of the per-rank B200 executor (C ABI: bfpp_exec_*).

Mirrors the reference's simulate entry points (``simulate_config``,
bindings/module.cpp:20-24) with a real ``execute``: the same
``place_stages``/``build_tasks`` graph is run on the GPU and a *measured*
``Timeline`` comes back, to which the reference's metrics
(``bubble_fraction``, ``throughput``, ``peak_inflight``) apply unchanged.

One process per GPU: rank = dp * n_pp + pp. NCCL unique ids are generated on
rank 0 and broadcast with torch.distributed (plumbing only).
"""
from __future__ import annotations

import ctypes as C
import os
from typing import List, Optional, Sequence

import numpy as np

from . import _native as N
from . import pipesim as ps
from .model import GPTConfig

SKIP_OPTIMIZER = 1
PROFILE_KERNELS = 2
RECOMPUTE = 4
MEMORY_CATEGORIES = ("weights", "grads", "optimizer", "grad_shards", "weight_shards", "activations", "pp_buffers",
                     "scratch")
KERNEL_CATEGORIES = ("gemm", "attention_fwd", "attention_bwd", "layernorm", "misc", "adam")


def _check(st):
    if st != 0:
        msg = N.lib().bfpp_last_error().decode()
        raise (ps.SpecError if st == 2 else ps.SimError)(msg)


def model_spec(cfg: GPTConfig) -> ps.ModelSpec:
    return ps.ModelSpec(n_layers=cfg.n_layers, s_hidden=cfg.s_hidden, n_heads=cfg.n_heads, s_seq=cfg.s_seq,
                        s_voc=cfg.s_voc)


def comm_ids(config: ps.ParallelConfig) -> bytes:
    """Fresh NCCL unique ids for every communicator of `config` (call on one rank)."""
    L = N.lib()
    n = L.bfpp_exec_n_comm_ids(C.byref(config._c()))
    buf = (C.c_char * (128 * n))()
    for i in range(n):
        _check(L.bfpp_nccl_unique_id(C.byref(buf, 128 * i)))
    return bytes(buf)


class Executor:
    def __init__(self, model, config: ps.ParallelConfig, *, rank: int = 0, world: int = 1,
                 device: Optional[int] = None, uids: Optional[bytes] = None, record_timeline: bool = False,
                 seed: int = 1234, lr: float = 1e-4, beta1: float = 0.9, beta2: float = 0.95,
                 eps: float = 1e-8, weight_decay: float = 0.0, init_std: float = 0.02,
                 skip_optimizer: bool = False, profile_kernels: bool = False, recompute: bool = False,
                 graph: Optional[ps.TaskGraph] = None):
        """graph: run this task graph (e.g. ``ps.build_accumulation_tasks``) instead of
        ``build_tasks(model, config)``; ``config`` then describes its placement (see
        ``accumulation_config``)."""
        if isinstance(model, GPTConfig):
            model = model_spec(model)
        self.model, self.config, self.rank, self.world = model, config, rank, world
        if device is None:
            device = int(os.environ.get("LOCAL_RANK", rank))
        opts = N.ExecOptsC(device, int(record_timeline), seed, lr, beta1, beta2, eps, weight_decay, init_std,
                           (SKIP_OPTIMIZER if skip_optimizer else 0) | (PROFILE_KERNELS if profile_kernels else 0)
                           | (RECOMPUTE if recompute else 0))
        h = C.c_void_p()
        ubuf = C.create_string_buffer(uids, len(uids)) if uids else None
        if graph is None:
            _check(N.lib().bfpp_exec_create(C.byref(model._c()), C.byref(config._c()), C.byref(opts), rank, world,
                                            ubuf, C.byref(h)))
        else:
            _check(N.lib().bfpp_exec_create_graph(C.byref(model._c()), C.byref(config._c()), graph.handle,
                                                  C.byref(opts), rank, world, ubuf, C.byref(h)))
        self._h = h
        g = C.c_void_p()
        _check(N.lib().bfpp_exec_graph(self._h, C.byref(g)))
        self.graph = ps.TaskGraph(g.value)
        self.pp_rank = rank % config.n_pp
        self.dp_rank = rank // config.n_pp
        L = N.lib()
        self.local_stages = [L.bfpp_exec_local_stage(self._h, c) for c in range(L.bfpp_exec_n_local_stages(self._h))]
        self.device_bytes = L.bfpp_exec_device_bytes(self._h)

    def memory(self) -> dict:
        """This rank's device bytes by category (+ pooled activation / logits set counts)."""
        return _memory_dict(lambda b, n: N.lib().bfpp_exec_memory(self._h, b, n))

    # ---- training step -------------------------------------------------------------------
    def step(self, tokens) -> float:
        """tokens: host int32 [n_mb, s_mb, s_seq+1] (numpy or pinned torch tensor) of this DP replica."""
        ptr = tokens.data_ptr() if hasattr(tokens, "data_ptr") else np.ascontiguousarray(tokens, np.int32).ctypes.data
        loss = C.c_float()
        _check(N.lib().bfpp_exec_step(self._h, C.c_void_p(ptr), C.byref(loss)))
        return loss.value

    def step_device(self, tokens_dev, loss_dev=None):
        _check(N.lib().bfpp_exec_step_device(self._h, C.c_void_p(tokens_dev.data_ptr()),
                                             C.c_void_p(loss_dev.data_ptr()) if loss_dev is not None else None))

    def sync(self):
        _check(N.lib().bfpp_exec_sync(self._h))

    # ---- state I/O -------------------------------------------------------------------------
    def stage_numel(self, stage: int) -> int:
        return N.lib().bfpp_exec_stage_numel(self._h, stage)

    def set_stage_params(self, stage: int, flat: np.ndarray):
        a = np.ascontiguousarray(flat, dtype=np.float32)
        _check(N.lib().bfpp_exec_set_params(self._h, stage, a.ctypes.data, a.size))

    def _get(self, fn, stage):
        n = self.stage_numel(stage)
        out = np.full(n, np.nan, dtype=np.float32)
        lo, hi = C.c_int64(), C.c_int64()
        _check(fn(self._h, stage, out.ctypes.data, n, C.byref(lo), C.byref(hi)))
        return out, lo.value, hi.value

    def get_stage_params(self, stage: int):
        """(full-size f32 array, NaN where another DP rank owns the element, lo, hi)."""
        return self._get(N.lib().bfpp_exec_get_params, stage)

    def get_stage_grads(self, stage: int):
        return self._get(N.lib().bfpp_exec_get_grads, stage)

    def get_stage_weights16(self, stage: int):
        """(bf16 compute weights as float32, lo, hi): the resident copy or this rank's DP_FS slices (NaN elsewhere)."""
        n = self.stage_numel(stage)
        raw = np.zeros(n, dtype=np.uint16)
        lo, hi = C.c_int64(), C.c_int64()
        _check(N.lib().bfpp_exec_get_weights16(self._h, stage, raw.ctypes.data, n, C.byref(lo), C.byref(hi)))
        return (raw.astype(np.uint32) << 16).view(np.float32), lo.value, hi.value

    def zero_grads(self):
        _check(N.lib().bfpp_exec_zero_grads(self._h))

    def task_times(self):
        n = len(self.graph.tasks)
        s = np.zeros(n)
        e = np.zeros(n)
        _check(N.lib().bfpp_exec_timeline(self._h, s.ctypes.data, e.ctypes.data))
        return s, e

    @property
    def stream_handle(self) -> int:
        """cudaStream_t of the executor's compute stream (every step starts and ends on it)."""
        return N.lib().bfpp_exec_stream(self._h)

    def set_flags(self, record_timeline: bool = False, profile_kernels: bool = False):
        _check(N.lib().bfpp_exec_set_flags(self._h, int(record_timeline), int(profile_kernels)))

    def kernel_stats(self):
        """{category: (launches, ms, work)} of the last step (ms/work need profile_kernels)."""
        out = {}
        for i, name in enumerate(KERNEL_CATEGORIES):
            n, ms, w = C.c_int64(), C.c_double(), C.c_double()
            _check(N.lib().bfpp_exec_kernel_stats(self._h, i, C.byref(n), C.byref(ms), C.byref(w)))
            out[name] = (n.value, ms.value, w.value)
        return out

    def close(self):
        if getattr(self, "_h", None):
            N.lib().bfpp_exec_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _memory_dict(fill) -> dict:
    b = (C.c_int64 * len(MEMORY_CATEGORIES))()
    n = (C.c_int64 * 2)()
    _check(fill(b, n))
    out = {k: int(b[i]) for i, k in enumerate(MEMORY_CATEGORIES)}
    out["total"] = sum(out.values())
    out["activation_sets"], out["head_sets"] = int(n[0]), int(n[1])
    return out


def memory_plan(model, config: ps.ParallelConfig, rank: int = 0, *, recompute: bool = False,
                skip_optimizer: bool = False) -> dict:
    """Device bytes rank `rank` of an executor for (model, config) would allocate, by category,
    computed on the host (the executor's own allocation code in sizing mode; no GPU needed)."""
    if isinstance(model, GPTConfig):
        model = model_spec(model)
    opts = N.ExecOptsC(0, 0, 0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0,
                       (RECOMPUTE if recompute else 0) | (SKIP_OPTIMIZER if skip_optimizer else 0))
    return _memory_dict(lambda b, n: N.lib().bfpp_exec_memory_plan(C.byref(model._c()), C.byref(config._c()),
                                                                   C.byref(opts), rank, b, n))


KERNEL_VARIANTS = ("gemm_1cta", "gemm_2cta", "gemm_2cta_pair", "gemm_2cta_nfast", "gemm_2cta_streamk",
                   "attn_fwd_multi", "attn_bwd_multi")


def kernel_variant_counts(reset: bool = False) -> dict:
    """Process-wide launch counts per kernel variant (bfpp_kernel_variant_count); reset=True
    zeroes them after reading."""
    L = N.lib()
    out = {name: int(L.bfpp_kernel_variant_count(i)) for i, name in enumerate(KERNEL_VARIANTS)}
    if reset:
        L.bfpp_kernel_variant_reset()
    return out


STREAMS = ("compute", "dp", "fwd_send", "fwd_recv", "bwd_send", "bwd_recv", "wgrad")


def plan_rank(graph: ps.TaskGraph, pp_rank: int, n_dp: int, dp_variant: ps.DpVariant = ps.DpVariant.DP0):
    """The executor's per-rank plan (host only): [(task id, stream, flags, slot, waits)] in enqueue
    order. dp_variant selects the gradient-buffer discipline (sharded variants pool the buffers)."""
    L = N.lib()
    nt, nw = C.c_int64(), C.c_int64()
    z = C.POINTER(C.c_int32)()
    v = int(dp_variant)
    _check(L.bfpp_plan_rank(graph.handle, pp_rank, n_dp, v, 0, 0, z, z, z, z, z, z, C.byref(nt), C.byref(nw)))
    n, m = nt.value, nw.value
    arr = lambda k: (C.c_int32 * max(1, k))()  # noqa: E731
    ids, streams, flags, slots, woff, wids = arr(n), arr(n), arr(n), arr(n), arr(n + 1), arr(m)
    _check(L.bfpp_plan_rank(graph.handle, pp_rank, n_dp, v, n, m, ids, streams, flags, slots, woff, wids,
                            C.byref(nt), C.byref(nw)))
    return [(ids[i], streams[i], flags[i], slots[i], list(wids[woff[i]:woff[i + 1]])) for i in range(n)]


def measured_timeline(graph: ps.TaskGraph, starts: Sequence[np.ndarray], ends: Sequence[np.ndarray]) -> ps.Timeline:
    """Merges per-rank task times (NaN where a rank does not own a task) into one Timeline."""
    s = np.full(len(graph.tasks), np.nan)
    e = np.full(len(graph.tasks), np.nan)
    for a, b in zip(starts, ends):
        a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
        m = ~np.isnan(a)
        s[m] = a[m]
        e[m] = b[m]
    if np.isnan(s).any():
        raise ps.SimError("measured timeline is missing tasks")
    return ps.Timeline.from_intervals(graph, list(s), list(e))


def accumulation_config(model, dp_variant: ps.DpVariant, n_mb: int, n_dp: int) -> ps.ParallelConfig:
    """Placement of ``build_accumulation_tasks`` graphs (schedule.cpp:454-500): one device, one layer
    per stage (n_loop = n_layers), n_mb micro-batches, data parallel over n_dp ranks."""
    if isinstance(model, GPTConfig):
        model = model_spec(model)
    return ps.ParallelConfig(n_dp=n_dp, n_pp=1, n_loop=model.n_layers, n_mb=n_mb, dp_variant=dp_variant,
                             schedule=ps.Schedule.BreadthFirst)


def execute_distributed(model, config: ps.ParallelConfig, **kw) -> Executor:
    """Creates this process's executor under torch.distributed (env RANK/WORLD_SIZE/LOCAL_RANK)."""
    import torch.distributed as dist
    rank, world = dist.get_rank(), dist.get_world_size()
    obj: List[Optional[bytes]] = [comm_ids(config) if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    return Executor(model, config, rank=rank, world=world, uids=obj[0], **kw)
