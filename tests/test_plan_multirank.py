"""Multi-rank host logic on CPU (gloo, world_size 2 and 4; no GPU).

Each rank process builds the task graph, computes its executor plan (libbfpp's
bfpp_plan_rank: stream assignment, cross-stream waits, host enqueue order) and
exchanges plans, NCCL unique ids and per-task times with torch.distributed
(gloo), exactly as bench.py / executor.execute_distributed do. Rank 0 then
emulates the executor's stream semantics across all ranks:

* every stream is FIFO in the plan's enqueue order; a task starts only when it is
  at the head of its stream and every event it waits on has been recorded;
* a pipeline transfer's receive completes once the sender's copy has run
  (copy-engine peer copy + flag write, csrc/exec/executor.cu);
* a DP collective (Reconstruct / Reduce) completes when it heads the DP stream of
  every rank in its DP group;

and checks that the step completes (no deadlock) and that every task ran after all
of its graph dependencies, on every rank. A second check merges per-rank measured
task times into one timeline and recovers the reference bubble fraction.
"""
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_2211_05953_b200 as ps
from paper_2211_05953_b200.executor import STREAMS, comm_ids, measured_timeline, plan_rank

S, V = ps.Schedule, ps.DpVariant
CASES = {
    "bf_pp2_dp1": (2, 1, 2, 4, V.DP_FS, S.BreadthFirst),
    "df_pp2_dp1": (2, 1, 2, 4, V.DP0, S.DepthFirst),
    "bf_pp2x2_dp2_fs": (2, 2, 2, 4, V.DP_FS, S.BreadthFirst),   # BASELINE configs[0] layout
    "bf_pp2x4_dp4_fs": (2, 4, 4, 2, V.DP_FS, S.BreadthFirst),   # bench.py layout at N = 8 (world 8)
    "gpipe_pp2_dp2_fs": (2, 2, 1, 2, V.DP_FS, S.GPipe),
    "1f1b_pp4_dp1": (4, 1, 1, 6, V.DP0, S.OneFOneB),
    "df_pp4x2_dp1": (4, 1, 2, 8, V.DP0, S.DepthFirst),
    "np_pp1_dp2_ps": (1, 2, 1, 3, V.DP_PS, S.NoPipeline),
    # gradient-accumulation graphs (build_accumulation_tasks; the schedule field is the order)
    "acc_bf_dp2_fs": (1, 2, None, 3, V.DP_FS, ps.AccumulationOrder.BreadthFirst),
    "acc_df_dp2_fs": (1, 2, None, 2, V.DP_FS, ps.AccumulationOrder.DepthFirst),
}


def _case_graph(name):
    n_pp, n_dp, loops, n_mb, variant, sched = CASES[name]
    if loops is None:  # accumulation: one layer per stage
        model = _model(1, 4)
        return ps.build_accumulation_tasks(model, variant, sched, n_mb)
    cfg = ps.ParallelConfig(n_dp=n_dp, n_pp=n_pp, n_loop=loops, n_mb=n_mb, dp_variant=variant, schedule=sched)
    return ps.build_tasks(_model(n_pp, loops), cfg)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _model(pp, loops):
    return ps.ModelSpec(n_layers=pp * loops * 2, s_hidden=128, n_heads=1, s_seq=64, s_voc=1000)


def emulate(graph, plans, n_pp, n_dp):
    """plans[rank] -> list of (id, stream, flags, slot, waits). Returns (completed order, error or None)."""
    tasks = graph.tasks
    world = n_pp * n_dp
    queues = {}
    for r in range(world):
        for item in plans[r]:
            queues.setdefault((r, item[1]), []).append(item)
    heads = {k: 0 for k in queues}
    done = [set() for _ in range(world)]           # task ids whose event is recorded on rank r
    sent = [set() for _ in range(n_dp)]            # transfers whose copy ran, per DP replica
    finished_order = []
    remaining = sum(len(q) for q in queues.values())
    while remaining:
        progressed = False
        for (r, st), q in queues.items():
            i = heads[(r, st)]
            if i >= len(q):
                continue
            tid, stream, flags, slot, waits = q[i]
            dp = r // n_pp
            if any(w not in done[r] for w in waits):
                continue
            t = tasks[tid]
            if t.kind == ps.TaskKind.Transfer and not (flags & 1) and tid not in sent[dp]:
                continue  # the receive waits for the peer's copy (flag write)
            if t.kind in (ps.TaskKind.Reconstruct, ps.TaskKind.Reduce):
                group = [d * n_pp + (r % n_pp) for d in range(n_dp)]
                if not all(heads.get((g, st), 0) < len(queues.get((g, st), [])) and
                           queues[(g, st)][heads[(g, st)]][0] == tid and
                           all(w in done[g] for w in queues[(g, st)][heads[(g, st)]][4]) for g in group):
                    continue
                for g in group:  # the collective completes on every member at once
                    done[g].add(tid)
                    heads[(g, st)] += 1
                    finished_order.append((g, tid))
                    remaining -= 1
                progressed = True
                continue
            if t.kind == ps.TaskKind.Transfer and (flags & 1):
                sent[dp].add(tid)
            done[r].add(tid)
            heads[(r, st)] += 1
            finished_order.append((r, tid))
            remaining -= 1
            progressed = True
        if not progressed:
            stuck = {f"rank{r}/{STREAMS[st]}": q[heads[(r, st)]][0] for (r, st), q in queues.items()
                     if heads[(r, st)] < len(q)}
            return finished_order, f"deadlock; stream heads: {stuck}"
    return finished_order, None


def check_dependencies(graph, order, n_pp, n_dp):
    """Every task ran after all of its graph dependencies (transfers count once on the sender)."""
    pos = {}
    for k, (r, tid) in enumerate(order):
        pos.setdefault((r // n_pp, tid), k)  # first completion within the replica
    for dp in range(n_dp):
        for t in graph.tasks:
            for d in t.deps:
                assert pos[(dp, d)] < pos[(dp, t.id)], (dp, t.id, d)


def _worker(rank, world, port, name, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n_pp, n_dp, loops, n_mb, variant, sched = CASES[name]
        graph = _case_graph(name)
        cfg = ps.ParallelConfig(n_dp=n_dp, n_pp=n_pp, n_loop=loops or 8, n_mb=n_mb, dp_variant=variant,
                                schedule=ps.Schedule.BreadthFirst if loops is None else sched)
        ids = [comm_ids(cfg) if rank == 0 else None]      # NCCL unique ids, as execute_distributed
        dist.broadcast_object_list(ids, src=0)
        plan = plan_rank(graph, rank % n_pp, n_dp, variant)
        # per-task "measured" times of this rank's tasks (simulated durations stand in for CUDA events)
        sim = ps.simulate(graph, ps.TimingModel(t_fwd_stage=1.0, bwd_ratio=2.0, t_pp_transfer=0.1,
                                                t_dp_reduce_stage=0.3, t_dp_reconstruct_stage=0.2))
        mine = {tid for tid, *_ in plan}
        starts = [sim.events[t.id].start if t.id in mine and (t.kind != ps.TaskKind.Transfer or t.device == rank % n_pp)
                  else float("nan") for t in graph.tasks]
        ends = [sim.events[t.id].end if s == s else float("nan") for t, s in zip(graph.tasks, starts)]
        gathered = [None] * world
        dist.all_gather_object(gathered, (rank, plan, len(ids[0]), starts, ends))
        if rank == 0:
            plans = {r: p for r, p, *_ in gathered}
            order, err = emulate(graph, plans, n_pp, n_dp)
            if err is None:
                check_dependencies(graph, order, n_pp, n_dp)
            rep0 = [(s, e) for r, _, _, s, e in gathered if r // n_pp == 0]
            tl = measured_timeline(graph, [s for s, _ in rep0], [e for _, e in rep0])
            q.put((err, len(ids[0]), {r: n for r, _, n, *_ in gathered}, ps.bubble_fraction(tl),
                   ps.bubble_fraction(sim)))
    except Exception as e:  # surface worker failures to the test
        if rank == 0:
            q.put((f"worker error: {e!r}", 0, {}, None, None))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name", list(CASES))
def test_multirank_plan_emulation(name):
    n_pp, n_dp = CASES[name][:2]
    world = n_pp * n_dp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    mp.start_processes(_worker, args=(world, _free_port(), name, q), nprocs=world, join=True, start_method="spawn")
    err, id_bytes, seen, bubble_measured, bubble_sim = q.get(timeout=60)
    assert err is None, err
    n_ids = 1 + n_pp  # world + one DP group per pipeline rank
    assert id_bytes == 128 * n_ids and set(seen.values()) == {128 * n_ids}
    assert bubble_measured == pytest.approx(bubble_sim, abs=1e-12)


def _local_plans(name):
    n_pp, n_dp = CASES[name][:2]
    graph = _case_graph(name)
    variant = CASES[name][4]
    return graph, {r: plan_rank(graph, r % n_pp, n_dp, variant) for r in range(n_pp * n_dp)}, n_pp, n_dp


def test_emulator_detects_mismatched_collective_order():
    """Sanity of the checker: DP collectives issued in a different order on two replicas deadlock."""
    graph, plans, n_pp, n_dp = _local_plans("bf_pp2x2_dp2_fs")
    dp_items = [i for i, it in enumerate(plans[2]) if it[1] == STREAMS.index("dp")]
    a, b = dp_items[0], dp_items[-1]
    plans[2][a], plans[2][b] = plans[2][b], plans[2][a]
    _, err = emulate(graph, plans, n_pp, n_dp)
    assert err is not None and "deadlock" in err


def test_emulator_detects_missing_wait():
    """Sanity of the checker: dropping the cross-stream waits lets a task run before its dependencies."""
    graph, plans, n_pp, n_dp = _local_plans("bf_pp2_dp1")
    plans = {r: [(tid, st, fl, sl, []) for tid, st, fl, sl, _ in p] for r, p in plans.items()}
    order, err = emulate(graph, plans, n_pp, n_dp)
    assert err is None
    with pytest.raises(AssertionError):
        check_dependencies(graph, order, n_pp, n_dp)


@pytest.mark.parametrize("name", ["bf_pp2x2_dp2_fs", "gpipe_pp2_dp2_fs", "acc_df_dp2_fs"])
def test_plan_marks_the_backward_completing_each_stage(name):
    """Flag 64 (last-unit backward: the executor reduces that stage layer by layer inside it) sits on
    exactly one backward per local stage -- the dependency of the stage's last Reduce; flag 128
    marks it when that Reduce is also the stage's first (BF: one unit per stage)."""
    graph, plans, n_pp, n_dp = _local_plans(name)
    tasks = graph.tasks
    for r in range(n_pp):
        plan = plans[r]
        flagged = {tasks[tid].stage: (tid, fl) for tid, st, fl, sl, w in plan if fl & 64}
        reduces = {}
        for tid, st, fl, sl, w in plan:
            if tasks[tid].kind == ps.TaskKind.Reduce:
                reduces.setdefault(tasks[tid].stage, []).append((tasks[tid].priority, tid))
        assert set(flagged) == set(reduces)
        for stage, (tid, fl) in flagged.items():
            rs = sorted(reduces[stage])
            assert tasks[rs[-1][1]].deps[0] == tid
            assert bool(fl & 128) == (len(rs) == 1)
