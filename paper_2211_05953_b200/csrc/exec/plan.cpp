// Per-rank execution plan of a TaskGraph (host only, no GPU): which stream each local task
// goes to, which cross-stream events it waits on, and the host enqueue order. Shared by the
// executor and by the CPU multi-rank emulation test (tests/test_plan_multirank.py).
#include "plan.hpp"

#include <algorithm>
#include <map>
#include <set>

namespace bfpp {

std::vector<PlanTask> plan_rank(const TaskGraph& g, i64 pp_rank, i64 n_dp, bool pooled_grads) {
    std::vector<PlanTask> order;
    // enqueue order = start order of a simulation with positive durations (a topological order
    // consistent with every lane's program/priority order on this device)
    TimingModel tm;
    tm.t_fwd_stage = 1.0;
    tm.bwd_ratio = 2.0;
    tm.t_pp_transfer = 0.01;
    tm.t_dp_reduce_stage = 0.05;
    tm.t_dp_reconstruct_stage = 0.05;
    const Timeline sim = simulate(g, tm);
    const size_t n = g.tasks.size();
    std::vector<TaskId> mine;
    for (const Task& t : g.tasks) {
        const bool local = t.device == pp_rank || (t.kind == TaskKind::Transfer && t.peer_device == pp_rank);
        if (local) mine.push_back(t.id);
    }
    std::stable_sort(mine.begin(), mine.end(), [&](TaskId a, TaskId b) {
        return sim.events[static_cast<size_t>(a)].start < sim.events[static_cast<size_t>(b)].start;
    });
    // reconstruct slot numbering (creation order per device) and Reduce unit bookkeeping
    std::map<TaskId, int> rec_slot;
    {
        int k = 0;
        for (const Task& t : g.tasks)
            if (t.kind == TaskKind::Reconstruct && t.device == pp_rank) rec_slot[t.id] = (k++) & 1;
    }
    std::map<TaskId, TaskId> reduce_of_last_bwd;      // last Bwd of a unit -> its Reduce
    std::map<i64, std::vector<TaskId>> reduces_of_stage;
    for (const Task& t : g.tasks)
        if (t.kind == TaskKind::Reduce && t.device == pp_rank) {
            reduce_of_last_bwd[t.deps[0]] = t.id;
            reduces_of_stage[t.stage].push_back(t.id);
        }
    for (auto& kv : reduces_of_stage)
        std::sort(kv.second.begin(), kv.second.end(), [&](TaskId a, TaskId b) {
            return g.tasks[static_cast<size_t>(a)].priority < g.tasks[static_cast<size_t>(b)].priority;
        });
    std::map<i64, TaskId> last_bwd_of_stage, prev_bwd;
    for (TaskId id : g.compute_program[static_cast<size_t>(pp_rank)]) {
        const Task& t = g.tasks[static_cast<size_t>(id)];
        if (t.kind == TaskKind::Bwd) last_bwd_of_stage[t.stage] = id;
    }
    auto stream_of = [&](const Task& t, bool* send) {
        if (t.lane == Lane::Compute) return static_cast<int>(S_COMPUTE);
        if (t.lane == Lane::DpNet) return static_cast<int>(S_DP);
        const bool fwd = g.tasks[static_cast<size_t>(t.deps[0])].kind == TaskKind::Fwd;
        *send = t.device == pp_rank;
        return static_cast<int>(fwd ? (*send ? S_FWD_SEND : S_FWD_RECV) : (*send ? S_BWD_SEND : S_BWD_RECV));
    };
    std::vector<int> stream_of_task(n, -1);
    for (TaskId id : mine) {
        bool send = false;
        stream_of_task[static_cast<size_t>(id)] = stream_of(g.tasks[static_cast<size_t>(id)], &send);
    }
    TaskId last_reduce = -1;  // Reduce of the latest unit-ending backward seen (program order)
    for (TaskId id : mine) {
        const Task& t = g.tasks[static_cast<size_t>(id)];
        PlanTask te;
        te.id = id;
        te.stream = stream_of(t, &te.send);
        for (TaskId d : t.deps) {
            const Task& dt = g.tasks[static_cast<size_t>(d)];
            if (t.kind == TaskKind::Transfer && !te.send) continue;  // the receive side has no local deps
            if (dt.kind == TaskKind::Reconstruct && t.lane == Lane::Compute) te.slot = rec_slot[d];
            if (stream_of_task[static_cast<size_t>(d)] == te.stream) continue;  // same stream: FIFO order
            if (stream_of_task[static_cast<size_t>(d)] < 0) continue;           // remote (reached via a transfer)
            te.waits.push_back(d);
        }
        if (t.kind == TaskKind::Reconstruct) te.slot = rec_slot[id];
        if (t.kind == TaskKind::Bwd) {
            // a new reduction unit of this stage may only start once the previous unit's
            // reduce-scatter has drained the stage's gradient buffer (pooled: per segment, by the
            // executor; the host enqueues this task after the rank's latest Reduce)
            auto pb = prev_bwd.find(t.stage);
            if (pb == prev_bwd.end()) te.first_in_unit = true;
            if (pb != prev_bwd.end()) {
                auto r = reduce_of_last_bwd.find(pb->second);
                if (r != reduce_of_last_bwd.end()) {
                    if (!pooled_grads) te.waits.push_back(r->second);
                    te.first_in_unit = true;
                }
            }
            if (pooled_grads && te.first_in_unit && last_reduce >= 0) te.after.push_back(last_reduce);
            prev_bwd[t.stage] = id;
            if (n_dp < 2 && last_bwd_of_stage[t.stage] == id) te.adam_after = true;
            auto red = reduce_of_last_bwd.find(id);
            if (n_dp >= 2 && red != reduce_of_last_bwd.end()) {
                const auto& rs = reduces_of_stage[t.stage];
                te.unit_end_bwd = true;
                te.last_unit_bwd = rs.back() == red->second;
                te.reduce_first_unit = rs.front() == red->second;
                last_reduce = red->second;
            }
        }
        if (t.kind == TaskKind::Reduce) {
            const auto& rs = reduces_of_stage[t.stage];
            te.first_unit = rs.front() == id;
            te.last_unit = rs.back() == id;
            te.adam_after = te.last_unit;
        }
        order.push_back(te);
    }
    // Host enqueue order: a topological order of this rank's tasks over the explicit waits
    // (graph deps on other streams + the executor's gradient-buffer resource deps) and the
    // per-stream FIFO order, ties broken by simulated start. Every event is then recorded
    // before any stream waits on it.
    {
        const size_t m = order.size();
        std::map<TaskId, size_t> pos;
        for (size_t i = 0; i < m; ++i) pos[order[i].id] = i;
        std::vector<std::vector<size_t>> succ(m);
        std::vector<int> indeg(m, 0);
        std::vector<long> last(S_N, -1);
        for (size_t i = 0; i < m; ++i) {
            const PlanTask& te = order[i];
            if (last[te.stream] >= 0) {
                succ[static_cast<size_t>(last[te.stream])].push_back(i);
                ++indeg[i];
            }
            last[te.stream] = static_cast<long>(i);
            for (TaskId w : te.waits) {
                succ[pos.at(w)].push_back(i);
                ++indeg[i];
            }
            for (TaskId w : te.after) {
                succ[pos.at(w)].push_back(i);
                ++indeg[i];
            }
        }
        std::set<size_t> ready;
        for (size_t i = 0; i < m; ++i)
            if (indeg[i] == 0) ready.insert(i);
        std::vector<PlanTask> sorted;
        while (!ready.empty()) {
            const size_t i = *ready.begin();
            ready.erase(ready.begin());
            sorted.push_back(order[i]);
            for (size_t j : succ[i])
                if (--indeg[j] == 0) ready.insert(j);
        }
        if (sorted.size() != m) throw SimError("executor: cyclic local dependencies");
        order = std::move(sorted);
        for (size_t i = order.size(); i-- > 0;)
            if (order[i].adam_after) {
                order[i].adam_tail = true;
                break;
            }
    }
    return order;
}

}  // namespace bfpp
