// Deterministic three-lane list scheduler and the schedule metrics.
//
// Semantics follow the reference simulator (simulate.cpp:41-158) exactly so
// that event times are bit-identical doubles: compute lanes run their program
// strictly in order, network lanes start the lowest-priority ready task whose
// lanes are free, a Transfer holds the PpNet lane of both endpoints, and all
// tasks finishing at the earliest end time retire together. The same metrics
// (bubble_fraction, peak_inflight; ref simulate.cpp:160-191) are applied to the
// executor's *measured* timelines.
#include <algorithm>
#include <cmath>
#include <functional>
#include <queue>
#include <set>
#include <sstream>

#include "schedule.hpp"

namespace bfpp {

static double duration(const Task& t, const TimingModel& tm) {
    switch (t.kind) {
    case TaskKind::Fwd: return tm.t_fwd_stage;
    case TaskKind::Bwd: return tm.bwd_ratio * tm.t_fwd_stage;
    case TaskKind::Transfer: return tm.t_pp_transfer + tm.pp_latency;
    case TaskKind::Reduce: return tm.t_dp_reduce_stage;
    case TaskKind::Reconstruct: return tm.t_dp_reconstruct_stage;
    }
    return 0.0;
}

namespace {
template <class Dur>
Timeline simulate_impl(const TaskGraph& g, Dur&& duration_of) {
    const size_t n = g.tasks.size();
    const size_t nd = static_cast<size_t>(g.n_devices);
    Timeline tl;
    tl.n_devices = g.n_devices;
    tl.events.assign(n, TimelineEvent{});
    tl.lane_busy.assign(nd, {0.0, 0.0, 0.0});

    std::vector<int> waiting(n);
    std::vector<std::vector<TaskId>> users(n);
    for (const Task& t : g.tasks) {
        waiting[static_cast<size_t>(t.id)] = static_cast<int>(t.deps.size());
        for (TaskId d : t.deps) users[static_cast<size_t>(d)].push_back(t.id);
    }
    std::vector<double> free_at(nd * 3, 0.0);
    auto lane_slot = [](i64 dev, Lane l) { return static_cast<size_t>(dev) * 3 + static_cast<size_t>(l); };
    std::vector<char> ready(n, 0), finished(n, 0);
    std::vector<size_t> pc(nd, 0);
    std::set<std::pair<int, TaskId>> net;  // ready network tasks by (priority, id)
    std::priority_queue<std::pair<double, TaskId>, std::vector<std::pair<double, TaskId>>,
                        std::greater<std::pair<double, TaskId>>>
        inflight;

    auto become_ready = [&](TaskId id) {
        ready[static_cast<size_t>(id)] = 1;
        const Task& t = g.tasks[static_cast<size_t>(id)];
        if (t.lane != Lane::Compute) net.insert({t.priority, id});
    };
    auto lanes_free = [&](const Task& t, double now) {
        if (free_at[lane_slot(t.device, t.lane)] > now) return false;
        if (t.kind == TaskKind::Transfer && free_at[lane_slot(t.peer_device, Lane::PpNet)] > now) return false;
        return true;
    };
    auto launch = [&](const Task& t, double now) {
        const double dur = duration_of(t);
        tl.events[static_cast<size_t>(t.id)] = {t.id, now, now + dur};
        free_at[lane_slot(t.device, t.lane)] = now + dur;
        tl.lane_busy[static_cast<size_t>(t.device)][static_cast<int>(t.lane)] += dur;
        if (t.kind == TaskKind::Transfer) {
            free_at[lane_slot(t.peer_device, Lane::PpNet)] = now + dur;
            tl.lane_busy[static_cast<size_t>(t.peer_device)][static_cast<int>(Lane::PpNet)] += dur;
        }
        inflight.push({now + dur, t.id});
    };

    for (size_t i = 0; i < n; ++i)
        if (waiting[i] == 0) become_ready(static_cast<TaskId>(i));

    size_t left = n;
    double now = 0.0;
    while (left > 0) {
        for (bool again = true; again;) {
            again = false;
            for (size_t d = 0; d < nd; ++d) {
                const auto& prog = g.compute_program[d];
                if (pc[d] >= prog.size()) continue;
                const Task& t = g.tasks[static_cast<size_t>(prog[pc[d]])];
                if (!ready[static_cast<size_t>(t.id)] || free_at[lane_slot(static_cast<i64>(d), Lane::Compute)] > now)
                    continue;
                launch(t, now);
                ++pc[d];
                again = true;
            }
            for (auto it = net.begin(); it != net.end();) {
                const Task& t = g.tasks[static_cast<size_t>(it->second)];
                if (lanes_free(t, now)) {
                    launch(t, now);
                    it = net.erase(it);
                    again = true;
                } else {
                    ++it;
                }
            }
        }
        if (inflight.empty()) {
            std::ostringstream os;
            os << "simulate: deadlock with " << left
               << " tasks pending (inconsistent program order and dependencies)";
            throw SimError(os.str());
        }
        now = inflight.top().first;
        while (!inflight.empty() && inflight.top().first <= now) {
            const TaskId id = inflight.top().second;
            inflight.pop();
            if (finished[static_cast<size_t>(id)]) continue;
            finished[static_cast<size_t>(id)] = 1;
            --left;
            for (TaskId u : users[static_cast<size_t>(id)])
                if (--waiting[static_cast<size_t>(u)] == 0) become_ready(u);
        }
        tl.makespan = std::max(tl.makespan, now);
    }
    return tl;
}
}  // namespace

Timeline simulate(const TaskGraph& g, const TimingModel& tm) {
    tm.validate();
    return simulate_impl(g, [&](const Task& t) { return duration(t, tm); });
}

// The same list scheduler with one duration per task (e.g. every task's measured duration): the
// makespan an executor with zero overhead would reach with those task times.
Timeline simulate_durations(const TaskGraph& g, const std::vector<double>& dur) {
    if (dur.size() != g.tasks.size()) throw SpecError("simulate_durations: one duration per task expected");
    for (double d : dur)
        if (!(d >= 0.0) || !std::isfinite(d)) throw SpecError("simulate_durations: durations must be finite and >= 0");
    return simulate_impl(g, [&](const Task& t) { return dur[static_cast<size_t>(t.id)]; });
}

Timeline timeline_from_intervals(const TaskGraph& g, const double* start, const double* end) {
    Timeline tl;
    tl.n_devices = g.n_devices;
    tl.lane_busy.assign(static_cast<size_t>(g.n_devices), {0.0, 0.0, 0.0});
    tl.events.resize(g.tasks.size());
    for (const Task& t : g.tasks) {
        const size_t i = static_cast<size_t>(t.id);
        const double dur = end[i] - start[i];
        tl.events[i] = {t.id, start[i], end[i]};
        tl.lane_busy[static_cast<size_t>(t.device)][static_cast<int>(t.lane)] += dur;
        if (t.kind == TaskKind::Transfer)
            tl.lane_busy[static_cast<size_t>(t.peer_device)][static_cast<int>(Lane::PpNet)] += dur;
        tl.makespan = std::max(tl.makespan, end[i]);
    }
    return tl;
}

double bubble_fraction(const Timeline& tl) {
    const double busy = tl.compute_busy_max();
    return busy <= 0.0 ? 0.0 : (tl.makespan - busy) / busy;
}

std::vector<i64> peak_inflight(const Timeline& tl, const TaskGraph& g, i64 layers_per_stage) {
    std::vector<std::vector<std::pair<double, int>>> marks(static_cast<size_t>(tl.n_devices));
    for (const Task& t : g.tasks) {
        if (t.lane != Lane::Compute) continue;
        marks[static_cast<size_t>(t.device)].push_back(
            {tl.events[static_cast<size_t>(t.id)].end, t.kind == TaskKind::Fwd ? 1 : -1});
    }
    std::vector<i64> peaks;
    for (auto& m : marks) {
        std::sort(m.begin(), m.end());  // releases sort before births at equal times
        i64 live = 0, peak = 0;
        for (const auto& e : m) peak = std::max(peak, live += e.second);
        peaks.push_back(peak * layers_per_stage);
    }
    return peaks;
}

}  // namespace bfpp
