// Schedule construction for the breadth-first pipeline executor.
//
// Behavioural contract (bit-exact, checked against the compiled reference in
// tests/test_schedule_parity.py):
//   * looping placement, stage s -> device s mod n_pp      (ref schedule.cpp:23-33)
//   * forward-first programs (BF / GPipe / NoPipeline)      (ref schedule.cpp:315-331)
//   * looped depth-first programs                           (ref schedule.cpp:335-375)
//   * non-looped 1F1B programs                              (ref schedule.cpp:377-392)
//   * task ids, deps (incl. their order) and priorities     (ref schedule.cpp:117-313)
//   * validation messages                                   (ref types.cpp:92-130)
// The implementation is organised differently from the reference (programs are
// produced by one generator keyed on the schedule, the graph is wired by a
// small set of free functions over a flat task vector).
#include "schedule.hpp"

#include <algorithm>
#include <cmath>
#include <map>
#include <sstream>
#include <tuple>

namespace bfpp {

const char* kind_name(TaskKind k) {
    static const char* names[] = {"Fwd", "Bwd", "Reduce", "Reconstruct", "Transfer"};
    int i = static_cast<int>(k);
    return (i >= 0 && i < 5) ? names[i] : "?";
}

const char* schedule_name(Schedule s) {
    static const char* names[] = {"no_pipeline", "gpipe", "1f1b", "depth_first", "breadth_first"};
    int i = static_cast<int>(s);
    return (i >= 0 && i < 5) ? names[i] : "?";
}

static void require(bool ok, const char* msg) {
    if (!ok) throw SpecError(msg);
}

void ModelSpec::validate() const {
    require(n_layers >= 1 && s_hidden >= 1 && n_heads >= 1 && s_head >= 1 && s_mlp >= 1 &&
                s_seq >= 1 && s_voc >= 1,
            "model: all size fields must be >= 1");
    require(n_heads * s_head == s_hidden, "model: n_heads * s_head must equal s_hidden");
}

void ClusterSpec::validate() const {
    require(n_node >= 1 && s_node >= 1, "cluster: node counts must be >= 1");
    require(peak_flops > 0, "cluster: peak_flops must be positive");
    require(bw_intra > 0 && bw_inter > 0, "cluster: bandwidths must be positive");
    require(pp_latency >= 0, "cluster: pp_latency must be non-negative");
    require(mem_capacity >= 0, "cluster: mem_capacity must be non-negative");
    require(kernel_efficiency > 0 && kernel_efficiency <= 1,
            "cluster: kernel_efficiency must be in (0, 1]");
    require(std::isfinite(peak_flops / bw_intra) && std::isfinite(peak_flops / bw_inter),
            "cluster: hardware intensities must be finite");
}

void ParallelConfig::validate() const {
    require(n_dp >= 1 && n_tp >= 1 && n_pp >= 1 && n_mb >= 1 && s_mb >= 1 && n_loop >= 1,
            "config: all grid and batching fields must be >= 1");
    const bool looped = schedule == Schedule::DepthFirst || schedule == Schedule::BreadthFirst;
    if (schedule == Schedule::NoPipeline) {
        require(n_pp == 1, "config: no_pipeline requires n_pp = 1");
        require(n_loop == 1, "config: no_pipeline requires n_loop = 1");
    }
    if (!looped && schedule != Schedule::NoPipeline)
        require(n_loop == 1, "config: non-looped schedules require n_loop = 1");
    if (schedule != Schedule::NoPipeline && n_pp > 1)
        require(n_mb >= n_pp, "config: pipelined schedules require n_mb >= n_pp");
    if (schedule == Schedule::DepthFirst)
        require(n_mb % n_pp == 0, "config: depth_first requires n_mb to be a multiple of n_pp");
}

void ParallelConfig::validate(const ModelSpec& m) const {
    validate();
    m.validate();
    if (m.n_layers % n_stage() != 0) {
        std::ostringstream os;
        os << "config: divisibility violated, n_stage = n_pp * n_loop = " << n_stage()
           << " does not divide n_layers = " << m.n_layers;
        throw SpecError(os.str());
    }
}

void ParallelConfig::validate(const ModelSpec& m, const ClusterSpec& c) const {
    validate(m);
    c.validate();
    if (grid_size() != c.n_gpu()) {
        std::ostringstream os;
        os << "config: grid mismatch, n_dp * n_tp * n_pp = " << grid_size()
           << " but the cluster has " << c.n_gpu() << " devices";
        throw SpecError(os.str());
    }
}

void TimingModel::validate() const {
    if (t_fwd_stage < 0 || t_pp_transfer < 0 || pp_latency < 0 || t_dp_reduce_stage < 0 ||
        t_dp_reconstruct_stage < 0)
        throw SpecError("timing: durations must be non-negative");
    if (bwd_ratio < 1.0) throw SpecError("timing: bwd_ratio must be >= 1");
}

double Timeline::compute_busy_max() const {
    double m = 0.0;
    for (const auto& l : lane_busy) m = std::max(m, l[0]);
    return m;
}

StagePlacement place_stages(const ModelSpec& m, const ParallelConfig& c) {
    c.validate(m);
    StagePlacement pl;
    pl.n_stage = c.n_stage();
    pl.n_pp = c.n_pp;
    pl.layers_per_stage = m.n_layers / pl.n_stage;
    pl.assignment.reserve(static_cast<size_t>(pl.n_stage));
    for (i64 s = 0; s < pl.n_stage; ++s) pl.assignment.push_back(s % c.n_pp);
    return pl;
}

namespace {

struct Step {
    TaskKind kind;
    i64 mb, stage;
};
using Program = std::vector<Step>;

// Which micro-batches share one sharded-DP reconstruction/reduction.
struct DpUnits {
    enum Mode { Stage, Group, MicroBatch } mode = Stage;
    i64 group = 1;
    i64 of(i64 mb) const { return mode == Stage ? 0 : mode == Group ? mb / group : mb; }
};

// Warm-up forwards, then one-forward-one-backward, then the backward drain.
Program alternate(const Program& f, const Program& b, size_t warm) {
    Program out;
    out.reserve(f.size() + b.size());
    warm = std::min(warm, f.size());
    size_t bi = 0;
    for (size_t k = 0; k < f.size(); ++k) {
        out.push_back(f[k]);
        if (k >= warm) out.push_back(b[bi++]);
    }
    while (bi < b.size()) out.push_back(b[bi++]);
    return out;
}

// Per-device compute programs; device d owns stages d, d+p, ..., d+(v-1)p.
std::vector<Program> make_programs(Schedule sched, i64 p, i64 v, i64 n_mb) {
    std::vector<Program> progs(static_cast<size_t>(p));
    for (i64 d = 0; d < p; ++d) {
        Program& prog = progs[static_cast<size_t>(d)];
        auto stage = [&](i64 loop) { return loop * p + d; };
        switch (sched) {
        case Schedule::NoPipeline:
        case Schedule::GPipe:
        case Schedule::BreadthFirst:
            // Every loop sweeps all micro-batches before the next loop starts.
            for (i64 c = 0; c < v; ++c)
                for (i64 mb = 0; mb < n_mb; ++mb) prog.push_back({TaskKind::Fwd, mb, stage(c)});
            for (i64 c = v - 1; c >= 0; --c)
                for (i64 mb = 0; mb < n_mb; ++mb) prog.push_back({TaskKind::Bwd, mb, stage(c)});
            break;
        case Schedule::OneFOneB: {
            Program f, b;
            for (i64 mb = 0; mb < n_mb; ++mb) {
                f.push_back({TaskKind::Fwd, mb, d});
                b.push_back({TaskKind::Bwd, mb, d});
            }
            prog = alternate(f, b, static_cast<size_t>(p - d - 1));
            break;
        }
        case Schedule::DepthFirst: {
            // Sequences of p micro-batches walk all loops before the next sequence.
            Program f, b;
            for (i64 g = 0; g * p < n_mb; ++g) {
                for (i64 c = 0; c < v; ++c)
                    for (i64 i = 0; i < p; ++i) f.push_back({TaskKind::Fwd, g * p + i, stage(c)});
                for (i64 c = v - 1; c >= 0; --c)
                    for (i64 i = 0; i < p; ++i) b.push_back({TaskKind::Bwd, g * p + i, stage(c)});
            }
            size_t warm = n_mb == p ? f.size() : static_cast<size_t>(2 * (p - d - 1) + (v - 1) * p);
            prog = alternate(f, b, warm);
            break;
        }
        }
    }
    return progs;
}

class Wiring {
public:
    Wiring(const StagePlacement& pl, i64 n_dev, i64 n_mb)
        : pl_(pl), n_stage_(pl.n_stage), n_mb_(n_mb),
          fwd_(static_cast<size_t>(n_mb * pl.n_stage), -1),
          bwd_(static_cast<size_t>(n_mb * pl.n_stage), -1) {
        g_.n_devices = n_dev;
        g_.compute_program.assign(static_cast<size_t>(n_dev), {});
    }

    TaskGraph graph() { return std::move(g_); }

    void compute(const std::vector<Program>& progs) {
        for (i64 d = 0; d < g_.n_devices; ++d) {
            auto& order = g_.compute_program[static_cast<size_t>(d)];
            for (const Step& st : progs[static_cast<size_t>(d)]) {
                TaskId id = emit(d, Lane::Compute, st.kind, st.mb, st.stage);
                TaskId& slot = (st.kind == TaskKind::Fwd ? fwd_ : bwd_)[at(st.mb, st.stage)];
                if (slot != -1) throw SpecError("schedule: duplicate compute step");
                slot = id;
                task(id).priority = static_cast<int>(order.size());
                order.push_back(id);
            }
        }
        for (TaskId f : fwd_)
            if (f == -1) throw SpecError("schedule: incomplete compute program");
        for (TaskId b : bwd_)
            if (b == -1) throw SpecError("schedule: incomplete compute program");
    }

    // Activation hand-offs: forward boundaries ascending, then backward
    // boundaries descending; transfers are numbered in creation order.
    void pipeline() {
        int seq = 0;
        auto boundary = [&](i64 from, i64 to, TaskKind k) {
            const i64 src = pl_.device_of(from), dst = pl_.device_of(to);
            for (i64 mb = 0; mb < n_mb_; ++mb) {
                TaskId producer = id_of(k, mb, from), consumer = id_of(k, mb, to);
                if (src == dst) {
                    task(consumer).deps.push_back(producer);
                    continue;
                }
                TaskId t = emit(src, Lane::PpNet, TaskKind::Transfer, mb, from);
                task(t).peer_device = dst;
                task(t).priority = seq++;
                task(t).deps.push_back(producer);
                task(consumer).deps.push_back(t);
            }
        };
        for (i64 s = 0; s + 1 < n_stage_; ++s) boundary(s, s + 1, TaskKind::Fwd);
        for (i64 s = n_stage_ - 1; s >= 1; --s) boundary(s, s - 1, TaskKind::Bwd);
        for (i64 mb = 0; mb < n_mb_; ++mb)
            for (i64 s = 0; s < n_stage_; ++s)
                task(id_of(TaskKind::Bwd, mb, s)).deps.push_back(id_of(TaskKind::Fwd, mb, s));
    }

    // Fully sharded weight all-gathers: one per (direction, unit, stage) in
    // first-use order; slot j is free once the last user of slot j-2 is done.
    void reconstructions(const DpUnits& u) {
        for (i64 d = 0; d < g_.n_devices; ++d) {
            std::vector<std::vector<TaskId>> users;
            std::map<std::tuple<int, i64, i64>, size_t> index;
            for (TaskId id : g_.compute_program[static_cast<size_t>(d)]) {
                const Task& t = task(id);
                auto key = std::make_tuple(t.kind == TaskKind::Fwd ? 0 : 1, u.of(t.micro_batch), t.stage);
                auto it = index.find(key);
                if (it == index.end()) {
                    it = index.emplace(key, users.size()).first;
                    users.emplace_back();
                }
                users[it->second].push_back(id);
            }
            for (size_t j = 0; j < users.size(); ++j) {
                const Task& head = task(users[j].front());
                TaskId r = emit(d, Lane::DpNet, TaskKind::Reconstruct, head.micro_batch, head.stage);
                for (TaskId user : users[j]) task(user).deps.push_back(r);
                int key = -2;
                if (j >= 2) {
                    TaskId release = users[j - 2].back();
                    task(r).deps.push_back(release);
                    key = 2 * task(release).priority;
                }
                dp_keys_.push_back({r, key});
            }
        }
    }

    // One gradient reduction per (stage, unit) after its last backward.
    void reductions(const DpUnits& u) {
        for (i64 d = 0; d < g_.n_devices; ++d) {
            std::map<std::pair<i64, i64>, TaskId> last;
            for (TaskId id : g_.compute_program[static_cast<size_t>(d)]) {
                const Task& t = task(id);
                if (t.kind == TaskKind::Bwd) last[{t.stage, u.of(t.micro_batch)}] = id;
            }
            for (const auto& kv : last) {
                const TaskId b = kv.second;
                const i64 mb = task(b).micro_batch;
                TaskId r = emit(d, Lane::DpNet, TaskKind::Reduce, mb, kv.first.first);
                task(r).deps.push_back(b);
                dp_keys_.push_back({r, 2 * task(b).priority + 1});
            }
        }
    }

    // DP lane order: stable by release key across all devices.
    void dp_priorities() {
        std::stable_sort(dp_keys_.begin(), dp_keys_.end(),
                         [](const std::pair<TaskId, int>& a, const std::pair<TaskId, int>& b) {
                             return a.second < b.second;
                         });
        for (size_t r = 0; r < dp_keys_.size(); ++r) task(dp_keys_[r].first).priority = static_cast<int>(r);
    }

private:
    size_t at(i64 mb, i64 s) const { return static_cast<size_t>(mb * n_stage_ + s); }
    TaskId id_of(TaskKind k, i64 mb, i64 s) const { return (k == TaskKind::Fwd ? fwd_ : bwd_)[at(mb, s)]; }
    Task& task(TaskId id) { return g_.tasks[static_cast<size_t>(id)]; }
    TaskId emit(i64 dev, Lane lane, TaskKind kind, i64 mb, i64 stage) {
        Task t;
        t.id = static_cast<TaskId>(g_.tasks.size());
        t.device = dev;
        t.lane = lane;
        t.kind = kind;
        t.micro_batch = mb;
        t.stage = stage;
        g_.tasks.push_back(std::move(t));
        return g_.tasks.back().id;
    }

    const StagePlacement& pl_;
    i64 n_stage_, n_mb_;
    TaskGraph g_;
    std::vector<TaskId> fwd_, bwd_;
    std::vector<std::pair<TaskId, int>> dp_keys_;
};

TaskGraph wire(const StagePlacement& pl, i64 n_dev, i64 n_mb, const std::vector<Program>& progs,
               bool dp_traffic, DpVariant variant, DpUnits units) {
    if (variant != DpVariant::DP_FS) units.mode = DpUnits::Stage;
    Wiring w(pl, n_dev, n_mb);
    w.compute(progs);
    w.pipeline();
    if (dp_traffic) {
        if (variant == DpVariant::DP_FS) w.reconstructions(units);
        w.reductions(units);
        w.dp_priorities();
    }
    return w.graph();
}

}  // namespace

TaskGraph build_tasks(const ModelSpec& m, const ParallelConfig& c, const StagePlacement& pl) {
    c.validate(m);
    if (pl.n_stage != c.n_stage() || pl.n_pp != c.n_pp)
        throw SpecError("schedule: placement does not match the configuration");
    DpUnits units;
    if (c.schedule == Schedule::DepthFirst) {
        units.mode = DpUnits::Group;
        units.group = c.n_pp;
    } else if (c.schedule != Schedule::BreadthFirst) {
        units.mode = DpUnits::MicroBatch;  // plain gradient accumulation
    }
    auto progs = make_programs(c.schedule, c.n_pp, pl.n_stage / c.n_pp, c.n_mb);
    return wire(pl, c.n_pp, c.n_mb, progs, c.n_dp >= 2, c.dp_variant, units);
}

TaskGraph build_accumulation_tasks(const ModelSpec& m, DpVariant v, AccumulationOrder o, i64 n_mb) {
    m.validate();
    if (n_mb < 1) throw SpecError("accumulation: n_mb must be >= 1");
    StagePlacement pl;
    pl.n_stage = m.n_layers;
    pl.n_pp = 1;
    pl.layers_per_stage = 1;
    pl.assignment.assign(static_cast<size_t>(m.n_layers), 0);
    std::vector<Program> progs(1);
    Program& prog = progs[0];
    const i64 L = m.n_layers;
    if (o == AccumulationOrder::DepthFirst) {
        for (i64 mb = 0; mb < n_mb; ++mb) {
            for (i64 l = 0; l < L; ++l) prog.push_back({TaskKind::Fwd, mb, l});
            for (i64 l = L - 1; l >= 0; --l) prog.push_back({TaskKind::Bwd, mb, l});
        }
    } else {
        for (i64 l = 0; l < L; ++l)
            for (i64 mb = 0; mb < n_mb; ++mb) prog.push_back({TaskKind::Fwd, mb, l});
        for (i64 l = L - 1; l >= 0; --l)
            for (i64 mb = 0; mb < n_mb; ++mb) prog.push_back({TaskKind::Bwd, mb, l});
    }
    DpUnits units;
    units.mode = o == AccumulationOrder::BreadthFirst ? DpUnits::Stage : DpUnits::MicroBatch;
    return wire(pl, 1, n_mb, progs, true, v, units);
}

i64 param_count(const ModelSpec& m) { return 12 * m.n_layers * m.s_hidden * m.s_hidden; }

double compute_per_gpu(const ModelSpec& m, const ParallelConfig& c) {
    // Eq. 11, evaluated in the reference's operation order for bit-equality.
    const double h = static_cast<double>(m.s_hidden);
    const double per_token = 96.0 * static_cast<double>(c.n_mb) * static_cast<double>(c.s_mb) *
                             static_cast<double>(m.n_layers) * h *
                             (h + static_cast<double>(m.s_seq) / 6.0 +
                              static_cast<double>(m.s_voc) / (16.0 * static_cast<double>(m.n_layers)));
    return static_cast<double>(m.s_seq) * per_token /
           (static_cast<double>(c.n_pp) * static_cast<double>(c.n_tp));
}

}  // namespace bfpp
