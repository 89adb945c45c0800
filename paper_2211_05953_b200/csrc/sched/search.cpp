// Configuration search (the reference's search.cpp:13-188, enumerate_configs / rank_configs with
// simulate scoring) restated for the executor's grid (n_tp = 1), plus a "measured" scoring mode:
// every candidate is simulated with a TimingModel built from per-kind task durations measured on
// B200s (a measured timeline's mean Fwd / Bwd / Transfer / Reconstruct / Reduce durations scaled
// to the candidate's stage size, micro-batch size and message sizes) instead of
// TimingModel::derive's peak * efficiency and nominal link bandwidths.
#include <algorithm>
#include <atomic>
#include <set>
#include <thread>
#include <tuple>

#include "schedule.hpp"

namespace bfpp {

namespace {

bool sharding_policy_allows(Schedule s, DpVariant v) {  // search.cpp:33-44
    switch (v) {
    case DpVariant::DP0: return true;
    case DpVariant::DP_PS: return s == Schedule::GPipe || s == Schedule::OneFOneB;
    case DpVariant::DP_FS: return s == Schedule::BreadthFirst || s == Schedule::NoPipeline;
    }
    return false;
}

bool looped(Schedule s) { return s == Schedule::DepthFirst || s == Schedule::BreadthFirst; }

using Key = std::tuple<i64, i64, i64, i64, i64, i64, int, int>;
Key config_key(const ParallelConfig& c) {  // search.cpp:46-57
    return {c.n_pp, c.n_tp, c.s_mb, c.n_mb, c.n_loop, c.n_dp, static_cast<int>(c.dp_variant),
            static_cast<int>(c.schedule)};
}

double stage_params(const ModelSpec& m, const ParallelConfig& c) {
    return 12.0 * static_cast<double>(m.s_hidden) * static_cast<double>(m.s_hidden) *
           static_cast<double>(m.n_layers) / (static_cast<double>(c.n_stage()) * static_cast<double>(c.n_tp));
}
double message_bytes(const ModelSpec& m, const ParallelConfig& c) {  // one [s_mb * seq, h] bf16 hand-off
    return 2.0 * static_cast<double>(m.s_hidden) * static_cast<double>(m.s_seq) * static_cast<double>(c.s_mb) /
           static_cast<double>(c.n_tp);
}

}  // namespace

// schedule.cpp:43-86 (n_tp = 1: no tensor-parallel blocking term); recompute defaults to true as in
// the reference (schedule.hpp:37-38)
TimingModel derive_timing(const ModelSpec& m, const ParallelConfig& c, const ClusterSpec& k, bool recompute) {
    c.validate(m, k);
    if (c.n_tp != 1) throw SpecError("derive_timing: tensor parallelism is not modelled (n_tp must be 1)");
    TimingModel t;
    t.bwd_ratio = recompute ? 3.0 : 2.0;
    const double effective = k.peak_flops * k.kernel_efficiency;
    t.t_fwd_stage = compute_per_gpu(m, c) /
                    (static_cast<double>(c.n_mb) * static_cast<double>(c.n_loop) * (1.0 + t.bwd_ratio) * effective);
    const double pp_bw = c.n_tp * c.n_pp <= k.s_node ? k.bw_intra : k.bw_inter;
    t.t_pp_transfer = 4.0 * static_cast<double>(m.s_hidden) * static_cast<double>(m.s_seq) *
                      static_cast<double>(c.s_mb) / (static_cast<double>(c.n_tp) * pp_bw);
    t.pp_latency = k.pp_latency;
    const double dp_bw = c.n_dp * c.n_tp * c.n_pp <= k.s_node ? k.bw_intra : k.bw_inter;
    if (c.n_dp >= 2) {
        t.t_dp_reduce_stage = 8.0 * stage_params(m, c) / dp_bw;
        t.t_dp_reconstruct_stage = 2.0 * stage_params(m, c) / dp_bw;
    } else {
        t.t_dp_reduce_stage = 0.0;
        t.t_dp_reconstruct_stage = 0.0;
    }
    return t;
}

MeasuredRates rates_from_timing(const ModelSpec& m, const ParallelConfig& c, const TimingModel& t) {
    c.validate(m);
    MeasuredRates r;
    const double layers = static_cast<double>(m.n_layers) / static_cast<double>(c.n_stage());
    r.fwd_layer_seq = t.t_fwd_stage / (layers * static_cast<double>(c.s_mb));
    r.bwd_ratio = t.bwd_ratio;
    r.pp_s_per_byte = t.t_pp_transfer / message_bytes(m, c);
    r.pp_latency = t.pp_latency;
    r.reduce_s_per_param = c.n_dp >= 2 ? t.t_dp_reduce_stage / stage_params(m, c) : 0.0;
    r.reconstruct_s_per_param = c.n_dp >= 2 ? t.t_dp_reconstruct_stage / stage_params(m, c) : 0.0;
    return r;
}

TimingModel timing_from_rates(const ModelSpec& m, const ParallelConfig& c, const MeasuredRates& r) {
    c.validate(m);
    TimingModel t;
    const double layers = static_cast<double>(m.n_layers) / static_cast<double>(c.n_stage());
    t.t_fwd_stage = r.fwd_layer_seq * layers * static_cast<double>(c.s_mb);
    t.bwd_ratio = r.bwd_ratio;
    t.t_pp_transfer = r.pp_s_per_byte * message_bytes(m, c);
    t.pp_latency = r.pp_latency;
    t.t_dp_reduce_stage = c.n_dp >= 2 ? r.reduce_s_per_param * stage_params(m, c) : 0.0;
    t.t_dp_reconstruct_stage = c.n_dp >= 2 ? r.reconstruct_s_per_param * stage_params(m, c) : 0.0;
    return t;
}

std::vector<ParallelConfig> enumerate_configs(const SearchSpace& sp, const ModelSpec& m, const ClusterSpec& k) {
    if (sp.schedules.empty() || sp.n_pp.empty() || sp.n_tp.empty() || sp.s_mb.empty() || sp.n_mb.empty() ||
        sp.n_loop.empty() || sp.dp_variants.empty() || sp.batch_sizes.empty())
        throw SpecError("search space: all choice sets must be nonempty");
    m.validate();
    k.validate();
    const i64 n_gpu = k.n_node * k.s_node;
    std::vector<ParallelConfig> out;
    std::set<Key> seen;
    const std::set<int> scheds(sp.schedules.begin(), sp.schedules.end()),
        variants(sp.dp_variants.begin(), sp.dp_variants.end());
    const std::set<i64> pps(sp.n_pp.begin(), sp.n_pp.end()), tps(sp.n_tp.begin(), sp.n_tp.end()),
        smbs(sp.s_mb.begin(), sp.s_mb.end()), mbs(sp.n_mb.begin(), sp.n_mb.end()),
        loops(sp.n_loop.begin(), sp.n_loop.end()), batches(sp.batch_sizes.begin(), sp.batch_sizes.end());
    for (int si : scheds)
        for (int vi : variants) {
            const Schedule s = static_cast<Schedule>(si);
            const DpVariant v = static_cast<DpVariant>(vi);
            if (!sharding_policy_allows(s, v)) continue;
            for (i64 pp : pps)
                for (i64 tp : tps)
                    for (i64 smb : smbs)
                        for (i64 mb : mbs)
                            for (i64 lp : loops)
                                for (i64 batch : batches) {
                                    ParallelConfig c;
                                    c.schedule = s;
                                    c.dp_variant = v;
                                    c.n_pp = s == Schedule::NoPipeline ? 1 : pp;
                                    c.n_loop = looped(s) ? lp : 1;
                                    c.n_tp = tp;
                                    c.s_mb = smb;
                                    c.n_mb = mb;
                                    if (c.n_tp * c.n_pp > n_gpu || n_gpu % (c.n_tp * c.n_pp) != 0) continue;
                                    c.n_dp = n_gpu / (c.n_tp * c.n_pp);
                                    if (c.batch_size() != batch) continue;
                                    try {
                                        c.validate(m, k);
                                    } catch (const SpecError&) {
                                        continue;
                                    }
                                    if (seen.insert(config_key(c)).second) out.push_back(c);
                                }
        }
    std::sort(out.begin(), out.end(),
              [](const ParallelConfig& a, const ParallelConfig& b) { return config_key(a) < config_key(b); });
    return out;
}

std::vector<RankedConfig> rank_configs(const std::vector<ParallelConfig>& configs, const ModelSpec& m,
                                       const ClusterSpec& k, bool measured, const MeasuredRates& rates,
                                       const MemoryOptions& mo, int threads) {
    std::vector<const ParallelConfig*> ok;
    for (const ParallelConfig& c : configs)
        if (feasible(m, c, k, mo)) ok.push_back(&c);
    std::vector<RankedConfig> scored(ok.size());
    auto eval = [&](size_t i) {
        RankedConfig rc;
        rc.config = *ok[i];
        rc.memory_bytes = total_memory(m, rc.config, mo).total_bytes;
        const StagePlacement pl = place_stages(m, rc.config);
        const TaskGraph g = build_tasks(m, rc.config, pl);
        // simulate_score derives with the default recompute = true (schedule.hpp:37-38: bwd_ratio 3)
        rc.timing = measured ? timing_from_rates(m, rc.config, rates) : derive_timing(m, rc.config, k);
        const Timeline tl = simulate(g, rc.timing);
        rc.config.validate(m, k);
        if (tl.makespan <= 0) throw SpecError("throughput: timeline has no extent");
        rc.score = compute_per_gpu(m, rc.config) / tl.makespan;  // perf.cpp:8-20
        rc.bubble = bubble_fraction(tl);
        scored[i] = rc;
    };
    unsigned n = threads > 0 ? static_cast<unsigned>(threads) : std::max(1u, std::thread::hardware_concurrency());
    n = std::min<unsigned>(n, static_cast<unsigned>(std::max<size_t>(1, scored.size())));
    if (n <= 1) {
        for (size_t i = 0; i < scored.size(); ++i) eval(i);
    } else {
        std::vector<std::thread> pool;
        std::atomic<size_t> next{0};
        for (unsigned t = 0; t < n; ++t)
            pool.emplace_back([&] {
                for (size_t i = next.fetch_add(1); i < scored.size(); i = next.fetch_add(1)) eval(i);
            });
        for (auto& th : pool) th.join();
    }
    // best first; ties toward lower memory, then less model parallelism (search.cpp:174-186)
    std::stable_sort(scored.begin(), scored.end(), [](const RankedConfig& a, const RankedConfig& b) {
        auto key = [](const RankedConfig& r) {
            return std::make_tuple(-r.score, r.memory_bytes, r.config.n_tp, r.config.n_pp, config_key(r.config));
        };
        return key(a) < key(b);
    });
    return scored;
}

}  // namespace bfpp
