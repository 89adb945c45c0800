// The reference's analytic per-device memory model (proj/src/memory.cpp:7-86) and cluster
// presets (types.cpp:206-231), restated so the executor's real allocations (Executor::memory_plan,
// bfpp_exec_memory_plan) can be held against it, plus a B200 preset the reference lacks.
#include <algorithm>
#include <string>

#include "schedule.hpp"

namespace bfpp {

// memory.cpp:7-31: training state per device. DP0 keeps opts.dp0_bytes_per_param per parameter
// of its pipeline slice; DP_PS 2 or 4 bytes (4 when gradients of several micro-batches wait for
// the reduction); DP_FS two reconstructed layers of bf16 weights + gradients (8 P / L).
double state_memory(const ModelSpec& m, const ParallelConfig& c, const MemoryOptions& o) {
    c.validate(m);
    const double P = static_cast<double>(param_count(m)), split = static_cast<double>(c.n_pp * c.n_tp);
    if (c.dp_variant == DpVariant::DP0) return o.dp0_bytes_per_param * P / split;
    if (c.dp_variant == DpVariant::DP_PS)
        return (c.schedule == Schedule::BreadthFirst || c.n_mb == 1 ? 2.0 : 4.0) * P / split;
    return 8.0 * P / (static_cast<double>(m.n_layers) * static_cast<double>(c.n_tp));
}

// memory.cpp:33-43: one micro-batch's full activations + gradients of one layer
// (s b h (10 + 24/t + 5 s a / (h t)) bytes).
double activation_memory(const ModelSpec& m, const ParallelConfig& c) {
    c.validate(m);
    const double t = static_cast<double>(c.n_tp), s = static_cast<double>(m.s_seq), h = static_cast<double>(m.s_hidden);
    return s * static_cast<double>(c.s_mb) * h * (10.0 + 24.0 / t + 5.0 * s * static_cast<double>(m.n_heads) / (h * t));
}

// memory.cpp:45-62: live layer-input checkpoints per device, capped per schedule.
double checkpoint_count(const ModelSpec& m, const ParallelConfig& c) {
    c.validate(m);
    const double L = static_cast<double>(m.n_layers), p = static_cast<double>(c.n_pp),
                 mb = static_cast<double>(c.n_mb);
    switch (c.schedule) {
    case Schedule::NoPipeline: return mb * L;
    case Schedule::GPipe:
    case Schedule::BreadthFirst: return mb * L / p;
    case Schedule::OneFOneB: return std::min(mb * L / p, (2.0 * p - 1.0) * L / p);
    case Schedule::DepthFirst: return std::min(mb * L / p, L + p - 1.0);
    }
    return 0.0;
}

// memory.cpp:64-70: one checkpoint = the layer input, 2 s b h / t bytes.
double checkpoint_memory(const ModelSpec& m, const ParallelConfig& c) {
    return checkpoint_count(m, c) * 2.0 * static_cast<double>(m.s_seq) * static_cast<double>(c.s_mb) *
           static_cast<double>(m.s_hidden) / static_cast<double>(c.n_tp);
}

MemoryBreakdown total_memory(const ModelSpec& m, const ParallelConfig& c, const MemoryOptions& o) {
    MemoryBreakdown b;
    b.state_bytes = state_memory(m, c, o);
    b.activation_bytes = activation_memory(m, c);
    b.checkpoint_bytes = checkpoint_memory(m, c);
    b.total_bytes = b.state_bytes + b.activation_bytes + b.checkpoint_bytes;
    return b;
}

// memory.cpp:82-86
bool feasible(const ModelSpec& m, const ParallelConfig& c, const ClusterSpec& k, const MemoryOptions& o) {
    return total_memory(m, c, o).total_bytes <= o.headroom * k.mem_capacity;
}

ClusterSpec cluster_preset(const std::string& name) {
    ClusterSpec k;
    if (name == "a100") {  // types.cpp:208-218
        k.n_node = 4, k.s_node = 8, k.peak_flops = 312e12, k.bw_intra = 600e9, k.bw_inter = 50e9;
        k.pp_latency = 20e-6, k.mem_capacity = 80.0 * (1ull << 30), k.kernel_efficiency = 0.6;
        return k;
    }
    if (name == "v100-dgx1") {  // types.cpp:219-229
        k.n_node = 8, k.s_node = 8, k.peak_flops = 125e12, k.bw_intra = 300e9, k.bw_inter = 32e9;
        k.pp_latency = 30e-6, k.mem_capacity = 32.0 * (1ull << 30), k.kernel_efficiency = 0.6;
        return k;
    }
    if (name == "b200") {
        // one 8 x B200 NVSwitch node: 2.25 PFLOP/s dense bf16, NVLink 5 900 GB/s per direction
        // (input + output, the reference's convention), 400 Gb/s NIC per GPU, 180 GB HBM3e;
        // kernel efficiency = the executor's measured GEMM rate in isolation over the spec peak
        // (1.2-1.33 PFLOP/s / 2.25); pp_latency = a measured small peer copy
        k.n_node = 1, k.s_node = 8, k.peak_flops = 2.25e15, k.bw_intra = 1.8e12, k.bw_inter = 100e9;
        k.pp_latency = 10e-6, k.mem_capacity = 180e9, k.kernel_efficiency = 0.55;
        return k;
    }
    throw SpecError("unknown cluster preset '" + name + "'");
}

}  // namespace bfpp
