// extern "C" boundary of the executor (include/bfpp.h, executor section).
#include <nccl.h>

#include <cstring>
#include <vector>

#include "../../../include/bfpp.h"
#include "../sched/capi_util.hpp"
#include "executor.hpp"
#include "plan.hpp"

struct bfpp_exec {
    std::unique_ptr<bfpp::Executor> x;
};

using namespace bfpp;

extern "C" {

int bfpp_nccl_unique_id(void* out) {
    return guarded([&] {
        static_assert(sizeof(ncclUniqueId) == BFPP_NCCL_UID_BYTES, "ncclUniqueId size");
        ncclUniqueId id;
        if (ncclGetUniqueId(&id) != ncclSuccess) throw std::runtime_error("ncclGetUniqueId failed");
        std::memcpy(out, &id, sizeof(id));
    });
}

int64_t bfpp_exec_n_comm_ids(const bfpp_parallel_config* c) { return 1 + c->n_pp; }

namespace {
int create(const bfpp_model_spec* m, const bfpp_parallel_config* c, const bfpp_graph* g, const bfpp_exec_opts* o,
           int32_t rank, int32_t world, const void* uids, bfpp_exec** out) {
    *out = nullptr;
    return guarded([&] {
        ExecOptions eo;
        eo.device = o->device;
        eo.record_timeline = o->record_timeline != 0;
        eo.seed = o->seed;
        eo.lr = o->lr;
        eo.beta1 = o->beta1;
        eo.beta2 = o->beta2;
        eo.eps = o->eps;
        eo.weight_decay = o->weight_decay;
        eo.init_std = o->init_std;
        eo.skip_optimizer = (o->flags & BFPP_EXEC_SKIP_OPTIMIZER) != 0;
        eo.profile_kernels = (o->flags & BFPP_EXEC_PROFILE_KERNELS) != 0;
        eo.recompute = (o->flags & BFPP_EXEC_RECOMPUTE) != 0;
        std::vector<ncclUniqueId> ids;
        if (uids) {
            const int64_t n = bfpp_exec_n_comm_ids(c);
            ids.resize(static_cast<size_t>(n));
            std::memcpy(ids.data(), uids, static_cast<size_t>(n) * sizeof(ncclUniqueId));
        }
        *out = new bfpp_exec{
            std::make_unique<Executor>(to_model(m), to_config(c), eo, rank, world, ids, g ? &g->g : nullptr)};
    });
}
}  // namespace

int bfpp_exec_create(const bfpp_model_spec* m, const bfpp_parallel_config* c, const bfpp_exec_opts* o, int32_t rank,
                     int32_t world, const void* uids, bfpp_exec** out) {
    return create(m, c, nullptr, o, rank, world, uids, out);
}

int bfpp_exec_create_graph(const bfpp_model_spec* m, const bfpp_parallel_config* c, const bfpp_graph* g,
                           const bfpp_exec_opts* o, int32_t rank, int32_t world, const void* uids,
                           bfpp_exec** out) {
    return create(m, c, g, o, rank, world, uids, out);
}

namespace {
void copy_plan(const MemoryPlan& mp, int64_t* bytes, int64_t* sets) {
    for (int k = 0; k < M_NCAT; ++k) bytes[k] = static_cast<int64_t>(mp.bytes[k]);
    sets[0] = mp.activation_sets;
    sets[1] = mp.head_sets;
}
}  // namespace

int bfpp_exec_memory_plan(const bfpp_model_spec* m, const bfpp_parallel_config* c, const bfpp_exec_opts* o,
                          int32_t rank, int64_t* bytes, int64_t* sets) {
    return guarded([&] {
        ExecOptions eo;
        eo.skip_optimizer = (o->flags & BFPP_EXEC_SKIP_OPTIMIZER) != 0;
        eo.recompute = (o->flags & BFPP_EXEC_RECOMPUTE) != 0;
        eo.dry_run = true;
        const ParallelConfig pc = to_config(c);
        Executor x(to_model(m), pc, eo, rank, static_cast<int>(pc.grid_size()), {}, nullptr);
        copy_plan(x.memory_plan(), bytes, sets);
    });
}

int bfpp_exec_memory(const bfpp_exec* e, int64_t* bytes, int64_t* sets) {
    return guarded([&] { copy_plan(e->x->memory_plan(), bytes, sets); });
}

int bfpp_exec_step(bfpp_exec* e, const int32_t* tokens_host, float* loss) {
    return guarded([&] { e->x->step(tokens_host, true, loss, nullptr); });
}

int bfpp_exec_step_device(bfpp_exec* e, const int32_t* tokens_dev, float* loss_dev) {
    return guarded([&] { e->x->step(tokens_dev, false, nullptr, loss_dev); });
}

int bfpp_exec_sync(bfpp_exec* e) {
    return guarded([&] { e->x->sync(); });
}

void bfpp_exec_destroy(bfpp_exec* e) { delete e; }

int bfpp_exec_graph(const bfpp_exec* e, bfpp_graph** out) {
    *out = nullptr;
    return guarded([&] { *out = new bfpp_graph{e->x->graph()}; });
}

int64_t bfpp_exec_n_local_stages(const bfpp_exec* e) { return e->x->n_local_stages(); }
int64_t bfpp_exec_local_stage(const bfpp_exec* e, int64_t c) { return e->x->local_stage(c); }
int64_t bfpp_exec_stage_numel(const bfpp_exec* e, int64_t stage) { return e->x->layout(stage).numel; }
int64_t bfpp_exec_device_bytes(const bfpp_exec* e) { return static_cast<int64_t>(e->x->device_bytes()); }

int bfpp_exec_set_params(bfpp_exec* e, int64_t stage, const float* host, int64_t n) {
    return guarded([&] { e->x->set_params(stage, host, n); });
}
int bfpp_exec_get_params(bfpp_exec* e, int64_t stage, float* host, int64_t n, int64_t* lo, int64_t* hi) {
    return guarded([&] { e->x->get_params(stage, host, n, lo, hi); });
}
int bfpp_exec_get_grads(bfpp_exec* e, int64_t stage, float* host, int64_t n, int64_t* lo, int64_t* hi) {
    return guarded([&] { e->x->get_grads(stage, host, n, lo, hi); });
}
int bfpp_exec_get_weights16(bfpp_exec* e, int64_t stage, uint16_t* host, int64_t n, int64_t* lo, int64_t* hi) {
    return guarded([&] { e->x->get_weights16(stage, host, n, lo, hi); });
}
int bfpp_exec_zero_grads(bfpp_exec* e) {
    return guarded([&] { e->x->zero_grads(); });
}
int bfpp_exec_timeline(const bfpp_exec* e, double* start, double* end) {
    return guarded([&] { e->x->timeline(start, end); });
}

int bfpp_plan_rank(const bfpp_graph* g, int64_t pp_rank, int64_t n_dp, int32_t dp_variant, int64_t cap,
                   int64_t wait_cap, int32_t* ids, int32_t* streams, int32_t* flags, int32_t* slots,
                   int32_t* wait_offsets, int32_t* wait_ids, int64_t* n_tasks, int64_t* n_waits) {
    return guarded([&] {
        if (pp_rank < 0 || pp_rank >= g->g.n_devices) throw SpecError("plan: pipeline rank out of range");
        if (dp_variant < 0 || dp_variant > 2) throw SpecError("plan: dp_variant out of range");
        // the executor pools the gradient buffers of the sharded variants (see plan.hpp)
        const bool pooled = n_dp >= 2 && dp_variant != static_cast<int32_t>(DpVariant::DP0);
        const std::vector<PlanTask> plan = plan_rank(g->g, pp_rank, n_dp, pooled);
        int64_t nw = 0;
        for (const PlanTask& p : plan) nw += static_cast<int64_t>(p.waits.size());
        *n_tasks = static_cast<int64_t>(plan.size());
        *n_waits = nw;
        if (cap == 0) return;
        if (cap < static_cast<int64_t>(plan.size())) throw SpecError("plan: task arrays smaller than n_tasks");
        if (wait_cap < nw) throw SpecError("plan: wait_ids smaller than n_waits");
        int32_t k = 0;
        for (size_t i = 0; i < plan.size(); ++i) {
            const PlanTask& p = plan[i];
            ids[i] = p.id;
            streams[i] = p.stream;
            flags[i] = (p.send ? 1 : 0) | (p.first_unit ? 2 : 0) | (p.last_unit ? 4 : 0) | (p.adam_after ? 8 : 0) |
                       (p.first_in_unit ? 16 : 0) | (p.adam_tail ? 32 : 0) | (p.last_unit_bwd ? 64 : 0) |
                       (p.reduce_first_unit ? 128 : 0) | (p.unit_end_bwd ? 256 : 0);
            slots[i] = p.slot;
            wait_offsets[i] = k;
            for (TaskId w : p.waits) wait_ids[k++] = w;
        }
        wait_offsets[plan.size()] = k;
    });
}

int bfpp_exec_set_flags(bfpp_exec* e, int32_t record_timeline, int32_t profile_kernels) {
    return guarded([&] { e->x->set_flags(record_timeline != 0, profile_kernels != 0); });
}

void* bfpp_exec_stream(const bfpp_exec* e) { return e->x->compute_stream(); }

int bfpp_exec_kernel_stats(const bfpp_exec* e, int32_t cat, int64_t* launches, double* ms, double* work) {
    return guarded([&] {
        if (cat < 0 || cat >= K_NCAT) throw SpecError("kernel_stats: unknown category");
        const KernelStats& k = e->x->kernel_stats();
        if (launches) *launches = k.launches[cat];
        if (ms) *ms = k.ms[cat];
        if (work) *work = k.work[cat];
    });
}

}  // extern "C"
