// Per-rank execution plan of a TaskGraph (see plan.cpp).
#pragma once

#include <vector>

#include "../sched/schedule.hpp"

namespace bfpp {

// Executor streams ("lanes" of the reference simulator, simulate.cpp:31-37, made concrete).
enum StreamId {
    S_COMPUTE = 0, S_DP = 1, S_FWD_SEND = 2, S_FWD_RECV = 3, S_BWD_SEND = 4, S_BWD_RECV = 5,
    S_WGRAD = 6,  // weight-gradient GEMMs of backward tasks (optional overlap with the data-gradient chain)
    S_N = 7
};

struct PlanTask {
    TaskId id = -1;
    int stream = S_COMPUTE;
    bool send = false;          // Transfer: this rank sends (else receives)
    int slot = -1;              // DP_FS weight slot used (compute) or filled (reconstruct)
    bool first_unit = false, last_unit = false;  // Reduce
    bool adam_after = false;    // Bwd (n_dp == 1) or Reduce (last unit): run the optimizer for this stage
    bool first_in_unit = false; // Bwd: first gradient contribution of its reduction unit (overwrite, no zeroing)
    bool adam_tail = false;     // the step's last optimizer update (nothing left to overlap it; informational)
    // Bwd that completes its stage's last reduction unit (n_dp >= 2): the executor may reduce and
    // update the stage segment by segment inside it; reduce_first_unit = that Reduce is also the
    // stage's first unit (its reduce-scatter overwrites the gradient shard)
    bool last_unit_bwd = false, reduce_first_unit = false;
    // Bwd that completes a reduction unit (any unit, n_dp >= 2): under pooled gradients its
    // segments are reduce-scattered as the backward produces them
    bool unit_end_bwd = false;
    std::vector<TaskId> waits;  // events to wait on (deps on other streams + resource deps)
    std::vector<TaskId> after;  // host enqueue order only (no GPU wait)
};

// Tasks of pipeline rank `pp_rank` (compute, DP and both ends of its transfers) in host
// enqueue order: a topological order over cross-stream waits and per-stream FIFO order.
// pooled_grads (sharded variants): the rank's stages share one f32 gradient buffer whose reuse the
// executor guards per segment; a unit's first backward is then only ordered on the host after the
// previous unit's Reduce (whose reduce-scatters record those segment events) instead of waiting
// for that Reduce on the GPU.
std::vector<PlanTask> plan_rank(const TaskGraph& g, i64 pp_rank, i64 n_dp, bool pooled_grads = false);

}  // namespace bfpp
